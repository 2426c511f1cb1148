// Host build of the product's key math header (paper_2005_07547_b200/csrc/pstf_keys.cuh) for
// CPU-side differential testing against the reference (tests/test_keys_host.py).  Test-only:
// the product computes keys on the GPU; this shim exists so millions of inputs can be checked
// against glibc without a GPU.  Compiled with -ffp-contract=off (no FMA contraction).
#include "../../paper_2005_07547_b200/csrc/pstf_keys.cuh"

using namespace pstf_b200;

// 28-byte SpatioDirectionalKey layout (field.h:32-42) for the Python side
struct Key28 {
    int32_t level, cell[3], dir[2];
    uint32_t checksum;
};
static Key28 k28(const Key &k) {
    Key28 o;
    o.level = k.level;
    for (int i = 0; i < 3; ++i) o.cell[i] = k.cell[i];
    o.dir[0] = k.dir[0];
    o.dir[1] = k.dir[1];
    o.checksum = k.checksum;
    return o;
}

extern "C" {
void kh_key_for_batch(double base, double k, int max_level, const double *pos, const double *dir,
                      const int32_t *level, int64_t n, Key28 *out) {
    KeyParams p{base, k, max_level};
    for (int64_t i = 0; i < n; ++i)
        out[i] = k28(key_for(p, pos[i], pos[n + i], pos[2 * n + i], dir[i], dir[n + i],
                             dir[2 * n + i], level[i]));
}
void kh_select_level_batch(double base, double k, int max_level, const double *fp, int64_t n,
                           int32_t *out) {
    KeyParams p{base, k, max_level};
    for (int64_t i = 0; i < n; ++i) out[i] = select_level(p, fp[i]);
}
void kh_atan2_cr_batch(const double *y, const double *x, int64_t n, double *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = atan2_cr_pos(y[i], x[i]);
}
void kh_sphere_to_square_batch(const double *dir, int64_t n, int exact, double *uv) {
    for (int64_t i = 0; i < n; ++i)
        sphere_to_square_impl(dir[i], dir[n + i], dir[2 * n + i], exact, &uv[i], &uv[n + i]);
}
}

// Fast shared-quantisation path of the fused vertex kernel (pstf_keys.cuh: select_level_fast,
// pos_q/cell_at, octa_f8/dir_cell_f8): approximate arithmetic with exact re-evaluation near
// cell boundaries.  negate=1 keys the direction -d through the shared octahedral magnitudes.
extern "C" void kh_key_for_shared_batch(double base, double k, int max_level, const double *pos,
                                        const double *dir, const int32_t *level, int64_t n,
                                        int negate, Key28 *out) {
    KeyParams p{base, k, max_level};
    FastParams f = make_fast_params(p);
    for (int64_t i = 0; i < n; ++i) {
        double px = pos[i], py = pos[n + i], pz = pos[2 * n + i];
        double dx = dir[i], dy = dir[n + i], dz = dir[2 * n + i];
        PosQ q = pos_q(f, px, py, pz);
        int l = level[i];
        DirF8 a, b;
        octa_f8(dx, dy, dz, 1, &a, &b);
        Key kk;
        kk.level = l;
        kk.cell[0] = cell_at(f, q.q[0], px, l);
        kk.cell[1] = cell_at(f, q.q[1], py, l);
        kk.cell[2] = cell_at(f, q.q[2], pz, l);
        kk.dir[0] = dir_cell_f8(negate ? b.u : a.u, l);
        kk.dir[1] = dir_cell_f8(negate ? b.v : a.v, l);
        kk.checksum = checksum_of(key_pack(kk));
        kk.pack_lo = 0;
        out[i] = k28(kk);
    }
}

extern "C" void kh_select_level_fast_batch(double base, double k, int max_level, const double *fp,
                                           int64_t n, int32_t *out) {
    KeyParams p{base, k, max_level};
    FastParams f = make_fast_params(p);
    for (int64_t i = 0; i < n; ++i) out[i] = select_level_fast(f, fp[i]);
}
