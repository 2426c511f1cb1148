// Host build of the product's key math header (paper_2005_07547_b200/csrc/pstf_keys.cuh) for
// CPU-side differential testing against the reference (tests/test_keys_host.py).  Test-only:
// the product computes keys on the GPU; this shim exists so millions of inputs can be checked
// against glibc without a GPU.  Compiled with -ffp-contract=off (no FMA contraction).
#include "../../paper_2005_07547_b200/csrc/pstf_keys.cuh"

using namespace pstf_b200;

extern "C" {
void kh_key_for_batch(double base, double k, int max_level, const double *pos, const double *dir,
                      const int32_t *level, int64_t n, Key *out) {
    KeyParams p{base, k, max_level};
    for (int64_t i = 0; i < n; ++i)
        out[i] = key_for(p, pos[i], pos[n + i], pos[2 * n + i], dir[i], dir[n + i], dir[2 * n + i],
                         level[i]);
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
