/*
 * pstf_keys.cuh — spatio-directional key quantisation for the B200 field cache.
 *
 * Bit-exact restatement (host+device) of the reference key math:
 *   selectLevel    proj/core/src/field.cpp:68-76
 *   cellSize       field.cpp:78-80,  dirResolution field.cpp:82-84
 *   keyFor         field.cpp:86-101, packKeyFields field.cpp:38-44, mixBits rng.h:61-68
 *   sphereToSquare proj/core/include/pstf/mappings.h:33-51
 * Exactness strategy:
 *   - compiled with -fmad=false (device) / -ffp-contract=off (host): no FMA contraction;
 *     explicit fma() appears only inside error-free transformations (two_prod).
 *   - floor(log2(s)) comes from the exponent bits plus an exact test of whether the correctly
 *     rounded log2(s) rounds up to the next integer (s a few ulps below a power of two).
 *   - atan2 is evaluated with a fast polynomial; only when the resulting octahedral
 *     coordinate lies within 1e-11 of a directional-cell boundary is it recomputed with a
 *     double-double atan2 that returns the correctly rounded result (what glibc returns on
 *     >99.8% of inputs, SURVEY.md Appendix B libm probe).  The fused vertex kernel also uses
 *     approximate divisions / square roots with exact re-evaluation near cell boundaries
 *     (see "fast shared per-vertex quantisation" below).
 *   - int32 conversions reproduce x86-64 cvttsd2si: NaN / out of range -> INT32_MIN.
 */
#pragma once
#include <stdint.h>
#include <math.h>

#if defined(__CUDACC__)
#define PSTF_HD __host__ __device__ __forceinline__
#define PSTF_HD_NOINLINE __host__ __device__ __noinline__
#else
#define PSTF_HD static inline
#define PSTF_HD_NOINLINE static
#endif

namespace pstf_b200 {

struct Key {
    int32_t level;
    int32_t cell[3];
    int32_t dir[2];
    uint32_t checksum;
    uint32_t pack_lo; /* low 32 bits of packKeyFields: home slot = pack_lo & mask */
};

struct KeyParams {
    double base_cell_size;
    double level_select_k;
    int32_t max_level;
};

PSTF_HD uint64_t mix_bits(uint64_t v) {
    v ^= v >> 30;
    v *= 0xbf58476d1ce4e5b9ULL;
    v ^= v >> 27;
    v *= 0x94d049bb133111ebULL;
    v ^= v >> 31;
    return v;
}

PSTF_HD uint64_t pack_key_fields(int32_t level, int32_t c0, int32_t c1, int32_t c2, int32_t d0,
                                 int32_t d1) {
    uint64_t h = (uint64_t)(uint32_t)level;
    h = mix_bits(h ^ (((uint64_t)(uint32_t)c0 << 32) | (uint32_t)c1));
    h = mix_bits(h ^ (((uint64_t)(uint32_t)c2 << 32) | (uint32_t)d0));
    h = mix_bits(h ^ (uint64_t)(uint32_t)d1);
    return h;
}

/* packKeyFields split after its first round: keys sharing (level, cell0, cell1) share h1 */
PSTF_HD uint64_t pack_h1(int32_t level, int32_t c0, int32_t c1) {
    return mix_bits((uint64_t)(uint32_t)level ^ (((uint64_t)(uint32_t)c0 << 32) | (uint32_t)c1));
}

PSTF_HD uint64_t pack_from_h1(uint64_t h1, int32_t c2, int32_t d0, int32_t d1) {
    uint64_t h = mix_bits(h1 ^ (((uint64_t)(uint32_t)c2 << 32) | (uint32_t)d0));
    return mix_bits(h ^ (uint64_t)(uint32_t)d1);
}

PSTF_HD uint32_t checksum_of(uint64_t packed) {
    uint32_t s = (uint32_t)mix_bits(packed ^ 0x5bf03635ULL);
    return s == 0 ? 1u : s;
}

/* x86-64 cvttsd2si: the reference's int32_t(double) on the reference platform */
PSTF_HD int32_t i32_x86(double x) {
    if (!(x >= -2147483648.0 && x < 2147483648.0)) return INT32_MIN;
    return (int32_t)x;
}

PSTF_HD uint64_t dbits(double x) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(x);
#else
    union { double d; uint64_t u; } c;
    c.d = x;
    return c.u;
#endif
}

PSTF_HD double bitsd(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)u);
#else
    union { double d; uint64_t u; } c;
    c.u = u;
    return c.d;
#endif
}

PSTF_HD double pow2d(int k) { /* 2^k, k in [-1022, 1023] */
    return bitsd((uint64_t)(k + 1023) << 52);
}

#define PSTF_INV_LN2 1.4426950408889634

/* field.cpp:68-76: clamp(floor(log2(footprint*K/base)), 0, maxLevel), with the rounding of a
 * correctly rounded log2 reproduced exactly. */
PSTF_HD int select_level(const KeyParams &p, double footprint) {
    if (!(footprint > 0.0)) return 0;
    double s = footprint * p.level_select_k / p.base_cell_size;
    if (s <= 1.0) return 0;
    int level;
    if (!(s <= 1.7976931348623157e308)) {
        level = INT32_MIN; /* log2(inf)=inf / log2(NaN)=NaN -> int32 on x86 -> INT32_MIN */
    } else {
        uint64_t b = dbits(s);
        int e = (int)((b >> 52) & 0x7ff) - 1023; /* s > 1 is a normal number */
        /* m = s / 2^(e+1) in [0.5, 1) exactly; delta = 1 - m exact (Sterbenz) */
        double m = bitsd((b & 0x000fffffffffffffULL) | (0x3feULL << 52));
        double delta = 1.0 - m;
        /* log2(s) = L + log2(1 - delta), L = e + 1; rounds to L iff the deficit
         * -log2(1-delta) ~= delta/ln2 (1 + delta/2) is <= half the gap below L */
        int L = e + 1;
        uint64_t lb = dbits((double)L);
        int pexp = (int)((lb >> 52) & 0x7ff) - 1023;
        int pow2 = (lb & 0x000fffffffffffffULL) == 0;
        double half_gap = pow2d(pexp - (pow2 ? 54 : 53));
        double deficit = delta * PSTF_INV_LN2 * (1.0 + 0.5 * delta);
        level = (deficit <= half_gap) ? L : e;
    }
    if (level < 0) level = 0;
    return level < p.max_level ? level : p.max_level;
}

PSTF_HD double cell_size(const KeyParams &p, int level) {
    return p.base_cell_size * (double)((uint64_t)1 << level); /* field.cpp:78-80 */
}

PSTF_HD int dir_resolution(int level) { return 8 >> (level < 2 ? level : 2); } /* field.cpp:82-84 */

/* ---------------- double-double atan2 (slow path, correctly rounded) ---------------- */
struct DD { double hi, lo; };

PSTF_HD DD dd_two_sum(double a, double b) {
    double s = a + b;
    double bb = s - a;
    double e = (a - (s - bb)) + (b - bb);
    DD r; r.hi = s; r.lo = e; return r;
}
PSTF_HD DD dd_quick(double a, double b) {
    double s = a + b;
    DD r; r.hi = s; r.lo = b - (s - a); return r;
}
PSTF_HD DD dd_two_prod(double a, double b) {
    double p = a * b;
    DD r; r.hi = p; r.lo = fma(a, b, -p); return r;
}
PSTF_HD DD dd_add(DD x, DD y) {
    DD s = dd_two_sum(x.hi, y.hi);
    DD t = dd_two_sum(x.lo, y.lo);
    s.lo += t.hi;
    s = dd_quick(s.hi, s.lo);
    s.lo += t.lo;
    return dd_quick(s.hi, s.lo);
}
PSTF_HD DD dd_neg(DD x) { x.hi = -x.hi; x.lo = -x.lo; return x; }
PSTF_HD DD dd_mul(DD x, DD y) {
    DD p = dd_two_prod(x.hi, y.hi);
    p.lo += x.hi * y.lo + x.lo * y.hi;
    return dd_quick(p.hi, p.lo);
}
PSTF_HD DD dd_div(DD x, DD y) {
    double q1 = x.hi / y.hi;
    DD r = dd_add(x, dd_neg(dd_mul(y, DD{q1, 0.0})));
    double q2 = r.hi / y.hi;
    r = dd_add(r, dd_neg(dd_mul(y, DD{q2, 0.0})));
    double q3 = r.hi / y.hi;
    DD q = dd_quick(q1, q2);
    return dd_add(q, DD{q3, 0.0});
}

#define PSTF_ATAN_TABLE \
    {0.0, 0.0}, \
    {0.015623728620476831, -4.913600136566304e-19}, \
    {0.031239833430268277, -1.188442711587748e-18}, \
    {0.046840712915969654, -1.655677442254952e-19}, \
    {0.06241880999595735, -1.5490756308295046e-18}, \
    {0.0779666338315423, 5.804551873143357e-18}, \
    {0.09347678115858947, -6.2844725995420954e-18}, \
    {0.10894195698986579, 6.8267122072409585e-18}, \
    {0.12435499454676144, -3.1253241424539383e-18}, \
    {0.13970887428916365, -2.9579864247315813e-18}, \
    {0.15499674192394097, 9.585415594114324e-18}, \
    {0.1702119252854744, -3.541164079802125e-18}, \
    {0.18534794999569476, 4.180692268843079e-18}, \
    {0.2003985538258785, 3.1399542871844493e-18}, \
    {0.21535769969773805, 4.738160130078733e-19}, \
    {0.23021958727684372, 1.2313404529142703e-17}, \
    {0.24497866312686414, 1.0698755618734451e-17}, \
    {0.2596296294082575, 1.9238754924615304e-17}, \
    {0.2741674511196588, 8.261353575163773e-18}, \
    {0.2885873618940774, -1.428369957377257e-17}, \
    {0.3028848683749714, -1.1010827903001369e-17}, \
    {0.31705575320914703, -1.893928924292642e-17}, \
    {0.3310960767041321, -7.952610375793799e-18}, \
    {0.34500217720710513, -2.2938804755578304e-17}, \
    {0.35877067027057225, -2.4623815582638635e-17}, \
    {0.3723984466767542, 1.9612311504845653e-17}, \
    {0.38588266939807375, 2.378822732491941e-17}, \
    {0.39922076957525254, 2.246598105617042e-17}, \
    {0.4124104415973873, -1.587652227770689e-17}, \
    {0.42544963737004227, 2.3315530741892885e-17}, \
    {0.43833655985795783, -2.494277030626541e-17}, \
    {0.4510696559885235, -2.2703795229420475e-17}, \
    {0.4636476090008061, 2.2698777452961687e-17}, \
    {0.4760693303227612, 1.4654487332256713e-17}, \
    {0.48833395105640554, -1.1373236189329585e-17}, \
    {0.5004408131472942, -4.7181675085518756e-17}, \
    {0.5123894603107377, -2.5462781472855804e-17}, \
    {0.5241796287829132, 5.520094119641666e-18}, \
    {0.5358112379604637, -4.0637956834825575e-18}, \
    {0.5472843809874369, 4.923709671396255e-17}, \
    {0.5585993153435624, -5.4556305485916264e-18}, \
    {0.5697564534829784, 1.2255062085054184e-17}, \
    {0.5807563535676704, -1.441464378193067e-17}, \
    {0.5915997103351114, 4.920495453686772e-17}, \
    {0.6022873461349642, 2.950430737228402e-17}, \
    {0.6128202021652414, -3.1552061848586226e-17}, \
    {0.6231993299340659, 2.672403885140095e-17}, \
    {0.6334258829691446, -2.7290767436015276e-17}, \
    {0.6435011087932844, 1.5834785051444286e-17}, \
    {0.6534263411807619, 3.5800634857340095e-17}, \
    {0.6632029927060933, -3.076054864429649e-17}, \
    {0.6728325475937632, -1.899315009714705e-17}, \
    {0.6823165548747481, 6.943223671560008e-18}, \
    {0.6916566218531999, -8.117151192285796e-18}, \
    {0.7008544078844502, -1.987626234335816e-17}, \
    {0.7099116184635249, -4.597166450584887e-17}, \
    {0.7188299996216245, -2.1478388444456983e-17}, \
    {0.7276113326265107, 2.569325697391839e-18}, \
    {0.7362574289814281, 3.473937648299457e-17}, \
    {0.7447701257160751, 3.708315849135547e-17}, \
    {0.7531512809621944, -2.4256934659182068e-17}, \
    {0.7614027698055784, 9.850030332752822e-18}, \
    {0.7695264804056583, -3.704991905602721e-17}, \
    {0.7775243103733478, -2.6676490951944502e-17}, \
    {0.7853981633974483, 3.061616997868383e-17}, \

#if defined(__CUDACC__)
__device__ __constant__ double pstf_atan_tab_dev[65][2] = {PSTF_ATAN_TABLE};
#endif
static const double pstf_atan_tab_host[65][2] = {PSTF_ATAN_TABLE};

PSTF_HD DD atan_tab(int i) {
#if defined(__CUDA_ARCH__)
    return DD{pstf_atan_tab_dev[i][0], pstf_atan_tab_dev[i][1]};
#else
    return DD{pstf_atan_tab_host[i][0], pstf_atan_tab_host[i][1]};
#endif
}

/* atan(t) for t = th + tl in [0, 1], double-double, ~2^-104 relative */
PSTF_HD_NOINLINE DD dd_atan01(DD t) {
    int i = (int)(t.hi * 64.0 + 0.5);
    if (i > 64) i = 64;
    double c = (double)i * 0.015625;
    DD num = dd_add(t, DD{-c, 0.0});
    DD tc = dd_mul(t, DD{c, 0.0});
    DD den = dd_add(DD{1.0, 0.0}, tc);
    DD r = dd_div(num, den);
    DD s = dd_mul(r, r);
    /* P(s) = sum_k (-1)^k s^k / (2k+1), k = 0..8 (|r| <= 2^-7) */
    const double ch[9] = {1.0, -0.3333333333333333, 0.2, -0.14285714285714285, 0.1111111111111111,
                          -0.09090909090909091, 0.07692307692307693, -0.06666666666666667,
                          0.058823529411764705};
    const double cl[9] = {0.0, -1.850371707708594e-17, -1.1102230246251566e-17,
                          -7.93016446160826e-18, 6.1679056923619804e-18, 2.523234146875356e-18,
                          -4.270088556250602e-18, -9.251858538542971e-19, 8.163404592832033e-19};
    DD acc = DD{ch[8], cl[8]};
    for (int k = 7; k >= 0; --k) acc = dd_add(dd_mul(acc, s), DD{ch[k], cl[k]});
    DD at = dd_mul(r, acc);
    return dd_add(atan_tab(i), at);
}

/* correctly rounded atan2(y, x) for x, y >= 0 (not both zero), incl. infinities */
PSTF_HD_NOINLINE double atan2_cr_pos(double y, double x) {
    const DD pio2 = DD{1.5707963267948966, 6.123233995736766e-17};
    if (x != x || y != y) return x + y;
    const double inf = HUGE_VAL;
    if (x == inf && y == inf) return 0.7853981633974483;
    if (x == inf) return 0.0;
    if (y == inf) return 1.5707963267948966;
    if (y == x) return 0.7853981633974483;
    int swap = y > x;
    double a = swap ? x : y, b = swap ? y : x; /* a < b */
    double th = a / b;
    double tl = fma(-th, b, a) / b;
    DD t = dd_quick(th, tl);
    DD r = dd_atan01(t);
    if (swap) r = dd_add(pio2, dd_neg(r));
    return r.hi + r.lo;
}

/* Approximate reciprocal / square root for the fast (non-deciding) path: single-precision
 * hardware estimate (relative error < 2^-22 incl. the rounding of the argument to float) + one
 * Newton step in fp64, relative error < 2^-43 (~1.2e-13) for den in [1e-30, 1e30].  The octahedral
 * coordinates built from them stay within ~1e-12 of the exact ones, well inside the 1e-11 margin
 * that sends a coordinate to the exact path. */
PSTF_HD double fast_rcp(double den) {
#if defined(__CUDA_ARCH__)
    double r = (double)__frcp_rn((float)den);
#else
    double r = (double)(1.0f / (float)den);
#endif
    return r * fma(-den, r, 2.0);
}

PSTF_HD double fast_sqrt01(double w) { /* w in [0, 1]; relative error < 2^-42 */
    if (!(w >= 1e-30)) return 0.0;
#if defined(__CUDA_ARCH__)
    double y = (double)rsqrtf((float)w);
#else
    double y = (double)(1.0f / sqrtf((float)w));
#endif
    y = y * fma(-0.5 * w, y * y, 1.5);
    return w * y;
}

/* Fast atan2 for x, y >= 0 (|error| < 1e-15 rad): octant reduction to |t| <= tan(pi/8) with one
 * approximate reciprocal, then a degree-9 polynomial in t^2 (Chebyshev-node fit).  Only used to
 * pick the directional cell; results within 1e-11 of a cell boundary are recomputed with the
 * correctly rounded atan2_cr_pos, so it never decides a key on its own near a boundary. */
PSTF_HD double atan2_fast(double y, double x) {
    if (!(x <= 1.7976931348623157e308 && y <= 1.7976931348623157e308)) return atan2_cr_pos(y, x);
    const int swap = y > x;
    const double a = swap ? x : y, b = swap ? y : x; /* 0 <= a <= b, b > 0 */
    double t, base;
    const bool small = a <= b * 0.41421356237309503;
    const double num = small ? a : a - b, den = small ? b : a + b;
    base = small ? 0.0 : 0.7853981633974483;
    if (den >= 1e-30 && den <= 1e30) t = num * fast_rcp(den);
    else t = num / den;
    const double z = t * t;
    double p = -0.025316479573776477;
    p = fma(p, z, 0.05024762118940128);
    p = fma(p, z, -0.0650598296717084);
    p = fma(p, z, 0.07673535428183285);
    p = fma(p, z, -0.09089529956562307);
    p = fma(p, z, 0.11111048853751296);
    p = fma(p, z, -0.14285712661684793);
    p = fma(p, z, 0.19999999978392663);
    p = fma(p, z, -0.3333333333322143);
    p = fma(p, z, 0.999999999999999);
    const double th = base + t * p;
    return swap ? 1.5707963267948966 - th : th;
}

/* mappings.h:33-51 with the reference's operation order; exact_atan selects the slow path */
PSTF_HD void sphere_to_square_impl(double dx, double dy, double dz, int exact_atan, double *uo,
                                   double *vo) {
    double x = fabs(dx), y = fabs(dy), z = fabs(dz);
    double omz = 1.0 - z;
    double r = sqrt((0.0 < omz) ? omz : 0.0); /* safeSqrt: std::max(0.0, x) vecmath.h:22 */
    double phi;
    if (x == 0.0 && y == 0.0) phi = 0.0;
    else phi = (exact_atan ? atan2_cr_pos(y, x) : atan2_fast(y, x)) * (2.0 / 3.14159265358979323846);
    double v = phi * r;
    double u = r - v;
    if (dz < 0.0) {
        double t = u;
        u = v;
        v = t;
        u = 1.0 - u;
        v = 1.0 - v;
    }
    u = copysign(u, dx);
    v = copysign(v, dy);
    *uo = 0.5 * (u + 1.0);
    *vo = 0.5 * (v + 1.0);
}

PSTF_HD int near_cell_boundary(double q) {
    if (!(q == q)) return 0;
    double f = floor(q);
    return (q - f) < 1e-11 || (f + 1.0 - q) < 1e-11;
}

/* dirCell (field.cpp:93-95) for resolution d */
PSTF_HD void dir_cells(double dx, double dy, double dz, int d, int32_t *d0, int32_t *d1) {
    double u, v;
    sphere_to_square_impl(dx, dy, dz, 0, &u, &v);
    double qu = u * (double)d, qv = v * (double)d;
    if (near_cell_boundary(qu) || near_cell_boundary(qv)) {
        sphere_to_square_impl(dx, dy, dz, 1, &u, &v);
        qu = u * (double)d;
        qv = v * (double)d;
    }
    int32_t a = i32_x86(qu), b = i32_x86(qv);
    *d0 = a < d - 1 ? a : d - 1;
    *d1 = b < d - 1 ? b : d - 1;
}

/* field.cpp:86-101 */
PSTF_HD Key key_for(const KeyParams &p, double px, double py, double pz, double dx, double dy,
                    double dz, int level) {
    Key k;
    k.level = level;
    double cs = cell_size(p, level);
    k.cell[0] = i32_x86(floor(px / cs));
    k.cell[1] = i32_x86(floor(py / cs));
    k.cell[2] = i32_x86(floor(pz / cs));
    dir_cells(dx, dy, dz, dir_resolution(level), &k.dir[0], &k.dir[1]);
    uint64_t pk = pack_key_fields(level, k.cell[0], k.cell[1], k.cell[2], k.dir[0], k.dir[1]);
    k.checksum = checksum_of(pk);
    k.pack_lo = (uint32_t)pk;
    return k;
}

PSTF_HD uint64_t key_pack(const Key &k) {
    return pack_key_fields(k.level, k.cell[0], k.cell[1], k.cell[2], k.dir[0], k.dir[1]);
}

/* ---------------- fast shared per-vertex quantisation (same results as key_for) -------------
 * Used by the fused vertex kernel.  Every key of a vertex uses the same position at the same
 * level, every level of a lookup uses the same position and direction, and d / -d share their
 * octahedral magnitudes.  Each quantity is first computed approximately (reciprocal multiply,
 * polynomial atan2, Newton sqrt) and the exact reference operation is re-run only when the
 * approximation lies within its error bound of a cell boundary:
 *  cells     x' = p * (1/base) * 2^-l is within 2^-51 |x| of fl(p / (base 2^l)); if x' is further
 *            than 2^-50 |x'| from every integer, floor(x') == floor(fl(p / cs)).
 *  level     s' = footprint * (K / base) is within a few ulps of fl(fl(fp K) / base); away from
 *            powers of two its exponent is floor(log2(s)); near them select_level runs exactly.
 *  dirCell   u, v to ~1e-15 absolute; within 1e-11 of k/8 the correctly rounded path re-runs.
 *            floor(U d) == floor(U 8) >> log2(8/d), so one floor per direction serves all
 *            levels (U is in [0, 1] or NaN). */
/* rare exact re-evaluations kept out of line (instruction-cache footprint of the hot kernel) */
PSTF_HD int select_level_exact(const KeyParams &p, double footprint) {
    return select_level(p, footprint);
}

PSTF_HD int32_t cell_exact(const KeyParams &p, double pcoord, int level) {
    if (pcoord == 0.0) return 0;
    return i32_x86(floor(pcoord / cell_size(p, level)));
}

struct FastParams {
    KeyParams kp;
    double inv_base;   /* fl(1 / base) */
    double k_inv_base; /* fl(K / base) */
};

PSTF_HD FastParams make_fast_params(const KeyParams &kp) {
    FastParams f;
    f.kp = kp;
    f.inv_base = 1.0 / kp.base_cell_size;
    f.k_inv_base = kp.level_select_k / kp.base_cell_size;
    return f;
}

/* Fast level: decided from the exponent of s' = footprint * fl(K / base), which lies within a few
 * ulps of the reference's fl(fl(footprint K) / base); sets *nx when s' is too close to a power of
 * two (or out of range) for that to be certain.  (*nx = "needs the exact reference operation") */
PSTF_HD int select_level_try(const FastParams &f, double footprint, int *nx) {
    /* branch-free (selects only): the caller's warp never diverges here */
    const bool pos = footprint > 0.0;
    const double s = footprint * f.k_inv_base;
    const bool low = s < 0.9999999999; /* exact s <= 1: level 0 (field.cpp:71) */
    const uint64_t b = dbits(s);
    const uint64_t mant = b & 0x000fffffffffffffULL;
    /* mantissa not within 2^-40 of either end of [1, 2): exponent == floor(log2(s)) */
    const bool mid = (s > 1.0000000001) & (s < 1e300) & (mant > (1ULL << 12)) &
                     (mant < 0x000fffffffffffffULL - (1ULL << 12));
    const int level = (int)((b >> 52) & 0x7ff) - 1023;
    *nx |= pos & !low & !mid;
    return (pos & !low & mid) ? (level < f.kp.max_level ? level : f.kp.max_level) : 0;
}

PSTF_HD int select_level_fast(const FastParams &f, double footprint) {
    int nx = 0;
    const int l = select_level_try(f, footprint, &nx);
    return nx ? select_level_exact(f.kp, footprint) : l;
}

struct PosQ {
    double q[3];
};

PSTF_HD PosQ pos_q(const FastParams &f, double px, double py, double pz) {
    PosQ r;
    r.q[0] = px * f.inv_base;
    r.q[1] = py * f.inv_base;
    r.q[2] = pz * f.inv_base;
    return r;
}

/* Fast cell coordinate floor(pcoord / (base 2^level)) from q = pcoord * fl(1 / base); sets *nx
 * when x' is within 2^-50 |x'| of an integer (or out of the plain range). */
PSTF_HD int32_t cell_try(double q, double pcoord, int level, int *nx) {
    /* branch-free: q == 0 exactly when pcoord == 0 (q = pcoord * fl(1/base), no underflow to 0
     * for nonzero pcoord above 2^-900), and then floor(+-0 / cs) == 0 like the fast path */
    (void)pcoord;
    const double x = q * pow2d(-level);
    const double ax = fabs(x);
    const double fl = floor(x);
    const double e = ax * 0x1p-50;
    /* non-short-circuit & and |: no branches, so the three coordinates of a position (and
     * the surrounding work) interleave */
    const bool ok = (ax < 2147483647.0) & ((ax >= 0x1p-900) | (ax == 0.0)) & (x - fl >= e) &
                    ((fl + 1.0) - x >= e); /* fl in [-2^31 + 1, 2^31 - 2]: exact conversion */
    /* far outside int32 (finite): the reference's conversion gives INT32_MIN */
    const bool far = (ax >= 4294967296.0) & (ax <= 1.7976931348623157e308);
    *nx |= !(ok | far);
    return ok ? (int32_t)fl : INT32_MIN;
}

PSTF_HD int32_t cell_at(const FastParams &f, double q, double pcoord, int level) {
    int nx = 0;
    const int32_t c = cell_try(q, pcoord, level, &nx);
    return nx ? cell_exact(f.kp, pcoord, level) : c; /* exact reference operation */
}

/* pre-swap octahedral coordinates from |x|, |y|, |z| (mappings.h:34-42) */
PSTF_HD void octa_base(double dx, double dy, double dz, int exact, double *u0, double *v0) {
    double x = fabs(dx), y = fabs(dy), z = fabs(dz);
    double omz = 1.0 - z;
    double w = (0.0 < omz) ? omz : 0.0; /* safeSqrt: std::max(0.0, x) vecmath.h:22 */
    double r = exact ? sqrt(w) : fast_sqrt01(w);
    double phi;
    if (x == 0.0 && y == 0.0) phi = 0.0;
    else phi = (exact ? atan2_cr_pos(y, x) : atan2_fast(y, x)) * (2.0 / 3.14159265358979323846);
    *v0 = phi * r;
    *u0 = r - *v0;
}

/* hemisphere swap + sign restoration + [0,1]^2 (mappings.h:43-50) */
PSTF_HD void octa_uv(double u0, double v0, double dx, double dy, double dz, double *U, double *V) {
    double u = u0, v = v0;
    if (dz < 0.0) {
        double t = u;
        u = v;
        v = t;
        u = 1.0 - u;
        v = 1.0 - v;
    }
    u = copysign(u, dx);
    v = copysign(v, dy);
    *U = 0.5 * (u + 1.0);
    *V = 0.5 * (v + 1.0);
}

/* floor(U * 8) with the reference's int32 conversion (NaN -> INT32_MIN); near = within 1e-11 of
 * an integer.  U lies in [-1e-12, 1 + 1e-12] or is NaN, so floor(U * 8) is in [-1, 8] or NaN;
 * f = q - fl is exact and 1 - f == fl + 1 - q wherever it is small. */
PSTF_HD int32_t f8_of(double U, int *near) {
    const double q = U * 8.0;
    const double fl = floor(q);
    *near |= fabs((q - fl) - 0.5) > 0.5 - 1e-11;
    return fl == fl ? (int32_t)fl : INT32_MIN;
}

struct DirF8 {
    int32_t u, v;
};

PSTF_HD void octa_f8_exact(double dx, double dy, double dz, int want_neg, DirF8 *pos,
                                    DirF8 *neg) {
    double u0, v0, U, V;
    int dummy = 0;
    octa_base(dx, dy, dz, 1, &u0, &v0);
    octa_uv(u0, v0, dx, dy, dz, &U, &V);
    pos->u = f8_of(U, &dummy);
    pos->v = f8_of(V, &dummy);
    if (want_neg) {
        octa_uv(u0, v0, -dx, -dy, -dz, &U, &V);
        neg->u = f8_of(U, &dummy);
        neg->v = f8_of(V, &dummy);
    }
}

/* atan2 for x, y >= 0 not both zero, no internal fallback: *nx set when the reduction's
 * denominator leaves [1e-30, 1e30] (infinities, NaN, denormal-scale directions) */
PSTF_HD double atan2_try(double y, double x, int *nx) {
    const int swap = y > x;
    const double a = swap ? x : y, b = swap ? y : x; /* 0 <= a <= b, b > 0 */
    const bool small = a <= b * 0.41421356237309503;
    const double num = small ? a : a - b, den = small ? b : a + b;
    *nx |= !(den >= 1e-30 && den <= 1e30);
    const double t = num * fast_rcp(den);
    const double z = t * t;
    double p = -0.025316479573776477;
    p = fma(p, z, 0.05024762118940128);
    p = fma(p, z, -0.0650598296717084);
    p = fma(p, z, 0.07673535428183285);
    p = fma(p, z, -0.09089529956562307);
    p = fma(p, z, 0.11111048853751296);
    p = fma(p, z, -0.14285712661684793);
    p = fma(p, z, 0.19999999978392663);
    p = fma(p, z, -0.3333333333322143);
    p = fma(p, z, 0.999999999999999);
    const double th = (small ? 0.0 : 0.7853981633974483) + t * p;
    return swap ? 1.5707963267948966 - th : th;
}

/* sqrt(w) for w in [0, 1] from the hardware reciprocal square root plus one fp32 Newton
 * correction: within 1.5 ulp (branch-free, 0 -> 0) */
PSTF_HD float sqrt_fast(float w) {
#if defined(__CUDA_ARCH__)
    const float y = rsqrtf(w);
#else
    const float y = 1.0f / sqrtf(w);
#endif
    const float r = w * y;
    const float e = fmaf(-r, r, w);
    const float s = fmaf(e, 0.5f * y, r);
    return w > 0.0f ? s : 0.0f;
}

/* floor(q) of q = 8 U in single precision; near when q is within 2e-5 of an integer (the
 * single-precision U below is within 1e-6 of the exact one, see octa_f8_try) */
PSTF_HD int32_t f8_of32(float U, int *near) {
    const float q = U * 8.0f;
    const float fl = floorf(q);
    *near |= fabsf((q - fl) - 0.5f) > 0.5f - 2e-5f;
    return (int32_t)fl;
}

/* octahedral cell coordinates (at resolution 8) of d and optionally -d from a single-precision
 * fast path; *nx set when any coordinate may lie within its error of a cell boundary or the
 * inputs are outside the fast path's domain (the caller then recomputes with octa_f8_exact).
 * Error budget (|.| in U units): w = 1 - |z| is formed in double precision and rounded once
 * (6e-8 relative), r = sqrt_fast(w) within 1.5 ulp, phi from a degree-4 minimax polynomial in t^2
 * (|error| < 3e-7) after an octant reduction with the hardware reciprocal estimate (t within
 * 3e-7 relative), then four rounded products/sums: |U' - U| < 1.5e-6, so q' = 8 U' is within
 * 1.2e-5 of q, inside the 2e-5 margin.  NaN, infinite and denormal-scale x, y (either one)
 * always take the exact path. */
PSTF_HD void octa_f8_try(double dx, double dy, double dz, int want_neg, DirF8 *pos, DirF8 *neg,
                         int *nx) {
    const double x = fabs(dx), y = fabs(dy), z = fabs(dz);
    /* safeSqrt(1 - |z|) (vecmath.h:22): the difference in double precision (exact for |z| in
     * [0.5, 1]), rounded once; NaN and negative -> 0 like std::max(0.0, .) */
    const float wf = fmaxf((float)(1.0 - z), 0.0f);
    const float r = sqrt_fast(wf);
    /* branch-free: phi is computed for x = y = 0 too and replaced by 0 there (mappings.h:39) */
    const bool zero = x == 0.0 && y == 0.0;
    const float xf = (float)x, yf = (float)y;
    /* fast-path domain: x and y finite (a NaN fails the comparisons) and the larger one in
     * [1e-30, 1e30] */
    *nx |= !zero & !(xf <= 1e30f && yf <= 1e30f && (xf >= 1e-30f || yf >= 1e-30f));
    const bool swap = yf > xf;
    const float a = swap ? xf : yf, b = swap ? yf : xf; /* 0 <= a <= b */
    const bool small = a <= b * 0.41421356f;
    const float num = small ? a : a - b, den = small ? b : a + b;
#if defined(__CUDA_ARCH__)
    float rc; /* hardware reciprocal estimate, relative error < 2^-22 (den is a normal) */
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(den));
    const float t = num * rc;
#else
    const float t = num * (1.0f / den);
#endif
    const float zz = t * t;
    float p = 0.07726402580738068f;
    p = fmaf(p, zz, -0.13751664757728577f);
    p = fmaf(p, zz, 0.19961561262607574f);
    p = fmaf(p, zz, -0.33332183957099915f);
    p = fmaf(p, zz, 0.9999998807907104f);
    const float th = (small ? 0.0f : 0.78539816f) + t * p;
    const float phi = zero ? 0.0f : (swap ? 1.57079633f - th : th) * 0.63661977f; /* * 2/pi */
    const float v0 = phi * r, u0 = r - v0;
    float u = u0, v = v0;
    if (dz < 0.0) { /* hemisphere swap (mappings.h:43-48) */
        u = 1.0f - v0;
        v = 1.0f - u0;
    }
    pos->u = f8_of32(0.5f * (copysignf(u, (float)dx) + 1.0f), nx);
    pos->v = f8_of32(0.5f * (copysignf(v, (float)dy) + 1.0f), nx);
    if (want_neg) {
        float un = u0, vn = v0;
        if (-dz < 0.0) {
            un = 1.0f - v0;
            vn = 1.0f - u0;
        }
        neg->u = f8_of32(0.5f * (copysignf(un, (float)-dx) + 1.0f), nx);
        neg->v = f8_of32(0.5f * (copysignf(vn, (float)-dy) + 1.0f), nx);
    }
}

/* octahedral cell coordinates (at resolution 8) of d and optionally -d, bit-identical to
 * min(int32(sphereToSquare(d) * 8), ...) before the per-level clamp */
PSTF_HD void octa_f8(double dx, double dy, double dz, int want_neg, DirF8 *pos, DirF8 *neg) {
    int nx = 0;
    octa_f8_try(dx, dy, dz, want_neg, pos, neg, &nx);
    if (nx) octa_f8_exact(dx, dy, dz, want_neg, pos, neg);
}

/* dirCell at a level from floor(U*8): min(floor(U*d), d-1) (field.cpp:93-95) */
PSTF_HD int32_t dir_cell_f8(int32_t f8, int level) {
    const int sh = level < 2 ? level : 2;
    const int32_t d = 8 >> sh;
    const int32_t c = f8 >> sh;
    const int32_t r = c < d - 1 ? c : d - 1;
    return f8 == INT32_MIN ? INT32_MIN : r; /* NaN direction (select, no branch) */
}

} // namespace pstf_b200
