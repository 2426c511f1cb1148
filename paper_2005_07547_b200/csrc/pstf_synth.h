/*
 * pstf_synth.h — synthetic PSTF vertex-stream generator (test/bench input, not the hot path).
 *
 * Produces the canonical 276 B/vertex SoA record that FieldRecorder::onVertex reads
 * (reference: proj/core/src/estimators.cpp:194-262, VertexRecord pathtracer.h:59-90),
 * for SURVEY.md §8d configs 2/4/5: a closed Cornell-class box [-1,1]x[0,2]x[-1,1]
 * (walls and albedos after proj/scenes/cornell.scene:11-83), a ceiling lamp patch
 * |x|,|z| <= 0.3 emitting 12, a pinhole camera looking down -z (vertical fov 40 deg,
 * cornell.scene:3-9) placed on the open front plane z = +1 so every camera ray hits a
 * wall, exactly B vertices per path (the last one is never extended, as at max depth,
 * pathtracer.cpp:203), cosine-sampled continuations, NEE towards the lamp, footprint
 * growth as pathtracer.cpp:120,198.
 *
 * Only IEEE-exact operations (+ - * / sqrt, integer hashing, comparisons) are used,
 * so host (C99, gcc -ffp-contract=off) and device (nvcc -fmad=false) produce
 * bit-identical streams.  Vertex (path p, bounce b) is stored at index b*n_paths + p
 * (wavefront order).  Header is plain C99 so the C oracle harness can include it.
 */
#ifndef PSTF_SYNTH_H
#define PSTF_SYNTH_H

#include <stdint.h>
#include <math.h>

#if defined(__CUDACC__)
#define PS_HD static __host__ __device__ __forceinline__
#else
#define PS_HD static inline
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Field indices of the contiguous fp64 SoA layout (34 fp64 arrays of n, then u32 flags[n]). */
enum {
    PS_POS = 0, PS_WO = 3, PS_WI = 6, PS_NPOS = 9, PS_NDIR = 12,
    PS_FP = 15, PS_NFP = 16, PS_RATIO = 17, PS_NMIS = 18,
    PS_EMIS = 19, PS_F = 22, PS_NEMIS = 25, PS_NEELOE = 28, PS_NEEFLI = 31,
    PS_NUM_F64 = 34
};
#define PS_FLAG_CONT 1u  /* contExtended  */
#define PS_FLAG_NEXT_SURF 2u /* nextIsSurface */
#define PS_FLAG_NEE 4u   /* nee.sampled   */
#define PS_BYTES_PER_VERTEX (PS_NUM_F64 * 8 + 4) /* 276 */

typedef struct {
    int width, height, bounces;
    uint64_t seed;
    uint64_t iter;
    double cam_shift_x; /* config 5: camera translated along x */
    uint64_t path0;     /* image stripe: paths [path0, path0 + n_local) ... */
    uint64_t n_local;   /* ... stored at b * n_local + (p - path0); 0 = whole image */
    int glossy;         /* config 3: floor and back wall are the glossy "steps" material of
                           staircase_glossy.scene:11-16 (see ps_material) */
} ps_params;

typedef struct { double x, y, z; } ps_v3;

PS_HD uint64_t ps_mix(uint64_t v) { /* SplitMix64 finaliser (same constants as rng.h:61-68) */
    v ^= v >> 30;
    v *= 0xbf58476d1ce4e5b9ULL;
    v ^= v >> 27;
    v *= 0x94d049bb133111ebULL;
    v ^= v >> 31;
    return v;
}

PS_HD double ps_rand(uint64_t base, uint32_t bounce, uint32_t dim) {
    uint64_t h = ps_mix(base ^ (((uint64_t)bounce << 32) | (uint64_t)dim) * 0x9e3779b97f4a7c15ULL);
    return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

PS_HD ps_v3 ps_v(double x, double y, double z) { ps_v3 r; r.x = x; r.y = y; r.z = z; return r; }
PS_HD double ps_dot(ps_v3 a, ps_v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

/* wall ids: 0 x=-1 (red), 1 x=+1 (green), 2 y=0 floor, 3 y=2 ceiling, 4 z=-1 back, 5 z=+1 front */
PS_HD ps_v3 ps_wall_normal(int w) {
    switch (w) {
    case 0: return ps_v(1.0, 0.0, 0.0);
    case 1: return ps_v(-1.0, 0.0, 0.0);
    case 2: return ps_v(0.0, 1.0, 0.0);
    case 3: return ps_v(0.0, -1.0, 0.0);
    case 4: return ps_v(0.0, 0.0, 1.0);
    default: return ps_v(0.0, 0.0, -1.0);
    }
}

PS_HD ps_v3 ps_albedo(int w) {
    if (w == 0) return ps_v(0.63, 0.065, 0.05);
    if (w == 1) return ps_v(0.14, 0.45, 0.091);
    return ps_v(0.73, 0.73, 0.73);
}

PS_HD int ps_is_lamp(int w, ps_v3 p) {
    return w == 3 && p.x >= -0.3 && p.x <= 0.3 && p.z >= -0.3 && p.z <= 0.3;
}

/* Closest wall hit from a point inside the box. Returns t, sets wall id and snaps the hit
 * coordinate onto the wall plane. */
PS_HD double ps_intersect(ps_v3 o, ps_v3 d, int *wall, ps_v3 *hit) {
    double t = 1e300;
    int w = -1;
    if (d.x < 0.0) { double tt = (-1.0 - o.x) / d.x; if (tt < t) { t = tt; w = 0; } }
    if (d.x > 0.0) { double tt = (1.0 - o.x) / d.x; if (tt < t) { t = tt; w = 1; } }
    if (d.y < 0.0) { double tt = (0.0 - o.y) / d.y; if (tt < t) { t = tt; w = 2; } }
    if (d.y > 0.0) { double tt = (2.0 - o.y) / d.y; if (tt < t) { t = tt; w = 3; } }
    if (d.z < 0.0) { double tt = (-1.0 - o.z) / d.z; if (tt < t) { t = tt; w = 4; } }
    if (d.z > 0.0) { double tt = (1.0 - o.z) / d.z; if (tt < t) { t = tt; w = 5; } }
    ps_v3 p = ps_v(o.x + d.x * t, o.y + d.y * t, o.z + d.z * t);
    /* snap + clamp to the box so rounding never leaves the walls */
    p.x = p.x < -1.0 ? -1.0 : (p.x > 1.0 ? 1.0 : p.x);
    p.y = p.y < 0.0 ? 0.0 : (p.y > 2.0 ? 2.0 : p.y);
    p.z = p.z < -1.0 ? -1.0 : (p.z > 1.0 ? 1.0 : p.z);
    if (w == 0) p.x = -1.0;
    if (w == 1) p.x = 1.0;
    if (w == 2) p.y = 0.0;
    if (w == 3) p.y = 2.0;
    if (w == 4) p.z = -1.0;
    if (w == 5) p.z = 1.0;
    *wall = w;
    *hit = p;
    return t;
}

/* local (a, b, c) with c along the wall normal -> world, exact +-1 frames */
PS_HD ps_v3 ps_to_world(int w, double a, double b, double c) {
    switch (w) {
    case 0: return ps_v(c, a, b);
    case 1: return ps_v(-c, a, b);
    case 2: return ps_v(a, c, b);
    case 3: return ps_v(a, -c, b);
    case 4: return ps_v(a, b, c);
    default: return ps_v(a, b, -c);
    }
}

#define PS_INV_PI 0.3183098861837907
#define PS_PI 3.141592653589793
#define PS_TAN_HALF_FOV 0.36397023426620234 /* tan(20 deg) */
#define PS_LAMP_EMISSION 12.0
#define PS_LAMP_PDF_AREA (1.0 / 0.36)

/* ---- glossy mode (BASELINE config 3): the materials of staircase_glossy.scene:11-22 ----
 * floor (wall 2) and back wall (4) are "steps": diffuse 0.2/0.18/0.15 + a Phong lobe of albedo
 * 0.6, exponent 48 around the mirror direction; the other walls are "wall" (diffuse 0.6).
 * BSDF value, pdf and lobe choice follow scene.cpp:326-389 (evalBsdf, pdfBsdf, sampleBsdf) with
 * IEEE-exact operations only: cos^48 by repeated squaring, and the power-cosine lobe sampled as
 * the maximum of 49 uniforms (P(max <= x) = x^49, exactly samplePowerCosine's distribution for
 * exponent 48) with a rejection-sampled azimuth. */
#define PS_GLOSSY_E 48.0

PS_HD int ps_is_steps(const ps_params *P, int w) { return P->glossy && (w == 2 || w == 4); }

PS_HD ps_v3 ps_diffuse_albedo(const ps_params *P, int w) {
    if (!P->glossy) return ps_albedo(w);
    if (ps_is_steps(P, w)) return ps_v(0.2, 0.18, 0.15);
    return ps_v(0.6, 0.6, 0.6);
}

PS_HD double ps_pow48(double c) { /* c^48 = c^32 c^16, one fixed product sequence */
    double c2 = c * c, c4 = c2 * c2, c8 = c4 * c4, c16 = c8 * c8, c32 = c16 * c16;
    return c32 * c16;
}

PS_HD ps_v3 ps_reflect(ps_v3 wo, ps_v3 n) { /* mirror of wo about n (vecmath reflect) */
    double k = 2.0 * ps_dot(wo, n);
    return ps_v(n.x * k - wo.x, n.y * k - wo.y, n.z * k - wo.z);
}

/* evalBsdf (scene.cpp:342-356) of a steps/wall vertex; lambertian Cornell walls otherwise */
PS_HD ps_v3 ps_eval_bsdf(const ps_params *P, int w, ps_v3 wi, ps_v3 wo, ps_v3 n) {
    double cosI = ps_dot(wi, n), cosO = ps_dot(wo, n);
    if (cosI <= 0.0 || cosO <= 0.0) return ps_v(0.0, 0.0, 0.0);
    ps_v3 a = ps_diffuse_albedo(P, w);
    ps_v3 f = ps_v(a.x * PS_INV_PI, a.y * PS_INV_PI, a.z * PS_INV_PI);
    if (ps_is_steps(P, w)) {
        double cosA = ps_dot(wi, ps_reflect(wo, n));
        if (cosA > 0.0) {
            double g = 0.6 * ((PS_GLOSSY_E + 2.0) * PS_INV_PI * 0.5 * ps_pow48(cosA));
            f = ps_v(f.x + g, f.y + g, f.z + g);
        }
    }
    return f;
}

PS_HD double ps_q_diffuse(const ps_params *P, int w) { /* lobeProbs (scene.cpp:331-338) */
    if (!ps_is_steps(P, w)) return 1.0;
    double ld = 0.2126 * 0.2 + 0.7152 * 0.18 + 0.0722 * 0.15, lg = 0.6;
    return ld / (ld + lg);
}

/* pdfBsdf (scene.cpp:358-368), per steradian */
PS_HD double ps_pdf_bsdf(const ps_params *P, int w, ps_v3 wi, ps_v3 wo, ps_v3 n) {
    if (ps_dot(wo, n) <= 0.0) return 0.0;
    double qd = ps_q_diffuse(P, w);
    double cosI = ps_dot(wi, n);
    double pdf = qd * (cosI > 0.0 ? cosI * PS_INV_PI : 0.0);
    if (qd < 1.0) {
        double cosA = ps_dot(wi, ps_reflect(wo, n));
        pdf += (1.0 - qd) * (cosA > 0.0 ? (PS_GLOSSY_E + 1.0) * (0.5 * PS_INV_PI) * ps_pow48(cosA) : 0.0);
    }
    return pdf;
}

/* an orthonormal frame around m (|m| = 1) with exact operations (buildFrame-like) */
PS_HD void ps_frame(ps_v3 m, ps_v3 *t, ps_v3 *b) {
    double sign = m.z >= 0.0 ? 1.0 : -1.0;
    double a = -1.0 / (sign + m.z);
    double bb = m.x * m.y * a;
    *t = ps_v(1.0 + sign * m.x * m.x * a, sign * bb, -sign * m.x);
    *b = ps_v(bb, sign + m.y * m.y * a, -m.y);
}

/* Writes the B vertices of one path into a contiguous SoA buffer of n_total vertices. */
PS_HD void ps_gen_path(const ps_params *P, uint64_t path, double *f64, uint32_t *flags,
                       uint64_t n_total) {
    const uint64_t n_paths = P->n_local ? P->n_local : (uint64_t)P->width * (uint64_t)P->height;
    const uint64_t lpath = P->n_local ? path - P->path0 : path;
    const uint64_t base = ps_mix(ps_mix(P->seed ^ (P->iter * 0xd1b54a32d192ed03ULL)) ^ path);
    const int px = (int)(path % (uint64_t)P->width);
    const int py = (int)(path / (uint64_t)P->width);
    const double pxAngle = 2.0 * PS_TAN_HALF_FOV / (double)P->height;
    const double aspect = (double)P->width / (double)P->height;

    double jx = ps_rand(base, 0, 100), jy = ps_rand(base, 0, 101);
    double ndcX = (((double)px + jx) / (double)P->width) * 2.0 - 1.0;
    double ndcY = 1.0 - (((double)py + jy) / (double)P->height) * 2.0;
    ps_v3 d = ps_v(ndcX * PS_TAN_HALF_FOV * aspect, ndcY * PS_TAN_HALF_FOV, -1.0);
    double len = sqrt(ps_dot(d, d));
    d = ps_v(d.x / len, d.y / len, d.z / len);
    ps_v3 o = ps_v(P->cam_shift_x, 1.0, 1.0);
    if (o.x > 0.999) o.x = 0.999;
    if (o.x < -0.999) o.x = -0.999;

    int wall;
    ps_v3 pos;
    double t = ps_intersect(o, d, &wall, &pos);
    double spread = pxAngle;
    double footprint = t * spread;
    double emis = ps_is_lamp(wall, pos) ? PS_LAMP_EMISSION : 0.0;

    for (int b = 0; b < P->bounces; ++b) {
        const uint64_t vi = (uint64_t)b * n_paths + lpath;
        ps_v3 n = ps_wall_normal(wall);
        ps_v3 alb = ps_diffuse_albedo(P, wall);
        ps_v3 wo = ps_v(-d.x, -d.y, -d.z);
        double cosO = ps_dot(wo, n);
        uint32_t fl = 0;

        /* ---- NEE towards the lamp (pathtracer.cpp:20-70 shape) ---- */
        double lx = -0.3 + 0.6 * ps_rand(base, (uint32_t)b, 0);
        double lz = -0.3 + 0.6 * ps_rand(base, (uint32_t)b, 1);
        ps_v3 toL = ps_v(lx - pos.x, 2.0 - pos.y, lz - pos.z);
        double distSq = ps_dot(toL, toL);
        ps_v3 ndir = ps_v(0.0, 0.0, 0.0);
        double neeLoe[3] = {0.0, 0.0, 0.0}, neeFli[3] = {0.0, 0.0, 0.0};
        if (distSq > 1e-12) {
            double dist = sqrt(distSq);
            ps_v3 dl = ps_v(toL.x / dist, toL.y / dist, toL.z / dist);
            double cosLight = dl.y;
            if (cosLight > 1e-9) {
                fl |= PS_FLAG_NEE;
                ndir = dl;
                double pdfSigma = PS_LAMP_PDF_AREA * distSq / cosLight;
                double cosX = ps_dot(dl, n);
                double fr = 0.0, fg = 0.0, fb = 0.0;
                double contPdf;
                if (P->glossy) {
                    ps_v3 fv = ps_eval_bsdf(P, wall, dl, wo, n);
                    fr = fv.x; fg = fv.y; fb = fv.z;
                    contPdf = ps_pdf_bsdf(P, wall, dl, wo, n);
                } else {
                    if (cosX > 0.0 && cosO > 0.0) {
                        fr = alb.x * PS_INV_PI; fg = alb.y * PS_INV_PI; fb = alb.z * PS_INV_PI;
                    }
                    contPdf = cosX > 0.0 ? cosX * PS_INV_PI : 0.0;
                }
                double mis = pdfSigma / (pdfSigma + contPdf);
                double rr = fr * PS_LAMP_EMISSION, rg = fg * PS_LAMP_EMISSION, rb = fb * PS_LAMP_EMISSION;
                neeFli[0] = rr * mis; neeFli[1] = rg * mis; neeFli[2] = rb * mis;
                if (pdfSigma > 0.0 && cosX > 0.0) {
                    double s = cosX * mis / pdfSigma;
                    neeLoe[0] = rr * s; neeLoe[1] = rg * s; neeLoe[2] = rb * s;
                }
            }
        }

        /* ---- cosine-sampled continuation (rejection in the unit disk: IEEE-exact) ---- */
        double a = 0.0, c2 = 0.0, r2 = 1.0;
        for (uint32_t k = 0; k < 64; ++k) {
            a = 2.0 * ps_rand(base, (uint32_t)b, 2 + 2 * k) - 1.0;
            c2 = 2.0 * ps_rand(base, (uint32_t)b, 3 + 2 * k) - 1.0;
            r2 = a * a + c2 * c2;
            if (r2 < 1.0) break;
        }
        if (!(r2 < 1.0)) { a = 0.0; c2 = 0.0; r2 = 0.0; }
        double cz = sqrt(1.0 - r2);
        ps_v3 wi = ps_to_world(wall, a, c2, cz);
        double cosI, pdfSigma;
        double fcont[3] = {alb.x * PS_INV_PI, alb.y * PS_INV_PI, alb.z * PS_INV_PI};
        if (P->glossy) {
            /* sampleBsdf (scene.cpp:370-389): lobe by luminance, Phong lobe about the mirror */
            if (ps_is_steps(P, wall) && ps_rand(base, (uint32_t)b, 200) >= ps_q_diffuse(P, wall)) {
                double ct = 0.0;
                for (uint32_t k = 0; k < 49; ++k) { /* cos(theta) = max of 49 uniforms */
                    double u = ps_rand(base, (uint32_t)b, 300 + k);
                    ct = u > ct ? u : ct;
                }
                double st = sqrt(1.0 - ct * ct);
                double len = sqrt(r2);
                double cp = len > 0.0 ? a / len : 1.0, sp = len > 0.0 ? c2 / len : 0.0;
                ps_v3 m = ps_reflect(wo, n), t, bt;
                ps_frame(m, &t, &bt);
                double lx = st * cp, ly = st * sp;
                wi = ps_v(t.x * lx + bt.x * ly + m.x * ct, t.y * lx + bt.y * ly + m.y * ct,
                          t.z * lx + bt.z * ly + m.z * ct);
                if (ps_dot(wi, n) <= 0.0) { /* below the horizon: mirrored back above (the
                                               synthetic paths keep exactly B vertices) */
                    double k2 = 2.0 * ps_dot(wi, n);
                    wi = ps_v(wi.x - n.x * k2, wi.y - n.y * k2, wi.z - n.z * k2);
                }
            }
            ps_v3 fv = ps_eval_bsdf(P, wall, wi, wo, n);
            fcont[0] = fv.x; fcont[1] = fv.y; fcont[2] = fv.z;
            cosI = ps_dot(wi, n);
            pdfSigma = ps_pdf_bsdf(P, wall, wi, wo, n);
        } else {
            cosI = ps_dot(wi, n);
            pdfSigma = cosI > 0.0 ? cosI * PS_INV_PI : 0.0;
        }
        double ratio = (cosI > 0.0 && pdfSigma > 0.0) ? cosI / (pdfSigma * 1.0) : 0.0;
        double pdfProj = cosI > 0.0 ? pdfSigma / cosI : 0.0;

        double nfp = 0.0, nemis = 0.0, nmis = 1.0;
        ps_v3 npos = ps_v(0.0, 0.0, 0.0);
        int nwall = wall;
        double nspread = spread;
        if (b + 1 < P->bounces) {
            fl |= PS_FLAG_CONT | PS_FLAG_NEXT_SURF;
            double pp = pdfProj > 1e-12 ? pdfProj : 1e-12;
            double sp = 1.0 / sqrt(pp * PS_PI);
            nspread = sp > pxAngle ? sp : pxAngle;
            double tn = ps_intersect(pos, wi, &nwall, &npos);
            nfp = footprint + tn * nspread;
            if (ps_is_lamp(nwall, npos)) {
                nemis = PS_LAMP_EMISSION;
                double cosL = wi.y;
                double lpdf = cosL > 1e-12 ? PS_LAMP_PDF_AREA * (tn * tn) / cosL : 0.0;
                nmis = pdfSigma / (pdfSigma + lpdf);
            }
        }

        double *F = f64;
#define PS_ST(field, value) F[(uint64_t)(field) * n_total + vi] = (value)
        PS_ST(PS_POS + 0, pos.x); PS_ST(PS_POS + 1, pos.y); PS_ST(PS_POS + 2, pos.z);
        PS_ST(PS_WO + 0, wo.x); PS_ST(PS_WO + 1, wo.y); PS_ST(PS_WO + 2, wo.z);
        PS_ST(PS_WI + 0, wi.x); PS_ST(PS_WI + 1, wi.y); PS_ST(PS_WI + 2, wi.z);
        PS_ST(PS_NPOS + 0, npos.x); PS_ST(PS_NPOS + 1, npos.y); PS_ST(PS_NPOS + 2, npos.z);
        PS_ST(PS_NDIR + 0, ndir.x); PS_ST(PS_NDIR + 1, ndir.y); PS_ST(PS_NDIR + 2, ndir.z);
        PS_ST(PS_FP, footprint);
        PS_ST(PS_NFP, nfp);
        PS_ST(PS_RATIO, ratio);
        PS_ST(PS_NMIS, nmis);
        PS_ST(PS_EMIS + 0, emis); PS_ST(PS_EMIS + 1, emis); PS_ST(PS_EMIS + 2, emis);
        PS_ST(PS_F + 0, fcont[0]); PS_ST(PS_F + 1, fcont[1]); PS_ST(PS_F + 2, fcont[2]);
        PS_ST(PS_NEMIS + 0, nemis); PS_ST(PS_NEMIS + 1, nemis); PS_ST(PS_NEMIS + 2, nemis);
        PS_ST(PS_NEELOE + 0, neeLoe[0]); PS_ST(PS_NEELOE + 1, neeLoe[1]); PS_ST(PS_NEELOE + 2, neeLoe[2]);
        PS_ST(PS_NEEFLI + 0, neeFli[0]); PS_ST(PS_NEEFLI + 1, neeFli[1]); PS_ST(PS_NEEFLI + 2, neeFli[2]);
#undef PS_ST
        flags[vi] = fl;

        /* advance */
        pos = npos;
        wall = nwall;
        d = wi;
        footprint = nfp;
        emis = nemis;
        spread = nspread;
    }
}

#ifdef __cplusplus
}
#endif
#endif /* PSTF_SYNTH_H */
