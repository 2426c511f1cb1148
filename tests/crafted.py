"""Crafted (adversarial) vertex streams for the fused vertex-pass parity tests.

The synthetic Cornell generator (csrc/pstf_synth.h) always sets contExtended and nextIsSurface
together and produces finite, well-conditioned values, so on its own it never reaches several
branches of FieldRecorder::onVertex (estimators.cpp:194-262) inside the fused kernels.  A
crafted stream starts from a synthetic frame and overwrites a seeded random subset of the
vertices with inputs that do:
  * flags: all eight {contExtended, nextIsSurface, nee.sampled} combinations, including the
    environment escape `contExtended && !nextIsSurface` (estimators.cpp:207-210);
  * value components NaN / +-inf / negative / -0.0 / denormal (rejected accumulates,
    field.cpp:160-163; the accepted ones must be folded like the reference);
  * transportRatio() <= 0, NaN or infinite on continued vertices (estimators.cpp:214, 227);
  * positions on and within an ulp of cell boundaries at every level, -0.0, and huge, infinite
    or NaN coordinates (int32 truncation edges);
  * directions on and near octahedral cell boundaries, axis-aligned, -0.0 components,
    unnormalised, NaN / infinite (mappings.h:33-51);
  * footprints straddling every level threshold by a few ulps, 0, negative, NaN, inf.
Everything is numpy-seeded, so the GPU and the reference replay see identical bytes."""
import numpy as np

import inputs

# canonical SoA field indices (csrc/pstf_synth.h PS_*)
POS, WO, WI, NPOS, NDIR, FP, NFP, RATIO, NMIS, EMIS, F, NEMIS, NEELOE, NEEFLI = (
    0, 3, 6, 9, 12, 15, 16, 17, 18, 19, 22, 25, 28, 31)
NF64 = 34

NAN, INF = float("nan"), float("inf")
# with extreme=False (ATOMIC parity: per-vertex aggregation reassociates the sums) the accepted
# values stay moderate so reassociation cannot overflow or cancel catastrophically
VALUES_EXTREME = np.array([NAN, INF, -INF, -1.5, -0.0, 0.0, 5e-324, 1e-300, 1e308, 3.25, -2e5])
VALUES_MODERATE = np.array([NAN, INF, -INF, -0.75, -0.0, 0.0, 5e-324, 1e-300, 0.5, 3.25])
RATIOS = np.array([0.0, -0.0, -0.5, NAN, -INF, INF, 5e-324, 0.25, 2.0])


def views(buf, n):
    return buf[:NF64 * n].reshape(NF64, n), buf[NF64 * n:].view(np.uint32)[:n]


def _boundary_positions(rng, m, base, max_level):
    """coordinates exactly on / one or two ulps around cell boundaries k * base * 2^l"""
    lvl = rng.integers(0, max_level + 1, size=m)
    k = rng.integers(-300, 300, size=m).astype(np.float64)
    x = k * (base * np.exp2(lvl))
    for _ in range(2):
        step = rng.integers(-1, 2, size=m)
        x = np.where(step > 0, np.nextafter(x, INF), np.where(step < 0, np.nextafter(x, -INF), x))
    return x


def _pick_dirs(rng, m):
    pool = np.concatenate([inputs.structured_dirs(), inputs.special_dirs(),
                           inputs.special_dirs_extra(), inputs.special_dirs_extra(),
                           inputs.boundary_dirs(rng, 256), inputs.random_dirs(rng, 64),
                           -inputs.boundary_dirs(rng, 64)])
    return pool[rng.integers(0, len(pool), size=m)]


def mutate(buf, n, seed, base, frac=0.3, extreme=False, max_level=4):
    """In place: overwrite about `frac` of the vertices of a contiguous SoA buffer (synthetic or
    captured) with the adversarial inputs listed in the module docstring."""
    rng = np.random.default_rng(seed)
    f, flags = views(buf, n)
    vals = VALUES_EXTREME if extreme else VALUES_MODERATE

    def sub(p):
        return np.nonzero(rng.random(n) < frac * p)[0]

    i = sub(0.5)  # flags: all eight combinations
    flags[i] = rng.integers(0, 8, size=len(i)).astype(np.uint32)
    for fld in (EMIS, F, NEMIS, NEELOE, NEEFLI):  # value components
        for c in range(3):
            i = sub(0.08)
            f[fld + c, i] = vals[rng.integers(0, len(vals), size=len(i))]
    i = sub(0.08)
    f[NMIS, i] = vals[rng.integers(0, len(vals), size=len(i))]
    i = sub(0.3)  # transport ratio
    f[RATIO, i] = RATIOS[rng.integers(0, len(RATIOS), size=len(i))]
    for fld in (POS, NPOS):  # positions
        for c in range(3):
            i = sub(0.25)
            f[fld + c, i] = _boundary_positions(rng, len(i), base, max_level)
            i = sub(0.02)
            f[fld + c, i] = rng.choice([-0.0, 0.0, NAN, INF, -INF, 1e12, -1e12, 2.0 ** 40],
                                       size=len(i))
    for fld in (WO, WI, NDIR):  # directions
        i = sub(0.25)
        f[fld:fld + 3, i] = _pick_dirs(rng, len(i)).T
    fps = inputs.level_footprints(base)
    for fld in (FP, NFP):  # footprints around every level threshold
        i = sub(0.4)
        f[fld, i] = fps[rng.integers(0, len(fps), size=len(i))]
    return buf


def pad_even(buf, n):
    """Copy of a contiguous SoA buffer whose field stride is n rounded up to even, so every
    field starts 16 B aligned (the fused kernel's TMA tile path requires it); returns
    (padded buffer, stride)"""
    m = n + (n & 1)
    f, flags = views(buf, n)
    out = np.zeros(NF64 * m + (m + 1) // 2, np.float64)
    fo = out[:NF64 * m].reshape(NF64, m)
    fo[:, :n] = f
    out[NF64 * m:].view(np.uint32)[:n] = flags
    return out, m
