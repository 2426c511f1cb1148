"""Seeded input generators shared by the oracle pin tests and the GPU parity tests."""
import math

import numpy as np

DIAMETER_CORNELL = math.sqrt(12.0)
BASE_CORNELL = DIAMETER_CORNELL / 256.0  # estimators.cpp:313, baseCellFraction 1/256


def structured_dirs():
    """Directions that sit exactly on octahedral bin boundaries or hit special cases."""
    s = 1.0 / math.sqrt(2.0)
    t = 1.0 / math.sqrt(3.0)
    out = []
    for x in (-1.0, -0.0, 0.0, 1.0):
        for y in (-1.0, -0.0, 0.0, 1.0):
            for z in (-1.0, -0.0, 0.0, 1.0):
                out.append((x, y, z))
    for a in (s, -s):
        for b in (s, -s):
            out += [(a, b, 0.0), (a, 0.0, b), (0.0, a, b), (a, b, -0.0)]
    for a in (t, -t):
        for b in (t, -t):
            for c in (t, -t):
                out.append((a, b, c))
    # half-angle style directions (phi = 1/2, r = 1/2 ...)
    for (x, y, z) in [(0.5, 0.5, math.sqrt(0.5)), (0.6, 0.8, 0.0), (0.8, 0.6, 0.0),
                      (0.28, 0.96, 0.0), (1e-300, 1.0, 0.0), (1.0, 1e-300, 0.0),
                      (5e-324, 5e-324, 1.0), (1e-17, 1e-17, -1.0)]:
        out += [(x, y, z), (-x, y, -z), (x, -y, z), (-x, -y, -z)]
    # octahedral bin boundaries: uv.x * d integral for d = 8 (v = k/8 in the upper hemisphere)
    for k in range(0, 9):
        phi = k / 8.0
        ang = phi * math.pi / 2
        for z in (0.0, 0.25, 0.5, 0.75):
            r = math.sqrt(1 - z * z)
            out.append((r * math.cos(ang), r * math.sin(ang), z))
            out.append((r * math.cos(ang), r * math.sin(ang), -z))
    return np.array(out, dtype=np.float64)


def special_dirs():
    nan, inf = float("nan"), float("inf")
    return np.array([(nan, 0, 1), (0, nan, 1), (0, 0, nan), (inf, 0, 0), (inf, inf, 0),
                     (-inf, 1, 0), (0, 0, 0), (2.0, 0.0, 0.0), (0.0, 0.0, 2.0), (3, 4, 12)],
                    dtype=np.float64)


def special_dirs_extra():
    """one non-finite component next to finite in-range ones (x NaN with y finite, ...): the
    fast octahedral path must hand them to the exact one (not in the golden fixtures)"""
    nan, inf = float("nan"), float("inf")
    return np.array([(nan, 0.5, 0.5), (nan, -0.6, -0.8), (0.6, nan, 0.8), (-0.6, nan, -0.8),
                     (0.3, 0.4, nan), (-inf, 0.5, 0.5), (0.5, -inf, 0.5), (1e-40, 0.6, 0.8),
                     (0.6, 1e-320, -0.8), (1e35, 1.0, 0.0), (nan, nan, 0.5)], dtype=np.float64)


def random_dirs(rng, n):
    v = rng.normal(size=(n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return v


def random_positions(rng, n, scale=3.0):
    p = rng.uniform(-scale, scale, size=(n, 3))
    # a slice exactly on cell boundaries
    m = n // 8
    p[:m] = np.round(p[:m] * 8.0) / 8.0
    return p


def special_positions():
    nan, inf = float("nan"), float("inf")
    return np.array([(0.0, -0.0, 1e-300), (nan, 0, 0), (inf, 0, 0), (-inf, 1, 1), (1e12, 0, 0),
                     (-1e12, 0, 0), (2.0 ** 31 * 0.5, 0, 0), (-(2.0 ** 31) * 0.5, 0, 0)],
                    dtype=np.float64)


def level_footprints(base, k=4.0, max_exp=8):
    """Footprints whose scaled value (fp*k/base) straddles powers of two by a few ulps."""
    out = [0.0, -0.0, -1.0, float("nan"), float("inf"), -float("inf"), 1e-300, 5e-324, 1e300,
           base / k, base / k * (1 + 2 ** -52), base / k * (1 - 2 ** -53)]
    for e in range(-2, max_exp + 1):
        target = 2.0 ** e
        fp = target * base / k
        x = fp
        for _ in range(70):
            out.append(x)
            x = np.nextafter(x, 0.0)
        x = fp
        for _ in range(70):
            out.append(x)
            x = np.nextafter(x, np.inf)
    return np.array(out, dtype=np.float64)


def random_footprints(rng, n, base):
    return base * np.exp(rng.uniform(-4, 8, size=n))


def boundary_dirs(rng, n):
    """Directions whose octahedral coordinates sit within a few ulps of directional-cell
    boundaries (phi = k/8 rays, perturbed by 0..4 ulps per component)."""
    k = rng.integers(0, 9, size=n)
    z = rng.choice([0.0, 0.0, 0.5, 0.25, 0.75, 1.0 / 3.0], size=n) * rng.choice([-1, 1], size=n)
    s = np.sqrt(1 - z * z)
    ang = k / 8.0 * (np.pi / 2)
    x = np.cos(ang) * s
    y = np.sin(ang) * s
    for _ in range(4):
        step = rng.integers(-1, 2, size=n)
        x = np.where(step > 0, np.nextafter(x, np.inf), np.where(step < 0, np.nextafter(x, -np.inf), x))
        step = rng.integers(-1, 2, size=n)
        y = np.where(step > 0, np.nextafter(y, np.inf), np.where(step < 0, np.nextafter(y, -np.inf), y))
    sx = rng.choice([-1.0, 1.0], size=n)
    sy = rng.choice([-1.0, 1.0], size=n)
    return np.stack([x * sx, y * sy, z], axis=1)
