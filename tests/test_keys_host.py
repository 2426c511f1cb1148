"""CPU differential test of the product's key math header (pstf_keys.cuh, host-compiled via
tests/native/keys_host.cpp) against the UNMODIFIED reference keyFor/selectLevel (oracle/_ref)
and the C restatement: 0 mismatches required on random, structured, special and
boundary-hugging inputs.  The GPU parity tests repeat this on the device."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import inputs
import pyoracle as po

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "native", "keys_host.cpp")
SO = os.path.join(HERE, "native", "libkeys_host.so")


@pytest.fixture(scope="module")
def kh():
    hdr = os.path.join(HERE, "..", "paper_2005_07547_b200", "csrc", "pstf_keys.cuh")
    if not os.path.exists(SO) or os.path.getmtime(SO) < max(os.path.getmtime(SRC),
                                                            os.path.getmtime(hdr)):
        subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                        "-o", SO, SRC], check=True)
    return C.CDLL(SO)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _keys(kh, cfg, pos, d, lv):
    n = len(lv)
    out = np.zeros(n, po.KEY_DTYPE)
    pT, dT = np.ascontiguousarray(pos.T), np.ascontiguousarray(d.T)
    lv = np.ascontiguousarray(lv, np.int32)
    kh.kh_key_for_batch(C.c_double(cfg.base_cell_size), C.c_double(cfg.level_select_k),
                        C.c_int(cfg.max_level), _p(pT), _p(dT), _p(lv), C.c_int64(n), _p(out))
    return out


def _mismatch(a, b):
    bad = np.zeros(len(a), bool)
    for f in ("level", "cell", "dir", "checksum"):
        bad |= (a[f] != b[f]).reshape(len(a), -1).any(1)
    return bad


def _checker(cfg):
    return po.RefStore(cfg) if po.ref_available() else po.OracleStore(cfg)


@pytest.mark.parametrize("base", [0.5, inputs.BASE_CORNELL, 0.01])
def test_keys_match_reference(kh, base):
    cfg = po.Config.make(capacity_log2=10, base_cell_size=base)
    ref = _checker(cfg)
    rng = np.random.default_rng(int(base * 1e6))
    d = np.concatenate([inputs.random_dirs(rng, 100000), inputs.boundary_dirs(rng, 100000),
                        inputs.structured_dirs(), inputs.special_dirs(),
                        inputs.special_dirs_extra()])
    n = len(d)
    pos = np.concatenate([inputs.random_positions(rng, n - 8), inputs.special_positions()])
    for level in range(cfg.max_level + 1):
        lv = np.full(n, level, np.int32)
        bad = _mismatch(_keys(kh, cfg, pos, d, lv), ref.keys_for(pos, d, lv))
        assert bad.sum() == 0, (level, np.nonzero(bad)[0][:10])


@pytest.mark.parametrize("max_level", [4, 60])
def test_select_level_matches_reference(kh, max_level):
    cfg = po.Config.make(capacity_log2=10, base_cell_size=inputs.BASE_CORNELL, max_level=max_level)
    ref = _checker(cfg)
    rng = np.random.default_rng(max_level)
    fp = np.concatenate([inputs.level_footprints(cfg.base_cell_size, max_exp=max_level + 2),
                         inputs.random_footprints(rng, 200000, cfg.base_cell_size)])
    out = np.zeros(len(fp), np.int32)
    kh.kh_select_level_batch(C.c_double(cfg.base_cell_size), C.c_double(4.0), C.c_int(max_level),
                             _p(fp), C.c_int64(len(fp)), _p(out))
    np.testing.assert_array_equal(out, ref.select_levels(fp))


def test_atan2_slow_path_is_correctly_rounded(kh):
    import mpmath as mp
    mp.mp.prec = 200
    rng = np.random.default_rng(3)
    y = np.abs(rng.normal(size=3000))
    x = np.abs(rng.normal(size=3000))
    y[:100] = x[:100] * np.nextafter(1.0, 2.0)
    out = np.zeros(len(y))
    kh.kh_atan2_cr_batch(_p(y), _p(x), C.c_int64(len(y)), _p(out))
    exact = np.array([float(mp.atan2(mp.mpf(a), mp.mpf(b))) for a, b in zip(y, x)])
    np.testing.assert_array_equal(out, exact)


@pytest.mark.parametrize("negate", [0, 1])
@pytest.mark.parametrize("base", [0.5, inputs.BASE_CORNELL, 1e-300, 1e300])
def test_shared_quantisation_identities(kh, negate, base):
    """The fast kernel's shared per-vertex quantisation (one division per coordinate for all
    levels; one atan2 for d and -d) gives exactly the reference keyFor keys."""
    cfg = po.Config.make(capacity_log2=10, base_cell_size=base, max_level=6)
    ref = _checker(cfg)
    rng = np.random.default_rng(77 + negate)
    d = np.concatenate([inputs.random_dirs(rng, 40000), inputs.boundary_dirs(rng, 40000),
                        inputs.structured_dirs(), inputs.special_dirs(),
                        inputs.special_dirs_extra()])
    n = len(d)
    pos = np.concatenate([inputs.random_positions(rng, n - 8), inputs.special_positions()])
    pos[:200] *= 1e-310  # subnormal positions exercise the direct-division fallback
    # positions on (or an ulp off) cell boundaries at every level exercise the exact re-check
    k = rng.integers(-300, 300, size=(3000, 3)).astype(np.float64)
    on = k * base * np.exp2(rng.integers(0, 7, size=(3000, 1)))
    pos[200:3200] = np.where(rng.random((3000, 3)) < 0.3, np.nextafter(on, np.inf), on)
    for level in range(cfg.max_level + 1):
        lv = np.full(n, level, np.int32)
        out = np.zeros(n, po.KEY_DTYPE)
        pT, dT = np.ascontiguousarray(pos.T), np.ascontiguousarray(d.T)
        kh.kh_key_for_shared_batch(C.c_double(base), C.c_double(4.0), C.c_int(6), _p(pT), _p(dT),
                                   _p(lv), C.c_int64(n), C.c_int(negate), _p(out))
        want = ref.keys_for(pos, -d if negate else d, lv)
        bad = _mismatch(out, want)
        assert bad.sum() == 0, (level, np.nonzero(bad)[0][:10])


@pytest.mark.parametrize("max_level", [4, 60])
def test_select_level_fast_matches_reference(kh, max_level):
    """select_level_fast (reciprocal multiply + exponent, exact path near powers of two)."""
    cfg = po.Config.make(capacity_log2=10, base_cell_size=inputs.BASE_CORNELL, max_level=max_level)
    ref = _checker(cfg)
    rng = np.random.default_rng(max_level + 5)
    fp = np.concatenate([inputs.level_footprints(cfg.base_cell_size, max_exp=max_level + 2),
                         inputs.random_footprints(rng, 300000, cfg.base_cell_size)])
    out = np.zeros(len(fp), np.int32)
    kh.kh_select_level_fast_batch(C.c_double(cfg.base_cell_size), C.c_double(4.0),
                                  C.c_int(max_level), _p(fp), C.c_int64(len(fp)), _p(out))
    np.testing.assert_array_equal(out, ref.select_levels(fp))
