"""CV-profile / guiding model store on the B200.

Python mirror of the reference's ``ModelStore`` (estimators.h:124-150, estimators.cpp:104-144)
with ``DirGrid`` (models.h:30-52, models.cpp:16-94), ``SphericalKdTree`` (models.h:59-109,
models.cpp:96-298) or ``Gmm`` models (models.h:113-177, models.cpp:427-702) over the C ABI
(``pstf_model_*`` in include/pstf_field.h).  Keys are the field's SpatioDirectionalKeys;
records are applied in the reference's deterministic order, so entries, weights and
accumulators are bitwise those of ``EstimatorRun`` in deterministic mode."""
from __future__ import annotations

import ctypes as C

import numpy as np

from .field import MODE_ATOMIC, MODE_ORDERED, PstfError, _check, _ptr, _soa3, _stream, _torch, _vec3, lib

MODEL_ENTRY_DTYPE = np.dtype([("level", "<i4"), ("cell", "<i4", (3,)), ("dir", "<i4", (2,)),
                              ("warm", "<u4"), ("c_old", "<f8"), ("c_new", "<f8"),
                              ("records", "<u8"), ("record_count", "<u8"), ("total", "<f8")],
                             align=True)
assert MODEL_ENTRY_DTYPE.itemsize == 72


MODEL_GRID, MODEL_KDTREE, MODEL_GMM = 0, 1, 2  # ModelKind (models.h:183)


class _ModelConfig(C.Structure):
    _fields_ = [("kind", C.c_int32), ("grid_resolution", C.c_int32),
                ("kd_leaf_count", C.c_int32), ("kd_split_threshold", C.c_double),
                ("gmm_components", C.c_int32), ("gmm_alpha_em", C.c_double),
                ("gmm_sigma_min_sq", C.c_double), ("gmm_sigma_max_sq", C.c_double),
                ("gmm_reseed_fraction", C.c_double),
                ("t_max", C.c_double), ("min_samples", C.c_int32), ("capacity_log2", C.c_uint32)]


class _ModelStats(C.Structure):
    _fields_ = [("entries", C.c_uint64), ("warm", C.c_uint64), ("dropped_records", C.c_uint64),
                ("capacity", C.c_uint64)]


class ModelStore:
    """ModelStore(ModelConfig{Grid, resolution}, tMax, minSamples) on cuda:device.

    Defaults are the CV-profile store of EstimatorRun (estimators.cpp:336-339 with
    estimators.h:32,56-57); capacity_log2 sizes the device table (the reference map grows)."""

    def __init__(self, grid_resolution=16, t_max=64.0, min_samples=32, capacity_log2=16,
                 device=0, kind=MODEL_GRID, kd_leaf_count=64, kd_split_threshold=4.0,
                 gmm_components=4, gmm_alpha_em=0.7, gmm_sigma_min_sq=2.5e-5,
                 gmm_sigma_max_sq=0.04, gmm_reseed_fraction=1e-4):
        self.kind = kind
        self.res = int(grid_resolution)
        self.r2 = (2 * kd_leaf_count - 1 if kind == MODEL_KDTREE else
                   21 * gmm_components + 3 if kind == MODEL_GMM else self.res * self.res)
        self.device = device
        self._h = C.c_void_p()
        cfg = _ModelConfig(int(kind), self.res, int(kd_leaf_count), float(kd_split_threshold),
                           int(gmm_components), float(gmm_alpha_em), float(gmm_sigma_min_sq),
                           float(gmm_sigma_max_sq), float(gmm_reseed_fraction),
                           float(t_max), int(min_samples), int(capacity_log2))
        _check(lib().pstf_model_create(C.byref(cfg), device, C.byref(self._h)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().pstf_model_destroy(h)
            except Exception:
                pass
            self._h = None

    def _dev(self):
        return _torch().device("cuda", self.device)

    def _f64(self, x):
        t = _torch()
        return t.as_tensor(x).to(device=self._dev(), dtype=t.float64).contiguous()

    def _keys(self, keys):
        """(n, 7) int32 key tensor (FieldStore.key_for_batch) or a KEY_DTYPE array"""
        t = _torch()
        if isinstance(keys, np.ndarray) and keys.dtype.names:
            keys = np.ascontiguousarray(keys).view(np.int32).reshape(-1, 7)
        return t.as_tensor(keys).to(device=self._dev(), dtype=t.int32).contiguous()

    def apply(self, keys, u, v, contribution, mode=MODE_ORDERED):
        """applyRecord for every record (estimators.cpp:109-117).  MODE_ORDERED: the
        deterministic order, bitwise; MODE_ATOMIC: no sort, sums within 1e-12 relative."""
        k = self._keys(keys)
        uu, vv, cc = self._f64(u), self._f64(v), self._f64(contribution)
        n = k.shape[0]
        if not (uu.numel() == vv.numel() == cc.numel() == n):
            raise PstfError("apply: keys, u, v and contribution must have one entry per record")
        _check(lib().pstf_model_apply(self._h, _ptr(k), _ptr(uu), _ptr(vv), _ptr(cc), n, mode,
                                      _stream()))

    def end_frame(self):
        _check(lib().pstf_model_end_frame(self._h, _stream()))

    endFrame = end_frame

    def lookup_warm(self, keys):
        """lookupWarm (estimators.cpp:104-107) -> int32 entry per key, -1 when cold/absent"""
        t = _torch()
        k = self._keys(keys)
        out = t.empty(k.shape[0], dtype=t.int32, device=self._dev())
        _check(lib().pstf_model_lookup_warm(self._h, _ptr(k), k.shape[0], _ptr(out), _stream()))
        return out

    def lookup_warm_levels(self, keyer, pos, direction, footprint):
        """the estimator's coarse-to-fine model search (estimators.cpp:464-469) with the keyer
        FieldStore's quantisation"""
        t = _torch()
        p, d = _soa3(pos, self._dev()), _soa3(direction, self._dev())
        fp = self._f64(footprint)
        n = fp.numel()
        out = t.empty(n, dtype=t.int32, device=self._dev())
        pv, dv = _vec3(p), _vec3(d)
        _check(lib().pstf_model_lookup_warm_levels(self._h, keyer.handle, C.byref(pv),
                                                   C.byref(dv), _ptr(fp), n, _ptr(out),
                                                   _stream()))
        return out

    def pdf(self, entry, u, v):
        """DirGrid::pdf (models.cpp:52-56); entry -1 -> 1.0"""
        t = _torch()
        e = t.as_tensor(entry).to(device=self._dev(), dtype=t.int32).contiguous()
        uu, vv = self._f64(u), self._f64(v)
        out = t.empty(e.numel(), dtype=t.float64, device=self._dev())
        _check(lib().pstf_model_pdf(self._h, _ptr(e), _ptr(uu), _ptr(vv), e.numel(), _ptr(out),
                                    _stream()))
        return out

    def sample(self, entry, u1, u2, u_select=None):
        """DirGrid / SphericalKdTree::sample(u), Gmm::sample(u_select, u) (models.cpp:58-92,
        176-200, 664-687) -> (u, v, pdf); entry -1 -> (u1, u2, 1.0)"""
        t = _torch()
        e = t.as_tensor(entry).to(device=self._dev(), dtype=t.int32).contiguous()
        a, b = self._f64(u1), self._f64(u2)
        us = None if u_select is None else self._f64(u_select)
        n = e.numel()
        su, sv, pdf = (t.empty(n, dtype=t.float64, device=self._dev()) for _ in range(3))
        _check(lib().pstf_model_sample(self._h, _ptr(e), _ptr(a), _ptr(b), _ptr(us), n, _ptr(su),
                                       _ptr(sv), _ptr(pdf), _stream()))
        return su, sv, pdf

    def stats(self) -> dict:
        s = _ModelStats()
        _check(lib().pstf_model_get_stats(self._h, C.byref(s)))
        return {f: int(getattr(s, f)) for f, _ in _ModelStats._fields_}

    def size(self) -> int:
        return self.stats()["entries"]

    def dump(self):
        """(entries sorted by key as MODEL_ENTRY_DTYPE, weights (n, R^2), accumulators (n, R^2))"""
        cnt = C.c_uint64()
        _check(lib().pstf_model_dump(self._h, None, None, None, 0, C.byref(cnt)))
        n = cnt.value
        e = np.zeros(max(n, 1), MODEL_ENTRY_DTYPE)
        w, a = np.zeros((max(n, 1), self.r2)), np.zeros((max(n, 1), self.r2))
        _check(lib().pstf_model_dump(self._h, e.ctypes.data_as(C.c_void_p),
                                     w.ctypes.data_as(C.c_void_p), a.ctypes.data_as(C.c_void_p),
                                     n, C.byref(cnt)))
        return e[:n], w[:n], a[:n]

    def dump_tree(self):
        """k-d tree topology in dump() order: (n, 2L-1, 5) int32 {leaf, axis, left, right,
        parent} and (n, 2L-1, 2) float64 {split, mass}"""
        cnt = C.c_uint64()
        _check(lib().pstf_model_dump(self._h, None, None, None, 0, C.byref(cnt)))
        n = cnt.value
        ti = np.zeros((max(n, 1), self.r2, 5), np.int32)
        tf = np.zeros((max(n, 1), self.r2, 2))
        _check(lib().pstf_model_dump_tree(self._h, ti.ctypes.data_as(C.c_void_p),
                                          tf.ctypes.data_as(C.c_void_p), n, C.byref(cnt)))
        return ti[:n], tf[:n]

