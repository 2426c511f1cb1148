"""ctypes/torch front-end of libpstf_b200.so, mirroring pstf::FieldStore (field.h:76-138) and
pstf::FieldUpdateQueue (field.h:143-167).

Scalar calls (``increment_counter``, ``accumulate``) are staged and flushed to the GPU in
SEQUENTIAL mode before anything observes the store, which reproduces the reference's
single-threaded scalar-call semantics bit-exactly (slot placement included).  Batched calls
take torch CUDA tensors and run on the current torch stream.  torch only provides device
memory and streams here; all field-cache arithmetic runs in the sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("PSTF_LIB_PATH") or os.path.join(_HERE, "lib", "libpstf_b200.so")

KIND_LO, KIND_LO_MINUS_E, KIND_LI, KIND_FLI = 0, 1, 2, 3
TECH_CAMERA, TECH_CONTINUATION, TECH_NEE, TECH_ALL = 1, 2, 4, 7
BLEND_SQRT, BLEND_LINEAR = 0, 1
MODE_ATOMIC, MODE_ORDERED, MODE_SEQUENTIAL = 0, 1, 2
VERTEX_F64_FIELDS = 34
VERTEX_BYTES = 276

KEY_DTYPE = np.dtype([("level", "<i4"), ("cell", "<i4", (3,)), ("dir", "<i4", (2,)),
                      ("checksum", "<u4")])
SNAPSHOT_DTYPE = np.dtype([("level", "<i4"), ("cell", "<i4", (3,)), ("dir", "<i4", (2,)),
                           ("checksum", "<u4"), ("value", "<f8", (3,)), ("c_old", "<f8")],
                          align=True)
SLOT_DTYPE = np.dtype([("checksum", "<u4"), ("level", "<i4"), ("cell", "<i4", (3,)),
                       ("dir", "<i4", (2,)), ("value_old", "<f8", (3,)), ("c_old", "<f8"),
                       ("accum", "<f8", (3,)), ("c_new", "<f8"), ("last_touched", "<u4")],
                      align=True)


class PstfError(RuntimeError):
    pass


class _Config(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("capacity_log2", C.c_uint32), ("max_level", C.c_int32),
                ("base_cell_size", C.c_double), ("level_select_k", C.c_double),
                ("t_max", C.c_double), ("blend", C.c_uint32), ("technique_mask", C.c_uint32),
                ("probe_window", C.c_uint32), ("evict_age_frames", C.c_uint32)]


class _Stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("frame", "rejected", "dropped", "internal_errors",
                                          "live", "touched_last", "new_keys_last",
                                          "evicted_last", "placement_rounds_last",
                                          "touched_total", "reds_total")]


class _Vec3(C.Structure):
    _fields_ = [("x", C.c_void_p), ("y", C.c_void_p), ("z", C.c_void_p)]


class _VertexSoa(C.Structure):
    _fields_ = [("position", _Vec3), ("wo", _Vec3), ("wi", _Vec3), ("next_position", _Vec3),
                ("nee_dir", _Vec3), ("footprint", C.c_void_p), ("next_footprint", C.c_void_p),
                ("ratio", C.c_void_p), ("next_emis_mis_weight", C.c_void_p),
                ("emission_here", _Vec3), ("f", _Vec3), ("next_emission", _Vec3),
                ("nee_loe", _Vec3), ("nee_fli", _Vec3), ("flags", C.c_void_p)]


_lib = None


def library_path() -> str:
    return _LIB_PATH


def lib():
    """Loads libpstf_b200.so; raises PstfError when the CUDA library is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise PstfError(f"{_LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; "
                        f"g.build()'` (the field cache has no CPU implementation)")
    L = C.CDLL(_LIB_PATH)
    vp, u64, i32, u32, d = C.c_void_p, C.c_uint64, C.c_int, C.c_uint32, C.c_double
    sig = {
        "pstf_abi_version": ([], i32),
        "pstf_last_error": ([], C.c_char_p),
        "pstf_kernel_launch_count": ([], u64),
        "pstf_field_create": ([vp, i32, vp], i32),
        "pstf_field_destroy": ([vp], i32),
        "pstf_field_get_config": ([vp, vp], i32),
        "pstf_select_level": ([vp, vp, vp, u64, vp], i32),
        "pstf_key_for": ([vp, vp, vp, vp, u64, vp, vp], i32),
        "pstf_field_apply": ([vp, vp, vp, vp, vp, u64, i32, vp], i32),
        "pstf_field_query": ([vp, vp, vp, vp, vp, u64, vp, vp, vp, vp, vp, vp, vp], i32),
        "pstf_field_end_frame": ([vp, vp], i32),
        "pstf_fields_end_frame": ([vp, i32, vp], i32),
        "pstf_field_invalidate": ([vp, vp, vp], i32),
        "pstf_field_get_stats": ([vp, vp], i32),
        "pstf_field_weighted_mean": ([vp, vp], i32),
        "pstf_field_snapshot": ([vp, vp, u64, vp], i32),
        "pstf_field_dump_snapshot": ([vp, C.c_char_p], i32),
        "pstf_read_snapshot": ([C.c_char_p, vp, u64, vp, vp], i32),
        "pstf_field_restore": ([vp, vp, u64], i32),
        "pstf_field_load_snapshot": ([vp, C.c_char_p], i32),
        "pstf_field_slots": ([vp, u64, u64, vp], i32),
        "pstf_vertex_pass": ([vp, vp, vp, vp, vp, u64, u32, u32, i32, vp], i32),
        "pstf_vertex_pass_host": ([vp, vp, vp, vp, vp, u64, u32, u32, i32, vp], i32),
        "pstf_vertex_pass_cv": ([vp, vp, vp, vp, vp, u64, u32, u32, i32, vp, vp, vp, vp, vp],
                                i32),
        "pstf_cv_lookup": ([vp, vp, u64, vp, vp, vp, vp, vp], i32),
        "pstf_synth_generate": ([i32, i32, i32, u64, u64, d, vp, vp], i32),
        "pstf_synth_generate_stripe": ([i32, i32, i32, u64, u64, d, u64, u64, vp, vp], i32),
        "pstf_synth_generate_scene": ([i32, i32, i32, i32, u64, u64, d, u64, u64, vp, vp], i32),
        "pstf_vertex_soa_from_buffer": ([vp, u64, vp], None),
        "pstf_profile_enable": ([i32], i32),
        "pstf_field_probe_histogram": ([vp, vp], i32),
        "pstf_diag_red_peak": ([i32, vp], i32),
        "pstf_profile_collect": ([vp, vp, vp, i32, vp], i32),
        "pstf_model_create": ([vp, i32, vp], i32),
        "pstf_model_destroy": ([vp], i32),
        "pstf_model_apply": ([vp, vp, vp, vp, vp, u64, i32, vp], i32),
        "pstf_model_end_frame": ([vp, vp], i32),
        "pstf_model_lookup_warm": ([vp, vp, u64, vp, vp], i32),
        "pstf_model_lookup_warm_levels": ([vp, vp, vp, vp, vp, u64, vp, vp], i32),
        "pstf_model_pdf": ([vp, vp, vp, vp, u64, vp, vp], i32),
        "pstf_model_sample": ([vp, vp, vp, vp, vp, u64, vp, vp, vp, vp], i32),
        "pstf_model_get_stats": ([vp, vp], i32),
        "pstf_model_dump": ([vp, vp, vp, vp, u64, vp], i32),
        "pstf_model_dump_tree": ([vp, vp, vp, u64, vp], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _check(rc):
    if rc != 0:
        raise PstfError(f"pstf error {rc}: {lib().pstf_last_error().decode()}")


def red_peak(device: int = 0) -> float:
    """Measured fp64 RED element updates/s (the vertex pass's pattern, L2-resident)."""
    out = C.c_double()
    _check(lib().pstf_diag_red_peak(device, C.byref(out)))
    return out.value


def kernel_launch_count() -> int:
    return int(lib().pstf_kernel_launch_count())


def profile_enable(on: bool = True):
    """Records CUDA events around every library launch on its stream (bench instrumentation)."""
    _check(lib().pstf_profile_enable(1 if on else 0))


def profile_collect() -> dict:
    """{kernel name: (total ms, launches)} since the last collect; synchronises."""
    n_max = 128
    names = C.create_string_buffer(64 * n_max)
    ms = (C.c_double * n_max)()
    cnt = (C.c_uint64 * n_max)()
    n = C.c_int()
    _check(lib().pstf_profile_collect(names, ms, cnt, n_max, C.byref(n)))
    out = {}
    for i in range(n.value):
        nm = names.raw[64 * i:64 * (i + 1)].split(b"\0")[0].decode()
        out[nm] = (float(ms[i]), int(cnt[i]))
    return out


def _torch():
    import torch
    return torch


def _stream():
    t = _torch()
    return C.c_void_p(t.cuda.current_stream().cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _vec3(t):
    """(3, n) contiguous CUDA fp64 tensor -> pstf_vec3_soa"""
    return _Vec3(t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr())


@dataclass
class FieldStoreConfig:
    """FieldStoreConfig (field.h:44-55) with the reference defaults."""
    kind: int = KIND_LO
    capacity_log2: int = 22
    max_level: int = 4
    base_cell_size: float = 0.01
    level_select_k: float = 4.0
    t_max: float = 64.0
    blend: int = BLEND_SQRT
    technique_mask: int = TECH_ALL
    probe_window: int = 32
    evict_age_frames: int = 64

    def _c(self):
        return _Config(self.kind, self.capacity_log2, self.max_level, self.base_cell_size,
                       self.level_select_k, self.t_max, self.blend, self.technique_mask,
                       self.probe_window, self.evict_age_frames)


@dataclass(frozen=True)
class SpatioDirectionalKey:
    """field.h:32-42; equality ignores the checksum like operator== (field.h:38-41)."""
    level: int
    cell: tuple
    dir_cell: tuple
    checksum: int

    def __eq__(self, o):
        return (self.level, tuple(self.cell), tuple(self.dir_cell)) == \
            (o.level, tuple(o.cell), tuple(o.dir_cell))

    def __hash__(self):
        return hash((self.level, tuple(self.cell), tuple(self.dir_cell)))


def _keys_to_tensor(keys, device):
    t = _torch()
    if isinstance(keys, t.Tensor):
        return keys.to(device=device, dtype=t.int32).contiguous()
    if isinstance(keys, np.ndarray) and keys.dtype == KEY_DTYPE:
        arr = keys.view(np.int32).reshape(-1, 7)
    else:
        arr = (np.array([[k.level, *k.cell, *k.dir_cell, k.checksum] for k in keys],
                        dtype=np.int64).reshape(-1, 7) & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
    return t.from_numpy(np.ascontiguousarray(arr)).to(device)


class FieldStore:
    """pstf::FieldStore (field.h:76-138) backed by libpstf_b200.so."""

    def __init__(self, config: FieldStoreConfig | None = None, device: int = 0):
        self._config = config or FieldStoreConfig()
        self.device = device
        self._h = C.c_void_p()
        cfg = self._config._c()
        _check(lib().pstf_field_create(C.byref(cfg), device, C.byref(self._h)))
        self._staged = []

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().pstf_field_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def config(self) -> FieldStoreConfig:
        return self._config

    @property
    def capacity(self) -> int:
        return 1 << self._config.capacity_log2

    def _dev(self):
        return _torch().device("cuda", self.device)

    # ---------------- key math (field.h:83-86) ----------------
    def select_level_batch(self, footprint):
        t = _torch()
        fp = footprint.to(device=self._dev(), dtype=t.float64).contiguous()
        out = t.empty(fp.numel(), dtype=t.int32, device=self._dev())
        _check(lib().pstf_select_level(self._h, _ptr(fp), _ptr(out), fp.numel(), _stream()))
        return out

    def key_for_batch(self, pos, direction, level):
        """pos, direction: (n, 3) or (3, n) fp64; level: (n,) int -> (n, 7) int32 key tensor"""
        t = _torch()
        p = _soa3(pos, self._dev())
        dd = _soa3(direction, self._dev())
        lv = t.as_tensor(level).to(device=self._dev(), dtype=t.int32).contiguous()
        n = lv.numel()
        out = t.empty((n, 7), dtype=t.int32, device=self._dev())
        pv, dv = _vec3(p), _vec3(dd)
        _check(lib().pstf_key_for(self._h, C.byref(pv), C.byref(dv), _ptr(lv), n, _ptr(out),
                                  _stream()))
        return out

    def selectLevel(self, footprint: float) -> int:
        t = _torch()
        return int(self.select_level_batch(t.tensor([float(footprint)], dtype=t.float64))[0])

    select_level = selectLevel

    def cellSize(self, level: int) -> float:
        return self._config.base_cell_size * float(1 << level)  # field.cpp:78-80

    def dirResolution(self, level: int) -> int:
        return 8 >> min(level, 2)  # field.cpp:82-84

    def keyFor(self, position, direction, level: int) -> SpatioDirectionalKey:
        t = _torch()
        k = self.key_for_batch(t.tensor([list(position)], dtype=t.float64),
                               t.tensor([list(direction)], dtype=t.float64), [int(level)])
        return keys_from_tensor(k)[0]

    key_for = keyFor

    # ---------------- updates (field.h:88-91, 157) ----------------
    def incrementCounter(self, key: SpatioDirectionalKey, w: float):
        self._staged.append((key, 0.0, 0.0, 0.0, float(w), 1))

    def accumulate(self, key: SpatioDirectionalKey, value, w: float):
        r, g, b = (float(x) for x in value)
        self._staged.append((key, r, g, b, float(w), 0))

    increment_counter = incrementCounter

    def flush(self):
        """Applies staged scalar calls (SEQUENTIAL mode == the reference's call sequence)."""
        if not self._staged:
            return
        t = _torch()
        staged, self._staged = self._staged, []
        keys = _keys_to_tensor([s[0] for s in staged], self._dev())
        v = t.tensor([[s[1] for s in staged], [s[2] for s in staged], [s[3] for s in staged]],
                     dtype=t.float64, device=self._dev())
        w = t.tensor([s[4] for s in staged], dtype=t.float64, device=self._dev())
        isc = t.tensor([s[5] for s in staged], dtype=t.uint8, device=self._dev())
        self.apply(keys, v, w, isc, MODE_SEQUENTIAL)

    def apply(self, keys, value, w, is_counter, mode=MODE_ATOMIC):
        """Batched updates: keys (n,7) int32, value (3,n) fp64 or None, w (n,), is_counter (n,)"""
        t = _torch()
        k = _keys_to_tensor(keys, self._dev())
        n = k.shape[0]
        vv = None
        if value is not None:
            v = value.to(device=self._dev(), dtype=t.float64).contiguous()
            vv = _vec3(v)
        ww = w.to(device=self._dev(), dtype=t.float64).contiguous()
        ic = None if is_counter is None else \
            is_counter.to(device=self._dev(), dtype=t.uint8).contiguous()
        _check(lib().pstf_field_apply(self._h, _ptr(k), C.byref(vv) if vv is not None else None,
                                      _ptr(ww), _ptr(ic), n, mode, _stream()))

    # ---------------- queries (field.h:93-94) ----------------
    def query_batch(self, pos, direction, footprint=None, level=None):
        self.flush()
        t = _torch()
        p = _soa3(pos, self._dev())
        dd = _soa3(direction, self._dev())
        n = p.shape[1]
        fp = None if footprint is None else \
            t.as_tensor(footprint).to(device=self._dev(), dtype=t.float64).contiguous()
        lv = None if level is None else \
            t.as_tensor(level).to(device=self._dev(), dtype=t.int32).contiguous()
        val = t.empty((3, n), dtype=t.float64, device=self._dev())
        valid = t.empty(n, dtype=t.uint8, device=self._dev())
        fb = t.empty(n, dtype=t.uint8, device=self._dev())
        ol = t.empty(n, dtype=t.int32, device=self._dev())
        pv, dv = _vec3(p), _vec3(dd)
        _check(lib().pstf_field_query(self._h, C.byref(pv), C.byref(dv), _ptr(fp), _ptr(lv), n,
                                      _ptr(val[0]), _ptr(val[1]), _ptr(val[2]), _ptr(valid),
                                      _ptr(fb), _ptr(ol), _stream()))
        return val, valid.bool(), fb.bool(), ol

    def queryFromLevel(self, position, direction, level: int):
        t = _torch()
        v, ok, fb, lv = self.query_batch(t.tensor([list(position)], dtype=t.float64),
                                         t.tensor([list(direction)], dtype=t.float64),
                                         level=[int(level)])
        return QueryResult(tuple(float(x) for x in v[:, 0].cpu()), bool(ok[0]), bool(fb[0]),
                           int(lv[0]))

    def query(self, position, direction, footprint: float):
        t = _torch()
        v, ok, fb, lv = self.query_batch(t.tensor([list(position)], dtype=t.float64),
                                         t.tensor([list(direction)], dtype=t.float64),
                                         footprint=[float(footprint)])
        return QueryResult(tuple(float(x) for x in v[:, 0].cpu()), bool(ok[0]), bool(fb[0]),
                           int(lv[0]))

    query_from_level = queryFromLevel

    # ---------------- frame barrier (field.h:100-103) ----------------
    def endFrame(self):
        self.flush()
        _check(lib().pstf_field_end_frame(self._h, _stream()))

    end_frame = endFrame

    def invalidate(self, region=None):
        """region: None or ((lo x, y, z), (hi x, y, z))"""
        self.flush()
        if region is None:
            _check(lib().pstf_field_invalidate(self._h, None, _stream()))
        else:
            box = (C.c_double * 6)(*[float(x) for x in (*region[0], *region[1])])
            _check(lib().pstf_field_invalidate(self._h, box, _stream()))

    # ---------------- observers (field.h:105-124) ----------------
    def stats(self) -> dict:
        self.flush()
        s = _Stats()
        _check(lib().pstf_field_get_stats(self._h, C.byref(s)))
        return {n: int(getattr(s, n)) for n, _ in _Stats._fields_}

    def frameIndex(self):
        return self.stats()["frame"]

    def rejectedUpdates(self):
        return self.stats()["rejected"]

    def droppedInserts(self):
        return self.stats()["dropped"]

    def internalErrors(self):
        return self.stats()["internal_errors"]

    def liveCellCount(self):
        return self.stats()["live"]

    def probe_histogram(self) -> np.ndarray:
        """hist[d] = live slots at probe distance d from their home slot (d >= 32 in [32])."""
        self.flush()
        h = np.zeros(33, np.uint64)
        _check(lib().pstf_field_probe_histogram(self._h, h.ctypes.data_as(C.c_void_p)))
        return h

    def weightedMeanValue(self):
        self.flush()
        out = (C.c_double * 3)()
        _check(lib().pstf_field_weighted_mean(self._h, out))
        return tuple(out)

    def snapshot(self) -> np.ndarray:
        """key-sorted records (field.cpp:311-337) as SNAPSHOT_DTYPE"""
        self.flush()
        live = self.liveCellCount()
        out = np.zeros(max(live, 1), SNAPSHOT_DTYPE)
        cnt = C.c_uint64()
        _check(lib().pstf_field_snapshot(self._h, out.ctypes.data_as(C.c_void_p), live,
                                         C.byref(cnt)))
        return out[:cnt.value]

    def dumpSnapshot(self, path: str):
        self.flush()
        _check(lib().pstf_field_dump_snapshot(self._h, path.encode()))

    dump_snapshot = dumpSnapshot

    @staticmethod
    def readSnapshot(path: str) -> np.ndarray:
        return read_snapshot(path)[1]

    def restore(self, records) -> None:
        """Insert snapshot records (SNAPSHOT_DTYPE, any order) and set their committed values;
        the semantics are pstf_field_restore's (include/pstf_field.h).  Extension: the
        reference writes snapshots (field.cpp:311-386) but cannot load them."""
        self.flush()
        r = np.ascontiguousarray(records, SNAPSHOT_DTYPE)
        _check(lib().pstf_field_restore(self._h, r.ctypes.data_as(C.c_void_p), len(r)))

    def loadSnapshot(self, path: str) -> None:
        """readSnapshot(path) + restore; the file's kind must be the store's"""
        self.flush()
        _check(lib().pstf_field_load_snapshot(self._h, path.encode()))

    load_snapshot = loadSnapshot

    def slots(self, begin=0, count=None) -> np.ndarray:
        self.flush()
        count = self.capacity - begin if count is None else count
        out = np.zeros(count, SLOT_DTYPE)
        _check(lib().pstf_field_slots(self._h, begin, count, out.ctypes.data_as(C.c_void_p)))
        return out


@dataclass
class QueryResult:
    """FieldQueryResult (field.h:57-62)"""
    value: tuple
    valid: bool
    fallback: bool
    level: int


class FieldUpdateQueue:
    """pstf::FieldUpdateQueue (field.h:143-167): apply() == ORDERED mode (bit-exact)."""

    def __init__(self):
        self._u = []

    def pushCounter(self, key, w):
        self._u.append((key, 0.0, 0.0, 0.0, float(w), 1))

    def pushValue(self, key, value, w):
        r, g, b = (float(x) for x in value)
        self._u.append((key, r, g, b, float(w), 0))

    def append(self, other: "FieldUpdateQueue"):
        self._u.extend(other._u)
        other._u = []

    def size(self):
        return len(self._u)

    def clear(self):
        self._u = []

    def apply(self, store: FieldStore):
        store.flush()
        if self._u:
            t = _torch()
            dev = store._dev()
            keys = _keys_to_tensor([s[0] for s in self._u], dev)
            v = t.tensor([[s[1] for s in self._u], [s[2] for s in self._u],
                          [s[3] for s in self._u]], dtype=t.float64, device=dev)
            w = t.tensor([s[4] for s in self._u], dtype=t.float64, device=dev)
            isc = t.tensor([s[5] for s in self._u], dtype=t.uint8, device=dev)
            store.apply(keys, v, w, isc, MODE_ORDERED)
        self._u = []


def keys_from_tensor(k) -> list:
    a = k.cpu().numpy().astype(np.int32)
    return [SpatioDirectionalKey(int(r[0]), (int(r[1]), int(r[2]), int(r[3])),
                                 (int(r[4]), int(r[5])), int(np.uint32(r[6].view(np.uint32))))
            for r in a]


def _soa3(x, device):
    """(n,3) or (3,n) -> contiguous (3,n) fp64 CUDA tensor (n==3 is read as (n,3))"""
    t = _torch()
    x = t.as_tensor(x, dtype=t.float64)
    if x.dim() == 2 and x.shape[1] == 3:
        x = x.t()
    return x.to(device).contiguous()


def end_frame_all(stores):
    """endFrame on up to 4 stores of one device with one pair of sweeps (frame barrier,
    estimators.cpp:647-651); identical to calling end_frame on each."""
    stores = [s for s in stores if s is not None]
    for s in stores:
        s.flush()
    arr = (C.c_void_p * len(stores))(*[s._h.value for s in stores])
    _check(lib().pstf_fields_end_frame(arr, len(stores), _stream()))


def read_snapshot(path: str):
    """FieldStore::readSnapshot (field.cpp:357-386) -> (kind, records)"""
    cnt = C.c_uint64()
    kind = C.c_uint32()
    _check(lib().pstf_read_snapshot(path.encode(), None, 0, C.byref(cnt), C.byref(kind)))
    out = np.zeros(max(cnt.value, 1), SNAPSHOT_DTYPE)
    _check(lib().pstf_read_snapshot(path.encode(), out.ctypes.data_as(C.c_void_p), cnt.value,
                                    C.byref(cnt), C.byref(kind)))
    return int(kind.value), out[:cnt.value]


def vertex_soa(buf, n) -> _VertexSoa:
    """pstf_vertex_soa view of a contiguous (34*n fp64 + n u32) buffer (torch tensor/ptr)."""
    v = _VertexSoa()
    p = buf.data_ptr() if hasattr(buf, "data_ptr") else int(buf)
    lib().pstf_vertex_soa_from_buffer(C.c_void_p(p), n, C.byref(v))
    return v


def synth_generate(width, height, bounces, seed=0x5EED, iteration=0, cam_shift_x=0.0, out=None,
                   path0=0, npaths=None, scene=0):
    """Synthetic Cornell stream on the device (pstf_synth.h) -> fp64 CUDA tensor buffer.
    path0/npaths select an image stripe (paths [path0, path0+npaths), all bounces); scene 1:
    the glossy materials of staircase_glossy.scene (BASELINE config 3)."""
    t = _torch()
    npaths = width * height - path0 if npaths is None else npaths
    n = npaths * bounces
    words = 34 * n + (n + 1) // 2
    if out is None:
        out = t.empty(words, dtype=t.float64, device="cuda")
    _check(lib().pstf_synth_generate_scene(scene, width, height, bounces, seed, iteration,
                                           cam_shift_x, path0, npaths, _ptr(out), _stream()))
    return out, n


def vertex_soa_from_fields(fields, flags) -> _VertexSoa:
    """pstf_vertex_soa from 34 separate fp64 device arrays (PS_* order: position xyz, wo, wi,
    next position, nee dir, footprint, next footprint, ratio, next MIS weight, emission, f,
    next emission, nee Lo\\E, nee FLi) and a u32 flags array (tensors or raw pointers)."""
    ptr = lambda t: t.data_ptr() if hasattr(t, "data_ptr") else int(t)
    v = _VertexSoa()
    k = 0
    for name, typ in _VertexSoa._fields_:
        if name == "flags":
            v.flags = ptr(flags)
        elif typ is _Vec3:
            setattr(v, name, _Vec3(ptr(fields[k]), ptr(fields[k + 1]), ptr(fields[k + 2])))
            k += 3
        else:
            setattr(v, name, ptr(fields[k]))
            k += 1
    return v


def vertex_pass(lo, loe, fli, li, buf, n, loe_mask=TECH_ALL, fli_mask=TECH_ALL,
                mode=MODE_ATOMIC, soa=None):
    """FieldRecorder::onVertex for n vertices in a device buffer (estimators.cpp:194-262);
    soa: a prebuilt pstf_vertex_soa (vertex_soa_from_fields) instead of buf."""
    for s in (lo, loe, fli, li):
        if s is not None:
            s.flush()
    v = soa if soa is not None else vertex_soa(buf, n)
    _check(lib().pstf_vertex_pass(lo._h, loe._h, fli._h, li._h if li is not None else None,
                                  C.byref(v), n, loe_mask, fli_mask, mode, _stream()))


def vertex_pass_host(lo, loe, fli, li, host_buf: np.ndarray, n, loe_mask=TECH_ALL,
                     fli_mask=TECH_ALL, mode=MODE_ATOMIC):
    """Same with a HOST buffer (pinned numpy/torch memory recommended)."""
    for s in (lo, loe, fli, li):
        if s is not None:
            s.flush()
    p = host_buf.data_ptr() if hasattr(host_buf, "data_ptr") else host_buf.ctypes.data
    v = vertex_soa(p, n)
    _check(lib().pstf_vertex_pass_host(lo._h, loe._h, fli._h, li._h if li is not None else None,
                                       C.byref(v), n, loe_mask, fli_mask, mode, _stream()))


def vertex_pass_cv(lo, loe, fli, li, buf, n, loe_mask=TECH_ALL, fli_mask=TECH_ALL,
                   mode=MODE_ATOMIC, out=None, soa=None):
    """vertex_pass plus the CV lookup of every vertex on the frame-start table, fused into the
    vertex kernel (== cv_lookup before vertex_pass) -> (value (3,n), valid (n,) uint8).
    out: optional preallocated (value, valid) pair."""
    t = _torch()
    for s in (lo, loe, fli, li):
        if s is not None:
            s.flush()
    v = soa if soa is not None else vertex_soa(buf, n)
    if out is None:
        dev = buf.device if buf is not None else "cuda"
        out = (t.empty((3, n), dtype=t.float64, device=dev), t.empty(n, dtype=t.uint8, device=dev))
    val, ok = out
    _check(lib().pstf_vertex_pass_cv(lo._h, loe._h, fli._h, li._h if li is not None else None,
                                     C.byref(v), n, loe_mask, fli_mask, mode, _ptr(val[0]),
                                     _ptr(val[1]), _ptr(val[2]), _ptr(ok), _stream()))
    return val, ok


def cv_lookup(loe, buf, n):
    """CV lookup at every vertex (estimators.cpp:453-462) -> (value (3,n), valid (n,))"""
    t = _torch()
    v = vertex_soa(buf, n)
    val = t.empty((3, n), dtype=t.float64, device=buf.device)
    ok = t.empty(n, dtype=t.uint8, device=buf.device)
    _check(lib().pstf_cv_lookup(loe._h, C.byref(v), n, _ptr(val[0]), _ptr(val[1]), _ptr(val[2]),
                                _ptr(ok), _stream()))
    return val, ok.bool()
