"""ctypes front-end for the parity checkers (TEST INFRASTRUCTURE ONLY).

Two interchangeable back-ends with one API:
  * ``OracleStore``  - the C restatement in oracle/pstf_oracle.c  (liboracle.so, always built)
  * ``RefStore``     - the UNMODIFIED reference field.cpp compiled from /root/reference into
                       oracle/_ref/libpstf_ref.so (present when built in this container)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
import this module.  The product package (paper_2005_07547_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpstf_ref.so")

KEY_DTYPE = np.dtype([("level", "<i4"), ("cell", "<i4", (3,)), ("dir", "<i4", (2,)),
                      ("checksum", "<u4")])
SLOT_DTYPE = np.dtype([("checksum", "<u4"), ("level", "<i4"), ("cell", "<i4", (3,)),
                       ("dir", "<i4", (2,)), ("value_old", "<f8", (3,)), ("c_old", "<f8"),
                       ("accum", "<f8", (3,)), ("c_new", "<f8"), ("last_touched", "<u4")],
                      align=True)
SNAP_DTYPE = np.dtype([("level", "<i4"), ("cell", "<i4", (3,)), ("dir", "<i4", (2,)),
                       ("checksum", "<u4"), ("value", "<f8", (3,)), ("c_old", "<f8")], align=True)
UPDATE_DTYPE = np.dtype([("key", KEY_DTYPE), ("value", "<f8", (3,)), ("w", "<f8"),
                         ("is_counter", "<i4")], align=True)
assert SLOT_DTYPE.itemsize == 104 and SNAP_DTYPE.itemsize == 64 and UPDATE_DTYPE.itemsize == 72

TECH_CAMERA, TECH_CONT, TECH_NEE = 1, 2, 4
TECH_ALL = 7
KIND_LO, KIND_LOE, KIND_LI, KIND_FLI = 0, 1, 2, 3


class Config(C.Structure):
    """FieldStoreConfig (field.h:44-55); same layout as po_config / pr_config."""
    _fields_ = [("kind", C.c_uint32), ("capacity_log2", C.c_uint32), ("max_level", C.c_int32),
                ("base_cell_size", C.c_double), ("level_select_k", C.c_double),
                ("t_max", C.c_double), ("blend", C.c_uint32), ("technique_mask", C.c_uint32),
                ("probe_window", C.c_uint32), ("evict_age_frames", C.c_uint32)]

    @classmethod
    def make(cls, kind=KIND_LO, capacity_log2=22, max_level=4, base_cell_size=0.01,
             level_select_k=4.0, t_max=64.0, blend=0, technique_mask=TECH_ALL, probe_window=32,
             evict_age_frames=64):
        return cls(kind, capacity_log2, max_level, base_cell_size, level_select_k, t_max, blend,
                   technique_mask, probe_window, evict_age_frames)


class Stats(C.Structure):
    _fields_ = [("frame", C.c_uint64), ("rejected", C.c_uint64), ("dropped", C.c_uint64),
                ("internal_errors", C.c_uint64), ("live", C.c_uint64)]


class _QR(C.Structure):
    _fields_ = [("value", C.c_double * 3), ("valid", C.c_int32), ("fallback", C.c_int32),
                ("level", C.c_int32)]


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_libs = {}


def _load(path):
    if path not in _libs:
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        _libs[path] = C.CDLL(path)
    return _libs[path]


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def oracle_lib():
    lib = _load(ORACLE_SO)
    if not getattr(lib, "_typed", False):
        vp, d, i32, u32, u64, sz = C.c_void_p, C.c_double, C.c_int, C.c_uint32, C.c_uint64, C.c_size_t
        lib.po_store_create.restype = vp
        lib.po_store_create.argtypes = [vp]
        lib.po_store_destroy.argtypes = [vp]
        lib.po_select_level.argtypes = [vp, d]
        lib.po_select_level.restype = i32
        lib.po_key_for.argtypes = [vp, vp, vp, i32]
        lib.po_key_for.restype = KeyStruct
        lib.po_increment_counter.argtypes = [vp, vp, d]
        lib.po_accumulate.argtypes = [vp, vp, vp, d]
        lib.po_query_from_level.argtypes = [vp, vp, vp, i32]
        lib.po_query_from_level.restype = _QR
        lib.po_query.argtypes = [vp, vp, vp, d]
        lib.po_query.restype = _QR
        lib.po_end_frame.argtypes = [vp]
        lib.po_invalidate_all.argtypes = [vp]
        lib.po_invalidate_box.argtypes = [vp, vp, vp]
        lib.po_stats_get.argtypes = [vp, vp]
        lib.po_weighted_mean.argtypes = [vp, vp]
        lib.po_slots.argtypes = [vp, vp]
        lib.po_snapshot.argtypes = [vp, vp, sz]
        lib.po_snapshot.restype = sz
        lib.po_restore.argtypes = [vp, vp, sz]
        lib.po_queue_apply.argtypes = [vp, vp, sz]
        lib.po_vertex_pass_contig.argtypes = [vp, vp, vp, vp, vp, sz, u32, u32, i32]
        lib.po_synth_generate.argtypes = [i32, i32, i32, u64, u64, d, vp, i32]
        lib.po_synth_generate_scene.argtypes = [i32, i32, i32, i32, u64, u64, d, vp, i32]
        lib.po_home_slot.argtypes = [vp, u32]
        lib.po_home_slot.restype = u32
        lib.po_key_for_batch.argtypes = [vp, vp, vp, vp, sz, vp]
        lib.po_select_level_batch.argtypes = [vp, vp, sz, vp]
        lib.po_query_batch.argtypes = [vp, vp, vp, vp, vp, sz, vp, vp]
        lib._typed = True
    return lib


def ref_lib():
    lib = _load(REF_SO)
    if not getattr(lib, "_typed", False):
        vp, d, i32, u32, i64 = C.c_void_p, C.c_double, C.c_int, C.c_uint32, C.c_int64
        lib.pr_store_create.restype = vp
        lib.pr_store_create.argtypes = [vp]
        lib.pr_store_destroy.argtypes = [vp]
        lib.pr_select_level.argtypes = [vp, d]
        lib.pr_select_level.restype = i32
        lib.pr_key_for.argtypes = [vp, vp, vp, i32, vp]
        lib.pr_key_for_batch.argtypes = [vp, vp, vp, vp, i64, vp]
        lib.pr_select_level_batch.argtypes = [vp, vp, i64, vp]
        lib.pr_sphere_to_square_batch.argtypes = [vp, i64, vp]
        lib.pr_home_slot.argtypes = [vp, vp]
        lib.pr_home_slot.restype = C.c_uint64
        lib.pr_increment.argtypes = [vp, vp, d]
        lib.pr_accumulate.argtypes = [vp, vp, vp, d]
        lib.pr_query_from_level.argtypes = [vp, vp, vp, i32, vp, vp]
        lib.pr_query.argtypes = [vp, vp, vp, d, vp, vp]
        lib.pr_query_batch.argtypes = [vp, vp, vp, vp, vp, i64, vp, vp]
        lib.pr_end_frame.argtypes = [vp]
        lib.pr_invalidate_all.argtypes = [vp]
        lib.pr_invalidate_box.argtypes = [vp, vp, vp]
        lib.pr_stats_get.argtypes = [vp, vp]
        lib.pr_weighted_mean.argtypes = [vp, vp]
        lib.pr_dump_snapshot.argtypes = [vp, C.c_char_p]
        lib.pr_dump_snapshot.restype = i32
        lib.pr_slots.argtypes = [vp, vp]
        lib.pr_restore.argtypes = [vp, vp, i64]
        lib.pr_queue_create.restype = vp
        lib.pr_queue_destroy.argtypes = [vp]
        lib.pr_queue_push_counter.argtypes = [vp, vp, d]
        lib.pr_queue_push_value.argtypes = [vp, vp, vp, d]
        lib.pr_queue_apply.argtypes = [vp, vp]
        lib.pr_vertex_pass.argtypes = [vp, vp, vp, vp, vp, i64, u32, u32, i32, i32, i64]
        lib.pr_hardware_concurrency.restype = i32
        lib._typed = True
    return lib


class KeyStruct(C.Structure):
    _fields_ = [("level", C.c_int32), ("cell", C.c_int32 * 3), ("dir", C.c_int32 * 2),
                ("checksum", C.c_uint32)]

    def as_tuple(self):
        return (self.level, tuple(self.cell), tuple(self.dir), self.checksum)


def key_from_np(k) -> KeyStruct:
    ks = KeyStruct()
    ks.level = int(k["level"])
    for i in range(3):
        ks.cell[i] = int(k["cell"][i])
    for i in range(2):
        ks.dir[i] = int(k["dir"][i])
    ks.checksum = int(k["checksum"])
    return ks


def _v3(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(3))


class _StoreBase:
    """Common API (mirrors pstf::FieldStore, field.h:76-138)."""

    def __init__(self, config: Config):
        self.config = config
        self.capacity = 1 << config.capacity_log2


class OracleStore(_StoreBase):
    def __init__(self, config: Config):
        super().__init__(config)
        self.lib = oracle_lib()
        self._cfg = Config.from_buffer_copy(config)
        self.h = self.lib.po_store_create(C.byref(self._cfg))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.po_store_destroy(self.h)
            self.h = None

    def select_level(self, fp):
        return self.lib.po_select_level(C.byref(self._cfg), float(fp))

    def key_for(self, pos, d, level) -> KeyStruct:
        p, q = _v3(pos), _v3(d)
        return self.lib.po_key_for(C.byref(self._cfg), _p(p), _p(q), int(level))

    def keys_for(self, pos, d, level):
        """pos, d: (n,3); level: (n,) -> structured KEY_DTYPE array"""
        pos = np.ascontiguousarray(np.asarray(pos, np.float64).T)
        d = np.ascontiguousarray(np.asarray(d, np.float64).T)
        level = np.ascontiguousarray(level, dtype=np.int32)
        out = np.zeros(len(level), KEY_DTYPE)
        self.lib.po_key_for_batch(C.byref(self._cfg), _p(pos), _p(d), _p(level), len(level),
                                  _p(out))
        return out

    def select_levels(self, fp):
        fp = np.ascontiguousarray(fp, dtype=np.float64)
        out = np.zeros(len(fp), np.int32)
        self.lib.po_select_level_batch(C.byref(self._cfg), _p(fp), len(fp), _p(out))
        return out

    def query_batch(self, pos, d, fp=None, level=None):
        n = len(pos)
        pos = np.ascontiguousarray(np.asarray(pos, np.float64).T)
        d = np.ascontiguousarray(np.asarray(d, np.float64).T)
        fp = None if fp is None else np.ascontiguousarray(fp, np.float64)
        level = None if level is None else np.ascontiguousarray(level, np.int32)
        v = np.zeros((3, n))
        f = np.zeros((3, n), np.int32)
        self.lib.po_query_batch(self.h, _p(pos), _p(d), _p(fp), _p(level), n, _p(v), _p(f))
        return v.T.copy(), f[0].astype(bool), f[1].astype(bool), f[2].copy()

    def increment_counter(self, key, w):
        self.lib.po_increment_counter(self.h, C.byref(key), float(w))

    def accumulate(self, key, v, w):
        vv = _v3(v)
        self.lib.po_accumulate(self.h, C.byref(key), _p(vv), float(w))

    def query_from_level(self, pos, d, level):
        r = self.lib.po_query_from_level(self.h, _p(_v3(pos)), _p(_v3(d)), int(level))
        return (tuple(r.value), bool(r.valid), bool(r.fallback), r.level)

    def query(self, pos, d, fp):
        r = self.lib.po_query(self.h, _p(_v3(pos)), _p(_v3(d)), float(fp))
        return (tuple(r.value), bool(r.valid), bool(r.fallback), r.level)

    def end_frame(self):
        self.lib.po_end_frame(self.h)

    def invalidate(self, lo=None, hi=None):
        if lo is None:
            self.lib.po_invalidate_all(self.h)
        else:
            self.lib.po_invalidate_box(self.h, _p(_v3(lo)), _p(_v3(hi)))

    def stats(self):
        s = Stats()
        self.lib.po_stats_get(self.h, C.byref(s))
        return dict(frame=s.frame, rejected=s.rejected, dropped=s.dropped,
                    internal_errors=s.internal_errors, live=s.live)

    def weighted_mean(self):
        out = np.zeros(3)
        self.lib.po_weighted_mean(self.h, _p(out))
        return out

    def slots(self):
        out = np.zeros(self.capacity, SLOT_DTYPE)
        self.lib.po_slots(self.h, _p(out))
        return out

    def snapshot(self):
        live = self.stats()["live"]
        out = np.zeros(max(live, 1), SNAP_DTYPE)
        n = self.lib.po_snapshot(self.h, _p(out), live)
        return out[:n]

    def restore(self, records):
        """snapshot restore (pstf_field_restore semantics, oracle/pstf_oracle.c po_restore)"""
        r = np.ascontiguousarray(records, SNAP_DTYPE)
        self.lib.po_restore(self.h, _p(r), len(r))

    def queue_apply(self, updates):
        u = np.ascontiguousarray(updates.copy())
        self.lib.po_queue_apply(self.h, _p(u), len(u))

    def home_slot(self, key):
        return self.lib.po_home_slot(C.byref(key), self.capacity - 1)


class RefStore(_StoreBase):
    def __init__(self, config: Config):
        super().__init__(config)
        self.lib = ref_lib()
        self._cfg = Config.from_buffer_copy(config)
        self.h = self.lib.pr_store_create(C.byref(self._cfg))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.pr_store_destroy(self.h)
            self.h = None

    def select_level(self, fp):
        return self.lib.pr_select_level(self.h, float(fp))

    def select_levels(self, fp):
        fp = np.ascontiguousarray(fp, dtype=np.float64)
        out = np.zeros(len(fp), np.int32)
        self.lib.pr_select_level_batch(self.h, _p(fp), len(fp), _p(out))
        return out

    def key_for(self, pos, d, level) -> KeyStruct:
        k = KeyStruct()
        self.lib.pr_key_for(self.h, _p(_v3(pos)), _p(_v3(d)), int(level), C.byref(k))
        return k

    def keys_for(self, pos, d, level):
        pos = np.ascontiguousarray(np.asarray(pos, np.float64).T)
        d = np.ascontiguousarray(np.asarray(d, np.float64).T)
        level = np.ascontiguousarray(level, dtype=np.int32)
        out = np.zeros(len(level), KEY_DTYPE)
        self.lib.pr_key_for_batch(self.h, _p(pos), _p(d), _p(level), len(level), _p(out))
        return out

    def increment_counter(self, key, w):
        self.lib.pr_increment(self.h, C.byref(key), float(w))

    def accumulate(self, key, v, w):
        self.lib.pr_accumulate(self.h, C.byref(key), _p(_v3(v)), float(w))

    def _q(self, fn, pos, d, arg):
        v = np.zeros(3)
        f = np.zeros(3, np.int32)
        fn(self.h, _p(_v3(pos)), _p(_v3(d)), arg, _p(v), _p(f))
        return (tuple(v), bool(f[0]), bool(f[1]), int(f[2]))

    def query_from_level(self, pos, d, level):
        return self._q(self.lib.pr_query_from_level, pos, d, int(level))

    def query(self, pos, d, fp):
        return self._q(self.lib.pr_query, pos, d, float(fp))

    def query_batch(self, pos, d, fp=None, level=None):
        n = len(pos)
        pos = np.ascontiguousarray(np.asarray(pos, np.float64).T)
        d = np.ascontiguousarray(np.asarray(d, np.float64).T)
        fp = None if fp is None else np.ascontiguousarray(fp, np.float64)
        level = None if level is None else np.ascontiguousarray(level, np.int32)
        v = np.zeros((3, n))
        f = np.zeros((3, n), np.int32)
        self.lib.pr_query_batch(self.h, _p(pos), _p(d), _p(fp), _p(level), n, _p(v), _p(f))
        return v.T.copy(), f[0].astype(bool), f[1].astype(bool), f[2].copy()

    def end_frame(self):
        self.lib.pr_end_frame(self.h)

    def invalidate(self, lo=None, hi=None):
        if lo is None:
            self.lib.pr_invalidate_all(self.h)
        else:
            self.lib.pr_invalidate_box(self.h, _p(_v3(lo)), _p(_v3(hi)))

    def stats(self):
        s = Stats()
        self.lib.pr_stats_get(self.h, C.byref(s))
        return dict(frame=s.frame, rejected=s.rejected, dropped=s.dropped,
                    internal_errors=s.internal_errors, live=s.live)

    def weighted_mean(self):
        out = np.zeros(3)
        self.lib.pr_weighted_mean(self.h, _p(out))
        return out

    def slots(self):
        out = np.zeros(self.capacity, SLOT_DTYPE)
        self.lib.pr_slots(self.h, _p(out))
        return out

    def dump_snapshot(self, path):
        if self.lib.pr_dump_snapshot(self.h, path.encode()) != 0:
            raise RuntimeError("dumpSnapshot failed")

    def snapshot(self):
        import tempfile
        with tempfile.NamedTemporaryFile(suffix=".snap") as f:
            self.dump_snapshot(f.name)
            return read_snapshot(f.name)[1]

    def restore(self, records):
        """restore through the reference's own findOrInsertSlot (oracle/ref_shim.cpp pr_restore)"""
        r = np.ascontiguousarray(records, SNAP_DTYPE)
        self.lib.pr_restore(self.h, _p(r), len(r))

    def queue_apply(self, updates):
        q = self.lib.pr_queue_create()
        try:
            for u in updates:
                k = key_from_np(u["key"])
                if u["is_counter"]:
                    self.lib.pr_queue_push_counter(q, C.byref(k), float(u["w"]))
                else:
                    v = np.ascontiguousarray(u["value"], np.float64)
                    self.lib.pr_queue_push_value(q, C.byref(k), _p(v), float(u["w"]))
            self.lib.pr_queue_apply(q, self.h)
        finally:
            self.lib.pr_queue_destroy(q)

    def home_slot(self, key):
        return int(self.lib.pr_home_slot(self.h, C.byref(key)))


def read_snapshot(path):
    """Parses the PSTFSNAP v1 file (field.cpp:311-386): returns (kind, records)."""
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 24 or data[:8] != b"PSTFSNAP":
        raise ValueError(f"{path}: not a field snapshot")
    version, kind = np.frombuffer(data[8:16], "<u4")
    count = int(np.frombuffer(data[16:24], "<u8")[0])
    if version != 1:
        raise ValueError("unsupported snapshot version")
    packed = np.dtype([("level", "<i4"), ("cell", "<i4", (3,)), ("dir", "<i4", (2,)),
                       ("checksum", "<u4"), ("value", "<f8", (3,)), ("c_old", "<f8")])
    recs = np.frombuffer(data[24:24 + count * packed.itemsize], packed)
    if len(recs) != count:
        raise ValueError("truncated snapshot")
    out = np.zeros(count, SNAP_DTYPE)
    for name in packed.names:
        out[name] = recs[name]
    return int(kind), out


def vertex_pass_oracle(lo, loe, fli, li, buf, n, loe_mask=TECH_ALL, fli_mask=TECH_ALL,
                       deterministic=True):
    lib = oracle_lib()
    lib.po_vertex_pass_contig(lo.h, loe.h, fli.h, li.h if li is not None else None, _p(buf), n,
                              loe_mask, fli_mask, 1 if deterministic else 0)


def vertex_pass_ref(lo, loe, fli, li, buf, n, loe_mask=TECH_ALL, fli_mask=TECH_ALL,
                    deterministic=True, threads=1, chunk=1920):
    lib = ref_lib()
    lib.pr_vertex_pass(lo.h, loe.h, fli.h, li.h if li is not None else None, _p(buf), n,
                       loe_mask, fli_mask, 1 if deterministic else 0, threads, chunk)


def vertex_pass_phases_ref(lo, loe, fli, buf, n, threads, loe_mask=TECH_ALL, fli_mask=TECH_ALL):
    """the reference replay timed by phase (keygen, lookup, insert; ms), SURVEY.md §8(d)"""
    lib = ref_lib()
    fn = lib.pr_vertex_pass_phases
    fn.argtypes = [C.c_void_p] * 4 + [C.c_int64, C.c_uint32, C.c_uint32, C.c_int, C.c_void_p]
    out = np.zeros(3)
    fn(lo.h, loe.h, fli.h, _p(buf), n, loe_mask, fli_mask, threads, _p(out))
    return {"keygen": float(out[0]), "lookup": float(out[1]), "insert": float(out[2])}


def host_info() -> dict:
    """CPU model, hardware threads and libc of this host (the CPU timing protocol's record)"""
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        libc = os.confstr("CS_GNU_LIBC_VERSION")
    except (ValueError, OSError):
        libc = ""
    return {"cpu_model": model, "hardware_concurrency": os.cpu_count(), "libc": libc}


def synth_generate(width, height, bounces, seed=0x5EED, iteration=0, cam_shift_x=0.0,
                   threads=None, scene=0):
    """Host generator (pstf_synth.h) -> contiguous buffer (34*n fp64 + n u32 as fp64 words).
    scene 1: the glossy materials (BASELINE config 3)."""
    n = width * height * bounces
    words = 34 * n + (n + 1) // 2
    buf = np.zeros(words, np.float64)
    threads = threads or min(os.cpu_count() or 1, 64)
    oracle_lib().po_synth_generate_scene(scene, width, height, bounces, seed, iteration,
                                         cam_shift_x, _p(buf), threads)
    return buf, n


def soa_views(buf, n):
    f64 = buf[:34 * n].reshape(34, n)
    flags = buf[34 * n:].view(np.uint32)[:n]
    return f64, flags


# ---------------------------------------------------------------- ModelStore<DirGrid> (§8f row 2)
MODEL_ENTRY_DTYPE = np.dtype([("level", "<i4"), ("cell", "<i4", (3,)), ("dir", "<i4", (2,)),
                              ("warm", "<u4"), ("c_old", "<f8"), ("c_new", "<f8"),
                              ("records", "<u8"), ("record_count", "<u8"), ("total", "<f8")],
                             align=True)
assert MODEL_ENTRY_DTYPE.itemsize == 72
MODEL_REF_SO = os.path.join(HERE, "_ref", "libpstf_model_ref.so")


def model_ref_available() -> bool:
    return os.path.exists(MODEL_REF_SO)


class _ModelBase:
    """ModelStore (estimators.h:124-150) with DirGrid models; the C restatement
    (OracleModelStore) or the reference compiled in place (RefModelStore)."""
    P = ""

    def __init__(self, res=16, t_max=64.0, min_samples=32, kind=0, leaves=64, tsplit=4.0,
                 comps=4, alpha_em=0.7, smin=2.5e-5, smax=0.04, reseed=1e-4):
        self.kind = kind
        self.res = res
        self.r2 = 2 * leaves - 1 if kind == 1 else (21 * comps + 3 if kind == 2 else res * res)
        self.h = self._fn("create")(kind, res, leaves, tsplit, comps, alpha_em, smin, smax, reseed,
                                    t_max, min_samples)

    def _fn(self, name):
        return getattr(self.lib, self.P + name)

    def __del__(self):
        try:
            self._fn("destroy")(self.h)
        except Exception:
            pass

    def apply(self, keys, u, v, c):
        k = np.ascontiguousarray(keys, KEY_DTYPE)
        u, v, c = (np.ascontiguousarray(x, np.float64) for x in (u, v, c))
        self._fn("apply")(self.h, _p(k), _p(u), _p(v), _p(c), len(k))

    def end_frame(self):
        self._fn("end_frame")(self.h)

    def pdf(self, keys, u, v):
        out, found = np.zeros(len(keys)), np.zeros(len(keys), bool)
        f = C.c_int()
        for i in range(len(keys)):
            ks = key_from_np(keys[i])
            out[i] = self._fn("pdf")(self.h, C.byref(ks), float(u[i]), float(v[i]), C.byref(f))
            found[i] = f.value
        return out, found

    def sample(self, keys, u1, u2, usel=None):
        n = len(keys)
        usel = np.zeros(n) if usel is None else usel
        su, sv, pdf, found = np.zeros(n), np.zeros(n), np.zeros(n), np.zeros(n, bool)
        a, b, p, f = C.c_double(), C.c_double(), C.c_double(), C.c_int()
        for i in range(n):
            ks = key_from_np(keys[i])
            self._fn("sample")(self.h, C.byref(ks), float(u1[i]), float(u2[i]), float(usel[i]),
                               C.byref(a), C.byref(b), C.byref(p), C.byref(f))
            su[i], sv[i], pdf[i], found[i] = a.value, b.value, p.value, f.value
        return su, sv, pdf, found

    def dump(self):
        """(entries sorted by key, weights (n, R^2), accumulators (n, R^2))"""
        n = self._fn("dump")(self.h, None, None, None, 0)
        e = np.zeros(max(n, 1), MODEL_ENTRY_DTYPE)
        w, a = np.zeros((max(n, 1), self.r2)), np.zeros((max(n, 1), self.r2))
        self._fn("dump")(self.h, _p(e), _p(w), _p(a), n)
        return e[:n], w[:n], a[:n]

    def _initial_parents(self, leaves):
        """parent of every node of the constructor's uniform tree (one fresh entry)"""
        k = np.zeros(1, KEY_DTYPE)
        self.apply(k, [0.5], [0.5], [0.0])
        return self.dump_tree()[0][0, :, 4]

    def dump_tree(self):
        """k-d tree topology: (n, 2L-1, 5) int32 {leaf, axis, left, right, parent},
        (n, 2L-1, 2) float64 {split, mass}"""
        n = self._fn("dump")(self.h, None, None, None, 0)
        ti = np.zeros((max(n, 1), self.r2, 5), np.int32)
        tf = np.zeros((max(n, 1), self.r2, 2))
        self._fn("dump_tree")(self.h, _p(ti), _p(tf), n)
        return ti[:n], tf[:n]


def _type_model_lib(lib, p, n_t):
    vp, d, i32 = C.c_void_p, C.c_double, C.c_int
    getattr(lib, p + "create").restype = vp
    getattr(lib, p + "create").argtypes = [i32, i32, i32, d, i32, d, d, d, d, d, i32]
    getattr(lib, p + "destroy").argtypes = [vp]
    getattr(lib, p + "apply").argtypes = [vp, vp, vp, vp, vp, n_t]
    getattr(lib, p + "end_frame").argtypes = [vp]
    getattr(lib, p + "pdf").argtypes = [vp, vp, d, d, vp]
    getattr(lib, p + "pdf").restype = d
    getattr(lib, p + "sample").argtypes = [vp, vp, d, d, d, vp, vp, vp, vp]
    getattr(lib, p + "dump").argtypes = [vp, vp, vp, vp, n_t]
    getattr(lib, p + "dump").restype = n_t
    getattr(lib, p + "dump_tree").argtypes = [vp, vp, vp, n_t]
    getattr(lib, p + "dump_tree").restype = n_t


class OracleModelStore(_ModelBase):
    P = "po_model_"

    def __init__(self, *a, **k):
        self.lib = oracle_lib()
        if not getattr(self.lib, "_model_typed", False):
            _type_model_lib(self.lib, self.P, C.c_size_t)
            self.lib._model_typed = True
        super().__init__(*a, **k)


class RefModelStore(_ModelBase):
    P = "pm_"

    def __init__(self, *a, **k):
        self.lib = _load(MODEL_REF_SO)
        if not getattr(self.lib, "_model_typed", False):
            _type_model_lib(self.lib, self.P, C.c_int64)
            self.lib._model_typed = True
        super().__init__(*a, **k)
