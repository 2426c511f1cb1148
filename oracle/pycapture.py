"""ctypes front-end for oracle/_ref/libpstf_capture.so (TEST INFRASTRUCTURE ONLY).

The UNMODIFIED reference renderer, compiled in place from /root/reference by oracle/Makefile:
  * ``capture_frame``  - one frame of the reference path tracer (pathtracer.cpp:80-239) with a
                         PathHooks collector (test_pathtracer.cpp:14-17); returns the canonical
                         276 B/vertex SoA buffer the B200 vertex pass consumes
  * ``RefEstimatorRun`` - EstimatorRun (estimators.cpp:308-655) with the reference's own field
                         stores: per-frame snapshots, slot arrays and counters (the ground truth)
The reference scenes are copied by the same recipe into oracle/_ref/scenes/ (build output).
Only tests/ and bench.py's reference legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from pyoracle import SLOT_DTYPE, Stats, _p, read_snapshot

HERE = os.path.dirname(os.path.abspath(__file__))
CAPTURE_SO = os.path.join(HERE, "_ref", "libpstf_capture.so")
SCENE_DIR = os.path.join(HERE, "_ref", "scenes")

# EstimatorKind ordinals (estimators.h:17)
PT, PT_NEE, IS, CV, IS_CV, B = range(6)

_lib = None


def available() -> bool:
    return os.path.exists(CAPTURE_SO) and os.path.isdir(SCENE_DIR)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(CAPTURE_SO)
        vp, i64, u64, d, i32, u32 = C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_int, C.c_uint32
        L.pc_last_error.restype = C.c_char_p
        L.pc_scene_load.restype = vp
        L.pc_scene_load.argtypes = [C.c_char_p, i32, i32]
        L.pc_scene_free.argtypes = [vp]
        L.pc_scene_diameter.restype = d
        L.pc_scene_diameter.argtypes = [vp]
        L.pc_capture.restype = vp
        L.pc_capture.argtypes = [vp, u64, u64, i32, i32, i32, C.POINTER(i64)]
        L.pc_capture_soa.argtypes = [vp, vp]
        L.pc_capture_depths.argtypes = [vp, vp]
        L.pc_capture_free.argtypes = [vp]
        L.pc_run_create.restype = vp
        L.pc_run_create.argtypes = [vp, i32, i32, i32, u64, u32, i32, u32, u32]
        L.pc_run_free.argtypes = [vp]
        L.pc_run_frame.argtypes = [vp]
        L.pc_run_store_config.argtypes = [vp, i32, vp, vp]
        L.pc_run_dump_snapshot.restype = i32
        L.pc_run_dump_snapshot.argtypes = [vp, i32, C.c_char_p]
        L.pc_run_stats.argtypes = [vp, i32, vp]
        L.pc_run_slots.argtypes = [vp, i32, vp]
        _lib = L
    return _lib


class Scene:
    """loadScene with the camera resolution overridden (acceptance_main.cpp:60-61)"""

    def __init__(self, name, width=0, height=0):
        path = name if os.path.isabs(name) else os.path.join(SCENE_DIR, name)
        self.h = lib().pc_scene_load(path.encode(), width, height)
        if not self.h:
            raise RuntimeError(lib().pc_last_error().decode())
        self.diameter = float(lib().pc_scene_diameter(self.h))

    def __del__(self):
        try:
            lib().pc_scene_free(self.h)
        except Exception:
            pass


def capture_frame(scene: Scene, frame: int, seed: int = 0, spp: int = 1, threads: int = 0,
                  max_depth: int = 0, with_depth: bool = False):
    """One reference frame's VertexRecords as the SoA buffer (34*n fp64, then n u32 flags packed
    into fp64 words, the layout of pstf_synth_generate / pstf_vertex_soa_from_buffer)."""
    L = lib()
    n = C.c_int64()
    cap = L.pc_capture(scene.h, frame, seed, spp, threads or (os.cpu_count() or 1), max_depth,
                       C.byref(n))
    try:
        n = n.value
        buf = np.zeros(34 * n + (n + 1) // 2, np.float64)
        L.pc_capture_soa(cap, _p(buf))
        depth = None
        if with_depth:
            depth = np.zeros(n, np.int32)
            L.pc_capture_depths(cap, _p(depth))
    finally:
        L.pc_capture_free(cap)
    return (buf, n, depth) if with_depth else (buf, n)


class RefEstimatorRun:
    """EstimatorRun (estimators.cpp:308-343) over the reference's own FieldStores"""

    def __init__(self, scene: Scene, kind=PT_NEE, deterministic=True, threads=0, seed=0,
                 capacity_log2=18, track_li=False, loe_mask=7, fli_mask=7):
        self.scene = scene
        self.track_li = track_li
        self.h = lib().pc_run_create(scene.h, kind, int(deterministic),
                                     threads or (os.cpu_count() or 1), seed, capacity_log2,
                                     int(track_li), loe_mask, fli_mask)

    def __del__(self):
        try:
            lib().pc_run_free(self.h)
        except Exception:
            pass

    def frame(self):
        lib().pc_run_frame(self.h)

    def store_config(self, which):
        """(base_cell_size, level_select_k, t_max, capacity_log2, max_level, probe_window,
        evict_age_frames) of store `which` (0 Lo, 1 Lo\\E, 2 FLi, 3 Li)"""
        d = np.zeros(3)
        i = np.zeros(4, np.int32)
        lib().pc_run_store_config(self.h, which, _p(d), _p(i))
        return dict(base_cell_size=float(d[0]), level_select_k=float(d[1]), t_max=float(d[2]),
                    capacity_log2=int(i[0]), max_level=int(i[1]), probe_window=int(i[2]),
                    evict_age_frames=int(i[3]))

    def dump_snapshot(self, which, path):
        if lib().pc_run_dump_snapshot(self.h, which, str(path).encode()):
            raise RuntimeError(lib().pc_last_error().decode())

    def snapshot(self, which, path):
        self.dump_snapshot(which, path)
        return read_snapshot(path)[1]

    def stats(self, which):
        s = Stats()
        lib().pc_run_stats(self.h, which, C.byref(s))
        return {k: int(getattr(s, k)) for k, _ in Stats._fields_}

    def slots(self, which):
        cap = 1 << self.store_config(which)["capacity_log2"]
        out = np.zeros(cap, SLOT_DTYPE)
        lib().pc_run_slots(self.h, which, _p(out))
        return out
