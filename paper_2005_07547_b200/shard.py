"""One field cache over several ranks (one process per GPU).

Every rank keeps a bitwise-identical replica of each store.  One progressive iteration on a
rank's vertices (its image stripe, or its own samples of the frame):

  1. phase 1 on the rank's vertices: lookups on the replica (committed state), REDs into the
     replica's accumulators, new keys pending                 (pstf_vertex_pass_local)
  2. the pending sizes and the live count, gathered on the device and read with the frame's
     ONE host synchronisation; all-gather the pending records; every rank places the union
     identically (the single-GPU deterministic placement) and adds its own records' sums
  3. the accumulators of the live slots, packed in slot order (the same slots in the same
     order on every rank), all-reduced (sum)                     (NCCL all-reduce)
  4. endFrame on every rank straight from the summed accumulators: identical inputs,
     identical committed state                                   (pstf_shard_end_frame)

Compared with owner-sharded blending plus a committed-delta all-gather, this moves one dense
array of (live slots x 32 B) per frame and needs no per-frame variable-size exchange besides the
(usually empty) new keys.  The protocol is written against a small backend interface so the
host-side logic runs on CPU (world-size-2/4 gloo tests with a numpy backend in tests/) as well
as on GPUs (`CudaBackend`: sm_100a kernels, device buffers, NCCL).  Slot placement, ages and
counts equal the single-GPU run; values differ from it only in fp64 summation order.
"""
from __future__ import annotations

import ctypes as C

PENDING_BYTES = 64


class Collectives:
    """The protocol's collectives over torch.distributed tensors (NCCL or gloo)."""

    def __init__(self, dist, device):
        self.dist = dist
        self.device = device
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()

    def gather_known(self, buf, sizes):
        """all-gather of byte buffers whose sizes every rank already knows (rank order)"""
        import torch
        mx = max(sizes)
        if mx == 0:
            return torch.empty(0, dtype=torch.uint8, device=self.device)
        if buf.numel() == mx:
            pad = buf.contiguous()
        else:
            pad = torch.zeros(mx, dtype=torch.uint8, device=self.device)
            pad[:buf.numel()] = buf
        out = torch.empty(self.world * mx, dtype=torch.uint8, device=self.device)
        self.dist.all_gather_into_tensor(out, pad)
        if all(sz == mx for sz in sizes):
            return out
        return torch.cat([out[r * mx:r * mx + sz] for r, sz in enumerate(sizes)])

    def all_gather_vec(self, v):
        """v: small 1-D int64 tensor on this rank; returns every rank's vector as host lists
        (rank order) — the frame's one host synchronisation"""
        import torch
        out = torch.empty(self.world * v.numel(), dtype=v.dtype, device=v.device)
        self.dist.all_gather_into_tensor(out, v.contiguous())
        flat = out.tolist()
        k = v.numel()
        return [flat[r * k:(r + 1) * k] for r in range(self.world)]

    def all_reduce_sum(self, t):
        """in-place sum over ranks of a tensor (device tensors: no host round trip)"""
        self.dist.all_reduce(t)
        return t


class ShardedFieldCache:
    """Drives one rank of the multi-GPU field cache.  backend: CudaBackend or a test backend."""

    def __init__(self, backend, coll: Collectives):
        self.b = backend
        self.c = coll

    def iteration(self, vertices):
        b, c = self.b, self.c
        b.vertex_pass_local(vertices)                                   # 1
        info = c.all_gather_vec(b.sync_vector())  # [pending records, live slots, pack overflow]
        if any(r[2] for r in info):
            raise RuntimeError("live-slot pack overflowed its bound")
        pend = [int(r[0]) for r in info]
        recs = c.gather_known(b.pending_bytes_n(pend[c.rank] * PENDING_BYTES),  # 2
                              [p * PENDING_BYTES for p in pend])
        b.resolve(recs)
        bound = int(info[0][1]) + sum(pend)  # live after placement <= live before + new keys
        packed = b.pack(bound)                                          # 3
        c.all_reduce_sum(packed)
        b.commit(packed)  # endFrame from the summed accumulators           # 4


def stripe_of(n_paths, bounces, rank, world):
    """Vertex indices (wavefront layout b*n_paths + p) of rank's image stripe: contiguous path
    range, all bounces, so next-vertex linkage stays on the rank."""
    p0 = n_paths * rank // world
    p1 = n_paths * (rank + 1) // world
    return [(b * n_paths + p0, b * n_paths + p1) for b in range(bounces)]


class CudaBackend:
    """The protocol's operations on the B200 library (device buffers throughout)."""

    def __init__(self, stores, rank, world, loe_mask=7, fli_mask=7):
        from . import field as F
        self.F = F
        self.L = F.lib()
        self.stores = [s for s in stores if s is not None]
        self.li = stores[3] if len(stores) > 3 else None
        self.masks = (loe_mask, fli_mask)
        self.world = world
        for s in self.stores:
            F._check(self.L.pstf_shard_set(s.handle, rank, world))
        self._arr = (C.c_void_p * len(self.stores))(*[s.handle.value for s in self.stores])
        L = self.L
        vp, u64, i32, u32 = C.c_void_p, C.c_uint64, C.c_int, C.c_uint32
        for name, args in {
            "pstf_vertex_pass_local": [vp, vp, vp, vp, vp, u64, u32, u32, vp],
            "pstf_pending_copy": [vp, vp, u64, vp],
            "pstf_resolve_records": [vp, i32, vp, u64, vp],
            "pstf_shard_info": [vp, i32, vp, vp],
            "pstf_shard_live_pack": [vp, i32, vp, u64, vp, vp],
            "pstf_shard_live_unpack": [vp, i32, vp, vp],
            "pstf_shard_end_frame": [vp, i32, vp, vp],
            "pstf_fields_end_frame": [vp, i32, vp], "pstf_shard_set": [vp, i32, i32],
        }.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = i32
        import torch
        self._info = torch.empty(3, dtype=torch.int64, device="cuda")
        self._live_total = torch.empty(1, dtype=torch.int64, device="cuda")
        self._packed = torch.empty(0, dtype=torch.float64, device="cuda")

    def vertex_pass_local(self, vertices):
        buf, n = vertices[:2]
        s = self.stores
        v = vertices[2] if len(vertices) > 2 else self.F.vertex_soa(buf, n)
        self.F._check(self.L.pstf_vertex_pass_local(
            s[0].handle, s[1].handle, s[2].handle, self.li.handle if self.li else None,
            C.byref(v), n, self.masks[0], self.masks[1], self.F._stream()))

    def sync_vector(self):
        """[pending records, live slots over the stores, pack overflows] (device int64[3])"""
        self.F._check(self.L.pstf_shard_info(self._arr, len(self.stores),
                                             C.c_void_p(self._info.data_ptr()), self.F._stream()))
        return self._info

    def pending_bytes_n(self, nbytes):
        """the pending records (nbytes known from the size exchange) as a uint8 device tensor"""
        import torch
        out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        n = nbytes // PENDING_BYTES
        if n:
            self.F._check(self.L.pstf_pending_copy(self.stores[0].handle,
                                                   C.c_void_p(out.data_ptr()), n,
                                                   self.F._stream()))
        return out

    def resolve(self, recs):
        n = recs.numel() // PENDING_BYTES
        self.F._check(self.L.pstf_resolve_records(self._arr, len(self.stores),
                                                  C.c_void_p(recs.data_ptr()) if n else None, n,
                                                  self.F._stream()))

    def pack(self, bound):
        """accumulators of the live slots (slot order, zero-padded): float64 tensor [bound*4]"""
        import torch
        if self._packed.numel() < 4 * bound:
            self._packed = torch.empty(max(4 * bound, 4 * 1024) * 5 // 4, dtype=torch.float64,
                                       device="cuda")
        out = self._packed[:4 * bound]
        self.F._check(self.L.pstf_shard_live_pack(self._arr, len(self.stores),
                                                  C.c_void_p(out.data_ptr()), bound,
                                                  C.c_void_p(self._live_total.data_ptr()),
                                                  self.F._stream()))
        return out

    def unpack(self, packed):
        self.F._check(self.L.pstf_shard_live_unpack(self._arr, len(self.stores),
                                                    C.c_void_p(packed.data_ptr()),
                                                    self.F._stream()))

    def end_frame(self):
        self.F._check(self.L.pstf_fields_end_frame(self._arr, len(self.stores), self.F._stream()))

    def commit(self, packed):
        """endFrame of every store from the all-reduced packed accumulators"""
        self.F._check(self.L.pstf_shard_end_frame(self._arr, len(self.stores),
                                                  C.c_void_p(packed.data_ptr()),
                                                  self.F._stream()))
