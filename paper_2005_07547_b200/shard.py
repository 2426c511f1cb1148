"""Key-owner sharding of the field cache across ranks (one process per GPU).

Every rank keeps a full replica of each store's occupancy and committed values; rank r owns the
slot range [r*cap/world, (r+1)*cap/world).  One progressive iteration on a rank's image stripe:

  1. phase 1 on the stripe: lookups on the replica, REDs into local partial accumulators,
     new keys pending                                          (pstf_vertex_pass_local)
  2. all-gather the pending records; every rank places the union identically (the
     single-GPU deterministic placement), adding only its own records' sums   (all_gather)
  3. partial accumulators of touched non-owned slots go to their owners       (all_to_all)
  4. pass 1 of endFrame reduced across ranks (global mean c_new)              (all_reduce)
  5. owners blend + evict their range and broadcast the committed slots       (all_gather)

The protocol is written against a small backend interface so the host-side logic runs on CPU
(world-size-2 gloo tests with a CPU reference backend in tests/) as well as on GPUs (the
`CudaBackend` below: sm_100a kernels, device buffers, NCCL).  Slot placement equals the
single-GPU layout; values differ from it only in fp64 summation order.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

PENDING_BYTES, PARTIAL_BYTES, DELTA_BYTES = 64, 40, 48


class Collectives:
    """Variable-length collectives over torch.distributed byte tensors (NCCL or gloo)."""

    def __init__(self, dist, device):
        self.dist = dist
        self.device = device
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()

    def _t(self, *a, **k):
        import torch
        return torch.tensor(*a, **k)

    def all_gather_bytes(self, buf):
        """buf: 1-D uint8 tensor; returns the concatenation of every rank's buffer (rank order)."""
        import torch
        n = self._t([buf.numel()], dtype=torch.int64, device=self.device)
        sizes = torch.empty(self.world, dtype=torch.int64, device=self.device)
        self.dist.all_gather_into_tensor(sizes, n)
        sizes = [int(x) for x in sizes.tolist()]  # one host round trip for all ranks
        mx = max(sizes)
        if mx == 0:
            return torch.empty(0, dtype=torch.uint8, device=self.device)
        if buf.numel() == mx:
            pad = buf.contiguous()
        else:
            pad = torch.zeros(mx, dtype=torch.uint8, device=self.device)
            pad[:buf.numel()] = buf
        out = torch.empty(self.world * mx, dtype=torch.uint8, device=self.device)
        self.dist.all_gather_into_tensor(out, pad)  # one contiguous collective
        if all(sz == mx for sz in sizes):
            return out
        return torch.cat([out[r * mx:r * mx + sz] for r, sz in enumerate(sizes)])

    def all_gather_counted(self, count, make_buf):
        """Variable-length all-gather when the local length is only known on the device:
        count is a 1-element int64 device tensor (bytes), make_buf(n) returns the local n-byte
        buffer.  One host synchronisation for every rank's size (instead of a local readback
        followed by the size exchange)."""
        import torch
        sizes = torch.empty(self.world, dtype=torch.int64, device=self.device)
        self.dist.all_gather_into_tensor(sizes, count)
        sizes = [int(x) for x in sizes.tolist()]
        return self._gather_known(make_buf(sizes[self.rank]), sizes)

    def _gather_known(self, buf, sizes):
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

    def all_to_all_bytes(self, buf, send_counts, rec_bytes):
        """buf holds world consecutive segments of send_counts[r] records (rec_bytes each)."""
        import torch
        sc = self._t(list(send_counts), dtype=torch.int64, device=self.device)
        rc = torch.empty_like(sc)
        self.dist.all_to_all_single(rc, sc)
        recv_counts = [int(x) for x in rc.tolist()]
        out = torch.empty(sum(recv_counts) * rec_bytes, dtype=torch.uint8, device=self.device)
        self.dist.all_to_all_single(out, buf[:sum(send_counts) * rec_bytes],
                                    [c * rec_bytes for c in recv_counts],
                                    [c * rec_bytes for c in send_counts])
        return out, recv_counts

    def all_to_all_counted(self, buf, send_counts_dev, rec_bytes):
        """all_to_all_bytes with the send counts (records per destination) on the device: the
        count exchange runs there too, and one host synchronisation reads both sides"""
        import torch
        rc = torch.empty_like(send_counts_dev)
        self.dist.all_to_all_single(rc, send_counts_dev)
        both = [int(x) for x in torch.cat([send_counts_dev, rc]).tolist()]
        send, recv = both[:self.world], both[self.world:]
        out = torch.empty(sum(recv) * rec_bytes, dtype=torch.uint8, device=self.device)
        self.dist.all_to_all_single(out, buf[:sum(send) * rec_bytes],
                                    [c * rec_bytes for c in recv], [c * rec_bytes for c in send])
        return out, recv

    def all_reduce_sum(self, arr):
        """Sum over ranks: a device tensor is reduced in place (no host round trip), anything
        else goes through a float64 device tensor and comes back as numpy."""
        import torch
        if isinstance(arr, torch.Tensor) and arr.device.type == "cuda":
            self.dist.all_reduce(arr)
            return arr
        t = torch.as_tensor(np.asarray(arr, np.float64), device=self.device)
        self.dist.all_reduce(t)
        return t.cpu().numpy()


class ShardedFieldCache:
    """Drives one rank of the sharded field cache.  backend: CudaBackend or a test backend."""

    def __init__(self, backend, coll: Collectives):
        self.b = backend
        self.c = coll

    def iteration(self, stripe):
        b, c = self.b, self.c
        counted = hasattr(b, "pending_count_dev") and hasattr(c, "all_gather_counted") and \
            hasattr(c, "all_to_all_counted")
        b.vertex_pass_local(stripe)                                    # 1
        if counted:  # device-side sizes: one host sync per variable-size exchange
            recs = c.all_gather_counted(b.pending_count_dev(), b.pending_bytes_n)
        else:
            recs = c.all_gather_bytes(b.pending_bytes())               # 2
        b.resolve(recs)
        if counted:                                                    # 3
            out, counts_dev = b.partials_export_async()
            recv, _ = c.all_to_all_counted(out, counts_dev, PARTIAL_BYTES)
        else:
            out, counts = b.partials_export()
            recv, _ = c.all_to_all_bytes(out, counts, PARTIAL_BYTES)
        b.partials_import(recv)
        sums = c.all_reduce_sum(b.end_frame_reduce())                  # 4
        if counted:                                                    # 5
            buf, nd = b.end_frame_commit_async(sums)
            b.deltas_import(c.all_gather_counted(nd, lambda n: buf[:n]))
        else:
            deltas = b.end_frame_commit(sums)
            b.deltas_import(c.all_gather_bytes(deltas))


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
            "pstf_pending_count": [vp, vp], "pstf_pending_copy": [vp, vp, u64, vp],
            "pstf_resolve_records": [vp, i32, vp, u64, vp],
            "pstf_partials_export": [vp, i32, vp, u64, vp, vp],
            "pstf_partials_import": [vp, i32, vp, u64, vp],
            "pstf_end_frame_reduce": [vp, i32, vp, vp],
            "pstf_end_frame_commit": [vp, i32, vp, vp, u64, vp, vp],
            "pstf_end_frame_reduce_dev": [vp, i32, vp, vp],
            "pstf_end_frame_commit_dev": [vp, i32, vp, vp, u64, vp, vp],
            "pstf_end_frame_commit_async": [vp, i32, vp, vp, u64, vp, vp],
            "pstf_pending_count_dev": [vp, vp, vp],
            "pstf_partials_export_async": [vp, i32, vp, u64, vp, vp],
            "pstf_deltas_import": [vp, i32, vp, u64, vp], "pstf_shard_set": [vp, i32, i32],
        }.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = i32

    def _torch(self):
        import torch
        return torch

    def vertex_pass_local(self, stripe):
        buf, n = stripe
        s = self.stores
        v = self.F.vertex_soa(buf, n)
        self.F._check(self.L.pstf_vertex_pass_local(
            s[0].handle, s[1].handle, s[2].handle, self.li.handle if self.li else None,
            C.byref(v), n, self.masks[0], self.masks[1], self.F._stream()))

    def pending_bytes(self):
        torch = self._torch()
        n = C.c_uint64()
        self.F._check(self.L.pstf_pending_count(self.stores[0].handle, C.byref(n)))
        out = torch.empty(n.value * PENDING_BYTES, dtype=torch.uint8, device="cuda")
        if n.value:
            self.F._check(self.L.pstf_pending_copy(self.stores[0].handle, C.c_void_p(out.data_ptr()),
                                                   n.value, self.F._stream()))
        return out

    def pending_count_dev(self):
        """pending-record bytes of this rank as a 1-element int64 device tensor"""
        torch = self._torch()
        n = torch.empty(1, dtype=torch.int64, device="cuda")
        self.F._check(self.L.pstf_pending_count_dev(self.stores[0].handle, C.c_void_p(n.data_ptr()),
                                                    self.F._stream()))
        return n * PENDING_BYTES

    def pending_bytes_n(self, nbytes):
        """the pending records (nbytes known from the size exchange) as a uint8 device tensor"""
        torch = self._torch()
        out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        n = nbytes // PENDING_BYTES
        if n:
            self.F._check(self.L.pstf_pending_copy(self.stores[0].handle, C.c_void_p(out.data_ptr()),
                                                   n, self.F._stream()))
        return out

    def end_frame_commit_async(self, sums):
        """owners blend + evict; (delta buffer, its byte count as a device int64 tensor)"""
        torch = self._torch()
        cap = sum(s.capacity // self.world for s in self.stores)
        out = torch.empty(max(cap, 1) * DELTA_BYTES, dtype=torch.uint8, device="cuda")
        nd = torch.empty(1, dtype=torch.int64, device="cuda")
        sums = sums.to(torch.float64).contiguous()
        self.F._check(self.L.pstf_end_frame_commit_async(self._arr, len(self.stores),
                                                         C.c_void_p(sums.data_ptr()),
                                                         C.c_void_p(out.data_ptr()), max(cap, 1),
                                                         C.c_void_p(nd.data_ptr()),
                                                         self.F._stream()))
        return out, nd * DELTA_BYTES

    def resolve(self, recs):
        n = recs.numel() // PENDING_BYTES
        self.F._check(self.L.pstf_resolve_records(self._arr, len(self.stores),
                                                  C.c_void_p(recs.data_ptr()) if n else None, n,
                                                  self.F._stream()))

    def partials_export(self):
        torch = self._torch()
        cap = sum(s.capacity for s in self.stores)
        out = torch.empty(cap * PARTIAL_BYTES, dtype=torch.uint8, device="cuda")
        counts = (C.c_uint64 * self.world)()
        self.F._check(self.L.pstf_partials_export(self._arr, len(self.stores),
                                                  C.c_void_p(out.data_ptr()), cap, counts,
                                                  self.F._stream()))
        return out, [int(x) for x in counts]

    def partials_export_async(self):
        """partial records (destination-major) and the per-rank counts as a device int64
        tensor, no host round trip"""
        torch = self._torch()
        cap = sum(s.capacity for s in self.stores)
        out = torch.empty(cap * PARTIAL_BYTES, dtype=torch.uint8, device="cuda")
        counts = torch.empty(self.world, dtype=torch.int64, device="cuda")
        self.F._check(self.L.pstf_partials_export_async(self._arr, len(self.stores),
                                                        C.c_void_p(out.data_ptr()), cap,
                                                        C.c_void_p(counts.data_ptr()),
                                                        self.F._stream()))
        return out, counts

    def partials_import(self, recs):
        n = recs.numel() // PARTIAL_BYTES
        if n:
            self.F._check(self.L.pstf_partials_import(self._arr, len(self.stores),
                                                      C.c_void_p(recs.data_ptr()), n,
                                                      self.F._stream()))

    def end_frame_reduce(self):
        """(sum c_new, count) per store as a device tensor (all-reduced in place next)"""
        torch = self._torch()
        sums = torch.empty(2 * len(self.stores), dtype=torch.float64, device="cuda")
        self.F._check(self.L.pstf_end_frame_reduce_dev(self._arr, len(self.stores),
                                                       C.c_void_p(sums.data_ptr()),
                                                       self.F._stream()))
        return sums

    def end_frame_commit(self, sums):
        torch = self._torch()
        cap = sum(s.capacity for s in self.stores) // self.world
        out = torch.empty(max(cap, 1) * DELTA_BYTES, dtype=torch.uint8, device="cuda")
        nd = C.c_uint64()
        if isinstance(sums, torch.Tensor) and sums.device.type == "cuda":
            sums = sums.to(torch.float64).contiguous()
            self.F._check(self.L.pstf_end_frame_commit_dev(self._arr, len(self.stores),
                                                           C.c_void_p(sums.data_ptr()),
                                                           C.c_void_p(out.data_ptr()), max(cap, 1),
                                                           C.byref(nd), self.F._stream()))
        else:
            sums = np.ascontiguousarray(sums, np.float64)
            self.F._check(self.L.pstf_end_frame_commit(self._arr, len(self.stores),
                                                       sums.ctypes.data_as(C.c_void_p),
                                                       C.c_void_p(out.data_ptr()), max(cap, 1),
                                                       C.byref(nd), self.F._stream()))
        return out[:nd.value * DELTA_BYTES]

    def deltas_import(self, recs):
        n = recs.numel() // DELTA_BYTES
        if n:
            self.F._check(self.L.pstf_deltas_import(self._arr, len(self.stores),
                                                    C.c_void_p(recs.data_ptr()), n,
                                                    self.F._stream()))
