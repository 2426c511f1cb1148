"""CPU reference backend for the multi-GPU protocol (TEST INFRASTRUCTURE ONLY).

Implements the operations of paper_2005_07547_b200.shard.CudaBackend on numpy replicas of the
Lo / Lo\\E / FLi stores, with the reference semantics (keys and levels from the C restatement in
oracle/, sequential insertion in key order, field.cpp:197-263 endFrame) and the same pending
record layout and live-slot packing order, so tests/test_shard_gloo.py can run the multi-rank
protocol with gloo on CPU and compare the result with a single-process oracle run."""
import numpy as np

import pyoracle as po

PEND_DT = np.dtype([("k", "<i4", (6,)), ("cs", "<u4"), ("meta", "<u4"), ("v", "<f8", (4,))])
assert PEND_DT.itemsize == 64
M64 = (1 << 64) - 1


def mix(v):
    v = int(v) & M64
    v ^= v >> 30
    v = (v * 0xbf58476d1ce4e5b9) & M64
    v ^= v >> 27
    v = (v * 0x94d049bb133111eb) & M64
    v ^= v >> 31
    return v


def pack(k):
    u = [int(x) & 0xffffffff for x in k]
    h = u[0]
    h = mix(h ^ ((u[1] << 32) | u[2]))
    h = mix(h ^ ((u[3] << 32) | u[4]))
    return mix(h ^ u[5])


class Replica:
    def __init__(self, cfg: po.Config, rank, world):
        self.cfg = cfg
        self.cap = 1 << cfg.capacity_log2
        self.mask = self.cap - 1
        self.chk = np.zeros(self.cap, np.uint32)
        self.lastb = np.zeros(self.cap, np.uint32)
        self.keyf = np.zeros((self.cap, 6), np.int32)
        self.acc = np.zeros((self.cap, 4))
        self.com = np.zeros((self.cap, 4))
        self.touched = np.zeros(self.cap, bool)
        self.frame = 0
        self.live = 0
        self.dropped = 0
        self.rank = rank
        self.internal = 0

    def touch(self, slot):
        self.lastb[slot] = (self.frame + 1) & 0xffffffff
        self.touched[slot] = True

    def probe_existing(self, home, cs):
        for i in range(self.cfg.probe_window):
            idx = (home + i) & self.mask
            c = self.chk[idx]
            if c == cs:
                return idx
            if c == 0:
                return -1
        return -2

    def find(self, home, cs):
        r = self.probe_existing(home, cs)
        return r if r >= 0 else -1


class CpuBackend:
    def __init__(self, cfgs, rank, world):
        self.reps = [Replica(c, rank, world) for c in cfgs]
        self.keycalc = po.OracleStore(cfgs[0])  # key math (all stores share the quantisation)
        self.rank, self.world = rank, world
        self.pending = np.zeros(0, PEND_DT)

    # ---------------------------------------------------------------- phase 1
    def _keys(self, pos, d, lv):
        k = self.keycalc.keys_for(pos, d, lv)
        return np.stack([k["level"], k["cell"][:, 0], k["cell"][:, 1], k["cell"][:, 2],
                         k["dir"][:, 0], k["dir"][:, 1]], 1), k["checksum"]

    def vertex_pass_local(self, stripe):
        buf, n = stripe
        f64, flags = po.soa_views(buf, n)
        F = lambda k: f64[k]
        cont = (flags & 1) != 0
        nsurf = (flags & 2) != 0
        nee = (flags & 4) != 0
        lv = self.keycalc.select_levels(F(15))
        pos = f64[0:3].T
        lo, loe, fli = self.reps
        # lookups at the next vertex on the replica (estimators.cpp:197-211)
        loN = np.zeros((n, 3))
        loeN = np.zeros((n, 3))
        look = cont & nsurf
        npos = f64[9:12].T
        mwi = -f64[6:9].T
        l0 = self.keycalc.select_levels(F(16))
        doneLo = ~look
        doneLoe = ~look
        for l in range(self.keycalc.config.max_level + 1):
            act = np.nonzero(look & (l0 <= l) & ~(doneLo & doneLoe))[0]
            if len(act) == 0:
                continue
            ks, cs = self._keys(npos[act], mwi[act], np.full(len(act), l, np.int32))
            for j, i in enumerate(act):
                home = pack(ks[j]) & lo.mask
                for rep, done, out in ((lo, doneLo, loN), (loe, doneLoe, loeN)):
                    if done[i]:
                        continue
                    idx = rep.find(home, cs[j])
                    if idx >= 0 and rep.com[idx, 3] > 0.0:
                        out[i] = rep.com[idx, :3]
                        done[i] = True
        env = cont & ~nsurf
        loN[env] = f64[25:28].T[env]
        # update values (field.cpp:13-25 order)
        ratio, nmis = F(17), F(18)
        fr = f64[22:25].T
        ne = f64[25:28].T
        transp = cont & (ratio > 0)
        le = ne * nmis[:, None]
        lin = le + loeN
        vlo = np.zeros((n, 4))
        vlo[:, 3] = 1.0
        vlo[:, :3] = f64[19:22].T + np.where(transp[:, None], ((0.0 + loN) * fr) * ratio[:, None], 0.0)
        vle = np.zeros((n, 4))
        vle[:, 3] = 1.0
        vle[:, :3] = np.where(transp[:, None], ((le + loeN) * fr) * ratio[:, None], 0.0) + \
            np.where(nee[:, None], f64[28:31].T, 0.0)
        vfc = np.zeros((n, 4))
        vfc[:, 3] = 1.0
        vfc[:, :3] = fr * lin
        vfn = np.zeros((n, 4))
        vfn[:, 3] = 1.0
        vfn[:, :3] = f64[31:34].T
        ncalls_lo = 2 + transp.astype(int)
        ncalls_le = 1 + transp.astype(int) + nee.astype(int)
        kLo, csLo = self._keys(pos, f64[3:6].T, lv)
        kFc, csFc = self._keys(pos, f64[6:9].T, lv)
        kFn, csFn = self._keys(pos, f64[12:15].T, lv)
        recs = []
        work = [(0, lo, kLo, csLo, vlo, ncalls_lo, np.ones(n, bool)),
                (1, loe, kLo, csLo, vle, ncalls_le, np.ones(n, bool)),
                (2, fli, kFc, csFc, vfc, np.full(n, 2), cont),
                (2, fli, kFn, csFn, vfn, np.full(n, 2), nee)]
        for sid, rep, ks, cs, vals, calls, has in work:
            for i in np.nonzero(has)[0]:
                home = pack(ks[i]) & rep.mask
                r = rep.probe_existing(home, cs[i])
                if r >= 0:
                    rep.acc[r] += vals[i]
                    rep.touch(r)
                elif r == -1:
                    rec = np.zeros(1, PEND_DT)
                    rec["k"] = ks[i]
                    rec["cs"] = cs[i]
                    rec["meta"] = sid | (self.rank << 3) | (int(calls[i]) << 8)
                    rec["v"] = vals[i]
                    recs.append(rec)
                else:
                    rep.dropped += int(calls[i])
        self.pending = np.concatenate(recs) if recs else np.zeros(0, PEND_DT)

    def sync_vector(self):
        import torch
        return torch.tensor([len(self.pending), sum(r.live for r in self.reps), 0],
                            dtype=torch.int64)

    def pending_bytes_n(self, nbytes):
        import torch
        assert nbytes == self.pending.nbytes
        return torch.from_numpy(self.pending.view(np.uint8).copy())

    # ---------------------------------------------------------------- placement
    def resolve(self, recs_t):
        recs = np.frombuffer(recs_t.numpy().tobytes(), PEND_DT)
        sid = recs["meta"] & 3
        origin = (recs["meta"] >> 3) & 31
        calls = recs["meta"] >> 8
        for s, rep in enumerate(self.reps):
            sel = np.nonzero(sid == s)[0]
            groups = {}
            for i in sel:
                groups.setdefault(tuple(int(x) for x in recs["k"][i]), []).append(i)
            for key in sorted(groups):  # sequential insertion in key order (field.cpp:402-406)
                idxs = groups[key]
                cs = int(recs["cs"][idxs[0]])
                home = pack(key) & rep.mask
                target = -1
                for j in range(rep.cfg.probe_window):
                    t = (home + j) & rep.mask
                    if rep.chk[t] == cs:
                        target = t
                        break
                    if rep.chk[t] == 0:
                        rep.chk[t] = cs
                        rep.keyf[t] = key
                        rep.live += 1
                        target = t
                        break
                own = [i for i in idxs if origin[i] == self.rank]
                own_calls = int(sum(calls[i] for i in own))
                if target < 0:
                    rep.dropped += own_calls
                    continue
                for i in own:
                    rep.acc[target] += recs["v"][i]
                if own_calls:
                    rep.touch(target)

    # ---------------------------------------------------------------- exchange
    def pack(self, bound):
        """accumulators of the live slots in (store, slot) order, zero-padded to bound"""
        import torch
        self.plist = [(s, int(slot)) for s, rep in enumerate(self.reps)
                      for slot in np.nonzero(rep.chk)[0]]
        assert len(self.plist) <= bound
        out = np.zeros((bound, 4))
        for i, (s, slot) in enumerate(self.plist):
            out[i] = self.reps[s].acc[slot]
        return torch.from_numpy(out.reshape(-1))

    def unpack(self, packed):
        v = packed.numpy().reshape(-1, 4)
        for i, (s, slot) in enumerate(self.plist):
            rep = self.reps[s]
            rep.acc[slot] = v[i]
            if (v[i] != 0).any():
                rep.touch(slot)

    # ---------------------------------------------------------------- endFrame
    def commit(self, packed):
        self.unpack(packed)
        self.end_frame()

    def end_frame(self):
        """field.cpp:197-263 on every store (all slots; untouched ones have zero accumulators)"""
        for rep in self.reps:
            live_snap = rep.live
            cn_all = rep.acc[:, 3]
            pos = (rep.chk != 0) & (cn_all > 0)
            mean = float(cn_all[pos].sum()) / pos.sum() if pos.any() else 0.0
            T = rep.cfg.t_max
            limited = T > 0 and np.isfinite(T)
            cap = (T * T - T) * mean if limited else 0.0
            for slot in np.nonzero(rep.chk)[0]:
                a = rep.acc[slot]
                cn = a[3]
                if cn > 0:
                    c = rep.com[slot]
                    cand = a[:3] / cn
                    alpha = np.sqrt(cn / (c[3] + cn)) if rep.cfg.blend == 0 else cn / (c[3] + cn)
                    if limited:
                        alpha = 1.0 / T if alpha < 1.0 / T else alpha  # std::max(alpha, 1/T)
                    c[:3] = c[:3] * (1.0 - alpha) + cand * alpha
                    c[3] = c[3] + cn
                    if limited:
                        c[3] = cap if cap < c[3] else c[3]
                elif (a[:3] != 0).any():
                    rep.internal += 1
                rep.acc[slot] = 0.0
            if live_snap * 4 > rep.cap * 3:
                for slot in np.nonzero(rep.chk)[0]:
                    if ((rep.frame - (int(rep.lastb[slot]) - 1)) & 0xffffffff) >= \
                            rep.cfg.evict_age_frames:
                        rep.chk[slot] = 0
                        rep.com[slot] = 0.0
                        rep.live -= 1
            rep.touched[:] = False
            rep.frame += 1
