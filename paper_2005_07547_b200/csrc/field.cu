/*
 * field.cu — B200-native PSTF field cache: sm_100a kernels + host orchestration + C ABI.
 *
 * Reference semantics: /root/reference/proj/core/src/field.cpp (FieldStore, FieldUpdateQueue)
 * and estimators.cpp:194-262 (FieldRecorder::onVertex).  Design: DESIGN.md.
 *
 * Per frame the update path is
 *   phase 1  one fused pass over the vertex (or update) stream: keys, committed-state lookups,
 *            update values; updates whose key already owns a slot reachable before any empty
 *            slot are added straight into the slot with warp-aggregated fp64 RED; updates of
 *            keys that would insert go to a pending buffer.
 *   phase 2  pending keys are sorted (priority order), de-duplicated and placed by a parallel
 *            deterministic deferred-acceptance loop whose fixpoint is exactly the slot layout of
 *            sequential insertion in priority order (field.cpp:116-146 applied in the order of
 *            FieldUpdateQueue::apply, field.cpp:396-420); then their sums are committed.
 *   endFrame two sweeps over the 8 B slot words of all stores of the batch: mean c_new of the
 *            slots touched this frame, then blend + cap + zero accumulators, fused with the
 *            age-eviction rule when the table is more than 3/4 full (field.cpp:197-263).
 */
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <tuple>
#include <mutex>
#include <new>
#include <set>
#include <string>
#include <vector>

#include <cooperative_groups.h>
#include <cub/cub.cuh>
namespace cg = cooperative_groups;

#include "../../include/pstf_field.h"
#include "kernels.cuh"
#include "pstf_keys.cuh"
#include "pstf_synth.h"
#include "store.cuh"

using namespace pstf_b200;

/* ------------------------------------------------------------------------------------------ */
/* errors, launch accounting                                                                   */

static thread_local std::string g_last_error;
static std::atomic<unsigned long long> g_launches{0};

static int set_err(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

#define CK(call)                                                                            \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return set_err(PSTF_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

/* Optional per-kernel CUDA-event timing on the launching stream (bench.py roofline). */
static std::atomic<int> g_prof{0};
static std::mutex g_prof_mu;
struct ProfRec {
    const char *name;
    cudaEvent_t a, b;
};
static std::vector<ProfRec> g_prof_recs;
static std::vector<cudaEvent_t> g_prof_pool;

static cudaEvent_t prof_event() {
    cudaEvent_t e = nullptr;
    if (!g_prof_pool.empty()) {
        e = g_prof_pool.back();
        g_prof_pool.pop_back();
    } else {
        cudaEventCreate(&e);
    }
    return e;
}

struct ProfScope {
    const char *name;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    ProfScope(const char *n, cudaStream_t s) : name(n), st(s) {
        if (g_prof.load(std::memory_order_relaxed)) {
            std::lock_guard<std::mutex> lk(g_prof_mu);
            a = prof_event();
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope() {
        if (a) {
            std::lock_guard<std::mutex> lk(g_prof_mu);
            cudaEvent_t b = prof_event();
            cudaEventRecord(b, st);
            g_prof_recs.push_back({name, a, b});
        }
    }
};

#define LAUNCH(kernel, grid, block, smem, stream, ...)                                      \
    do {                                                                                    \
        ProfScope ps_(#kernel, (stream));                                                   \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                         \
        g_launches.fetch_add(1, std::memory_order_relaxed);                                 \
        cudaError_t e_ = cudaGetLastError();                                                \
        if (e_ != cudaSuccess)                                                              \
            return set_err(PSTF_E_CUDA, std::string(#kernel) + ": " + cudaGetErrorString(e_)); \
    } while (0)

static unsigned grid_for(uint64_t n, unsigned block) {
    uint64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > 0x7fffffffULL) g = 0x7fffffffULL;
    return (unsigned)g;
}

static int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

/* ------------------------------------------------------------------------------------------ */
/* device buffers                                                                              */

struct DBuf {
    void *p = nullptr;
    size_t bytes = 0;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t ensure(size_t need) {
        if (need <= bytes) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        size_t nb = std::max(need, (size_t)256);
        nb = nb + nb / 4;
        cudaError_t e = cudaMalloc(&p, nb);
        if (e == cudaSuccess) bytes = nb;
        return e;
    }
    template <class T> T *as() const { return reinterpret_cast<T *>(p); }
};

#define ENSURE(buf, nbytes) CK((buf).ensure(nbytes))

struct Scratch {
    DBuf pend, pend_seq, pend_count;
    DBuf valid, scan;                       // apply(): order-preserving compaction
    DBuf ranges;                            // int32 min/max of 7 key fields
    DBuf words;                             // packed sort words [nw][N]
    DBuf ktmp0, ktmp1, perm0, perm1, cub;   // radix sort
    DBuf head, uid, ufirst, ukey, ucs, usid, uhome, ucalls, usum, ures0, ures1, rank, csr, useq;
    DBuf changed;
    DBuf ddtab, rep_of, uidx, ukw, nudev;   // sort-free ATOMIC phase 2
    DBuf ftgt, fperm, fkey_out, fperm_out;  // ORDERED / SEQUENTIAL fold
    DBuf snap;                              // snapshot gather
    DBuf fterms, fisc, fstart, fnruns;      // ORDERED/SEQUENTIAL fold: terms, run starts
    DBuf winner;                            // snapshot restore: last record per slot
    DBuf hio;                               // host-pointer API staging
    DBuf ulist, overflow;                   // sharding: packed live list, pack-overflow flag
    DBuf ef_done;                           // one-pass endFrame: blocks done (last rolls)
    DBuf pend2_key, pend2_val, pend2_count; // ORDERED: value calls of existing slots
    DBuf o_key, o_key2, o_idx, o_idx2, o_tgt, o_flag; // their slot-grouped sort (o_tgt: run marks)
    DBuf o_fp, o_fk;                                  // its marked runs' re-sort
    DBuf cn_cnt, cn_vals;                             // endFrame: Σc_new in slot order
    DBuf iota;                                        // 0, 1, 2, ... (iota_n entries written)
    uint64_t iota_n = 0;
    uint64_t live_bound = 0;
    long long *live_total_dev = nullptr;
    bool overflow_zeroed = false;
    unsigned long long *h_small = nullptr;  // pinned readback
    ~Scratch() {
        if (h_small) cudaFreeHost(h_small);
    }
};

/* A vertex pass whose phase 2 (new-key placement) may still be owed: pstf_vertex_pass returns
 * right after phase 1 with the pending count on its way to pinned host memory, and the next
 * entry point that touches one of its stores settles it.  pstf_fields_end_frame settles it for
 * free in the common case: it enqueues endFrame guarded by the device-side count (the kernels
 * return at once when new keys are pending), so when there are none the GPU never idles. */
struct DeferredPass {
    bool active = false;
    pstf_field *fs[4] = {nullptr, nullptr, nullptr, nullptr};
    int nf = 0, mode = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t ev = nullptr;
    unsigned long long *h_count = nullptr; /* pinned */
};

struct pstf_field {
    pstf_field_config cfg;
    int device = 0;
    uint64_t frame = 0;
    DevStore d;
    uint32_t *hold[2] = {nullptr, nullptr};
    void *arena = nullptr;
    Scratch sc;
    std::mutex host_mu; /* serialises the host-pointer (scalar facade) entry points */
    int world = 1;      /* key-owner sharding */
    DBuf hold64;                  /* 2 x capacity 64-bit priority holds (sort-free phase 2) */
    DeferredPass dp;              /* owned by the Lo store of a deferred vertex pass */
    pstf_field *owed_by = nullptr; /* the Lo store whose deferred pass involves this store */
    /* every update of the current frame carried unit counter weights and was counted in
     * C_F_CN (tiled ATOMIC vertex passes + their placement): endFrame may run in one pass
     * (k_ef_onepass + k_ef_tail).  Any other update path clears it until the next endFrame. */
    bool unit_frame = true;
    /* pstf_field_apply with counter calls this frame: their weights may make Σc_new inexact */
    bool counted_apply = false;
    /* hot-slot detection for the tiled vertex pass (this store as its Lo store): the last
     * frame's REDs per touched slot, copied back asynchronously after endFrame */
    unsigned long long *rd_host = nullptr; /* mapped pinned: {reds_total, touched slots} */
    cudaEvent_t rd_ev = nullptr;
    bool rd_pending = false, rd_probe = false, agg = false;
    /* Twin stores: a Lo and a Lo\E store created alike and, since creation, updated only by
     * the same vertex passes and end-framed together receive the same keys, counters and
     * touches (estimators.cpp:219,227: Lo\E's key is the Lo key), so their occupancy and
     * touch marks are identical and the tiled kernel takes Lo\E's probes from Lo's (one probe
     * and one lookup word fewer per vertex).  Any other update of either store, or a pass
     * pairing it differently, ends the relation for good (twin_break). */
    pstf_field *twin = nullptr;
    bool pristine = true; /* nothing has touched the store since creation */
    ~pstf_field() {
        if (dp.ev) cudaEventDestroy(dp.ev);
        if (dp.h_count) cudaFreeHost(dp.h_count);
        if (rd_ev) cudaEventDestroy(rd_ev);
        if (rd_host) cudaFreeHost(rd_host);
    }
};

static DevStore dev_view(const pstf_field *f) {
    DevStore s = f->d;
    s.frame = (uint32_t)f->frame;
    return s;
}

/* ------------------------------------------------------------------------------------------ */
/* K1: select_level / key_for batch                                                            */

__global__ void k_select_level(KeyParams kp, const double *fp, int32_t *out, uint64_t n) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = select_level(kp, fp[i]);
}

__global__ void k_key_for(KeyParams kp, pstf_vec3_soa pos, pstf_vec3_soa dir, const int32_t *level,
                          uint64_t n, pstf_key *out) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    Key k = key_for(kp, pos.x[i], pos.y[i], pos.z[i], dir.x[i], dir.y[i], dir.z[i], level[i]);
    pstf_key o;
    o.level = k.level;
    o.cell[0] = k.cell[0];
    o.cell[1] = k.cell[1];
    o.cell[2] = k.cell[2];
    o.dir_cell[0] = k.dir[0];
    o.dir_cell[1] = k.dir[1];
    o.checksum = k.checksum;
    out[i] = o;
}

/* ------------------------------------------------------------------------------------------ */
/* K4: hierarchical lookup (queryFromLevel, field.cpp:179-195)                                 */

__device__ __forceinline__ bool lookup_level_chain(const DevStore &s, double px, double py,
                                                   double pz, double dx, double dy, double dz,
                                                   int level, double3 *val, int *lev_out) {
    for (int l = level; l <= s.kp.max_level; ++l) {
        Key k = key_for(s.kp, px, py, pz, dx, dy, dz, l);
        int idx = probe_find(s, (uint32_t)key_pack(k) & s.mask, k.checksum);
        if (idx >= 0) {
            double4 c = ld4_ro(com_ptr(s, idx));
            if (c.w > 0.0) {
                *val = make_double3(c.x, c.y, c.z);
                *lev_out = l;
                return true;
            }
        }
    }
    *lev_out = level;
    return false;
}

__global__ void k_query(DevStore s, pstf_vec3_soa pos, pstf_vec3_soa dir, const double *fp,
                        const int32_t *level, uint64_t n, double *vr, double *vg, double *vb,
                        uint8_t *valid, uint8_t *fallback, int32_t *olevel) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int l0 = fp ? select_level(s.kp, fp[i]) : level[i];
    double3 v = make_double3(0.0, 0.0, 0.0);
    int lo;
    bool ok = lookup_level_chain(s, pos.x[i], pos.y[i], pos.z[i], dir.x[i], dir.y[i], dir.z[i], l0,
                                 &v, &lo);
    if (!ok) v = make_double3(0.0, 0.0, 0.0);
    if (vr) vr[i] = v.x;
    if (vg) vg[i] = v.y;
    if (vb) vb[i] = v.z;
    if (valid) valid[i] = ok;
    if (fallback) fallback[i] = ok && lo != l0;
    if (olevel) olevel[i] = lo;
}

/* ------------------------------------------------------------------------------------------ */
/* K5: fused vertex pass (phase 1)                                                             */

struct VPArgs {
    Stores4 st;
    int has_li;
    int same_lo_loe, same_fli_lo, same_li_fli;
    uint32_t loe_mask, fli_mask;
    pstf_vertex_soa v;
    uint64_t n;
    PendRec *pend;
    unsigned long long *pend_count;
    uint64_t pend_cap;
    /* ORDERED: value calls whose key already owns a slot (phase 1 found it) go here as (sort
     * key, value) pairs for the slot-grouped fold (fold_slot_records) */
    uint64_t *pend2_key;
    double4 *pend2_val;
    unsigned long long *pend2_count; /* [0] calls, [1] checksum alias seen */
    uint64_t pend2_cap;
    int pend2_capl; /* the stores' largest capacity_log2 (the key's slot field width) */
};

#define VP_BLOCK 256
#define WARPS_PER_BLOCK (VP_BLOCK / 32)

struct PendSink {
    PendRec *pend;
    unsigned long long *count;
    uint64_t cap;
};

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

/* isfinite(a) && isfinite(b) && isfinite(c) on the exponent fields (integer pipe) */
__device__ __forceinline__ bool finite3(double a, double b, double c) {
    const int ea = __double2hiint(a) & 0x7ff00000, eb = __double2hiint(b) & 0x7ff00000,
              ec = __double2hiint(c) & 0x7ff00000;
    return max(ea, max(eb, ec)) != 0x7ff00000;
}

/* Reserves pending-record positions with one atomic per warp; all 32 lanes must call it.
 * Returns this lane's record, or nullptr (not wanted / buffer full: the host sees the count). */
__device__ __forceinline__ PendRec *warp_reserve(const PendSink &a, bool want) {
    unsigned m = __ballot_sync(0xffffffffu, want);
    if (!m) return nullptr;
    unsigned lane = lane_id();
    int leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if ((int)lane == leader) base = atomicAdd(a.count, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    const unsigned long long pos = base + __popc(m & ((1u << lane) - 1u));
    return want && pos < a.cap ? a.pend + pos : nullptr;
}

/* one 64 B record written as four 16 B stores straight from registers (no local-memory copy) */
__device__ __forceinline__ void put_record(PendRec *p, const Key &k, uint32_t meta, double v0,
                                           double v1, double v2, double v3) {
    int4 *q = reinterpret_cast<int4 *>(p);
    q[0] = make_int4(k.level, k.cell[0], k.cell[1], k.cell[2]);
    q[1] = make_int4(k.dir[0], k.dir[1], (int)k.checksum, (int)meta);
    reinterpret_cast<double2 *>(p)[2] = make_double2(v0, v1);
    reinterpret_cast<double2 *>(p)[3] = make_double2(v2, v3);
}

/* One update slot of the vertex (ATOMIC mode), executed by all 32 lanes in lock-step:
 * probe the frame-start table; existing slot -> warp-aggregated RED; empty-first -> pending;
 * exhausted -> dropped. */
__device__ __forceinline__ void red_add4(double4 *dst, double4 t) {
    if (t.x != 0.0) atomicAdd(&dst->x, t.x);
    if (t.y != 0.0) atomicAdd(&dst->y, t.y);
    if (t.z != 0.0) atomicAdd(&dst->z, t.z);
    if (t.w != 0.0) atomicAdd(&dst->w, t.w);
}

/* res: >= 0 existing slot, -1 new key, -2 dropped, -3 no update; mark = slot's meta.y */
template <class Store>
__device__ __forceinline__ void apply_contribution(const Store &s, const PendSink &a,
                                                   double4 *sm, int sid, const Key &k, double4 v,
                                                   uint32_t ncalls, int res, uint32_t mark,
                                                   bool do_red = true, bool aggregate = true,
                                                   uint32_t *nred = nullptr) {
    unsigned lane = lane_id();
    unsigned long long gk = res >= 0 ? (((unsigned long long)sid << 32) | (unsigned)res)
                                     : (0xffffffff00000000ull | lane);
    unsigned peers = aggregate ? __match_any_sync(0xffffffffu, gk) : (1u << lane);
    if (!aggregate) {
        /* Sector-coalesced REDs: the warp's 32 cells x 4 components are transposed through
         * shared memory so each RED instruction covers 8 cells x {r,g,b,c}; the 4 lanes of a
         * cell hit one 32 B sector, so L1 sends 8 sector requests per instruction, not 32. */
        int *rsm = reinterpret_cast<int *>(sm + 32);
        sm[lane] = v;
        rsm[lane] = do_red ? res : -3;
        __syncwarp();
        const double *flat = reinterpret_cast<const double *>(sm);
        const int comp = lane & 3;
        uint32_t cnt = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int cell = 8 * k + (lane >> 2);
            const int rs = rsm[cell];
            const double val = flat[4 * cell + comp];
            const bool on = rs >= 0 && val != 0.0;
            if (on) atomicAdd(reinterpret_cast<double *>(acc_ptr(s, rs)) + comp, val);
            cnt += on;
        }
        if (nred) *nred += cnt;
        __syncwarp();
        if (res >= 0) touch_slot(s, (uint32_t)res, mark);
    } else if (__all_sync(0xffffffffu, peers == (1u << lane))) {
        /* no two lanes share a slot: one RED per component, no shared-memory round trip */
        if (res >= 0) {
            if (do_red) red_add4(acc_ptr(s, res), v);
            touch_slot(s, (uint32_t)res, mark);
        }
    } else {
        sm[lane] = v;
        __syncwarp();
        if (res >= 0 && (int)lane == __ffs(peers) - 1) {
            double4 t = make_double4(0.0, 0.0, 0.0, 0.0);
            unsigned m = peers;
            while (m) {
                int j = __ffs(m) - 1;
                m &= m - 1;
                double4 x = sm[j];
                t.x += x.x;
                t.y += x.y;
                t.z += x.z;
                t.w += x.w;
            }
            if (do_red) red_add4(acc_ptr(s, res), t);
            touch_slot(s, (uint32_t)res, mark);
        }
        __syncwarp();
    }
    if (PendRec *p = warp_reserve(a, res == -1))
        put_record(p, k, PSTF_META(sid, 0, ncalls) | ((uint32_t)s.rank << 3), v.x, v.y, v.z, v.w);
    if (res == -2) atomicAdd(&s.ctr[C_DROPPED], (unsigned long long)ncalls);
}

__device__ __forceinline__ void contribute_atomic(const DevStore &s, const PendSink &a, double4 *sm,
                                                  int sid, bool has, const Key &k, double4 v,
                                                  uint32_t ncalls, bool do_red = true) {
    int res = -3;
    uint32_t mark = 0;
    if (has) res = probe_existing(s, k.pack_lo & s.mask, k.checksum, &mark);
    apply_contribution(s, a, sm, sid, k, v, ncalls, res, mark, do_red);
}

/* ORDERED mode, counter calls of the vertex pass (weight 1.0, estimators.cpp:219,227,243,249):
 * cNew only ever receives whole numbers, so its sum is exact in any order.  An existing key's
 * counter is therefore applied in place (cNew += 1, lastTouched = frame: field.cpp:122-124,
 * 157) and only a new key's counter becomes a record (its placement needs one); a full window
 * counts the drop (field.cpp:145).  A key that matches a slot's checksum but not its key fields
 * (a checksum alias: the reference shares the slot, field.cpp:103-113) returns -4 and raises
 * *alias: its value calls become full records, and the pass takes the general path. */
__device__ __forceinline__ int count_call(const DevStore &s, const PendSink &a, bool want,
                                          int sid, const Key &k, unsigned long long *alias) {
    int res = -3;
    uint32_t mark = 0;
    if (want) res = probe_existing(s, k.pack_lo & s.mask, k.checksum, &mark);
    if (res >= 0) {
        atomicAdd(&acc_ptr(s, res)->w, 1.0);
        touch_slot(s, (uint32_t)res, mark);
        const KeyFields kf = s.keyf[res];
        if (kf.level != k.level || kf.c0 != k.cell[0] || kf.c1 != k.cell[1] ||
            kf.c2 != k.cell[2] || kf.d0 != k.dir[0] || kf.d1 != k.dir[1]) {
            atomicOr(alias, 1ull);
            res = -4;
        }
    }
    if (PendRec *p = warp_reserve(a, res == -1))
        put_record(p, k, PSTF_META(sid, 1, 1) | ((uint32_t)s.rank << 3), 0.0, 0.0, 0.0, 1.0);
    if (res == -2) atomicAdd(&s.ctr[C_DROPPED], 1ull);
    return res;
}

/* ORDERED mode, the vertex's value calls (weight 1.0), all 32 lanes together.  Calls of a key
 * whose counter call found its slot become (sort key, value) pairs, one reservation per warp
 * for all seven call sites (an all-zero value is a no-op on the accumulator — it starts at +0.0
 * and can never become -0.0 — and is not emitted); a new key's (or an alias's) calls become
 * full pending records; a call whose window is full counts one drop (field.cpp:145). */
struct VCall {
    bool want;
    int res;
    double r, g, b;
};

__device__ __forceinline__ void value_calls(const VPArgs &a, const PendSink &ps, const VCall *c,
                                            const Key &kLo, const Key &kLoe, const Key &kFc,
                                            const Key &kFn, const Key &kLi) {
    const unsigned lane = lane_id(), lt = (1u << lane) - 1u;
    const int capl = a.pend2_capl, S = capl + 2;
    unsigned m[7], tot = 0;
#pragma unroll
    for (int q = 0; q < 7; ++q) {
        const bool zero = c[q].r == 0.0 && c[q].g == 0.0 && c[q].b == 0.0;
        m[q] = __ballot_sync(0xffffffffu, c[q].want && c[q].res >= 0 && !zero);
        tot += __popc(m[q]);
    }
    if (tot) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(a.pend2_count, (unsigned long long)tot);
        base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
        for (int q = 0; q < 7; ++q) {
            if ((m[q] >> lane) & 1u) {
                const unsigned long long pos = base + __popc(m[q] & lt);
                if (pos < a.pend2_cap) {
                    const uint64_t sid = q < 2 ? 0 : q < 4 ? 1 : q < 6 ? 2 : 3;
                    const uint64_t sk = (sid << capl) | (uint32_t)c[q].res;
                    a.pend2_key[pos] = (sk << (64 - S)) | (dbits(c[q].r) >> S);
                    a.pend2_val[pos] = make_double4(c[q].r, c[q].g, c[q].b, 0.0);
                }
            }
            base += __popc(m[q]);
        }
    }
#pragma unroll
    for (int q = 0; q < 7; ++q) {
        const int sid = q < 2 ? 0 : q < 4 ? 1 : q < 6 ? 2 : 3;
        const Key &k = q < 2 ? kLo : q < 4 ? kLoe : q == 4 ? kFc : q == 5 ? kFn : kLi;
        if (PendRec *p = warp_reserve(ps, c[q].want && (c[q].res == -1 || c[q].res == -4)))
            put_record(p, k, PSTF_META(sid, 0, 1), c[q].r, c[q].g, c[q].b, 1.0);
        if (c[q].want && c[q].res == -2) atomicAdd(&a.st.s[sid].ctr[C_DROPPED], 1ull);
    }
}


template <int MODE>
__global__ void __launch_bounds__(VP_BLOCK) k_vertex_pass(VPArgs a) {
    __shared__ double4 smem[WARPS_PER_BLOCK][36];
    double4 *sm = smem[threadIdx.x >> 5];
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const bool live = i < a.n;
    const uint64_t ii = live ? i : 0;
    const pstf_vertex_soa &V = a.v;
    const DevStore &sLo = a.st.s[0];
    const DevStore &sLoe = a.st.s[1];
    const DevStore &sFli = a.st.s[2];
    const DevStore &sLi = a.st.s[3];

    uint32_t fl = live ? __ldg(&V.flags[ii]) : 0u;
    const bool cont = (fl & PSTF_VERTEX_CONT_EXTENDED) != 0;
    const bool nsurf = (fl & PSTF_VERTEX_NEXT_IS_SURFACE) != 0;
    const bool nee = (fl & PSTF_VERTEX_NEE_SAMPLED) != 0;

    const double px = __ldg(&V.position.x[ii]), py = __ldg(&V.position.y[ii]),
                 pz = __ldg(&V.position.z[ii]);
    const double wox = __ldg(&V.wo.x[ii]), woy = __ldg(&V.wo.y[ii]), woz = __ldg(&V.wo.z[ii]);
    const double wix = __ldg(&V.wi.x[ii]), wiy = __ldg(&V.wi.y[ii]), wiz = __ldg(&V.wi.z[ii]);
    const double fp = __ldg(&V.footprint[ii]);
    const int level = select_level(sLo.kp, fp); /* estimators.cpp:195 */

    /* next-vertex lookups on committed state (estimators.cpp:197-211) */
    double3 loNext = make_double3(0.0, 0.0, 0.0), loeNext = make_double3(0.0, 0.0, 0.0);
    const double nex = __ldg(&V.next_emission.x[ii]), ney = __ldg(&V.next_emission.y[ii]),
                 nez = __ldg(&V.next_emission.z[ii]);
    if (live && cont) {
        if (nsurf) {
            const double qx = __ldg(&V.next_position.x[ii]), qy = __ldg(&V.next_position.y[ii]),
                         qz = __ldg(&V.next_position.z[ii]);
            const double nfp = __ldg(&V.next_footprint[ii]);
            const double dx = -wix, dy = -wiy, dz = -wiz;
            int lq;
            double3 r;
            if (a.same_lo_loe) {
                /* Lo and LoE share the quantisation: one key per level, two probes */
                int l0 = select_level(sLo.kp, nfp);
                bool doneLo = false, doneLoe = false;
                for (int l = l0; l <= sLo.kp.max_level && !(doneLo && doneLoe); ++l) {
                    Key k = key_for(sLo.kp, qx, qy, qz, dx, dy, dz, l);
                    uint64_t pk = key_pack(k);
                    if (!doneLo) {
                        int idx = probe_find(sLo, (uint32_t)pk & sLo.mask, k.checksum);
                        if (idx >= 0) {
                            double4 c = ld4_ro(com_ptr(sLo, idx));
                            if (c.w > 0.0) {
                                loNext = make_double3(c.x, c.y, c.z);
                                doneLo = true;
                            }
                        }
                    }
                    if (!doneLoe) {
                        int idx = probe_find(sLoe, (uint32_t)pk & sLoe.mask, k.checksum);
                        if (idx >= 0) {
                            double4 c = ld4_ro(com_ptr(sLoe, idx));
                            if (c.w > 0.0) {
                                loeNext = make_double3(c.x, c.y, c.z);
                                doneLoe = true;
                            }
                        }
                    }
                }
            } else {
                if (lookup_level_chain(sLo, qx, qy, qz, dx, dy, dz, select_level(sLo.kp, nfp), &r, &lq))
                    loNext = r;
                if (lookup_level_chain(sLoe, qx, qy, qz, dx, dy, dz, select_level(sLoe.kp, nfp), &r, &lq))
                    loeNext = r;
            }
        } else {
            loNext = make_double3(nex, ney, nez);
        }
    }
    const double ratio = __ldg(&V.ratio[ii]);
    const double fr = __ldg(&V.f.x[ii]), fg = __ldg(&V.f.y[ii]), fb = __ldg(&V.f.z[ii]);
    const double nmis = __ldg(&V.next_emis_mis_weight[ii]);
    const double ehx = __ldg(&V.emission_here.x[ii]), ehy = __ldg(&V.emission_here.y[ii]),
                 ehz = __ldg(&V.emission_here.z[ii]);

    /* ---- Lo (estimators.cpp:215-221) ---- */
    Key kLo = key_for(sLo.kp, px, py, pz, wox, woy, woz, level);
    const bool transp = cont && ratio > 0.0;
    double ulx = ((0.0 + loNext.x) * fr) * ratio, uly = ((0.0 + loNext.y) * fg) * ratio,
           ulz = ((0.0 + loNext.z) * fb) * ratio; /* computeUpdateValue(Lo) field.cpp:17-18 */
    /* ---- LoE (226-234) ---- */
    Key kLoe = a.same_lo_loe ? kLo : key_for(sLoe.kp, px, py, pz, wox, woy, woz, level);
    const double lex = nex * nmis, ley = ney * nmis, lez = nez * nmis;
    double uex = ((lex + loeNext.x) * fr) * ratio, uey = ((ley + loeNext.y) * fg) * ratio,
           uez = ((lez + loeNext.z) * fb) * ratio;
    const bool loeCont = transp && (a.loe_mask & PSTF_TECH_CONTINUATION);
    const bool loeNee = nee && (a.loe_mask & PSTF_TECH_NEE);
    double nlx = 0, nly = 0, nlz = 0;
    if (loeNee) {
        nlx = __ldg(&V.nee_loe.x[ii]);
        nly = __ldg(&V.nee_loe.y[ii]);
        nlz = __ldg(&V.nee_loe.z[ii]);
    }
    /* lIncoming (237) */
    const double lix = lex + loeNext.x, liy = ley + loeNext.y, liz = lez + loeNext.z;
    /* ---- FLi continuation (241-246) ---- */
    Key kFc = key_for(sFli.kp, px, py, pz, wix, wiy, wiz, level);
    const bool fliCont = cont && (a.fli_mask & PSTF_TECH_CONTINUATION);
    const double fcx = fr * lix, fcy = fg * liy, fcz = fb * liz;
    /* ---- FLi NEE (247-254) ---- */
    Key kFn;
    double nfx = 0, nfy = 0, nfz = 0;
    const bool fliNee = nee && (a.fli_mask & PSTF_TECH_NEE);
    if (nee) {
        kFn = key_for(sFli.kp, px, py, pz, nee ? __ldg(&V.nee_dir.x[ii]) : 0.36,
                      nee ? __ldg(&V.nee_dir.y[ii]) : 0.48, nee ? __ldg(&V.nee_dir.z[ii]) : 0.8,
                      level);
        if (fliNee) {
            nfx = __ldg(&V.nee_fli.x[ii]);
            nfy = __ldg(&V.nee_fli.y[ii]);
            nfz = __ldg(&V.nee_fli.z[ii]);
        }
    } else {
        kFn = kFc;
    }
    /* ---- Li (256-261) ---- */
    Key kLi = kFc;
    if (a.has_li && !a.same_li_fli) kLi = key_for(sLi.kp, px, py, pz, wix, wiy, wiz, level);
    const double lvx = lix * 1.0, lvy = liy * 1.0, lvz = liz * 1.0;

    if (MODE == PSTF_MODE_ATOMIC) {
        /* per-(vertex, store, key) aggregation of the reference's separate calls; non-finite
         * accumulates are rejected and counted like field.cpp:161-163 */
        unsigned rej = 0;
        double4 vlo = make_double4(0.0, 0.0, 0.0, 1.0);
        uint32_t nlo = 1;
        if (finite3(ehx, ehy, ehz)) { vlo.x += ehx; vlo.y += ehy; vlo.z += ehz; ++nlo; } else ++rej;
        if (transp) {
            if (finite3(ulx, uly, ulz)) { vlo.x += ulx; vlo.y += uly; vlo.z += ulz; ++nlo; } else ++rej;
        }
        double4 vle = make_double4(0.0, 0.0, 0.0, 1.0);
        uint32_t nle = 1;
        unsigned rejLoe = 0;
        if (loeCont) {
            if (finite3(uex, uey, uez)) { vle.x += uex; vle.y += uey; vle.z += uez; ++nle; } else ++rejLoe;
        }
        if (loeNee) {
            if (finite3(nlx, nly, nlz)) { vle.x += nlx; vle.y += nly; vle.z += nlz; ++nle; } else ++rejLoe;
        }
        double4 vfc = make_double4(0.0, 0.0, 0.0, 1.0);
        uint32_t nfc = 1;
        unsigned rejFli = 0;
        if (fliCont) {
            if (finite3(fcx, fcy, fcz)) { vfc.x += fcx; vfc.y += fcy; vfc.z += fcz; ++nfc; } else ++rejFli;
        }
        double4 vfn = make_double4(0.0, 0.0, 0.0, 1.0);
        uint32_t nfn = 1;
        if (fliNee) {
            if (finite3(nfx, nfy, nfz)) { vfn.x += nfx; vfn.y += nfy; vfn.z += nfz; ++nfn; } else ++rejFli;
        }
        double4 vli = make_double4(0.0, 0.0, 0.0, 1.0);
        uint32_t nli = 1;
        unsigned rejLi = 0;
        if (finite3(lvx, lvy, lvz)) { vli.x += lvx; vli.y += lvy; vli.z += lvz; ++nli; } else ++rejLi;

        if (live) {
            if (rej) atomicAdd(&sLo.ctr[C_REJECTED], (unsigned long long)rej);
            if (rejLoe) atomicAdd(&sLoe.ctr[C_REJECTED], (unsigned long long)rejLoe);
            if (rejFli) atomicAdd(&sFli.ctr[C_REJECTED], (unsigned long long)rejFli);
            if (a.has_li && cont && rejLi) atomicAdd(&sLi.ctr[C_REJECTED], (unsigned long long)rejLi);
        }
        const PendSink ps{a.pend, a.pend_count, a.pend_cap};
        contribute_atomic(sLo, ps, sm, 0, live, kLo, vlo, nlo);
        contribute_atomic(sLoe, ps, sm, 1, live, kLoe, vle, nle);
        contribute_atomic(sFli, ps, sm, 2, live && cont, kFc, vfc, nfc);
        contribute_atomic(sFli, ps, sm, 2, live && nee, kFn, vfn, nfn);
        if (a.has_li) contribute_atomic(sLi, ps, sm, 3, live && cont, kLi, vli, nli);
    } else {
        /* ORDERED: the reference's individual calls, in any order (the sort canonicalises) */
        const PendSink ps{a.pend, a.pend_count, a.pend_cap};
        unsigned long long *alias = a.pend2_count + 1;
        unsigned rejLo = 0, rejLoe = 0, rejFli = 0, rejLi = 0;
        const int rLo = count_call(sLo, ps, live, 0, kLo, alias);
        const int rLoe = count_call(sLoe, ps, live, 1, kLoe, alias);
        const int rFc = count_call(sFli, ps, live && cont, 2, kFc, alias);
        const int rFn = count_call(sFli, ps, live && nee, 2, kFn, alias);
        const int rLi = a.has_li ? count_call(sLi, ps, live && cont, 3, kLi, alias) : -3;
        VCall vc[7];
        bool ok = finite3(ehx, ehy, ehz);
        rejLo += live && !ok;
        vc[0] = {live && ok, rLo, ehx, ehy, ehz};
        ok = finite3(ulx, uly, ulz);
        rejLo += live && transp && !ok;
        vc[1] = {live && transp && ok, rLo, ulx, uly, ulz};
        ok = finite3(uex, uey, uez);
        rejLoe += live && loeCont && !ok;
        vc[2] = {live && loeCont && ok, rLoe, uex, uey, uez};
        ok = finite3(nlx, nly, nlz);
        rejLoe += live && loeNee && !ok;
        vc[3] = {live && loeNee && ok, rLoe, nlx, nly, nlz};
        ok = finite3(fcx, fcy, fcz);
        rejFli += live && fliCont && !ok;
        vc[4] = {live && fliCont && ok, rFc, fcx, fcy, fcz};
        ok = finite3(nfx, nfy, nfz);
        rejFli += live && fliNee && !ok;
        vc[5] = {live && fliNee && ok, rFn, nfx, nfy, nfz};
        ok = finite3(lvx, lvy, lvz);
        rejLi += a.has_li && live && cont && !ok;
        vc[6] = {a.has_li && live && cont && ok, rLi, lvx, lvy, lvz};
        value_calls(a, ps, vc, kLo, kLoe, kFc, kFn, kLi);
        if (rejLo) atomicAdd(&sLo.ctr[C_REJECTED], (unsigned long long)rejLo);
        if (rejLoe) atomicAdd(&sLoe.ctr[C_REJECTED], (unsigned long long)rejLoe);
        if (rejFli) atomicAdd(&sFli.ctr[C_REJECTED], (unsigned long long)rejFli);
        if (rejLi) atomicAdd(&sLi.ctr[C_REJECTED], (unsigned long long)rejLi);
    }
}

/* ------------------------------------------------------------------------------------------ */
/* K5 (fast path): persistent, TMA-staged fused vertex pass (ATOMIC mode, shared quantisation) */
/*
 * Each CTA (VT threads, one vertex per thread per tile) loops over tiles of VT vertices.  The 35
 * SoA field segments of the next tiles are fetched by one elected thread with 1-D bulk async
 * copies (cp.async.bulk, L2 evict-first: the stream is read once) into a 2-stage shared-memory
 * ring guarded by mbarriers, so the 276 B/vertex input stream never stalls the warps; lanes read
 * their fields from shared memory just in time.  Per vertex the position is divided by the base
 * cell once and each direction goes through atan2 once (pos_q / octa_pair), shared by the Lo,
 * Lo\E, FLi and Li keys and by every level of the next-vertex lookup chain.
 */
#ifndef PSTF_VP_DBG_BUILD
#define PSTF_VP_DBG_BUILD 0 /* experiment builds: 1 no lookups, 2 no RED, 4 keys only, 32 stream */
#endif
#ifndef PSTF_PRED_RED
#define PSTF_PRED_RED 1
#endif

#ifndef PSTF_FLI_NEXT_WORD
#define PSTF_FLI_NEXT_WORD 1
#endif
#ifndef VT_THREADS
#define VT_THREADS 128 /* vertices (= threads) per tile and CTA */
#endif
#define VT VT_THREADS
#define VT_MINB (512 / VT) /* resident CTAs per SM of the default single-stage config */
#ifndef PSTF_VT_EXPERIMENT
static_assert(VT_MINB == 4, "the vertex-pass launch table names 4 CTAs/SM (VT = 128)");
#endif

struct TileStage {
    double f[PS_NUM_F64][VT];
    uint32_t flags[VT];
};

struct VPArgs2 {
    Stores4 st;
    FastParams fp;
    int dbg; /* unused: the experiment switches are compile-time (PSTF_VP_DBG_BUILD) */
    int pf;  /* L2 prefetch distance in tiles of this CTA (PSTF_VP_PF, default 1) */
    int has_li;
    uint32_t loe_mask, fli_mask;
    const double *fld[PS_NUM_F64];
    const uint32_t *flags;
    uint64_t n;
    PendRec *pend;
    unsigned long long *pend_count;
    uint64_t pend_cap;
    double *cv[3];     /* fused CV lookup outputs (estimators.cpp:453-462), CV instantiation only */
    uint8_t *cv_valid;
    /* ORDERED instantiation: the slot-grouped value calls (as VPArgs) */
    uint64_t *pend2_key;
    double4 *pend2_val;
    unsigned long long *pend2_count; /* [0] calls, [1] checksum alias seen */
    uint64_t pend2_cap;
    int pend2_capl;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    for (;;) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (done) break; /* try_wait suspends the warp in hardware until the phase flips */
    }
}

__device__ __forceinline__ void prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void issue_tile(const VPArgs2 &a, TileStage *st, uint64_t *bar,
                                           uint64_t tile, uint64_t policy) {
    mbar_expect_tx(bar, (uint32_t)(PS_NUM_F64 * VT * 8 + VT * 4));
    const uint64_t v0 = tile * VT;
#if PSTF_ISSUE_ROLLED
#pragma unroll 1
#endif
    for (int k = 0; k < PS_NUM_F64; ++k) bulk_g2s(&st->f[k][0], a.fld[k] + v0, VT * 8, bar, policy);
    bulk_g2s(&st->flags[0], a.flags + v0, VT * 4, bar, policy);
}

/* Uniformly strided inputs (all 34 f64 fields of one buffer at a fixed field stride, the layout
 * of pstf_synth_generate and pstf_vertex_soa_from_buffer): one 2-D tensor copy moves a tile's
 * [34][VT] block, one 1-D bulk copy its flags, instead of 35 per-field copies. */
__device__ __forceinline__ void issue_tile_tmap(const VPArgs2 &a, const CUtensorMap *tm,
                                                TileStage *st, uint64_t *bar, uint64_t tile,
                                                uint64_t policy) {
    mbar_expect_tx(bar, (uint32_t)(PS_NUM_F64 * VT * 8 + VT * 4));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(&st->f[0][0])),
        "l"(tm), "r"((int)(tile * VT)), "r"(0), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
    bulk_g2s(&st->flags[0], a.flags + tile * VT, VT * 4, bar, policy);
}

__device__ __forceinline__ void prefetch_tile_tmap(const VPArgs2 &a, const CUtensorMap *tm,
                                                   uint64_t tile, uint64_t policy) {
    /* evict-first like the copies themselves: the prefetched stream must not push the hash
     * tables' lines out of L2 */
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile.L2::cache_hint [%0, {%1, %2}], %3;"
                 ::"l"(tm), "r"((int)(tile * VT)), "r"(0), "l"(policy)
                 : "memory");
    prefetch_l2(a.flags + tile * VT, VT * 4);
}

/* pull a later tile's segments into L2 so its shared-memory copy completes at L2 latency */
__device__ __forceinline__ void prefetch_tile(const VPArgs2 &a, uint64_t tile) {
    const uint64_t v0 = tile * VT;
#if PSTF_ISSUE_ROLLED
#pragma unroll 1
#endif
    for (int k = 0; k < PS_NUM_F64; ++k) prefetch_l2(a.fld[k] + v0, VT * 8);
    prefetch_l2(a.flags + v0, VT * 4);
}

struct SmemSrc {
    const TileStage *t;
    int j;
    uint64_t v; /* global vertex index */
    __device__ __forceinline__ double f(int k) const { return t->f[k][j]; }
    __device__ __forceinline__ uint32_t flags() const { return t->flags[j]; }
    __device__ __forceinline__ uint64_t index() const { return v; }
};


__device__ __forceinline__ Key make_key(uint64_t h1, int level, int32_t c0, int32_t c1, int32_t c2,
                                        int32_t d0, int32_t d1) {
    Key k;
    k.level = level;
    k.cell[0] = c0;
    k.cell[1] = c1;
    k.cell[2] = c2;
    k.dir[0] = d0;
    k.dir[1] = d1;
    const uint64_t pk = pack_from_h1(h1, c2, d0, d1);
    k.checksum = checksum_of(pk);
    k.pack_lo = (uint32_t)pk;
    return k;
}

/* Pipe hooks of vertex_body, called by all 32 lanes of every warp:
 *   key_inputs_done()  every key input (fields 0..PS_NA-1 and the flags) has been read
 *   wait_values()      before the first value input (fields PS_NA..) is read
 *   values_done()      every value input has been read
 * The single-stage tiled kernel needs none of them (NoPipe).  A split-stage kernel that refilled
 * its key-input stage early and its value-input stage late through them (no CTA barrier per
 * tile) measured 0.99 ms against 0.91 ms for the synchronized single stage on config 2. */
struct NoPipe {
    __device__ __forceinline__ void key_inputs_done() const {}
    __device__ __forceinline__ void wait_values() const {}
    __device__ __forceinline__ void values_done() const {}
};

/* ORDERED tiled kernel: each warp reserves the (sort key, value) pair buffer in chunks of
 * PAIR_CHUNK entries (one atomic per chunk instead of one per contribution: the counter is a
 * single hot address); a chunk's unused tail is filled with holes, key ~0 (above every real
 * key: the slot-grouped sort moves them to the end), counted in pend2_count[2] */
#define PAIR_CHUNK 256
struct PairChunk {
    unsigned long long base = 0;
    uint32_t used = PAIR_CHUNK; /* full: the first need reserves */
    uint64_t holes = 0;
    bool any = false;
};

__device__ __forceinline__ void pair_close(const VPArgs2 &a, PairChunk &pc) {
    if (pc.any) {
        for (uint32_t i = pc.used + lane_id(); i < PAIR_CHUNK; i += 32)
            if (pc.base + i < a.pend2_cap) a.pend2_key[pc.base + i] = ~0ull;
        pc.holes += PAIR_CHUNK - pc.used;
    }
    pc.used = PAIR_CHUNK;
}

/* the warp's positions for `need` (<= 64) pairs; warp-uniform */
__device__ __forceinline__ unsigned long long pair_reserve(const VPArgs2 &a, PairChunk &pc,
                                                           uint32_t need) {
    if (pc.used + need > PAIR_CHUNK) {
        pair_close(a, pc);
        unsigned long long b = 0;
        if (lane_id() == 0) b = atomicAdd(a.pend2_count, (unsigned long long)PAIR_CHUNK);
        pc.base = __shfl_sync(0xffffffffu, b, 0);
        pc.used = 0;
        pc.any = true;
    }
    const unsigned long long pos = pc.base + pc.used;
    pc.used += need;
    return pos;
}

/* ORD (ORDERED mode): every counter call of an existing key is added in place (the RED of
 * {0, 0, 0, 1}), every value call becomes a (sort key, value) pair for the slot-grouped fold, a
 * new key's (or a checksum alias's) calls become one full pending record each; see
 * value_calls() for the per-thread kernel's version of the same rules */
template <bool CV, bool ORD, bool AGG, bool TWIN, class Src, class Pipe = NoPipe>
__device__ __forceinline__ void vertex_body(const VPArgs2 &a, const Src &S, bool live,
                                            double4 *sm, uint32_t &nred, uint64_t &ef_cn,
                                            PairChunk &pc, const Pipe &pipe = Pipe()) {
    const DevStore &sLo = a.st.s[0];
    const DevStore &sLoe = a.st.s[1];
    const DevStore &sFli = a.st.s[2];
    const DevStore &sLi = a.st.s[3];
    const KeyParams &kp = sLo.kp;
    const FastParams &fq = a.fp;
    const uint32_t fl = live ? S.flags() : 0u;
    const bool cont = (fl & PSTF_VERTEX_CONT_EXTENDED) != 0;
    const bool nsurf = (fl & PSTF_VERTEX_NEXT_IS_SURFACE) != 0;
    const bool nee = (fl & PSTF_VERTEX_NEE_SAMPLED) != 0;
    const bool look = cont && nsurf && !(PSTF_VP_DBG_BUILD & 1);
    /* Lo\E shares Lo's occupancy (twin stores, see pstf_field::twin): its probes are Lo's */
    constexpr bool TWINQ = TWIN;

    /* ---- keys (estimators.cpp:195, 215, 226, 242, 248, 257): one level, one cell triple and
     * one packKeyFields prefix for all update keys of the vertex ---- */
    int nx = 0; /* set when any quantity lies too close to a cell boundary for the fast path */
    DirF8 fo, fi, fin, fn, ftmp;
    const uint2 z = make_uint2(0u, 0u);
    const double4 z4 = make_double4(0.0, 0.0, 0.0, 0.0);
    /* the first lookup key at the next vertex goes first (estimators.cpp:198-206): its home words
     * and speculative committed records then travel while the update keys are built */
    const double wix = S.f(PS_WI), wiy = S.f(PS_WI + 1), wiz = S.f(PS_WI + 2);
    octa_f8_try(wix, wiy, wiz, look, &fi, &fin, &nx);
    const double qx = S.f(PS_NPOS), qy = S.f(PS_NPOS + 1), qz = S.f(PS_NPOS + 2);
    const PosQ nq = pos_q(fq, qx, qy, qz);
    int l0 = select_level_try(fq, S.f(PS_NFP), &nx);
    int32_t n0 = cell_try(nq.q[0], qx, l0, &nx), n1 = cell_try(nq.q[1], qy, l0, &nx),
            n2 = cell_try(nq.q[2], qz, l0, &nx);
    uint64_t qpk = pack_key_fields(l0, n0, n1, n2, dir_cell_f8(fin.u, l0), dir_cell_f8(fin.v, l0));
    uint32_t ql = (uint32_t)qpk & sLo.mask, qe = (uint32_t)qpk & sLoe.mask;
    uint32_t wl = look ? ld_meta(&sLo.meta[ql]).x : 0u;
    uint32_t we = TWINQ ? wl : (look ? ld_meta(&sLoe.meta[qe]).x : 0u);
    double4 sl = look ? ld4_ro(com_ptr(sLo, ql)) : z4, se = look ? ld4_ro(com_ptr(sLoe, qe)) : z4;

    /* ---- the update keys: one level, one cell triple, one packKeyFields prefix ---- */
    int level = select_level_try(fq, S.f(PS_FP), &nx);
    const double px = S.f(PS_POS), py = S.f(PS_POS + 1), pz = S.f(PS_POS + 2);
    const PosQ q = pos_q(fq, px, py, pz);
    int32_t c0 = cell_try(q.q[0], px, level, &nx), c1 = cell_try(q.q[1], py, level, &nx),
            c2 = cell_try(q.q[2], pz, level, &nx);
    const double wox = S.f(PS_WO), woy = S.f(PS_WO + 1), woz = S.f(PS_WO + 2);
    /* lanes without NEE use a fixed generic direction so a speculated evaluation never lands
     * near a boundary for their zero nee.dir */
    const double ndx = nee ? S.f(PS_NDIR) : 0.36, ndy = nee ? S.f(PS_NDIR + 1) : 0.48,
                 ndz = nee ? S.f(PS_NDIR + 2) : 0.8;
    octa_f8_try(wox, woy, woz, 0, &fo, &ftmp, &nx);
    octa_f8_try(ndx, ndy, ndz, 0, &fn, &ftmp, &nx);
    if (nx) { /* rare: the vertex's quantities through the exact reference operations (one
               * out-of-the-way block instead of a fallback at every use) */
        level = select_level(kp, S.f(PS_FP));
        c0 = cell_exact(kp, px, level);
        c1 = cell_exact(kp, py, level);
        c2 = cell_exact(kp, pz, level);
        octa_f8_exact(wox, woy, woz, 0, &fo, &ftmp);
        octa_f8_exact(wix, wiy, wiz, look, &fi, &fin);
        octa_f8_exact(ndx, ndy, ndz, 0, &fn, &ftmp);
        l0 = select_level(kp, S.f(PS_NFP));
        n0 = cell_exact(kp, qx, l0);
        n1 = cell_exact(kp, qy, l0);
        n2 = cell_exact(kp, qz, l0);
        qpk = pack_key_fields(l0, n0, n1, n2, dir_cell_f8(fin.u, l0), dir_cell_f8(fin.v, l0));
        ql = (uint32_t)qpk & sLo.mask;
        qe = (uint32_t)qpk & sLoe.mask;
        wl = look ? ld_meta(&sLo.meta[ql]).x : 0u;
        we = look ? ld_meta(&sLoe.meta[qe]).x : 0u;
        sl = look ? ld4_ro(com_ptr(sLo, ql)) : z4;
        se = look ? ld4_ro(com_ptr(sLoe, qe)) : z4;
    }
    pipe.key_inputs_done();
    const uint64_t h1 = pack_h1(level, c0, c1);
    const Key kLo = make_key(h1, level, c0, c1, c2, dir_cell_f8(fo.u, level), dir_cell_f8(fo.v, level));
    const Key kFc = make_key(h1, level, c0, c1, c2, dir_cell_f8(fi.u, level), dir_cell_f8(fi.v, level));
    const Key kFn = make_key(h1, level, c0, c1, c2, dir_cell_f8(fn.u, level), dir_cell_f8(fn.v, level));

    /* ---- the five update home words in one round trip ---- */
    const bool has2 = live && cont, has3 = live && nee, has4 = a.has_li && live && cont;
    const uint32_t h0 = kLo.pack_lo & sLo.mask, h1s = kLo.pack_lo & sLoe.mask,
                   h2 = kFc.pack_lo & sFli.mask, h3 = kFn.pack_lo & sFli.mask,
                   h4 = kFc.pack_lo & sLi.mask;
    const uint2 m0 = live ? ld_meta(&sLo.meta[h0]) : z,
                m1 = TWINQ ? m0 : (live ? ld_meta(&sLoe.meta[h1s]) : z),
                m2 = has2 ? ld_meta(&sFli.meta[h2]) : z, m3 = has3 ? ld_meta(&sFli.meta[h3]) : z,
                m4 = has4 ? ld_meta(&sLi.meta[h4]) : z;
#if PSTF_FLI_NEXT_WORD
    /* the FLi store is the crowded one: its two probes also preload the word after home */
    const uint2 m2b = has2 ? ld_meta(&sFli.meta[(h2 + 1) & sFli.mask]) : z,
                m3b = has3 ? ld_meta(&sFli.meta[(h3 + 1) & sFli.mask]) : z;
#endif
    /* CV lookup at this vertex = Lo\E query of the Lo key: speculate its home record too */
    const double4 scv = CV && live ? ld4_ro(com_ptr(sLoe, h1s)) : z4;

    double3 loNext = make_double3(0.0, 0.0, 0.0), loeNext = make_double3(0.0, 0.0, 0.0);
    if (look) {
        const uint32_t cs = checksum_of(qpk);
        bool doneLo = false, doneLoe = false;
        if (wl == cs) { /* speculation hit: sl is the committed record of the slot */
            if (sl.w > 0.0) loNext = make_double3(sl.x, sl.y, sl.z);
            doneLo = sl.w > 0.0;
        }
        if (we == cs) {
            if (se.w > 0.0) loeNext = make_double3(se.x, se.y, se.z);
            doneLoe = se.w > 0.0;
        }
        /* general path: rest of the probe window at l0 (unless the home word settled it), then
         * the coarser levels (queryFromLevel, field.cpp:179-195) */
        const bool homeLo = wl == cs || wl == 0u, homeLoe = we == cs || we == 0u;
        if (!(doneLo && doneLoe)) {
            for (int l = l0; l <= kp.max_level && !(doneLo && doneLoe); ++l) {
                uint64_t pk = qpk;
                if (l != l0) {
                    int lx = 0;
                    int32_t a0 = cell_try(nq.q[0], qx, l, &lx), a1 = cell_try(nq.q[1], qy, l, &lx),
                            a2 = cell_try(nq.q[2], qz, l, &lx);
                    if (lx) {
                        a0 = cell_exact(kp, qx, l);
                        a1 = cell_exact(kp, qy, l);
                        a2 = cell_exact(kp, qz, l);
                    }
                    pk = pack_key_fields(l, a0, a1, a2, dir_cell_f8(fin.u, l), dir_cell_f8(fin.v, l));
                }
                const uint32_t ccs = checksum_of(pk);
                const uint32_t hl = (uint32_t)pk & sLo.mask, he = (uint32_t)pk & sLoe.mask;
                int il = -1, ie = -1;
                if (!doneLo) {
                    if (l == l0 && homeLo) il = -1; /* home word: empty, or match not > 0 */
                    else il = resolve_find(sLo, hl, ccs, l == l0 ? wl : ld_meta(&sLo.meta[hl]).x);
                }
                if (!doneLoe) {
                    if (l == l0 && homeLoe) ie = -1;
                    else if (TWINQ && !doneLo) ie = il;
                    else ie = resolve_find(sLoe, he, ccs, l == l0 ? we : ld_meta(&sLoe.meta[he]).x);
                }
                const double4 cl = il >= 0 ? ld4_ro(com_ptr(sLo, il)) : z4;
                const double4 ce = ie >= 0 ? ld4_ro(com_ptr(sLoe, ie)) : z4;
                if (il >= 0 && cl.w > 0.0) {
                    loNext = make_double3(cl.x, cl.y, cl.z);
                    doneLo = true;
                }
                if (ie >= 0 && ce.w > 0.0) {
                    loeNext = make_double3(ce.x, ce.y, ce.z);
                    doneLoe = true;
                }
            }
        }
    }

    if (PSTF_VP_DBG_BUILD & 4) {
        if ((m0.x ^ m1.x ^ m2.x ^ m3.x ^ m4.x ^ kLo.checksum ^ kFc.checksum ^ kFn.checksum) ==
                0x12345u && loNext.x + loeNext.y == 1.2345)
            atomicAdd(&sLo.ctr[C_INTERNAL], 1ull);
        pipe.wait_values();
        pipe.values_done();
        return;
    }

    /* ---- probes of the five update keys: settle the frame-start table first, so the home
     * words die before the values are built ---- */
    uint32_t k0 = 0, k1 = 0, k2 = 0, k3 = 0, k4 = 0;
    const int r0 = live ? resolve_probe(sLo, h0, kLo.checksum, m0, &k0) : -3;
    int r1 = -3;
    if (TWINQ) {
        r1 = r0;
        k1 = k0;
    } else {
        r1 = live ? resolve_probe(sLoe, h1s, kLo.checksum, m1, &k1) : -3;
    }
#if PSTF_FLI_NEXT_WORD
    const int r2 = has2 ? resolve_probe2(sFli, h2, kFc.checksum, m2, m2b, &k2) : -3;
    const int r3 = has3 ? resolve_probe2(sFli, h3, kFn.checksum, m3, m3b, &k3) : -3;
#else
    const int r2 = has2 ? resolve_probe(sFli, h2, kFc.checksum, m2, &k2) : -3;
    const int r3 = has3 ? resolve_probe(sFli, h3, kFn.checksum, m3, &k3) : -3;
#endif
    const int r4 = has4 ? resolve_probe(sLi, h4, kFc.checksum, m4, &k4) : -3;
    const PendSink ps{a.pend, a.pend_count, a.pend_cap};
    /* ORD: a slot whose checksum matches but whose key fields do not (a checksum alias) */
    uint32_t amask = 0;
    if (ORD) { /* 0.15 ms of the ORDERED tiled pass on config 2 */
        const auto alias_of = [](const DevStore &s, int r, const Key &k) -> uint32_t {
            if (r < 0) return 0u;
            const KeyFields kf = s.keyf[r];
            return (kf.level != k.level || kf.c0 != k.cell[0] || kf.c1 != k.cell[1] ||
                    kf.c2 != k.cell[2] || kf.d0 != k.dir[0] || kf.d1 != k.dir[1]) ? 1u : 0u;
        };
        amask = alias_of(sLo, r0, kLo) | alias_of(sLoe, r1, kLo) << 1 |
                alias_of(sFli, r2, kFc) << 2 | alias_of(sFli, r3, kFn) << 3 |
                alias_of(sLi, r4, kFc) << 4;
        if (amask) atomicOr(a.pend2_count + 1, 1ull);
    }

    if (CV && live) {
        /* ---- fused CV lookup (estimators.cpp:453-462; k_cv_lookup semantics): the Lo\E query
         * at (position, wo, footprint) on the frame-start table.  Its first level's key is the
         * Lo key, whose Lo\E probe r1 is already settled ---- */
        double3 cv = make_double3(0.0, 0.0, 0.0);
        bool ok = false;
        if (r1 >= 0) {
            const double4 c = r1 == (int)h1s ? scv : ld4_ro(com_ptr(sLoe, r1));
            ok = c.w > 0.0;
            if (ok) cv = make_double3(c.x, c.y, c.z);
        }
        for (int l = level + 1; !ok && l <= kp.max_level; ++l) {
            const double px = S.f(PS_POS), py = S.f(PS_POS + 1), pz = S.f(PS_POS + 2);
            const PosQ q = pos_q(fq, px, py, pz);
            int lx = 0;
            int32_t a0 = cell_try(q.q[0], px, l, &lx), a1 = cell_try(q.q[1], py, l, &lx),
                    a2 = cell_try(q.q[2], pz, l, &lx);
            if (lx) {
                a0 = cell_exact(kp, px, l);
                a1 = cell_exact(kp, py, l);
                a2 = cell_exact(kp, pz, l);
            }
            const uint64_t pk =
                pack_key_fields(l, a0, a1, a2, dir_cell_f8(fo.u, l), dir_cell_f8(fo.v, l));
            const int idx = probe_find(sLoe, (uint32_t)pk & sLoe.mask, checksum_of(pk));
            if (idx >= 0) {
                const double4 c = ld4_ro(com_ptr(sLoe, idx));
                ok = c.w > 0.0;
                if (ok) cv = make_double3(c.x, c.y, c.z);
            }
        }
        const uint64_t i = S.index();
        a.cv[0][i] = cv.x;
        a.cv[1][i] = cv.y;
        a.cv[2][i] = cv.z;
        a.cv_valid[i] = ok ? 1 : 0;
    }

    /* ---- update values (field.cpp:13-25 evaluation order), each built from the staged inputs
     * just before its contribution; one rolled loop over the five contributions keeps a single
     * copy of the probe/RED/pending code in the instruction stream ---- */
    pipe.wait_values();
    if (cont && !nsurf) /* environment (estimators.cpp:209) */
        loNext = make_double3(S.f(PS_NEMIS), S.f(PS_NEMIS + 1), S.f(PS_NEMIS + 2));
    const bool transp = cont && S.f(PS_RATIO) > 0.0;
    /* Li = Le + Lo\E(next) (estimators.cpp:239) */
    const auto li = [&](int c, double lo_e) {
        return S.f(PS_NEMIS + c) * S.f(PS_NMIS) + lo_e;
    };
    /* ORD: the contribution's individual value calls (at most two) */
    double3 call0 = make_double3(0.0, 0.0, 0.0), call1 = call0;
    const auto add3 = [&](double4 &v, uint32_t &nc, unsigned &rej, double x, double y, double z2) {
        if (finite3(x, y, z2)) {
            if (ORD) {
                if (nc == 1) call0 = make_double3(x, y, z2);
                else call1 = make_double3(x, y, z2);
            } else {
                v.x += x;
                v.y += y;
                v.z += z2;
            }
            ++nc;
        } else {
            ++rej;
        }
    };
    /* contribution c: store sid(c) = {Lo, Lo\E, FLi, FLi, Li}; its probe result and touch mark
     * shift down one register per iteration (no select chains) */
    int rr0 = r0, rr1 = r1, rr2 = r2, rr3 = r3, rr4 = r4;
    uint32_t kk0 = k0, kk1 = k1, kk2 = k2, kk3 = k3, kk4 = k4;
    uint32_t rejpack = 0; /* rejected calls per store, one byte each (at most 3 per vertex) */
    /* the TWIN instantiations run only without an Li store and with every technique on
     * (loe_mask = fli_mask = all, the default): the Li branch and the mask tests are compiled
     * out (a smaller rolled loop: 0.9% and 0.7% on config 2) */
    constexpr bool MASKS_ALL = TWIN;
    const int ncontrib = !TWIN && a.has_li ? 5 : 4;
#pragma unroll 1
    for (int c = 0; c < ncontrib; ++c) {
        double4 v = make_double4(0.0, 0.0, 0.0, 1.0); /* the counter call */
        uint32_t nc = 1;
        unsigned rej = 0;
        if (c == 0) { /* Lo: emission, transport (estimators.cpp:210-224) */
            add3(v, nc, rej, S.f(PS_EMIS), S.f(PS_EMIS + 1), S.f(PS_EMIS + 2));
            if (transp) {
                const double ratio = S.f(PS_RATIO);
                add3(v, nc, rej, ((0.0 + loNext.x) * S.f(PS_F)) * ratio,
                     ((0.0 + loNext.y) * S.f(PS_F + 1)) * ratio,
                     ((0.0 + loNext.z) * S.f(PS_F + 2)) * ratio);
            }
        } else if (c == 1) { /* Lo\E (226-234); its key is the Lo key */
            if (transp && (MASKS_ALL || (a.loe_mask & PSTF_TECH_CONTINUATION))) {
                const double nmis = S.f(PS_NMIS), ratio = S.f(PS_RATIO);
                add3(v, nc, rej, ((S.f(PS_NEMIS) * nmis + loeNext.x) * S.f(PS_F)) * ratio,
                     ((S.f(PS_NEMIS + 1) * nmis + loeNext.y) * S.f(PS_F + 1)) * ratio,
                     ((S.f(PS_NEMIS + 2) * nmis + loeNext.z) * S.f(PS_F + 2)) * ratio);
            }
            if (nee && (MASKS_ALL || (a.loe_mask & PSTF_TECH_NEE)))
                add3(v, nc, rej, S.f(PS_NEELOE), S.f(PS_NEELOE + 1), S.f(PS_NEELOE + 2));
        } else if (c == 2) { /* FLi continuation (241-246) */
            if (cont && (MASKS_ALL || (a.fli_mask & PSTF_TECH_CONTINUATION)))
                add3(v, nc, rej, S.f(PS_F) * li(0, loeNext.x), S.f(PS_F + 1) * li(1, loeNext.y),
                     S.f(PS_F + 2) * li(2, loeNext.z));
        } else if (c == 3) { /* FLi NEE (247-254) */
            if (nee && (MASKS_ALL || (a.fli_mask & PSTF_TECH_NEE)))
                add3(v, nc, rej, S.f(PS_NEEFLI), S.f(PS_NEEFLI + 1), S.f(PS_NEEFLI + 2));
        } else if (!TWIN) { /* Li (256-261) */
            if (cont)
                add3(v, nc, rej, li(0, loeNext.x) * 1.0, li(1, loeNext.y) * 1.0,
                     li(2, loeNext.z) * 1.0);
        }
        const int sid = c < 2 ? c : (c < 4 ? 2 : 3);
        rejpack += rej << (8 * sid);
        const DevStore &s = a.st.s[sid];
        const int res = rr0;
        const uint32_t mark = kk0;
        /* sector-coalesced REDs: the warp's 32 cells x 4 components are transposed through
         * shared memory so each RED instruction covers 8 cells x {r,g,b,c}; the 4 lanes of a
         * cell hit one 32 B sector, so L1 sends 8 sector requests per instruction, not 32 */
        int *rsm = reinterpret_cast<int *>(sm + 32);
        const unsigned lane = lane_id();
        /* the RED element updates of this lane's own contribution (before any aggregation:
         * the hot-slot measure must not depend on the variant that measured it) */
        const uint32_t own = AGG && res >= 0 ? (uint32_t)(v.x != 0.0) + (v.y != 0.0) +
                                                   (v.z != 0.0) + (v.w != 0.0)
                                             : 0u;
        if (AGG) {
            /* hot slots (chosen per launch from the last frame's RED density): lanes whose
             * contributions hit one slot are summed first and only the lowest of them issues
             * the REDs (profiles/round2_match_any_ab.md) */
            const unsigned peers =
                __match_any_sync(0xffffffffu, res >= 0 ? (uint32_t)res : 0x80000000u | lane);
            const int leader = __ffs(peers) - 1;
            sm[lane] = v;
            __syncwarp();
            if (__popc(peers) > 1 && (int)lane == leader) {
                unsigned m = peers & (peers - 1);
                while (m) {
                    const double4 o = sm[__ffs(m) - 1];
                    m &= m - 1;
                    v.x += o.x;
                    v.y += o.y;
                    v.z += o.z;
                    v.w += o.w;
                }
            }
            __syncwarp();
            sm[lane] = v;
            rsm[lane] = (PSTF_VP_DBG_BUILD & 2) || (int)lane != leader ? -3 : res;
        } else {
            sm[lane] = v;
            rsm[lane] = (PSTF_VP_DBG_BUILD & 2) ? -3 : res;
        }
        __syncwarp();
        const double *flat = reinterpret_cast<const double *>(sm);
        const int comp = lane & 3;
        double *const accc = reinterpret_cast<double *>(s.acc) + comp; /* component column */
        uint32_t cnt = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int cell = 8 * q + (lane >> 2);
            const int rs = rsm[cell];
            const double val = flat[4 * cell + comp];
            const bool on = rs >= 0 && val != 0.0;
#if PSTF_PRED_RED
            /* predicated RED, no branch around it (no memory clobber: the RED is unordered
             * with the thread's other accesses, which never touch acc this pass); 32-bit slot
             * index, one wide multiply-add for the address */
            double *dst = accc + (uint64_t)(on ? (uint32_t)rs : 0u) * 4u;
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
                         "@p red.relaxed.gpu.global.add.f64 [%0], %1;\n\t}" ::"l"(dst),
                         "d"(val), "r"((uint32_t)on));
#else
            if (on) atomicAdd(reinterpret_cast<double *>(acc_ptr(s, rs)) + comp, val);
#endif
            cnt += on;
        }
        nred += AGG ? own : cnt;
        __syncwarp();
        /* unit-weight frame accounting (k_ef_onepass): one counter call of weight 1 per
         * contribution with a slot; 16-bit fields per store */
        if (res >= 0) {
            touch_slot(s, (uint32_t)res, mark);
            if (!ORD) ef_cn += 1ull << (16 * sid);
        }
        if (ORD) {
            const bool al = (amask >> c) & 1u;
            const uint32_t nv = nc - 1; /* value calls of this contribution */
            const auto nz = [](double3 q) { return q.x != 0.0 || q.y != 0.0 || q.z != 0.0; };
            const bool p0 = res >= 0 && !al && nv > 0 && nz(call0);
            const bool p1 = res >= 0 && !al && nv > 1 && nz(call1);
            const unsigned b0 = __ballot_sync(0xffffffffu, p0), b1 = __ballot_sync(0xffffffffu, p1);
            const unsigned tot = __popc(b0) + __popc(b1);
            if (tot) {
                const unsigned long long base = pair_reserve(a, pc, tot);
                const int capl = a.pend2_capl, S2 = capl + 2;
                const uint64_t sk = ((uint64_t)sid << capl) | (uint32_t)(res >= 0 ? res : 0);
                const unsigned lt = (1u << lane) - 1u;
                if (p0) {
                    const unsigned long long pos = base + __popc(b0 & lt);
                    if (pos < a.pend2_cap) {
                        a.pend2_key[pos] = (sk << (64 - S2)) | (dbits(call0.x) >> S2);
                        a.pend2_val[pos] = make_double4(call0.x, call0.y, call0.z, 0.0);
                    }
                }
                if (p1) {
                    const unsigned long long pos = base + __popc(b0) + __popc(b1 & lt);
                    if (pos < a.pend2_cap) {
                        a.pend2_key[pos] = (sk << (64 - S2)) | (dbits(call1.x) >> S2);
                        a.pend2_val[pos] = make_double4(call1.x, call1.y, call1.z, 0.0);
                    }
                }
            }
            const Key k = c < 2 ? kLo : (c == 3 ? kFn : kFc);
            const bool full = res == -1 || al;
            if (PendRec *p = warp_reserve(ps, res == -1)) /* a new key's counter call */
                put_record(p, k, PSTF_META(sid, 1, 1) | ((uint32_t)s.rank << 3), 0.0, 0.0, 0.0,
                           1.0);
            if (PendRec *p = warp_reserve(ps, full && nv > 0))
                put_record(p, k, PSTF_META(sid, 0, 1), call0.x, call0.y, call0.z, 1.0);
            if (PendRec *p = warp_reserve(ps, full && nv > 1))
                put_record(p, k, PSTF_META(sid, 0, 1), call1.x, call1.y, call1.z, 1.0);
        } else if (PendRec *p = warp_reserve(ps, res == -1)) { /* a new key (rare after warm-up) */
            const Key k = c < 2 ? kLo : (c == 3 ? kFn : kFc);
            put_record(p, k, PSTF_META(sid, 0, nc) | ((uint32_t)s.rank << 3), v.x, v.y, v.z, v.w);
        }
        if (res == -2) atomicAdd(&s.ctr[C_DROPPED], (unsigned long long)nc); /* per call */
        rr0 = rr1;
        rr1 = rr2;
        rr2 = rr3;
        rr3 = rr4;
        kk0 = kk1;
        kk1 = kk2;
        kk2 = kk3;
        kk3 = kk4;
    }
    if (__any_sync(0xffffffffu, live && rejpack != 0) && live) /* non-finite values (rare) */
        for (int q = 0; q < 4; ++q) {
            const unsigned r = (rejpack >> (8 * q)) & 0xffu;
            if (r) atomicAdd(&a.st.s[q].ctr[C_REJECTED], (unsigned long long)r);
        }
    pipe.values_done();
}

template <int STAGES, int MINB, bool TMAP, bool CV = false, bool ORD = false, bool AGG = false,
          bool TWIN = false>
__global__ void __launch_bounds__(VT, MINB)
    k_vertex_pass_tiled(VPArgs2 a, const __grid_constant__ CUtensorMap tm) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TileStage *stages = reinterpret_cast<TileStage *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + STAGES * sizeof(TileStage));
    __shared__ double4 wsm[VT / 32][36]; /* 32 cells + 32 ints of probe results */
    const int tid = threadIdx.x;
    double4 *sm = wsm[tid >> 5];
    const uint64_t nfull = a.n / VT;
    uint64_t policy = 0;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (int s = 0; s < STAGES; ++s) {
            uint64_t t = blockIdx.x + (uint64_t)s * gridDim.x;
            if (t < nfull) {
                if (TMAP) issue_tile_tmap(a, &tm, &stages[s], &bars[s], t, policy);
                else issue_tile(a, &stages[s], &bars[s], t, policy);
            }
            for (int d = 1; d <= a.pf; ++d)
                if (t + (uint64_t)d * gridDim.x < nfull) {
                    if (TMAP) prefetch_tile_tmap(a, &tm, t + (uint64_t)d * gridDim.x, policy);
                    else prefetch_tile(a, t + (uint64_t)d * gridDim.x);
                }
        }
    uint32_t it = 0, nred = 0;
    uint64_t ef_cn = 0; /* per-store 16-bit counters, flushed every 1024 tiles */
    PairChunk pc;       /* ORD only */
    const auto flush_ef = [&]() {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const unsigned c = __reduce_add_sync(0xffffffffu, (unsigned)(ef_cn >> (16 * q)) & 0xffffu);
            if ((tid & 31) == 0 && c) atomicAdd(&a.st.s[q].ctr[C_F_CN], (unsigned long long)c);
        }
        ef_cn = 0;
    };
    const uint64_t ntiles = (a.n + VT - 1) / VT;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int s = (int)(it % STAGES);
        bool live = true;
        if (tile < nfull) {
            mbar_wait(&bars[s], (it / STAGES) & 1u);
        } else {
            /* the partial last tile: plain loads into this lane's own column of the stage (no
             * bulk copy is in flight any more), so the one inlined body serves every tile */
            const uint64_t v = tile * VT + tid;
            live = v < a.n;
            for (int k = 0; k < PS_NUM_F64; ++k) stages[s].f[k][tid] = live ? a.fld[k][v] : 0.0;
            stages[s].flags[tid] = live ? a.flags[v] : 0u;
        }
        SmemSrc src{&stages[s], tid, tile * VT + tid};
        const uint64_t nt = tile + (uint64_t)STAGES * gridDim.x;
        const auto issue_next = [&]() {
            if (nt < nfull) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const uint64_t pt = nt + (uint64_t)a.pf * gridDim.x;
                if (TMAP) {
                    issue_tile_tmap(a, &tm, &stages[s], &bars[s], nt, policy);
                    if (pt < nfull) prefetch_tile_tmap(a, &tm, pt, policy);
                } else {
                    issue_tile(a, &stages[s], &bars[s], nt, policy);
                    if (pt < nfull) prefetch_tile(a, pt);
                }
            }
        };
        if (PSTF_VP_DBG_BUILD & 32) { /* experiment: stream only */
            if (src.f(PS_FP) == -12345.0) atomicAdd(&a.st.s[0].ctr[C_INTERNAL], 1ull);
        } else {
            vertex_body<CV, ORD, AGG, TWIN>(a, src, live, sm, nred, ef_cn, pc);
        }
        __syncthreads(); /* every lane is done with stage s */
        if (tid == 0) issue_next();
        if ((it & 1023u) == 1023u) flush_ef();
    }
    flush_ef();
    if (ORD) {
        pair_close(a, pc);
        if ((tid & 31) == 0 && pc.holes) atomicAdd(a.pend2_count + 2, (unsigned long long)pc.holes);
    }
    /* RED element updates issued (atomic-roofline accounting, one atomic per warp) */
    for (int o = 16; o; o >>= 1) nred += __shfl_xor_sync(0xffffffffu, nred, o);
    if ((tid & 31) == 0 && nred) atomicAdd(&a.st.s[0].ctr[C_REDS], (unsigned long long)nred);
}

/* CV lookup at the current vertex (estimators.cpp:453-462) */
__global__ void k_cv_lookup(DevStore s, pstf_vertex_soa V, uint64_t n, double *vr, double *vg,
                            double *vb, uint8_t *valid) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double3 v = make_double3(0.0, 0.0, 0.0);
    int lo;
    bool ok = lookup_level_chain(s, V.position.x[i], V.position.y[i], V.position.z[i], V.wo.x[i],
                                 V.wo.y[i], V.wo.z[i], select_level(s.kp, V.footprint[i]), &v, &lo);
    if (!ok) v = make_double3(0.0, 0.0, 0.0);
    if (vr) vr[i] = v.x;
    if (vg) vg[i] = v.y;
    if (vb) vb[i] = v.z;
    if (valid) valid[i] = ok;
}

/* ------------------------------------------------------------------------------------------ */
/* apply(): batched incrementCounter / accumulate / FieldUpdateQueue::apply                    */

__device__ __forceinline__ bool update_valid(bool is_counter, double r, double g, double b,
                                             double w) {
    if (is_counter) return (w >= 0.0) && isfinite(w); /* field.cpp:149 */
    return finite3(r, g, b) && isfinite(w) && !(w < 0.0); /* field.cpp:161 */
}

struct ApplyArgs {
    DevStore s;
    const pstf_key *keys;
    const double *vr, *vg, *vb;
    const double *w;
    const uint8_t *isc;
    uint64_t n;
};

/* ATOMIC: existing slot -> RED, new key -> pending, exhausted -> dropped */
__global__ void k_apply_atomic(ApplyArgs a, PendRec *pend, unsigned long long *pend_count,
                               uint64_t cap) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    const bool isc = a.isc ? a.isc[i] != 0 : false;
    const double w = a.w[i];
    const double r = (isc || !a.vr) ? 0.0 : a.vr[i], g = (isc || !a.vg) ? 0.0 : a.vg[i],
                 b = (isc || !a.vb) ? 0.0 : a.vb[i];
    if (!update_valid(isc, r, g, b, w)) {
        atomicAdd(&a.s.ctr[C_REJECTED], 1ull);
        return;
    }
    pstf_key k = a.keys[i];
    uint64_t pk = pack_key_fields(k.level, k.cell[0], k.cell[1], k.cell[2], k.dir_cell[0],
                                  k.dir_cell[1]);
    double4 v = isc ? make_double4(0.0, 0.0, 0.0, w > 0.0 ? w : 0.0)
                    : make_double4(r * w, g * w, b * w, 0.0);
    uint32_t mark = 0;
    int res = probe_existing(a.s, (uint32_t)pk & a.s.mask, k.checksum, &mark);
    if (res >= 0) {
        red_add4(acc_ptr(a.s, res), v);
        touch_slot(a.s, (uint32_t)res, mark);
    } else if (res == -2) {
        atomicAdd(&a.s.ctr[C_DROPPED], 1ull);
    } else {
        unsigned long long pos = atomicAdd(pend_count, 1ull);
        if (pos < cap) {
            PendRec rr;
            rr.k[0] = k.level;
            rr.k[1] = k.cell[0];
            rr.k[2] = k.cell[1];
            rr.k[3] = k.cell[2];
            rr.k[4] = k.dir_cell[0];
            rr.k[5] = k.dir_cell[1];
            rr.cs = k.checksum;
            rr.meta = PSTF_META(0, 0, 1);
            rr.v[0] = v.x;
            rr.v[1] = v.y;
            rr.v[2] = v.z;
            rr.v[3] = v.w;
            pend[pos] = rr;
        }
    }
}

/* ORDERED / SEQUENTIAL: validity flags, then an order-preserving compaction */
__global__ void k_apply_flags(ApplyArgs a, uint32_t *valid) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    const bool isc = a.isc ? a.isc[i] != 0 : false;
    const double w = a.w[i];
    const double r = (isc || !a.vr) ? 0.0 : a.vr[i], g = (isc || !a.vg) ? 0.0 : a.vg[i],
                 b = (isc || !a.vb) ? 0.0 : a.vb[i];
    bool ok = update_valid(isc, r, g, b, w);
    valid[i] = ok ? 1u : 0u;
    if (!ok) atomicAdd(&a.s.ctr[C_REJECTED], 1ull);
}

__global__ void k_apply_records(ApplyArgs a, const uint32_t *valid, const uint32_t *scan,
                                PendRec *pend, uint64_t *seq) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= a.n || !valid[i]) return;
    const bool isc = a.isc ? a.isc[i] != 0 : false;
    pstf_key k = a.keys[i];
    PendRec rr;
    rr.k[0] = k.level;
    rr.k[1] = k.cell[0];
    rr.k[2] = k.cell[1];
    rr.k[3] = k.cell[2];
    rr.k[4] = k.dir_cell[0];
    rr.k[5] = k.dir_cell[1];
    rr.cs = k.checksum;
    rr.meta = PSTF_META(0, isc ? 1 : 0, 1);
    /* a counter call keeps its value: the queue orders a key's calls by (isCounter, bits r, g,
     * b, w) whatever they are (field.cpp:402-410); the fold ignores it (field.cpp:413-414) */
    rr.v[0] = a.vr ? a.vr[i] : 0.0;
    rr.v[1] = a.vg ? a.vg[i] : 0.0;
    rr.v[2] = a.vb ? a.vb[i] : 0.0;
    rr.v[3] = a.w[i];
    uint32_t pos = scan[i];
    pend[pos] = rr;
    if (seq) seq[pos] = i;
}

/* ------------------------------------------------------------------------------------------ */
/* phase 2: sort pending records into priority order                                           */

#define NF_KEY 7 /* store, level, c0, c1, c2, d0, d1 */
enum { F_STORE = 0, F_LEVEL, F_C0, F_C1, F_C2, F_D0, F_D1, F_ISC, F_R, F_G, F_B, F_W, F_SEQ, F_MAX };

struct Layout {
    int nfields;
    int fid[F_MAX];
    int word[F_MAX];
    int shift[F_MAX];
    int bits[F_MAX];
    long long minv[F_MAX];
    int nwords;
    int begin_bit[F_MAX];
};

__device__ __forceinline__ int rec_field_i(const PendRec &r, int f) {
    return f == F_STORE ? (int)PSTF_META_SID(r.meta) : r.k[f - 1];
}

/* min/max of the 7 key fields over the pending records; out[2f] = min, out[2f+1] = max */
__global__ void k_ranges(const PendRec *pend, const unsigned long long *count, uint64_t cap,
                         int *out) {
    uint64_t n = *count;
    if (n > cap) n = cap;
    int mn[NF_KEY], mx[NF_KEY];
    for (int f = 0; f < NF_KEY; ++f) {
        mn[f] = INT32_MAX;
        mx[f] = INT32_MIN;
    }
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        PendRec r = pend[i];
        for (int f = 0; f < NF_KEY; ++f) {
            int v = rec_field_i(r, f);
            mn[f] = min(mn[f], v);
            mx[f] = max(mx[f], v);
        }
    }
    /* warp, then block reduction: one pair of atomics per field per block (the 14 global
     * words are shared by every block, so per-warp atomics serialise) */
    __shared__ int smn[NF_KEY], smx[NF_KEY];
    if (threadIdx.x < NF_KEY) {
        smn[threadIdx.x] = INT32_MAX;
        smx[threadIdx.x] = INT32_MIN;
    }
    __syncthreads();
    for (int f = 0; f < NF_KEY; ++f) {
        int a = __reduce_min_sync(0xffffffffu, mn[f]);
        int b = __reduce_max_sync(0xffffffffu, mx[f]);
        if (lane_id() == 0) {
            atomicMin(&smn[f], a);
            atomicMax(&smx[f], b);
        }
    }
    __syncthreads();
    if (threadIdx.x < NF_KEY) {
        atomicMin(&out[2 * threadIdx.x], smn[threadIdx.x]);
        atomicMax(&out[2 * threadIdx.x + 1], smx[threadIdx.x]);
    }
}

__global__ void k_encode(const PendRec *pend, const uint64_t *seq, uint64_t n, Layout L,
                         uint64_t *words) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    PendRec r = pend[i];
    uint64_t w[F_MAX];
    for (int k = 0; k < L.nwords; ++k) w[k] = 0;
    for (int q = 0; q < L.nfields; ++q) {
        int f = L.fid[q];
        uint64_t v;
        if (f < NF_KEY) v = (uint64_t)((long long)rec_field_i(r, f) - L.minv[q]);
        else if (f == F_ISC) v = PSTF_META_ISC(r.meta);
        else if (f == F_SEQ) v = seq[i];
        else v = dbits(r.v[f - F_R]);
        w[L.word[q]] |= L.bits[q] == 64 ? v : (v << L.shift[q]);
    }
    for (int k = 0; k < L.nwords; ++k) words[(uint64_t)k * n + i] = w[k];
}

__global__ void k_iota(uint32_t *p, uint64_t n) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = (uint32_t)i;
}

__global__ void k_gather_u64(const uint64_t *src, const uint32_t *perm, uint64_t n, uint64_t *dst) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[perm[i]];
}

/* head[j] = 1 where the (store, key) of sorted position j differs from j-1 */
__global__ void k_heads(const PendRec *pend, const uint32_t *perm, uint64_t n, uint32_t *head) {
    uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    if (j == 0) {
        head[0] = 1;
        return;
    }
    PendRec a = pend[perm[j - 1]], b = pend[perm[j]];
    bool same = PSTF_META_SID(a.meta) == PSTF_META_SID(b.meta);
    for (int f = 0; f < 6; ++f) same = same && a.k[f] == b.k[f];
    head[j] = same ? 0u : 1u;
}

struct UniqArgs {
    uint32_t *ufirst;
    KeyFields *ukey;
    uint32_t *ucs, *usid, *uhome;
    uint32_t *ucalls;
    double4 *usum;
    uint64_t *useq; // first submission seq (SEQUENTIAL)
};

__global__ void k_unique_build(const PendRec *pend, const uint32_t *perm, const uint32_t *head,
                               const uint32_t *uid, const uint64_t *seq, uint64_t n, Stores4 st,
                               UniqArgs u) {
    uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j >= n || !head[j]) return;
    uint32_t q = uid[j] - 1u;
    uint32_t r = perm[j];
    PendRec p = pend[r];
    u.ufirst[q] = (uint32_t)j;
    KeyFields kf = {p.k[0], p.k[1], p.k[2], p.k[3], p.k[4], p.k[5]};
    u.ukey[q] = kf;
    u.ucs[q] = p.cs;
    uint32_t sid = PSTF_META_SID(p.meta);
    u.usid[q] = sid;
    uint64_t pk = pack_key_fields(p.k[0], p.k[1], p.k[2], p.k[3], p.k[4], p.k[5]);
    u.uhome[q] = (uint32_t)pk & st.s[sid].mask;
    if (u.useq) u.useq[q] = seq[r];
}

/* per-unique sums (ATOMIC) and call counts (all modes), warp-aggregated over sorted runs */
__global__ void k_unique_sums(const PendRec *pend, const uint32_t *perm, const uint32_t *uid,
                              uint64_t n, int atomic_mode, UniqArgs u, int own_origin) {
    __shared__ double4 smem[8][32];
    double4 *sm = smem[threadIdx.x >> 5];
    uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    bool live = j < n;
    uint32_t q = live ? uid[j] - 1u : 0xffffffffu;
    double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
    uint32_t calls = 0;
    if (live) {
        PendRec p = pend[perm[j]];
        /* sharded: only this rank's records add values / count drops here (the other ranks'
         * records are present so that every replica places every new key identically) */
        if (own_origin < 0 || (int)PSTF_META_ORIGIN(p.meta) == own_origin) {
            v = make_double4(p.v[0], p.v[1], p.v[2], p.v[3]);
            calls = PSTF_META_CALLS(p.meta);
        }
    }
    unsigned peers = __match_any_sync(0xffffffffu, q);
    sm[lane_id()] = v;
    __syncwarp();
    if (live && (int)lane_id() == __ffs(peers) - 1) {
        double4 t = make_double4(0.0, 0.0, 0.0, 0.0);
        unsigned m = peers;
        while (m) {
            int l = __ffs(m) - 1;
            m &= m - 1;
            double4 x = sm[l];
            t.x += x.x;
            t.y += x.y;
            t.z += x.z;
            t.w += x.w;
        }
        if (atomic_mode) {
            if (t.x != 0.0) atomicAdd(&u.usum[q].x, t.x);
            if (t.y != 0.0) atomicAdd(&u.usum[q].y, t.y);
            if (t.z != 0.0) atomicAdd(&u.usum[q].z, t.z);
            if (t.w != 0.0) atomicAdd(&u.usum[q].w, t.w);
        }
    }
    /* call counts: integer, any order */
    unsigned c = __reduce_add_sync(peers, calls);
    if (live && (int)lane_id() == __ffs(peers) - 1) atomicAdd(&u.ucalls[q], c);
}

__global__ void k_rank_scatter(const uint32_t *sorted_uid, uint64_t nu, uint32_t *rank,
                               const uint32_t *ucs, uint32_t *cs_by_rank) {
    uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (r >= nu) return;
    uint32_t u = sorted_uid[r];
    rank[u] = (uint32_t)r;
    cs_by_rank[r] = ucs[u];
}

/* ------------------------------------------------------------------------------------------ */
/* phase 2: deterministic placement (deferred acceptance, Jacobi rounds)                       */

struct PlaceArgs {
    Stores4 st;
    uint64_t nu;
    const uint32_t *usid, *uhome, *ucs;
    const uint32_t *rank;       // NULL -> rank = u
    const uint32_t *cs_by_rank; // checksum of the key holding rank r
    int parity;                 // which hold array is "prev"
    const unsigned *nu_dev;     // unique count on the device (sort-free path), else NULL
};

__device__ __forceinline__ uint64_t place_nu(const PlaceArgs &a) {
    return a.nu_dev ? (uint64_t)*a.nu_dev : a.nu;
}

/* sort-free ATOMIC phase 2: dedup hash table over the records' order-preserving key words */
struct Dedup {
    const uint64_t *words; /* words[i]: (store, level, cells, dirs) of record i, key order */
    const uint32_t *tab;   /* open addressing, record index of the representative, ~0 empty */
    uint32_t mask;
    const PendRec *pend;
};

__device__ __forceinline__ uint32_t dd_hash(uint64_t w) { return (uint32_t)mix_bits(w); }

/* checksum of the unique key whose key word is w (present in the table) */
__device__ __forceinline__ uint32_t dd_checksum(const Dedup &d, uint64_t w) {
    for (uint32_t h = dd_hash(w) & d.mask;; h = (h + 1) & d.mask) {
        const uint32_t r = d.tab[h];
        if (r == 0xffffffffu) return 0u; /* not reachable: every hold value is a present key */
        if (d.words[r] == w) return d.pend[r].cs;
    }
}

/* One key's step of a placement round (deferred acceptance over the frame-start table): the
 * first equal-checksum resident (FIXED), else the first slot held by a higher-priority key with
 * an equal checksum (MERGE), else the first free slot not held by a higher-priority key
 * (PROPOSE), else DROP.  The window's home words are loaded 8 at a time (independent loads:
 * one round trip per 8 probes on crowded tables). */
__device__ __forceinline__ unsigned long long place_step(const PlaceArgs &a, uint64_t u,
                                                         int parity) {
    const DevStore &s = a.st.s[a.usid[u]];
    const uint32_t *hold_prev = parity ? s.hold1 : s.hold0;
    const uint32_t r = a.rank ? a.rank[u] : (uint32_t)u;
    const uint32_t cs = a.ucs[u];
    const uint32_t home = a.uhome[u];
    for (uint32_t i0 = 0; i0 < s.window; i0 += 8) {
        uint32_t c[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            c[j] = i0 + j < s.window ? s.meta[(home + i0 + j) & s.mask].x : 0xffffffffu;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (i0 + j >= s.window) return PSTF_RES(R_DROP, 0);
            const uint32_t idx = (home + i0 + j) & s.mask;
            if (c[j] != 0) {
                if (c[j] == cs) return PSTF_RES(R_FIXED, idx); /* older resident (field.cpp:122) */
                continue;
            }
            const uint32_t h = hold_prev[idx];
            if (h < r) {
                if (a.cs_by_rank[h] == cs) return PSTF_RES(R_MERGE, idx); /* higher-priority twin */
                continue;
            }
            return PSTF_RES(R_PROPOSE, idx);
        }
    }
    return PSTF_RES(R_DROP, 0);
}

__device__ __forceinline__ uint32_t *hold_array(const DevStore &s, int which) {
    return which ? s.hold1 : s.hold0;
}

/* All placement rounds in one cooperative launch (grid-wide barriers instead of host round
 * trips): round k reads hold[parity_k] and res[k&1], proposes into hold[parity_k^1] and writes
 * res[(k+1)&1]; then the previous round's proposals are cleared from hold[parity_k].  Stops at
 * the fixpoint (no result changed).  Epilogue: the final results land in r0, the last round's
 * proposals are cleared, and every store of the batch records the round count. */
__global__ void __launch_bounds__(256) k_place_loop(PlaceArgs a, unsigned long long *r0,
                                                    unsigned long long *r1, int *ctl,
                                                    uint32_t max_rounds) {
    cg::grid_group g = cg::this_grid();
    const uint64_t tid0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    int parity = a.parity;
    unsigned long long *prev = r0, *next = r1;
    uint32_t k = 0;
    for (;; ++k) {
        bool changed = false;
        for (uint64_t u = tid0; u < a.nu; u += stride) {
            const unsigned long long res = place_step(a, u, parity);
            if (PSTF_RES_T(res) == R_PROPOSE)
                atomicMin(&hold_array(a.st.s[a.usid[u]], parity ^ 1)[PSTF_RES_SLOT(res)],
                          a.rank ? a.rank[u] : (uint32_t)u);
            next[u] = res;
            changed |= res != prev[u];
        }
        if (__syncthreads_or(changed) && threadIdx.x == 0) atomicOr(&ctl[k & 1], 1);
        g.sync();
        for (uint64_t u = tid0; u < a.nu; u += stride) { /* clear the previous round's holds */
            const unsigned long long res = prev[u];
            if (PSTF_RES_T(res) == R_PROPOSE)
                hold_array(a.st.s[a.usid[u]], parity)[PSTF_RES_SLOT(res)] = PSTF_HOLD_NONE;
        }
        const int ch = *(volatile int *)&ctl[k & 1];
        g.sync(); /* everyone has read the flag before it is reset for round k + 2 */
        if (tid0 == 0) ctl[k & 1] = 0;
        unsigned long long *t = prev;
        prev = next;
        next = t;
        parity ^= 1;
        if (!ch) break;
        if (k + 1 > max_rounds) {
            if (tid0 == 0) ctl[3] = 1;
            break;
        }
    }
    /* prev = the last round's results; its proposals sit in hold[parity ^ 1] */
    for (uint64_t u = tid0; u < a.nu; u += stride) {
        const unsigned long long res = prev[u];
        if (prev != r0) r0[u] = res;
        if (PSTF_RES_T(res) == R_PROPOSE)
            hold_array(a.st.s[a.usid[u]], parity ^ 1)[PSTF_RES_SLOT(res)] = PSTF_HOLD_NONE;
    }
    if (tid0 == 0) {
        ctl[2] = (int)(k + 1);
        for (int i = 0; i < 4; ++i)
            if (a.st.s[i].ctr) a.st.s[i].ctr[C_ROUNDS] = k + 1;
    }
}

/* ---- sort-free ATOMIC phase 2 ------------------------------------------------------------ */
/* every record finds (or becomes) the representative of its key word */
__global__ void k_dd_insert(const uint64_t *words, uint64_t n, uint32_t *tab, uint32_t mask,
                            uint32_t *rep_of) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t w = words[i];
    for (uint32_t h = dd_hash(w) & mask;; h = (h + 1) & mask) {
        uint32_t cur = tab[h];
        if (cur == 0xffffffffu) {
            cur = atomicCAS(&tab[h], 0xffffffffu, (uint32_t)i);
            if (cur == 0xffffffffu) {
                rep_of[i] = (uint32_t)i;
                return;
            }
        }
        if (words[cur] == w) {
            rep_of[i] = cur;
            return;
        }
    }
}

/* representatives become unique keys (unique ids in arbitrary order; priority = key word) */
__global__ void k_dd_unique(const PendRec *pend, const uint64_t *words, const uint32_t *rep_of,
                            uint64_t n, Stores4 st, UniqArgs u, uint64_t *ukw, uint32_t *uidx,
                            unsigned *nu) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const bool rep = i < n && rep_of[i] == (uint32_t)i;
    const unsigned m = __ballot_sync(0xffffffffu, rep);
    if (!m) return;
    unsigned base = 0;
    if ((int)lane_id() == __ffs(m) - 1) base = atomicAdd(nu, (unsigned)__popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (!rep) return;
    const uint32_t q = base + __popc(m & ((1u << lane_id()) - 1u));
    uidx[i] = q;
    const PendRec p = pend[i];
    u.ufirst[q] = (uint32_t)i;
    u.ukey[q] = KeyFields{p.k[0], p.k[1], p.k[2], p.k[3], p.k[4], p.k[5]};
    u.ucs[q] = p.cs;
    const uint32_t sid = PSTF_META_SID(p.meta);
    u.usid[q] = sid;
    u.uhome[q] = (uint32_t)pack_key_fields(p.k[0], p.k[1], p.k[2], p.k[3], p.k[4], p.k[5]) &
                 st.s[sid].mask;
    u.ucalls[q] = 0u;
    u.usum[q] = make_double4(0.0, 0.0, 0.0, 0.0);
    ukw[q] = words[i];
}

/* per-unique sums and call counts (ATOMIC: any order) */
__global__ void k_dd_sums(const PendRec *pend, const uint32_t *rep_of, const uint32_t *uidx,
                          uint64_t n, UniqArgs u, int own_origin) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const PendRec p = pend[i];
    /* sharded: only this rank's records add values / count calls (see k_unique_sums) */
    if (own_origin >= 0 && (int)PSTF_META_ORIGIN(p.meta) != own_origin) return;
    const uint32_t q = uidx[rep_of[i]];
    if (p.v[0] != 0.0) atomicAdd(&u.usum[q].x, p.v[0]);
    if (p.v[1] != 0.0) atomicAdd(&u.usum[q].y, p.v[1]);
    if (p.v[2] != 0.0) atomicAdd(&u.usum[q].z, p.v[2]);
    if (p.v[3] != 0.0) atomicAdd(&u.usum[q].w, p.v[3]);
    atomicAdd(&u.ucalls[q], PSTF_META_CALLS(p.meta));
}

/* placement with 64-bit key-word priorities: the same deferred acceptance as k_place_loop
 * (sequential insertion in ascending key order), the holder of a slot identified by its key
 * word, its checksum found through the dedup table */
__device__ __forceinline__ unsigned long long place_step64(const PlaceArgs &a, const uint64_t *ukw,
                                                           const Dedup &dd, uint64_t u,
                                                           int parity) {
    const DevStore &s = a.st.s[a.usid[u]];
    const unsigned long long *hold_prev = parity ? s.hold64_1 : s.hold64_0;
    const uint64_t r = ukw[u];
    const uint32_t cs = a.ucs[u];
    const uint32_t home = a.uhome[u];
    for (uint32_t i0 = 0; i0 < s.window; i0 += 8) {
        uint32_t c[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            c[j] = i0 + j < s.window ? s.meta[(home + i0 + j) & s.mask].x : 0xffffffffu;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (i0 + j >= s.window) return PSTF_RES(R_DROP, 0);
            const uint32_t idx = (home + i0 + j) & s.mask;
            if (c[j] != 0) {
                if (c[j] == cs) return PSTF_RES(R_FIXED, idx); /* older resident (field.cpp:122) */
                continue;
            }
            const unsigned long long h = hold_prev[idx];
            if (h < r) {
                if (dd_checksum(dd, h) == cs) return PSTF_RES(R_MERGE, idx); /* higher-priority twin */
                continue;
            }
            return PSTF_RES(R_PROPOSE, idx);
        }
    }
    return PSTF_RES(R_DROP, 0);
}

__device__ __forceinline__ unsigned long long *hold64(const DevStore &s, int which) {
    return which ? s.hold64_1 : s.hold64_0;
}

__global__ void __launch_bounds__(256) k_place_loop64(PlaceArgs a, const uint64_t *ukw, Dedup dd,
                                                      unsigned long long *r0,
                                                      unsigned long long *r1, int *ctl,
                                                      uint32_t max_rounds) {
    cg::grid_group g = cg::this_grid();
    const uint64_t tid0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t nu = place_nu(a);
    int parity = a.parity;
    unsigned long long *prev = r0, *next = r1;
    uint32_t k = 0;
    for (;; ++k) {
        bool changed = false;
        for (uint64_t u = tid0; u < nu; u += stride) {
            const unsigned long long res = place_step64(a, ukw, dd, u, parity);
            if (PSTF_RES_T(res) == R_PROPOSE)
                atomicMin(&hold64(a.st.s[a.usid[u]], parity ^ 1)[PSTF_RES_SLOT(res)],
                          (unsigned long long)ukw[u]);
            next[u] = res;
            changed |= res != prev[u];
        }
        if (__syncthreads_or(changed) && threadIdx.x == 0) atomicOr(&ctl[k & 1], 1);
        g.sync();
        for (uint64_t u = tid0; u < nu; u += stride) {
            const unsigned long long res = prev[u];
            if (PSTF_RES_T(res) == R_PROPOSE)
                hold64(a.st.s[a.usid[u]], parity)[PSTF_RES_SLOT(res)] = ~0ull;
        }
        const int ch = *(volatile int *)&ctl[k & 1];
        g.sync();
        if (tid0 == 0) ctl[k & 1] = 0;
        unsigned long long *t = prev;
        prev = next;
        next = t;
        parity ^= 1;
        if (!ch) break;
        if (k + 1 > max_rounds) {
            if (tid0 == 0) ctl[3] = 1;
            break;
        }
    }
    for (uint64_t u = tid0; u < nu; u += stride) {
        const unsigned long long res = prev[u];
        if (prev != r0) r0[u] = res;
        if (PSTF_RES_T(res) == R_PROPOSE)
            hold64(a.st.s[a.usid[u]], parity ^ 1)[PSTF_RES_SLOT(res)] = ~0ull;
    }
    if (tid0 == 0) {
        ctl[2] = (int)(k + 1);
        for (int i = 0; i < 4; ++i)
            if (a.st.s[i].ctr) a.st.s[i].ctr[C_ROUNDS] = k + 1;
    }
}

__global__ void k_commit(PlaceArgs a, const unsigned long long *res, const KeyFields *ukey,
                         const uint32_t *ucalls, const double4 *usum, int atomic_mode) {
    uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (u >= place_nu(a)) return;
    const DevStore &s = a.st.s[a.usid[u]];
    unsigned long long r = res[u];
    uint32_t t = PSTF_RES_T(r), slot = PSTF_RES_SLOT(r);
    if (t == R_DROP) {
        atomicAdd(&s.ctr[C_DROPPED], (unsigned long long)ucalls[u]);
        return;
    }
    if (t == R_PROPOSE) {
        s.meta[slot].x = a.ucs[u]; /* (k_place_loop has released the slot's hold) */
        atomicOr(&s.lbits[slot >> 5], 1u << (slot & 31u));
        s.keyf[slot] = ukey[u];
        /* live / new-key counters: one atomic per group of lanes of the same store */
        const unsigned grp = __match_any_sync(__activemask(), a.usid[u]);
        if ((int)lane_id() == __ffs(grp) - 1) {
            atomicAdd(&s.ctr[C_LIVE], (unsigned long long)__popc(grp));
            atomicAdd(&s.ctr[C_NEW_KEYS], (unsigned long long)__popc(grp));
        }
    }
    if (atomic_mode) {
        double4 v = usum[u];
        double4 *dst = acc_ptr(s, slot);
        if (v.x != 0.0) atomicAdd(&dst->x, v.x);
        if (v.y != 0.0) atomicAdd(&dst->y, v.y);
        if (v.z != 0.0) atomicAdd(&dst->z, v.z);
        if (v.w != 0.0) atomicAdd(&dst->w, v.w);
    }
    /* sharded: a replica touches a slot for its own records only (the all-reduce of the
     * accumulators marks the slots the other ranks touched) */
    if (ucalls[u] != 0) {
        /* unit-weight frame accounting (k_ef_onepass): the counter calls of these records */
        touch_slot(s, slot);
        if (atomic_mode) atomicAdd(&s.ctr[C_F_CN], (unsigned long long)usum[u].w);
    }
}

/* ORDERED / SEQUENTIAL: per-record fold target (store << 32 | slot), dropped -> ~0 */
__global__ void k_fold_targets(const uint32_t *perm, const uint32_t *uid, uint64_t n,
                               const unsigned long long *res, const uint32_t *usid,
                               int by_record, uint64_t *tgt, uint32_t *order) {
    uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    uint32_t u = uid[j] - 1u;
    unsigned long long r = res[u];
    uint64_t t = PSTF_RES_T(r) == R_DROP
                     ? ~0ull
                     : (((uint64_t)usid[u] << 32) | (uint64_t)PSTF_RES_SLOT(r));
    uint32_t rec = perm[j];
    if (by_record) { /* SEQUENTIAL: position = record index = submission order */
        tgt[rec] = t;
        order[rec] = rec;
    } else { /* ORDERED: position = canonical sorted position */
        tgt[j] = t;
        order[j] = rec;
    }
}

/* one thread per run of equal targets: sequential fold in the sorted order (field.cpp:413-418) */
/* the fold's terms in final (slot, canonical) order, computed in parallel: value.c * w of an
 * accumulate (field.cpp:168-170), w of a counter (field.cpp:157); contiguous, so the
 * sequential per-slot fold below streams instead of gathering 64 B records */
__global__ void k_fold_terms(const PendRec *pend, const uint32_t *recs, uint64_t n, double4 *T,
                             uint8_t *isc) {
    uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (q >= n) return;
    const PendRec r = pend[recs[q]];
    const double w = r.v[3];
    const bool c = PSTF_META_ISC(r.meta) != 0;
    T[q] = c ? make_double4(0.0, 0.0, 0.0, w)
             : make_double4(r.v[0] * w, r.v[1] * w, r.v[2] * w, 0.0);
    isc[q] = c;
}

/* run starts of the target-sorted terms: head flags, then (after a scan) their positions */
__global__ void k_fold_heads(const uint64_t *tgt, uint64_t n, uint32_t *head) {
    uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (p < n) head[p] = p == 0 || tgt[p] != tgt[p - 1];
}

__global__ void k_fold_starts(const uint32_t *head, const uint32_t *run, uint64_t n,
                              uint32_t *start) {
    uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (p < n && head[p]) start[run[p]] = (uint32_t)p;
    if (p == n - 1) start[run[p] + head[p]] = (uint32_t)n; /* sentinel: end of the last run */
}

__global__ void k_fold_nruns(const uint32_t *head, const uint32_t *run, uint64_t n, uint32_t *nr) {
    nr[0] = run[n - 1] + head[n - 1];
}

/* sequential fold per target slot in canonical order (FieldUpdateQueue::apply, field.cpp:
 * 396-420), one thread per run.  The run's bounds are known, so the term loads are issued 8
 * at a time ahead of the dependent fp64 adds (the hottest slots take tens of thousands of
 * calls: their chains would otherwise wait on a load per call). */
__device__ __forceinline__ void fold_one(double4 &acc, const double4 v, bool c) {
    if (c) {
        if (v.w > 0.0) acc.w += v.w; /* field.cpp:157 */
    } else {
        acc.x += v.x; /* field.cpp:168-170 */
        acc.y += v.y;
        acc.z += v.z;
    }
}

#define FOLD_LONG 256 /* runs at least this long are folded by a warp (k_fold_long) */

__global__ void k_fold(const double4 *__restrict__ T, const uint8_t *__restrict__ isc,
                       const uint64_t *tgt, const uint32_t *start, const uint32_t *nruns,
                       Stores4 st) {
    const uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (r >= *nruns) return;
    const uint32_t q0 = start[r], q1 = start[r + 1];
    if (q1 - q0 >= FOLD_LONG) return;
    const uint64_t t = tgt[q0];
    if (t == ~0ull) return;
    const DevStore &s = st.s[t >> 32];
    const uint32_t slot = (uint32_t)t;
    double4 acc = *acc_ptr(s, slot);
    uint32_t q = q0;
    for (; q + 8 <= q1; q += 8) {
        double4 v[8];
        bool c[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            v[k] = T[q + k];
            c[k] = isc[q + k] != 0;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) fold_one(acc, v[k], c[k]);
    }
    for (; q < q1; ++q) fold_one(acc, T[q], isc[q] != 0);
    *acc_ptr(s, slot) = acc;
}

/* the long runs, one warp each: lanes load 32 consecutive terms (one memory latency per 32
 * calls instead of per call, the next 32 prefetched), every lane applies them in order from
 * broadcasts, so each lane carries the same sequential sum */
__global__ void k_fold_long(const double4 *__restrict__ T, const uint8_t *__restrict__ isc,
                            const uint64_t *tgt, const uint32_t *start, const uint32_t *nruns,
                            Stores4 st) {
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t nr = *nruns;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < nr;
         r += nwarps) {
        const uint32_t q0 = start[r], q1 = start[r + 1];
        if (q1 - q0 < FOLD_LONG) continue; /* warp-uniform */
        const uint64_t t = tgt[q0];
        if (t == ~0ull) continue;
        const DevStore &s = st.s[t >> 32];
        const uint32_t slot = (uint32_t)t;
        double4 acc = *acc_ptr(s, slot);
        double4 nv = q0 + lane < q1 ? T[q0 + lane] : make_double4(0.0, 0.0, 0.0, 0.0);
        int nc = q0 + lane < q1 ? isc[q0 + lane] : 0;
        for (uint32_t b = q0; b < q1; b += 32) {
            const double4 v = nv;
            const int c = nc;
            const uint32_t nb = b + 32; /* prefetch the next 32 */
            if (nb + lane < q1) {
                nv = T[nb + lane];
                nc = isc[nb + lane];
            }
            const int k = (int)min(32u, q1 - b);
            /* fully unrolled: the broadcasts do not depend on acc, so they run ahead of the
             * dependent adds */
#pragma unroll
            for (int l = 0; l < 32; ++l) {
                const double4 u = make_double4(__shfl_sync(0xffffffffu, v.x, l),
                                               __shfl_sync(0xffffffffu, v.y, l),
                                               __shfl_sync(0xffffffffu, v.z, l),
                                               __shfl_sync(0xffffffffu, v.w, l));
                const int cu = __shfl_sync(0xffffffffu, c, l);
                if (l < k) fold_one(acc, u, cu != 0);
            }
        }
        if (lane == 0) *acc_ptr(s, slot) = acc;
    }
}


/* ------------------------------------------------------------------------------------------ */
/* K3: endFrame (field.cpp:197-263), all stores of a batch in one launch per pass            */

__device__ __forceinline__ double warp_sum_d(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

#define EF_BLOCK 256

/* Pass 1 (field.cpp:205-216) for every store of the batch: compact the touched-slot bitmap into
 * tlist (clearing it), sum c_new over those slots (untouched slots have zero accumulators by
 * construction) and snapshot `live` for the eviction rule. */
#define PICK4(a, j) ((j) == 0 ? (a)[0] : (j) == 1 ? (a)[1] : (j) == 2 ? (a)[2] : (a)[3])

/* store j of a batch with segment boundaries seg[1..3] (seg[nst..3] = the total) */
#define SEG_OF(i, seg) (((i) >= (seg)[1]) + ((i) >= (seg)[2]) + ((i) >= (seg)[3]))

/* endFrame pass 1 for every store of the batch at once: the touched bitmaps become touched lists
 * (tbits cleared) and Σ c_new / #(c_new > 0) are reduced (field.cpp:201-214).  The stores'
 * bitmap words form one flat index space, each store's range padded to whole warps, so a warp
 * never straddles two stores; the c_new gathers of a word's set bits are issued 8 at a time. */
__device__ __forceinline__ void ef_reduce_body(const Stores4 &st, int nst);
__device__ __forceinline__ void ef_blend_body(const Stores4 &st, int nst);
__device__ __forceinline__ void ef_evict_body(const Stores4 &st, int nst, int finish);

__global__ void __launch_bounds__(EF_BLOCK) k_ef_reduce(Stores4 st, int nst,
                                                        const unsigned long long *guard) {
    if (guard && *guard) return; /* new keys still pending: the host places them first */
    ef_reduce_body(st, nst);
}
__global__ void __launch_bounds__(EF_BLOCK) k_ef_blend(Stores4 st, int nst,
                                                       const unsigned long long *guard) {
    if (guard && *guard) return;
    ef_blend_body(st, nst);
}
__global__ void __launch_bounds__(EF_BLOCK) k_ef_evict(Stores4 st, int nst, int finish,
                                                       const unsigned long long *guard) {
    if (guard && *guard) return;
    ef_evict_body(st, nst, finish);
}

/* the three endFrame passes in one cooperative launch (grid barriers between them) */
__global__ void __launch_bounds__(EF_BLOCK) k_ef_fused(Stores4 st, int nst,
                                                       const unsigned long long *guard) {
    if (guard && *guard) return; /* uniform across the grid: every block returns */
    cg::grid_group g = cg::this_grid();
    ef_reduce_body(st, nst);
    g.sync();
    ef_blend_body(st, nst);
    g.sync();
    ef_evict_body(st, nst, 1);
}

__device__ __forceinline__ void ef_reduce_body(const Stores4 &st, int nst) {
    __shared__ double ssum[4][EF_BLOCK / 32];
    __shared__ unsigned long long scnt[4][EF_BLOCK / 32];
    uint64_t seg[4], nw[4];
    uint64_t acc_w = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) { /* static indices only: the arrays stay in registers */
        nw[j] = j < nst ? ((uint64_t)st.s[j].mask + 32) / 32 : 0;
        seg[j] = acc_w;
        acc_w += (nw[j] + 31) & ~31ull;
    }
    const uint64_t total = acc_w; /* stores >= nst have no words: seg[j >= nst] == total */
    if (blockIdx.x == 0 && threadIdx.x < (unsigned)nst) {
        const DevStore &s = st.s[threadIdx.x];
        s.ctr[C_LIVE_SNAP] = s.ctr[C_LIVE];
        s.ctr[C_EVICTED] = 0;
    }
    double sum[4] = {0.0, 0.0, 0.0, 0.0};
    unsigned cnt[4] = {0u, 0u, 0u, 0u};
    const unsigned lane = lane_id();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t iters = (total + stride - 1) / stride;
    for (uint64_t it = 0; it < iters; ++it) { /* warp-uniform trip count (shuffles below) */
        const uint64_t gi = it * stride + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
        const int j = min(SEG_OF(gi, seg), nst - 1);
        const uint64_t wi = gi - PICK4(seg, j);
        const DevStore &s = st.s[j];
        uint32_t w = gi < total && wi < PICK4(nw, j) ? s.tbits[wi] : 0u;
        if (w) s.tbits[wi] = 0u;
        const unsigned c = __popc(w);
        unsigned incl = c;
        for (int o = 1; o < 32; o <<= 1) {
            unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)lane >= o) incl += t;
        }
        const unsigned wtotal = __shfl_sync(0xffffffffu, incl, 31);
        if (!wtotal) continue;
        unsigned long long base = 0;
        if (lane == 31) base = atomicAdd(&s.ctr[C_TOUCHED_N], (unsigned long long)wtotal);
        base = __shfl_sync(0xffffffffu, base, 31);
        unsigned long long pos = base + (incl - c);
        double lsum = 0.0;
        unsigned lcnt = 0;
        while (w) {
            uint32_t sl[8];
            double cn[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                sl[q] = w ? (uint32_t)(wi * 32 + (uint64_t)(__ffs(w) - 1)) : 0xffffffffu;
                w &= w - 1;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) cn[q] = sl[q] != 0xffffffffu ? acc_ptr(s, sl[q])->w : 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (sl[q] != 0xffffffffu) {
                    s.tlist[pos++] = sl[q];
                    if (cn[q] > 0.0) {
                        lsum += cn[q];
                        ++lcnt;
                    }
                }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q == j) {
                sum[q] += lsum;
                cnt[q] += lcnt;
            }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const double t = warp_sum_d(sum[q]);
        const unsigned cc = __reduce_add_sync(0xffffffffu, cnt[q]);
        if (lane == 0) {
            ssum[q][threadIdx.x >> 5] = t;
            scnt[q][threadIdx.x >> 5] = cc;
        }
    }
    __syncthreads();
    if (threadIdx.x < (unsigned)nst) {
        const int q = threadIdx.x;
        double t = 0.0;
        unsigned long long c = 0;
        for (int w = 0; w < EF_BLOCK / 32; ++w) {
            t += ssum[q][w];
            c += scnt[q][w];
        }
        if (c) {
            /* an inexact frame's sum is already there, summed in slot order (k_cn_seq) */
            if (!st.s[q].ctr[C_CN_INEXACT]) atomicAdd(st.s[q].cn_sum, t);
            atomicAdd(&st.s[q].ctr[C_CN_COUNT], c);
        }
    }
}

/* ---- Σc_new in the reference's order (field.cpp:201-213: slot order, left to right) ----
 * A frame whose counter weights are whole numbers <= 2^20 (every vertex pass: weight 1) has an
 * exact Σc_new, so the reduce pass sums it in any order.  Otherwise (C_CN_INEXACT, raised by
 * pstf_field_apply) the touched slots' c_new values are compacted in slot order and summed by
 * one thread, so the mean, and with it the c_old cap, is bitwise the reference's for any
 * weights.  Every kernel here returns at once in exact frames. */
__global__ void k_cn_flag(const double *w, const uint8_t *isc, uint64_t n,
                          unsigned long long *ctr) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    bool bad = false;
    if (i < n && isc[i]) {
        const double x = w[i];
        bad = x >= 0.0 && isfinite(x) && (x != floor(x) || x > 1048576.0); /* counted calls */
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31u) == 0) atomicOr(&ctr[C_CN_INEXACT], 1ull);
}

__global__ void k_cn_words(DevStore s, const unsigned long long *guard, uint32_t *cnt) {
    if ((guard && *guard) || !s.ctr[C_CN_INEXACT]) return;
    const uint64_t nw = ((uint64_t)s.mask + 32) / 32;
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < nw) cnt[i] = __popc(s.tbits[i]);
}

__global__ void k_cn_scatter(DevStore s, const unsigned long long *guard, const uint32_t *pos,
                             double *V) {
    if ((guard && *guard) || !s.ctr[C_CN_INEXACT]) return;
    const uint64_t nw = ((uint64_t)s.mask + 32) / 32;
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= nw) return;
    uint32_t w = s.tbits[i], p = pos[i];
    while (w) {
        const uint32_t slot = (uint32_t)(i * 32 + (uint64_t)(__ffs(w) - 1));
        w &= w - 1;
        /* live slots only (field.cpp:205-206); c_new <= 0 adds nothing to a sum that starts at
         * +0.0 and only ever grows */
        const double cn = s.meta[slot].x != 0u ? acc_ptr(s, slot)->w : 0.0;
        V[p++] = cn > 0.0 ? cn : 0.0;
    }
}

__global__ void k_cn_seq(DevStore s, const unsigned long long *guard, const uint32_t *pos,
                         const uint32_t *cnt, const double *V) {
    if ((guard && *guard) || !s.ctr[C_CN_INEXACT]) return;
    const uint64_t nw = ((uint64_t)s.mask + 32) / 32;
    const uint64_t n = (uint64_t)pos[nw - 1] + cnt[nw - 1];
    double sum = 0.0, nx[16];
    uint64_t i = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) nx[k] = (uint64_t)k < n ? V[k] : 0.0;
    for (; i + 16 <= n; i += 16) {
        double cur[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) cur[k] = nx[k];
#pragma unroll
        for (int k = 0; k < 16; ++k) nx[k] = i + 16 + k < n ? V[i + 16 + k] : 0.0;
#pragma unroll
        for (int k = 0; k < 16; ++k) sum += cur[k];
    }
    for (int k = 0; i < n; ++i, ++k) sum += nx[k];
    *s.cn_sum = sum;
}

/* the blend of one slot with c_new > 0 (field.cpp:218-241): candidate, alpha with the 1/T floor,
 * mix, cOld capped at (T^2 - T) * mean c_new; mean: the frame's Σc_new / count, read from the
 * store's reduce-pass scratch unless given (use_mean); with use_mean false and mean 0 the cap is
 * skipped (callers that know it cannot apply) */
__device__ __forceinline__ double4 blend_one(const DevStore &s, double4 a, double4 c,
                                            double mean = 0.0, bool use_mean = false,
                                            bool from_scratch = true) {
    const double cn = a.w;
    const double tMax = s.t_max;
    const bool limited = tMax > 0.0 && isfinite(tMax);
    double meanCNew = mean;
    if (!use_mean && from_scratch) {
        const unsigned long long cnt = s.ctr[C_CN_COUNT];
        meanCNew = cnt > 0 ? *s.cn_sum / (double)cnt : 0.0;
    }
    const double capc = limited ? (tMax * tMax - tMax) * meanCNew : 0.0;
    const double cx = a.x / cn, cy = a.y / cn, cz = a.z / cn;
    double alpha = s.blend == PSTF_BLEND_SQRT ? sqrt(cn / (c.w + cn)) : cn / (c.w + cn);
    if (limited) {
        const double fl = 1.0 / tMax;
        alpha = (alpha < fl) ? fl : alpha; /* std::max(alpha, 1/tMax) */
    }
    const double oma = 1.0 - alpha;
    c.x = c.x * oma + cx * alpha;
    c.y = c.y * oma + cy * alpha;
    c.z = c.z * oma + cz * alpha;
    c.w = c.w + cn;
    if (limited && (use_mean || from_scratch))
        c.w = (capc < c.w) ? capc : c.w; /* std::min(cOld, cap) */
    return c;
}

/* endFrame pass 2 (field.cpp:216-246) over every store's touched list at once (one flat index
 * space), two entries per thread per iteration with their acc/com loads in flight together */
__device__ __forceinline__ void ef_blend_body(const Stores4 &st, int nst) {
    uint64_t seg[4];
    uint64_t total = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        seg[j] = total;
        total += j < nst ? st.s[j].ctr[C_TOUCHED_N] : 0;
    }
    unsigned internal[4] = {0u, 0u, 0u, 0u};
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += 2 * stride) {
        const bool two = i + stride < total;
        int jj[2];
        uint32_t sl[2];
        double4 av[2], cv[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const uint64_t e = k == 0 || !two ? i : i + stride;
            jj[k] = min(SEG_OF(e, seg), nst - 1);
            sl[k] = st.s[jj[k]].tlist[e - PICK4(seg, jj[k])];
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            av[k] = ld4(acc_ptr(st.s[jj[k]], sl[k]));
            cv[k] = ld4(com_ptr(st.s[jj[k]], sl[k]));
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            if (k == 1 && !two) break;
            const DevStore &s = st.s[jj[k]];
            const uint32_t slot = sl[k];
            const double4 a = av[k];
            const double cn = a.w;
            if (cn > 0.0) {
                st4(com_ptr(s, slot), blend_one(s, a, cv[k]));
            } else if (!(a.x == 0.0 && a.y == 0.0 && a.z == 0.0)) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (q == jj[k]) ++internal[q];
            }
            if (cn != 0.0 || a.x != 0.0 || a.y != 0.0 || a.z != 0.0)
                st4(acc_ptr(s, slot), make_double4(0.0, 0.0, 0.0, 0.0));
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const unsigned t = __reduce_add_sync(0xffffffffu, internal[q]);
        if (lane_id() == 0 && t) atomicAdd(&st.s[q].ctr[C_INTERNAL], (unsigned long long)t);
    }
}
__device__ __forceinline__ void ef_evict_body(const Stores4 &st, int nst, int finish) {
    if (finish && blockIdx.x == 0 && threadIdx.x < nst) { /* roll the per-frame scratch */
        const DevStore &s = st.s[threadIdx.x];
        s.ctr[C_TOUCHED_LAST] = s.ctr[C_TOUCHED_N];
        s.ctr[C_TOUCHED_TOTAL] += s.ctr[C_TOUCHED_N];
        s.ctr[C_TOUCHED_N] = 0;
        s.ctr[C_CN_COUNT] = 0;
        s.ctr[C_F_CN] = 0;
        s.ctr[C_F_DEFER] = 0;
        s.ctr[C_CN_INEXACT] = 0;
        s.ctr[C_REDS_MARK] = s.ctr[C_REDS];
        *s.cn_sum = 0.0;
    }
    for (int j = 0; j < nst; ++j) {
        const DevStore &s = st.s[j];
        const uint64_t cap = (uint64_t)s.mask + 1;
        if (!(s.ctr[C_LIVE_SNAP] * 4ull > (unsigned long long)cap * 3ull)) continue;
        unsigned ev = 0;
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap;
             i += (uint64_t)gridDim.x * blockDim.x) {
            const uint2 m = s.meta[i];
            if (m.x != 0 && (uint32_t)(s.frame - (m.y - 1u)) >= s.evict_age) {
                s.meta[i].x = 0;
                atomicAnd(&s.lbits[i >> 5], ~(1u << (i & 31u)));
                *com_ptr(s, i) = make_double4(0.0, 0.0, 0.0, 0.0);
                ++ev;
            }
        }
        ev = __reduce_add_sync(0xffffffffu, ev);
        if (lane_id() == 0 && ev) {
            atomicAdd(&s.ctr[C_EVICTED], (unsigned long long)ev);
            atomicAdd(&s.ctr[C_LIVE], (unsigned long long)(-(long long)ev));
        }
    }
}

/* endFrame (field.cpp:197-263) in one pass over the touched slots, for a frame whose updates
 * all carried unit counter weights (tiled ATOMIC vertex passes and their placement).  Only the
 * cOld cap min(cOld + c_new, (T^2 - T) * mean c_new) needs the frame's mean c_new; Σc_new was
 * counted while updating (C_F_CN: whole numbers, exact in any order) and at most `live` slots are
 * touched, so mean c_new = Σc_new / touched >= Σc_new / live.  A touched slot whose cOld + c_new stays within
 * (T^2 - T) * Σc_new / live is therefore never capped: it is blended as soon as the walk over
 * the touched bitmap finds it (acc and com gathered together; no touched list, no grid
 * barrier).  The few that may be capped go to a short list that k_ef_tail blends with the
 * exact mean once every touched slot has been counted.  The alpha / mix arithmetic is the
 * reference's (blend_one), so the result is bitwise the two-pass endFrame's. */
__global__ void __launch_bounds__(EF_BLOCK) k_ef_onepass(Stores4 st, int nst,
                                                         const unsigned long long *guard) {
    if (guard && *guard) return; /* new keys still pending: the host places them first */
    __shared__ uint32_t wlist[EF_BLOCK / 32][1024]; /* a warp's touched slots of 32 words */
    uint64_t seg[4], nw[4];
    uint64_t acc_w = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        nw[j] = j < nst ? ((uint64_t)st.s[j].mask + 32) / 32 : 0;
        seg[j] = acc_w;
        acc_w += (nw[j] + 31) & ~31ull; /* whole 32-word chunks per store */
    }
    const uint64_t total = acc_w;
    if (blockIdx.x == 0 && threadIdx.x < (unsigned)nst) {
        const DevStore &s = st.s[threadIdx.x];
        s.ctr[C_LIVE_SNAP] = s.ctr[C_LIVE];
        s.ctr[C_EVICTED] = 0;
    }
    const unsigned lane = lane_id();
    uint32_t *list = wlist[threadIdx.x >> 5];
    unsigned internal[4] = {0u, 0u, 0u, 0u}, tch[4] = {0u, 0u, 0u, 0u};
    const uint64_t nchunks = total / 32;
    const uint64_t wstride = (uint64_t)gridDim.x * (EF_BLOCK / 32);
    /* one warp per chunk of 32 bitmap words: the chunk's touched slots are compacted into
     * shared memory, then blended 32 at a time (every lane gathers one slot's acc and com:
     * full memory-level parallelism whatever the bits per word) */
    for (uint64_t ch = blockIdx.x * (uint64_t)(EF_BLOCK / 32) + (threadIdx.x >> 5); ch < nchunks;
         ch += wstride) {
        const uint64_t gi = ch * 32 + lane;
        const int j = min(SEG_OF(ch * 32, seg), nst - 1); /* warp-uniform */
        const DevStore &s = st.s[j];
        const uint64_t wi = gi - PICK4(seg, j);
        uint32_t w = wi < PICK4(nw, j) ? s.tbits[wi] : 0u;
        if (w) s.tbits[wi] = 0u;
        const unsigned c = __popc(w);
        unsigned incl = c;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)lane >= o) incl += t;
        }
        const unsigned T = __shfl_sync(0xffffffffu, incl, 31);
        if (!T) continue;
        unsigned pos = incl - c;
        while (w) {
            list[pos++] = (uint32_t)(wi * 32 + (uint64_t)(__ffs(w) - 1));
            w &= w - 1;
        }
        __syncwarp();
        /* no slot with cOld + c_new <= capLo is capped (mean c_new >= Σc_new / live) */
        const double tMax = s.t_max;
        const bool limited = tMax > 0.0 && isfinite(tMax);
        const unsigned long long live = s.ctr[C_LIVE];
        const double capLo = limited && live ? (tMax * tMax - tMax) *
                                                   ((double)s.ctr[C_F_CN] / (double)live)
                                             : HUGE_VAL;
        for (unsigned i = lane; i < T; i += 32) {
            const uint32_t slot = list[i];
            const double4 a = ld4(acc_ptr(s, slot));
            const double4 cv = ld4(com_ptr(s, slot));
            if (a.w > 0.0) {
                if (limited && !(cv.w + a.w <= capLo)) { /* may be capped: k_ef_tail */
                    s.tlist[atomicAdd(&s.ctr[C_F_DEFER], 1ull)] = slot;
                    continue;
                }
                st4(com_ptr(s, slot), blend_one(s, a, cv, 0.0, false, false)); /* uncapped */
            } else if (!(a.x == 0.0 && a.y == 0.0 && a.z == 0.0)) {
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    if (r == j) ++internal[r];
            }
            if (a.w != 0.0 || a.x != 0.0 || a.y != 0.0 || a.z != 0.0)
                st4(acc_ptr(s, slot), make_double4(0.0, 0.0, 0.0, 0.0));
        }
        __syncwarp();
        if (lane == 0) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if (r == j) tch[r] += T;
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const unsigned t = __reduce_add_sync(0xffffffffu, internal[q]);
        const unsigned tc = __reduce_add_sync(0xffffffffu, tch[q]);
        if (lane == 0 && t) atomicAdd(&st.s[q].ctr[C_INTERNAL], (unsigned long long)t);
        if (lane == 0 && tc) atomicAdd(&st.s[q].ctr[C_TOUCHED_N], (unsigned long long)tc);
    }
}

/* the rest of a one-pass endFrame: the deferred slots blended with the exact mean c_new
 * (Σc_new / touched slots, field.cpp:205-216), the age eviction when crowded, and the roll of
 * the per-frame counters by the last block to finish */
__device__ __forceinline__ void ef_tail_body(const Stores4 &st, int nst) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    for (int j = 0; j < nst; ++j) {
        const DevStore &s = st.s[j];
        const uint64_t nd = s.ctr[C_F_DEFER];
        if (!nd) continue;
        const unsigned long long cnt = s.ctr[C_TOUCHED_N];
        const double mean = cnt > 0 ? (double)s.ctr[C_F_CN] / (double)cnt : 0.0;
        for (uint64_t i = t0; i < nd; i += stride) {
            const uint32_t slot = s.tlist[i];
            const double4 a = ld4(acc_ptr(s, slot));
            st4(com_ptr(s, slot), blend_one(s, a, ld4(com_ptr(s, slot)), mean, true));
            st4(acc_ptr(s, slot), make_double4(0.0, 0.0, 0.0, 0.0));
        }
    }
    ef_evict_body(st, nst, 0);
}

/* roll the per-frame counters of a store (nobody reads them any more this frame) */
__device__ __forceinline__ void ef_roll(const DevStore &s) {
    s.ctr[C_TOUCHED_LAST] = s.ctr[C_TOUCHED_N];
    s.ctr[C_TOUCHED_TOTAL] += s.ctr[C_TOUCHED_N];
    s.ctr[C_TOUCHED_N] = 0;
    s.ctr[C_CN_COUNT] = 0;
    s.ctr[C_F_CN] = 0;
    s.ctr[C_F_DEFER] = 0;
    s.ctr[C_CN_INEXACT] = 0;
    s.ctr[C_REDS_MARK] = s.ctr[C_REDS];
    *s.cn_sum = 0.0;
}

__global__ void __launch_bounds__(EF_BLOCK) k_ef_tail(Stores4 st, int nst,
                                                      const unsigned long long *guard,
                                                      unsigned int *done, int rd_lo,
                                                      unsigned long long *rd_out) {
    if (guard && *guard) return;
    ef_tail_body(st, nst);
    /* last block: roll the per-frame counters */
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && rd_out && threadIdx.x == 0) {
        /* hot-slot measure of the tiled vertex pass whose Lo store is rd_lo: its RED element
         * updates so far and the frame's touched slots, straight into mapped host memory */
        unsigned long long t = 0;
        for (int i = 0; i < nst; ++i) t += st.s[i].ctr[C_TOUCHED_N];
        volatile unsigned long long *o = rd_out;
        o[0] = st.s[rd_lo].ctr[C_REDS] - st.s[rd_lo].ctr[C_REDS_MARK]; /* this frame's */
        o[1] = t;
        __threadfence_system();
    }
    __syncthreads();
    if (last && threadIdx.x < (unsigned)nst) {
        ef_roll(st.s[threadIdx.x]);
        if (threadIdx.x == 0) *done = 0u;
    }
}

/* ---------------- multi-GPU: replicated stores, all-reduced accumulators ----
 * Every rank holds a bitwise-identical replica of each store.  After phase 1 on its own
 * vertices and the identical placement of every rank's new keys, the ranks all-reduce the
 * accumulators of the live slots — packed in slot order, so entry i is the same slot on every
 * rank — and every rank then runs the ordinary endFrame on identical inputs. */

struct WSeg { /* word offsets of the stores in one flat word space; o[nst] = total */
    uint32_t o[5];
};

/* live-slot counts of the 32-slot words of the stores' flat word space (store j's words at
 * [wseg.o[j], wseg.o[j+1])), from the live bitmaps; cnt has one extra trailing word so the
 * exclusive scan also yields the total */
__global__ void k_live_count(Stores4 st, int nst, WSeg wseg, uint32_t *cnt) {
    const uint64_t total = wseg.o[nst];
    const uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (w > total) return;
    if (w == total) {
        cnt[w] = 0;
        return;
    }
    int j = 0;
    while (j + 1 < nst && w >= wseg.o[j + 1]) ++j;
    cnt[w] = (uint32_t)__popc(st.s[j].lbits[w - wseg.o[j]]);
}

/* entry scan[w] + k of the packed list = the k-th live slot of word w: its (store, slot) and
 * its accumulators (a word per thread, its set bits in slot order); entries
 * [live_total, bound) are zero */
__global__ void k_live_pack(Stores4 st, int nst, WSeg wseg, const uint32_t *scan,
                            uint64_t bound, unsigned long long *list, double4 *packed,
                            long long *live_total, unsigned long long *overflow) {
    const uint64_t total = wseg.o[nst];
    const uint64_t n = scan[total];
    const uint64_t t0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    if (t0 == 0) {
        *live_total = (long long)n;
        if (n > bound) atomicAdd(overflow, 1ull);
    }
    for (uint64_t w = t0; w < total; w += stride) {
        int j = 0;
        while (j + 1 < nst && w >= wseg.o[j + 1]) ++j;
        const DevStore &s = st.s[j];
        const uint64_t wl = w - wseg.o[j];
        uint32_t bits = s.lbits[wl];
        uint64_t pos = scan[w];
        while (bits && pos < bound) {
            const uint32_t slot = (uint32_t)(wl * 32 + (uint64_t)(__ffs(bits) - 1));
            bits &= bits - 1;
            list[pos] = ((unsigned long long)j << 32) | slot;
            st4(&packed[pos], ld4(acc_ptr(s, slot)));
            ++pos;
        }
    }
    for (uint64_t i = n + t0; i < bound; i += stride) packed[i] = make_double4(0.0, 0.0, 0.0, 0.0);
}

/* the all-reduced accumulators back into every replica; a slot touched on any rank (a nonzero
 * sum: every update call of a vertex pass carries weight 1 in c_new) gets lastTouched = frame
 * and its touched bit, exactly as a local touch would have set them */
__global__ void k_live_unpack(Stores4 st, const unsigned long long *list, const double4 *packed,
                              const long long *live_total, uint64_t bound) {
    const uint64_t n = min((uint64_t)*live_total, bound);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long e = list[i];
        const DevStore &s = st.s[(e >> 32) & 3];
        const uint32_t slot = (uint32_t)e;
        const double4 v = packed[i];
        *acc_ptr(s, slot) = v;
        if (v.x != 0.0 || v.y != 0.0 || v.z != 0.0 || v.w != 0.0) touch_slot(s, slot);
    }
}

/* endFrame (field.cpp:197-263) of a multi-GPU frame straight from the all-reduced packed
 * accumulators (one cooperative launch, no unpack into acc): pass 1 sums c_new per store over
 * the packed entries; pass 2 blends the touched entries (a nonzero sum: every update call of a
 * vertex pass carries weight 1 in c_new), marks them touched this frame and zeroes the
 * replica's own partial accumulators; pass 3 is the usual age eviction (identical on every
 * replica: same live counts, same ages). */
__global__ void __launch_bounds__(EF_BLOCK) k_ef_packed(Stores4 st, int nst,
                                                        const unsigned long long *list,
                                                        const double4 *packed,
                                                        const long long *live_total,
                                                        uint64_t bound) {
    cg::grid_group g = cg::this_grid();
    __shared__ double ssum[4][EF_BLOCK / 32];
    __shared__ unsigned long long scnt[4][EF_BLOCK / 32], stch[4][EF_BLOCK / 32];
    const uint64_t n = min((uint64_t)*live_total, bound);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (blockIdx.x == 0 && threadIdx.x < (unsigned)nst) {
        const DevStore &s = st.s[threadIdx.x];
        s.ctr[C_LIVE_SNAP] = s.ctr[C_LIVE];
        s.ctr[C_EVICTED] = 0;
    }
    double sum[4] = {0.0, 0.0, 0.0, 0.0};
    unsigned cnt[4] = {0u, 0u, 0u, 0u}, tch[4] = {0u, 0u, 0u, 0u};
    for (uint64_t i = t0; i < n; i += stride) {
        const int j = (int)((list[i] >> 32) & 3);
        const double4 v = packed[i];
        const bool touched = v.x != 0.0 || v.y != 0.0 || v.z != 0.0 || v.w != 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q == j) {
                if (v.w > 0.0) {
                    sum[q] += v.w;
                    ++cnt[q];
                }
                tch[q] += touched;
            }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const double t = warp_sum_d(sum[q]);
        const unsigned cc = __reduce_add_sync(0xffffffffu, cnt[q]);
        const unsigned tt = __reduce_add_sync(0xffffffffu, tch[q]);
        if (lane_id() == 0) {
            ssum[q][threadIdx.x >> 5] = t;
            scnt[q][threadIdx.x >> 5] = cc;
            stch[q][threadIdx.x >> 5] = tt;
        }
    }
    __syncthreads();
    if (threadIdx.x < (unsigned)nst) {
        const int q = threadIdx.x;
        double t = 0.0;
        unsigned long long c = 0, tc = 0;
        for (int w = 0; w < EF_BLOCK / 32; ++w) {
            t += ssum[q][w];
            c += scnt[q][w];
            tc += stch[q][w];
        }
        if (c) {
            /* an inexact frame's sum is already there, summed in slot order (k_cn_seq) */
            if (!st.s[q].ctr[C_CN_INEXACT]) atomicAdd(st.s[q].cn_sum, t);
            atomicAdd(&st.s[q].ctr[C_CN_COUNT], c);
        }
        if (tc) atomicAdd(&st.s[q].ctr[C_TOUCHED_N], tc);
    }
    g.sync();
    unsigned internal[4] = {0u, 0u, 0u, 0u};
    for (uint64_t i = t0; i < n; i += stride) {
        const unsigned long long e = list[i];
        const int j = (int)((e >> 32) & 3);
        const DevStore &s = st.s[j];
        const uint32_t slot = (uint32_t)e;
        const double4 v = packed[i];
        if (!(v.x != 0.0 || v.y != 0.0 || v.z != 0.0 || v.w != 0.0)) continue;
        if (v.w > 0.0) {
            st4(com_ptr(s, slot), blend_one(s, v, ld4(com_ptr(s, slot))));
        } else if (!(v.x == 0.0 && v.y == 0.0 && v.z == 0.0)) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (q == j) ++internal[q];
        }
        s.meta[slot].y = s.frame + 1u; /* lastTouched = frame (field.cpp:123,133,137) */
        st4(acc_ptr(s, slot), make_double4(0.0, 0.0, 0.0, 0.0));
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const unsigned t = __reduce_add_sync(0xffffffffu, internal[q]);
        if (lane_id() == 0 && t) atomicAdd(&st.s[q].ctr[C_INTERNAL], (unsigned long long)t);
    }
    g.sync();
    ef_evict_body(st, nst, 1);
}

/* the vector the one host synchronisation of a multi-GPU frame reads: {pending records of this
 * rank, live slots over the stores (after the last endFrame), pack overflows} */
__global__ void k_shard_info(Stores4 st, int nst, const unsigned long long *pend_count,
                             uint64_t pend_cap, const unsigned long long *overflow,
                             long long *out) {
    if (threadIdx.x != 0) return;
    const unsigned long long pc = pend_count ? *pend_count : 0ull;
    out[0] = (long long)(pc < pend_cap ? pc : pend_cap);
    long long live = 0;
    for (int j = 0; j < nst; ++j) live += (long long)st.s[j].ctr[C_LIVE];
    out[1] = live;
    out[2] = (long long)(overflow ? *overflow : 0ull);
}

/* ------------------------------------------------------------------------------------------ */
/* invalidate / weighted mean / snapshot / slots                                               */

__global__ void k_invalidate(DevStore s, int use_box, double lx, double ly, double lz, double hx,
                             double hy, double hz) {
    uint64_t cap = (uint64_t)s.mask + 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (s.meta[i].x == 0) continue;
        if (use_box) {
            KeyFields k = s.keyf[i];
            double cs = cell_size(s.kp, k.level); /* field.cpp:278-283 */
            double cx = ((double)k.c0 + 0.5) * cs, cy = ((double)k.c1 + 0.5) * cs,
                   cz = ((double)k.c2 + 0.5) * cs;
            if (!(cx >= lx && cx <= hx && cy >= ly && cy <= hy && cz >= lz && cz <= hz)) continue;
        }
        com_ptr(s, i)->w = 0.0;
    }
}

__global__ void k_weighted_mean(DevStore s, double *out4) {
    uint64_t cap = (uint64_t)s.mask + 1;
    double r = 0, g = 0, b = 0, w = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (s.meta[i].x == 0) continue;
        double4 c = *com_ptr(s, i);
        if (c.w <= 0.0) continue; /* field.cpp:299 */
        r += c.x * c.w;
        g += c.y * c.w;
        b += c.z * c.w;
        w += c.w;
    }
    r = warp_sum_d(r);
    g = warp_sum_d(g);
    b = warp_sum_d(b);
    w = warp_sum_d(w);
    if (lane_id() == 0 && w != 0.0) {
        atomicAdd(&out4[0], r);
        atomicAdd(&out4[1], g);
        atomicAdd(&out4[2], b);
        atomicAdd(&out4[3], w);
    }
}

__global__ void k_snap_gather(DevStore s, pstf_snapshot_record *out, unsigned long long *count) {
    uint64_t cap = (uint64_t)s.mask + 1;
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    bool live = i < cap && s.meta[i].x != 0;
    unsigned m = __ballot_sync(0xffffffffu, live);
    if (!m) return;
    unsigned long long base = 0;
    int leader = __ffs(m) - 1;
    if ((int)lane_id() == leader) base = atomicAdd(count, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (!live) return;
    /* slot order is kept by sorting on (key, slot) afterwards */
    unsigned long long pos = base + __popc(m & ((1u << lane_id()) - 1u));
    KeyFields k = s.keyf[i];
    double4 c = *com_ptr(s, i);
    pstf_snapshot_record r;
    r.level = k.level;
    r.cell[0] = k.c0;
    r.cell[1] = k.c1;
    r.cell[2] = k.c2;
    r.dir_cell[0] = k.d0;
    r.dir_cell[1] = k.d1;
    r.checksum = s.meta[i].x;
    r.value[0] = c.x;
    r.value[1] = c.y;
    r.value[2] = c.z;
    r.c_old = c.w;
    out[pos] = r;
}

/* snapshot sort words: 3 x u64 = (level,c0) (c1,c2) (d0,d1), signed -> biased */
__global__ void k_snap_words(const pstf_snapshot_record *r, uint64_t n, uint64_t *words) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    auto b = [](int32_t v) { return (uint64_t)((uint32_t)v ^ 0x80000000u); };
    pstf_snapshot_record x = r[i];
    words[i] = (b(x.level) << 32) | b(x.cell[0]);
    words[n + i] = (b(x.cell[1]) << 32) | b(x.cell[2]);
    words[2 * n + i] = (b(x.dir_cell[0]) << 32) | b(x.dir_cell[1]);
}

__global__ void k_snap_permute(const pstf_snapshot_record *src, const uint32_t *perm, uint64_t n,
                               pstf_snapshot_record *dst) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[perm[i]];
}

/* ------------------------------------------------------------------------------------------ */
/* synthetic stream                                                                            */

__global__ void k_synth(ps_params P, double *buf, uint64_t n_total) {
    uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t n_paths = P.n_local ? P.n_local : (uint64_t)P.width * (uint64_t)P.height;
    if (p >= n_paths) return;
    ps_gen_path(&P, p + P.path0, buf, (uint32_t *)(buf + 34 * n_total), n_total);
}

/* ========================================================================================== */
/* host orchestration                                                                          */

static int sort_multiword(Scratch &sc, const uint64_t *words, const int *begin_bits, int nw,
                          uint64_t n, uint32_t **perm_out, cudaStream_t st) {
    ENSURE(sc.perm0, n * 4);
    ENSURE(sc.perm1, n * 4);
    ENSURE(sc.ktmp0, n * 8);
    ENSURE(sc.ktmp1, n * 8);
    uint32_t *pa = sc.perm0.as<uint32_t>(), *pb = sc.perm1.as<uint32_t>();
    LAUNCH(k_iota, grid_for(n, 256), 256, 0, st, pa, n);
    for (int k = nw - 1; k >= 0; --k) {
        const uint64_t *src = words + (uint64_t)k * n;
        uint64_t *kin = sc.ktmp0.as<uint64_t>();
        if (k == nw - 1) {
            CK(cudaMemcpyAsync(kin, src, n * 8, cudaMemcpyDeviceToDevice, st));
        } else {
            LAUNCH(k_gather_u64, grid_for(n, 256), 256, 0, st, src, pa, n, kin);
        }
        size_t bytes = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, sc.ktmp1.as<uint64_t>(), pa, pb,
                                           (int64_t)n, begin_bits[k], 64, st));
        ENSURE(sc.cub, bytes);
        bytes = sc.cub.bytes;
        { ProfScope ps_("cub::DeviceRadixSort", st);
        CK(cub::DeviceRadixSort::SortPairs(sc.cub.p, bytes, kin, sc.ktmp1.as<uint64_t>(), pa, pb,
                                           (int64_t)n, begin_bits[k], 64, st));
        g_launches.fetch_add(4, std::memory_order_relaxed); }
        std::swap(pa, pb);
    }
    *perm_out = pa;
    return PSTF_OK;
}

static int bits_for(unsigned long long range) {
    return range == 0 ? 0 : 64 - __builtin_clzll(range);
}

static void add_field(Layout &L, int fid, int bits, long long minv, int &word, int &free_bits) {
    if (bits <= 0) return;
    if (bits > free_bits) {
        L.begin_bit[word] = free_bits;
        ++word;
        free_bits = 64;
    }
    int q = L.nfields++;
    L.fid[q] = fid;
    L.bits[q] = bits;
    L.word[q] = word;
    L.shift[q] = free_bits - bits;
    L.minv[q] = minv;
    free_bits -= bits;
}

static Stores4 stores4(pstf_field *const *fs, int nf) {
    Stores4 s;
    memset(&s, 0, sizeof(s));
    for (int i = 0; i < nf && i < 4; ++i)
        if (fs[i]) s.s[i] = dev_view(fs[i]);
    return s;
}

/* cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link) */
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

/* the dynamic shared-memory limit is an attribute of a kernel on one device: set once per
 * (kernel, device) pair */
static int smem_attr(const void *fn, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({fn, dev})) return PSTF_OK;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.insert({fn, dev});
    return PSTF_OK;
}
#define SMEM_ATTR(fn, bytes)                                                                       \
    do {                                                                                           \
        int rc_ = smem_attr((const void *)(fn), (int)(bytes));                                   \
        if (rc_) return rc_;                                                                       \
    } while (0)

static int read_small(Scratch &sc, const void *dev, size_t bytes, cudaStream_t st) {
    if (!sc.h_small) CK(cudaMallocHost(&sc.h_small, 4096));
    CK(cudaMemcpyAsync(sc.h_small, dev, bytes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return PSTF_OK;
}

/* Sort-free phase 2 for ATOMIC mode (one 64-bit key word per record): a dedup hash table
 * groups the records by key, the unique keys take ids in any order, and the placement compares
 * the order-preserving key words themselves (64-bit holds), which is the ascending-key priority
 * the sorted path derives from its ranks.  No sort, no host round trip for the unique count. */
static int phase2_atomic_fast(Scratch &sc, pstf_field *const *fs, int nf, uint64_t n,
                              const PendRec *pend, int own_origin, cudaStream_t st) {
    uint64_t T = 64;
    while (T < 2 * n) T <<= 1;
    ENSURE(sc.ddtab, T * 4);
    ENSURE(sc.rep_of, n * 4);
    ENSURE(sc.uidx, n * 4);
    ENSURE(sc.ukw, n * 8);
    ENSURE(sc.nudev, 16);
    ENSURE(sc.ufirst, n * 4);
    ENSURE(sc.ukey, n * sizeof(KeyFields));
    ENSURE(sc.ucs, n * 4);
    ENSURE(sc.usid, n * 4);
    ENSURE(sc.uhome, n * 4);
    ENSURE(sc.ucalls, n * 4);
    ENSURE(sc.usum, n * sizeof(double4));
    ENSURE(sc.ures0, n * 8);
    ENSURE(sc.ures1, n * 8);
    ENSURE(sc.changed, 16);
    for (int i = 0; i < nf; ++i) { /* 64-bit holds, all "none" between passes */
        pstf_field *f = fs[i];
        if (!f || f->d.hold64_0) continue;
        const uint64_t cap = (uint64_t)f->d.mask + 1;
        CK(f->hold64.ensure(2 * cap * 8));
        CK(cudaMemsetAsync(f->hold64.p, 0xff, 2 * cap * 8, st));
        f->d.hold64_0 = f->hold64.as<unsigned long long>();
        f->d.hold64_1 = f->hold64.as<unsigned long long>() + cap;
    }
    Stores4 S = stores4(fs, nf);
    CK(cudaMemsetAsync(sc.ddtab.p, 0xff, T * 4, st));
    CK(cudaMemsetAsync(sc.nudev.p, 0, 16, st));
    UniqArgs U;
    U.ufirst = sc.ufirst.as<uint32_t>();
    U.ukey = sc.ukey.as<KeyFields>();
    U.ucs = sc.ucs.as<uint32_t>();
    U.usid = sc.usid.as<uint32_t>();
    U.uhome = sc.uhome.as<uint32_t>();
    U.ucalls = sc.ucalls.as<uint32_t>();
    U.usum = sc.usum.as<double4>();
    U.useq = nullptr;
    const uint64_t *words = sc.words.as<uint64_t>();
    LAUNCH(k_dd_insert, grid_for(n, 256), 256, 0, st, words, n, sc.ddtab.as<uint32_t>(),
           (uint32_t)(T - 1), sc.rep_of.as<uint32_t>());
    LAUNCH(k_dd_unique, grid_for(n, 256), 256, 0, st, pend, words,
           (const uint32_t *)sc.rep_of.as<uint32_t>(), n, S, U, sc.ukw.as<uint64_t>(),
           sc.uidx.as<uint32_t>(), sc.nudev.as<unsigned>());
    LAUNCH(k_dd_sums, grid_for(n, 256), 256, 0, st, pend, (const uint32_t *)sc.rep_of.as<uint32_t>(),
           (const uint32_t *)sc.uidx.as<uint32_t>(), n, U, own_origin);
    PlaceArgs P;
    memset(&P, 0, sizeof(P));
    P.st = S;
    P.nu = n; /* upper bound; the kernels read the count from nu_dev */
    P.usid = U.usid;
    P.uhome = U.uhome;
    P.ucs = U.ucs;
    P.parity = 0;
    P.nu_dev = sc.nudev.as<unsigned>();
    Dedup dd{words, sc.ddtab.as<uint32_t>(), (uint32_t)(T - 1), pend};
    unsigned long long *r0 = sc.ures0.as<unsigned long long>(), *r1 = sc.ures1.as<unsigned long long>();
    CK(cudaMemsetAsync(r0, 0, n * 8, st));
    CK(cudaMemsetAsync(sc.changed.p, 0, 16, st));
    {
        static int blocks_per_sm = -1;
        if (blocks_per_sm < 0) {
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_place_loop64, 256, 0));
            blocks_per_sm = std::max(1, std::min(blocks_per_sm, 4));
        }
        const unsigned grid = (unsigned)std::min<uint64_t>(grid_for(n, 256),
                                                           (uint64_t)sm_count() * blocks_per_sm);
        const uint64_t *ukw = sc.ukw.as<uint64_t>();
        int *ctl = sc.changed.as<int>();
        uint32_t max_rounds = (uint32_t)std::min<uint64_t>(n + 2, 0x7fffffffu);
        void *args[] = {&P, &ukw, &dd, &r0, &r1, &ctl, &max_rounds};
        ProfScope ps_("k_place_loop64", st);
        CK(cudaLaunchCooperativeKernel((const void *)k_place_loop64, grid, 256, args, 0, st));
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    LAUNCH(k_commit, grid_for(n, 256), 256, 0, st, P, r0, U.ukey, U.ucalls, U.usum, 1);
    return PSTF_OK;
}

/* Phase 2 for the records sitting in sc.pend (count on device in sc.pend_count).
 * fs[0..nf) are the stores addressed by record store ids. */
static int resolve_pending(Scratch &sc, pstf_field *const *fs, int nf, int mode, uint64_t n_known,
                           cudaStream_t st, int own_origin = -1) {
    uint64_t n = n_known;
    if (n == (uint64_t)-1) {
        int rc = read_small(sc, sc.pend_count.p, 8, st);
        if (rc) return rc;
        n = sc.h_small[0];
    }
    for (int i = 0; i < nf; ++i)
        if (fs[i]) {
            CK(cudaMemsetAsync(&fs[i]->d.ctr[C_NEW_KEYS], 0, 8, st));
            CK(cudaMemsetAsync(&fs[i]->d.ctr[C_ROUNDS], 0, 8, st));
        }
    if (n == 0) return PSTF_OK;
    if (n > sc.pend.bytes / sizeof(PendRec))
        return set_err(PSTF_E_NOMEM, "pending-update buffer overflow");
    if (n >= 0xffffffffULL) return set_err(PSTF_E_INVALID, "too many pending updates");
    const PendRec *pend = sc.pend.as<PendRec>();
    const uint64_t *seq = mode == PSTF_MODE_SEQUENTIAL ? sc.pend_seq.as<uint64_t>() : nullptr;
    Stores4 S = stores4(fs, nf);

    /* 1. key-field ranges -> compact sort layout */
    ENSURE(sc.ranges, 2 * NF_KEY * 4);
    {
        int init[2 * NF_KEY];
        for (int f = 0; f < NF_KEY; ++f) {
            init[2 * f] = INT32_MAX;
            init[2 * f + 1] = INT32_MIN;
        }
        if (!sc.h_small) CK(cudaMallocHost(&sc.h_small, 4096));
        memcpy(sc.h_small, init, sizeof(init));
        CK(cudaMemcpyAsync(sc.ranges.p, sc.h_small, sizeof(init), cudaMemcpyHostToDevice, st));
        unsigned g = std::min<uint64_t>(grid_for(n, 256), (uint64_t)sm_count() * 8);
        LAUNCH(k_ranges, g, 256, 0, st, pend, sc.pend_count.as<unsigned long long>(), n,
               sc.ranges.as<int>());
    }
    int rng[2 * NF_KEY];
    {
        int rc = read_small(sc, sc.ranges.p, sizeof(rng), st);
        if (rc) return rc;
        memcpy(rng, sc.h_small, sizeof(rng));
    }
    Layout L;
    memset(&L, 0, sizeof(L));
    int word = 0, free_bits = 64;
    for (int f = 0; f < NF_KEY; ++f) {
        long long mn = rng[2 * f], mx = rng[2 * f + 1];
        add_field(L, f, bits_for((unsigned long long)(mx - mn)), mn, word, free_bits);
    }
    if (mode == PSTF_MODE_ORDERED) { /* field.cpp:407-410 tie-break: (isCounter, r, g, b, w) */
        add_field(L, F_ISC, 1, 0, word, free_bits);
        for (int c = 0; c < 4; ++c) add_field(L, F_R + c, 64, 0, word, free_bits);
    } else if (mode == PSTF_MODE_SEQUENTIAL) {
        add_field(L, F_SEQ, std::max(1, bits_for(n)), 0, word, free_bits);
    }
    if (L.nfields == 0) add_field(L, F_STORE, 1, 0, word, free_bits);
    L.begin_bit[word] = free_bits;
    L.nwords = word + 1;

    ENSURE(sc.words, (size_t)L.nwords * n * 8);
    LAUNCH(k_encode, grid_for(n, 256), 256, 0, st, pend, seq, n, L, sc.words.as<uint64_t>());
    static const bool no_fast = getenv("PSTF_NO_FAST_PHASE2") != nullptr;
    if (mode == PSTF_MODE_ATOMIC && L.nwords == 1 && !no_fast)
        return phase2_atomic_fast(sc, fs, nf, n, pend, own_origin, st);
    uint32_t *perm = nullptr;
    {
        int rc = sort_multiword(sc, sc.words.as<uint64_t>(), L.begin_bit, L.nwords, n, &perm, st);
        if (rc) return rc;
    }

    /* 2. unique keys (segments of equal (store, key)) */
    ENSURE(sc.head, n * 4);
    ENSURE(sc.uid, n * 4);
    LAUNCH(k_heads, grid_for(n, 256), 256, 0, st, pend, perm, n, sc.head.as<uint32_t>());
    {
        size_t bytes = 0;
        CK(cub::DeviceScan::InclusiveSum(nullptr, bytes, sc.head.as<uint32_t>(),
                                         sc.uid.as<uint32_t>(), (int64_t)n, st));
        ENSURE(sc.cub, bytes);
        bytes = sc.cub.bytes;
        { ProfScope ps_("cub::DeviceScan", st);
        CK(cub::DeviceScan::InclusiveSum(sc.cub.p, bytes, sc.head.as<uint32_t>(),
                                         sc.uid.as<uint32_t>(), (int64_t)n, st));
        g_launches.fetch_add(2, std::memory_order_relaxed); }
    }
    uint64_t nu;
    {
        int rc = read_small(sc, sc.uid.as<uint32_t>() + (n - 1), 4, st);
        if (rc) return rc;
        nu = ((uint32_t *)sc.h_small)[0];
    }
    if (getenv("PSTF_DEBUG_PHASE2")) fprintf(stderr, "phase2: %llu records, %llu unique keys\n",
                                            (unsigned long long)n, (unsigned long long)nu);
    ENSURE(sc.ufirst, nu * 4);
    ENSURE(sc.ukey, nu * sizeof(KeyFields));
    ENSURE(sc.ucs, nu * 4);
    ENSURE(sc.usid, nu * 4);
    ENSURE(sc.uhome, nu * 4);
    ENSURE(sc.ucalls, nu * 4);
    ENSURE(sc.usum, nu * sizeof(double4));
    ENSURE(sc.ures0, nu * 8);
    ENSURE(sc.ures1, nu * 8);
    ENSURE(sc.changed, 16);
    UniqArgs U;
    U.ufirst = sc.ufirst.as<uint32_t>();
    U.ukey = sc.ukey.as<KeyFields>();
    U.ucs = sc.ucs.as<uint32_t>();
    U.usid = sc.usid.as<uint32_t>();
    U.uhome = sc.uhome.as<uint32_t>();
    U.ucalls = sc.ucalls.as<uint32_t>();
    U.usum = sc.usum.as<double4>();
    U.useq = nullptr;
    if (mode == PSTF_MODE_SEQUENTIAL) {
        ENSURE(sc.useq, nu * 8);
        U.useq = sc.useq.as<uint64_t>();
    }
    CK(cudaMemsetAsync(U.ucalls, 0, nu * 4, st));
    CK(cudaMemsetAsync(U.usum, 0, nu * sizeof(double4), st));
    LAUNCH(k_unique_build, grid_for(n, 256), 256, 0, st, pend, perm, sc.head.as<uint32_t>(),
           sc.uid.as<uint32_t>(), seq, n, S, U);
    LAUNCH(k_unique_sums, grid_for(n, 256), 256, 0, st, pend, perm, sc.uid.as<uint32_t>(), n,
           mode == PSTF_MODE_ATOMIC ? 1 : 0, U, own_origin);

    /* 3. priority ranks */
    PlaceArgs P;
    memset(&P, 0, sizeof(P));
    P.st = S;
    P.nu = nu;
    P.usid = U.usid;
    P.uhome = U.uhome;
    P.ucs = U.ucs;
    P.rank = nullptr;
    P.cs_by_rank = U.ucs;
    if (mode == PSTF_MODE_SEQUENTIAL) { /* priority = first submission (scalar-call order) */
        ENSURE(sc.rank, nu * 4);
        ENSURE(sc.csr, nu * 4);
        uint32_t *ids_in = nullptr, *ids = nullptr;
        ENSURE(sc.fperm, nu * 4);
        ENSURE(sc.fperm_out, nu * 4);
        ENSURE(sc.fkey_out, nu * 8);
        ids_in = sc.fperm.as<uint32_t>();
        ids = sc.fperm_out.as<uint32_t>();
        LAUNCH(k_iota, grid_for(nu, 256), 256, 0, st, ids_in, nu);
        size_t bytes = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, U.useq, sc.fkey_out.as<uint64_t>(),
                                           ids_in, ids, (int64_t)nu, 0, 64, st));
        ENSURE(sc.cub, bytes);
        bytes = sc.cub.bytes;
        { ProfScope ps_("cub::DeviceRadixSort", st);
        CK(cub::DeviceRadixSort::SortPairs(sc.cub.p, bytes, U.useq, sc.fkey_out.as<uint64_t>(),
                                           ids_in, ids, (int64_t)nu, 0, 64, st));
        g_launches.fetch_add(4, std::memory_order_relaxed); }
        LAUNCH(k_rank_scatter, grid_for(nu, 256), 256, 0, st, ids, nu, sc.rank.as<uint32_t>(),
               U.ucs, sc.csr.as<uint32_t>());
        P.rank = sc.rank.as<uint32_t>();
        P.cs_by_rank = sc.csr.as<uint32_t>();
    }

    /* 4. deterministic placement: Jacobi rounds to the unique fixpoint, on the device */
    unsigned long long *rprev = sc.ures0.as<unsigned long long>();
    CK(cudaMemsetAsync(rprev, 0, nu * 8, st));
    CK(cudaMemsetAsync(sc.changed.p, 0, 16, st));
    P.parity = 0;
    {
        static int blocks_per_sm = -1;
        if (blocks_per_sm < 0) {
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_place_loop, 256, 0));
            blocks_per_sm = std::max(1, std::min(blocks_per_sm, 4));
        }
        const unsigned grid = (unsigned)std::min<uint64_t>(grid_for(nu, 256),
                                                           (uint64_t)sm_count() * blocks_per_sm);
        unsigned long long *r1 = sc.ures1.as<unsigned long long>();
        int *ctl = sc.changed.as<int>();
        uint32_t max_rounds = (uint32_t)std::min<uint64_t>(nu + 2, 0x7fffffffu);
        void *args[] = {&P, &rprev, &r1, &ctl, &max_rounds};
        ProfScope ps_("k_place_loop", st);
        CK(cudaLaunchCooperativeKernel((const void *)k_place_loop, grid, 256, args, 0, st));
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    P.parity = -1;
    LAUNCH(k_commit, grid_for(nu, 256), 256, 0, st, P, rprev, U.ukey, U.ucalls, U.usum,
           mode == PSTF_MODE_ATOMIC ? 1 : 0);

    /* 5. ORDERED / SEQUENTIAL: sequential fold per slot */
    if (mode != PSTF_MODE_ATOMIC) {
        ENSURE(sc.ftgt, n * 8);
        ENSURE(sc.fperm, n * 4);
        ENSURE(sc.fkey_out, n * 8);
        ENSURE(sc.fperm_out, n * 4);
        LAUNCH(k_fold_targets, grid_for(n, 256), 256, 0, st, perm, sc.uid.as<uint32_t>(), n, rprev,
               U.usid, mode == PSTF_MODE_SEQUENTIAL ? 1 : 0, sc.ftgt.as<uint64_t>(),
               sc.fperm.as<uint32_t>());
        size_t bytes = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, sc.ftgt.as<uint64_t>(),
                                           sc.fkey_out.as<uint64_t>(), sc.fperm.as<uint32_t>(),
                                           sc.fperm_out.as<uint32_t>(), (int64_t)n, 0, 64, st));
        ENSURE(sc.cub, bytes);
        bytes = sc.cub.bytes;
        { ProfScope ps_("cub::DeviceRadixSort", st);
        CK(cub::DeviceRadixSort::SortPairs(sc.cub.p, bytes, sc.ftgt.as<uint64_t>(),
                                           sc.fkey_out.as<uint64_t>(), sc.fperm.as<uint32_t>(),
                                           sc.fperm_out.as<uint32_t>(), (int64_t)n, 0, 64, st));
        g_launches.fetch_add(4, std::memory_order_relaxed); }
        ENSURE(sc.fterms, n * sizeof(double4));
        ENSURE(sc.fisc, n);
        LAUNCH(k_fold_terms, grid_for(n, 256), 256, 0, st, pend, sc.fperm_out.as<uint32_t>(), n,
               sc.fterms.as<double4>(), sc.fisc.as<uint8_t>());
        /* runs of equal targets: heads -> scan -> start positions (+ sentinel) */
        ENSURE(sc.head, n * 4);
        ENSURE(sc.uid, n * 4);
        ENSURE(sc.fstart, (n + 1) * 4);
        const uint64_t *ftgt = sc.fkey_out.as<uint64_t>();
        LAUNCH(k_fold_heads, grid_for(n, 256), 256, 0, st, ftgt, n, sc.head.as<uint32_t>());
        {
            size_t bytes = 0;
            CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, sc.head.as<uint32_t>(),
                                             sc.uid.as<uint32_t>(), (int64_t)n, st));
            ENSURE(sc.cub, bytes);
            bytes = sc.cub.bytes;
            ProfScope ps_("cub::DeviceScan", st);
            CK(cub::DeviceScan::ExclusiveSum(sc.cub.p, bytes, sc.head.as<uint32_t>(),
                                             sc.uid.as<uint32_t>(), (int64_t)n, st));
            g_launches.fetch_add(2, std::memory_order_relaxed);
        }
        LAUNCH(k_fold_starts, grid_for(n, 256), 256, 0, st, sc.head.as<uint32_t>(),
               sc.uid.as<uint32_t>(), n, sc.fstart.as<uint32_t>());
        ENSURE(sc.fnruns, 8);
        LAUNCH(k_fold_nruns, 1, 1, 0, st, sc.head.as<uint32_t>(), sc.uid.as<uint32_t>(), n,
               sc.fnruns.as<uint32_t>());
        LAUNCH(k_fold, grid_for(n, 256), 256, 0, st, sc.fterms.as<double4>(), sc.fisc.as<uint8_t>(),
               ftgt, sc.fstart.as<uint32_t>(), sc.fnruns.as<uint32_t>(), S);
        LAUNCH(k_fold_long, (unsigned)sm_count() * 8, 256, 0, st, sc.fterms.as<double4>(),
               sc.fisc.as<uint8_t>(), ftgt, sc.fstart.as<uint32_t>(), sc.fnruns.as<uint32_t>(), S);
    }
    return PSTF_OK;
}

__global__ void k_set_u64(unsigned long long *p, unsigned long long v) { *p = v; }

/* ---- ORDERED vertex passes: the value calls of keys that already own a slot ----
 * FieldUpdateQueue::apply (field.cpp:396-420) sorts every call by (key, isCounter, bits r, g, b,
 * w) and applies them in that order; a slot's accumulator therefore sums its value calls in the
 * order of their value bits (all of one key, weight 1.0).  These calls need no placement:
 *   1. one 64-bit sort key per record: store and slot in the top S bits, the leading 64 - S bits
 *      of bits(r) below (one CUB radix sort of (key, index));
 *   2. the components gathered in that order (three arrays r | g | b);
 *   3. the only calls that can be out of (r, g, b) order are inside runs of equal sort keys
 *      (equal leading bits of r: r values an ulp apart, or equal r with different g, b): each
 *      run holding an out-of-order neighbour pair is re-sorted in place, by one warp (rank sort
 *      through shuffles, <= 32 calls; bitonic in shared memory, <= 256) or one block (the same,
 *      <= 4096), or, longer, compacted with the other such runs and radix-sorted least
 *      significant word first (b, g, then run start with the low bits of r);
 *   4. the terms folded sequentially per slot (a warp per long slot: three lanes carry the r, g
 *      and b sums).
 * A record whose key is not its slot's (a checksum alias sharing the slot: the queue would order
 * the two keys' calls apart) or whose weight is not 1 sends all of them through the general
 * path, decided before anything is folded. */
__global__ void k_iota32(uint32_t *idx, uint64_t n) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) idx[i] = (uint32_t)i;
}

/* the general path's full record of a slot-grouped call (the slot's key: no alias reached
 * this list), exactly as the vertex pass writes a new key's value call */
__global__ void k_slot_expand(const uint64_t *__restrict__ key, const double4 *__restrict__ val,
                              uint64_t n, int capl, Stores4 st, PendRec *out,
                              unsigned long long *cnt) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const bool real = i < n && key[i] != ~0ull; /* holes: unused tails of the tiled kernel's chunks */
    const unsigned m = __ballot_sync(0xffffffffu, real);
    if (!m) return;
    unsigned long long base = 0;
    if (lane_id() == (unsigned)(__ffs(m) - 1)) base = atomicAdd(cnt, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (!real) return;
    const int S = capl + 2;
    const uint64_t sk = key[i] >> (64 - S);
    const uint32_t sid = (uint32_t)(sk >> capl), slot = (uint32_t)(sk & ((1ull << capl) - 1ull));
    const DevStore &s = st.s[sid];
    const KeyFields kf = s.keyf[slot];
    Key k;
    k.level = kf.level;
    k.cell[0] = kf.c0;
    k.cell[1] = kf.c1;
    k.cell[2] = kf.c2;
    k.dir[0] = kf.d0;
    k.dir[1] = kf.d1;
    k.checksum = s.meta[slot].x;
    const double4 v = val[i];
    put_record(out + base + __popc(m & ((1u << lane_id()) - 1u)), k, PSTF_META(sid, 0, 1), v.x,
               v.y, v.z, 1.0);
}

/* own position at each run head of the sorted keys (0 elsewhere: a max-scan gives every position
 * its run's start), and the heads of the slots' segments */
__global__ void k_run_heads(const uint64_t *key, uint64_t n, int S, uint32_t *hp, uint32_t *sh) {
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint64_t k = key[j], kp = j ? key[j - 1] : ~k;
    hp[j] = (j == 0 || k != kp) ? (uint32_t)j : 0u;
    sh[j] = j == 0 || (k >> (64 - S)) != (kp >> (64 - S));
}

/* the value calls' components in the sorted order, one array each (r, g, b) */
__global__ void k_slot_terms(const double4 *__restrict__ val, const uint32_t *__restrict__ idx,
                             uint64_t n, double *__restrict__ T) {
    const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (q >= n) return;
    const double4 v = val[idx[q]];
    T[q] = v.x;
    T[n + q] = v.y;
    T[2 * n + q] = v.z;
}

/* the run check on the sorted terms: a call that sorts before its neighbour inside a run of
 * equal keys marks the run (bit at its start); each run's length is written at its start */
__global__ void k_run_check(const double *__restrict__ T, const uint64_t *__restrict__ key,
                            const uint32_t *__restrict__ rstart, uint64_t n, uint32_t *claim,
                            uint32_t *runlen) {
    const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (q >= n) return;
    const uint64_t k = key[q];
    const uint32_t s0 = rstart[q];
    if (q > 0 && k == key[q - 1]) {
        const uint64_t a0 = dbits(T[q]), b0 = dbits(T[q - 1]), a1 = dbits(T[n + q]),
                       b1 = dbits(T[n + q - 1]), a2 = dbits(T[2 * n + q]),
                       b2 = dbits(T[2 * n + q - 1]);
        if (a0 != b0 ? a0 < b0 : a1 != b1 ? a1 < b1 : a2 < b2)
            atomicOr(&claim[s0 >> 5], 1u << (s0 & 31u));
    }
    if (q == n - 1 || key[q + 1] != k) runlen[s0] = (uint32_t)(q + 1 - s0);
}

#define FIX_THREAD 32  /* marked runs up to this long: rank sort by one warp */
#define FIX_WARP 256   /* up to this long: bitonic sort in shared memory by one warp */
#define FIX_BLOCK 4096 /* up to this long: the same by one block */

/* the marked runs (the claim bitmap of k_run_check, a 32-position word per thread), by length:
 * (start, length) lists for the warp rank sort, the warp bitonic and the block bitonic sorters
 * (cnt[4], cnt[7], cnt[5]; one global reservation per block and list); longer runs are marked
 * again (claim2) for the radix path and counted (flag bit 2, cnt[3]) */
__global__ void __launch_bounds__(256) k_marked_lists(const uint32_t *__restrict__ claim, uint64_t nw,
                                                      const uint32_t *__restrict__ runlen,
                                                      uint2 *lst8, uint2 *lst16, uint2 *lst_t,
                                                      uint2 *lst_w, uint2 *lst_b,
                                                      unsigned int *cnt, uint32_t *claim2) {
    __shared__ unsigned bc[5], bb[5];
    if (threadIdx.x < 5) bc[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint32_t bits = w < nw ? claim[w] : 0u;
    /* classes: <= 8, <= 16, <= 32 calls (the grouped rank sorts), <= FIX_WARP, <= FIX_BLOCK */
    const auto cls = [](uint32_t len) {
        return len <= 8 ? 0 : len <= 16 ? 1 : len <= FIX_THREAD ? 2 : len <= FIX_WARP ? 3
                                                                   : len <= FIX_BLOCK ? 4 : 5;
    };
    unsigned mine[5] = {0u, 0u, 0u, 0u, 0u};
    for (uint32_t m = bits; m; m &= m - 1) { /* count this word's runs per class */
        const uint32_t j = (uint32_t)(w * 32 + (uint64_t)(__ffs(m) - 1)), len = runlen[j];
        const int c = cls(len);
#pragma unroll
        for (int q = 0; q < 5; ++q)
            if (q == c) ++mine[q];
        if (c == 5) {
            atomicOr(&claim2[j >> 5], 1u << (j & 31u));
            atomicOr(&cnt[0], 2u);
            atomicAdd(&cnt[3], len);
        }
    }
    unsigned off[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) off[c] = mine[c] ? atomicAdd(&bc[c], mine[c]) : 0u;
    __syncthreads();
    if (threadIdx.x < 5 && bc[threadIdx.x]) {
        const int cidx[5] = {1, 2, 4, 7, 5};
        bb[threadIdx.x] = atomicAdd(&cnt[cidx[threadIdx.x]], bc[threadIdx.x]);
    }
    __syncthreads();
    uint2 *const lists[5] = {lst8, lst16, lst_t, lst_w, lst_b};
    for (uint32_t m = bits; m; m &= m - 1) {
        const uint32_t j = (uint32_t)(w * 32 + (uint64_t)(__ffs(m) - 1)), len = runlen[j];
        const int c = cls(len);
        if (c == 5) continue;
        unsigned o = 0;
#pragma unroll
        for (int q = 0; q < 5; ++q)
            if (q == c) o = off[q]++;
        lists[c][bb[c] + o] = make_uint2(j, len);
    }
}

/* bitonic sort of N (a power of two) (r, g, b) bit triples in shared memory by the threads
 * [t0, t0 + nt); sync() between the steps */
template <class Sync>
__device__ __forceinline__ void bitonic3(uint64_t *kr, uint64_t *kg, uint64_t *kb, uint32_t N,
                                         uint32_t t0, uint32_t nt, Sync sync) {
    for (uint32_t k = 2; k <= N; k <<= 1)
        for (uint32_t h = k >> 1; h > 0; h >>= 1) {
            for (uint32_t i = t0; i < N; i += nt) {
                const uint32_t q = i ^ h;
                if (q <= i) continue;
                const bool gt = kr[i] != kr[q] ? kr[i] > kr[q]
                                : kg[i] != kg[q] ? kg[i] > kg[q] : kb[i] > kb[q];
                if (gt == ((i & k) == 0)) {
                    uint64_t t = kr[i]; kr[i] = kr[q]; kr[q] = t;
                    t = kg[i]; kg[i] = kg[q]; kg[q] = t;
                    t = kb[i]; kb[i] = kb[q]; kb[q] = t;
                }
            }
            sync();
        }
}

/* one warp per marked run of up to FIX_WARP calls */
__global__ void __launch_bounds__(256) k_fix_warp(double *T, uint64_t n, const uint2 *lst,
                                                  const unsigned int *cnt) {
    __shared__ uint64_t wsm[8][3][FIX_WARP];
    const unsigned lane = lane_id(), w = threadIdx.x >> 5;
    uint64_t *kr = wsm[w][0], *kg = wsm[w][1], *kb = wsm[w][2];
    const uint32_t nl = cnt[7];
    for (uint64_t e = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; e < nl;
         e += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t j0 = lst[e].x, len = lst[e].y;
        uint32_t N = 64;
        while (N < len) N <<= 1;
        for (uint32_t i = lane; i < N; i += 32) {
            const bool in = i < len;
            kr[i] = in ? dbits(T[j0 + i]) : ~0ull;
            kg[i] = in ? dbits(T[n + j0 + i]) : ~0ull;
            kb[i] = in ? dbits(T[2 * n + j0 + i]) : ~0ull;
        }
        __syncwarp();
        bitonic3(kr, kg, kb, N, lane, 32, [] { __syncwarp(); });
        for (uint32_t i = lane; i < len; i += 32) {
            T[j0 + i] = __longlong_as_double((long long)kr[i]);
            T[n + j0 + i] = __longlong_as_double((long long)kg[i]);
            T[2 * n + j0 + i] = __longlong_as_double((long long)kb[i]);
        }
        __syncwarp();
    }
}

/* marked runs of up to W calls (W = 8, 16, 32), 32 / W of them per warp: each lane of a W-lane
 * group holds one call of its run and counts the calls before it (rank sort through shuffles
 * within the group), then stores it at its rank */
template <int W>
__global__ void __launch_bounds__(256) k_fix_small(double *T, uint64_t n, const uint2 *lst,
                                                   const unsigned int *count) {
    const unsigned lane = lane_id(), sub = lane % W, grp = lane / W;
    const uint32_t nl = *count;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t base = ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5) * (32 / W);
         base < nl; base += nwarps * (32 / W)) {
        const uint64_t e = base + grp;
        const uint32_t j0 = e < nl ? lst[e].x : 0u, len = e < nl ? lst[e].y : 0u;
        const bool in = sub < len;
        const uint64_t r = in ? dbits(T[j0 + sub]) : ~0ull;
        const uint64_t g = in ? dbits(T[n + j0 + sub]) : ~0ull;
        const uint64_t b = in ? dbits(T[2 * n + j0 + sub]) : ~0ull;
        uint32_t rank = 0;
#pragma unroll 4
        for (uint32_t i = 0; i < (uint32_t)W; ++i) {
            const uint64_t ri = __shfl_sync(0xffffffffu, r, i, W);
            const uint64_t gi = __shfl_sync(0xffffffffu, g, i, W);
            const uint64_t bi = __shfl_sync(0xffffffffu, b, i, W);
            const bool lt = i < len && (ri != r ? ri < r : gi != g ? gi < g : bi != b ? bi < b
                                                                             : i < sub);
            rank += lt;
        }
        if (in) {
            T[j0 + rank] = __longlong_as_double((long long)r);
            T[n + j0 + rank] = __longlong_as_double((long long)g);
            T[2 * n + j0 + rank] = __longlong_as_double((long long)b);
        }
    }
}

/* one block per marked run of up to FIX_BLOCK calls: bitonic sort of the (r, g, b) bit triples
 * in shared memory (padded with all-ones: never a finite value) */
__global__ void __launch_bounds__(512) k_fix_block(double *T, uint64_t n, const uint2 *lst,
                                                   const unsigned int *cnt) {
    extern __shared__ uint64_t fsm[];
    uint64_t *kr = fsm, *kg = fsm + FIX_BLOCK, *kb = fsm + 2 * FIX_BLOCK;
    const uint32_t nl = cnt[5];
    for (uint32_t e = blockIdx.x; e < nl; e += gridDim.x) {
        const uint32_t j0 = lst[e].x, len = lst[e].y;
        uint32_t N = 512;
        while (N < len) N <<= 1;
        for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
            const bool in = i < len;
            kr[i] = in ? dbits(T[j0 + i]) : ~0ull;
            kg[i] = in ? dbits(T[n + j0 + i]) : ~0ull;
            kb[i] = in ? dbits(T[2 * n + j0 + i]) : ~0ull;
        }
        __syncthreads();
        bitonic3(kr, kg, kb, N, threadIdx.x, blockDim.x, [] { __syncthreads(); });
        for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) {
            T[j0 + i] = __longlong_as_double((long long)kr[i]);
            T[n + j0 + i] = __longlong_as_double((long long)kg[i]);
            T[2 * n + j0 + i] = __longlong_as_double((long long)kb[i]);
        }
        __syncthreads();
    }
}

/* records in the runs too long for a block (claim2 at their start): flags for the compaction */
__global__ void k_run_marked(const uint32_t *__restrict__ rstart, const uint32_t *__restrict__ claim,
                             uint64_t n, uint8_t *in) {
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint32_t s0 = rstart[j];
    in[j] = (claim[s0 >> 5] >> (s0 & 31u)) & 1u;
}

/* their radix key for the pass c: 0 bits(b), 1 bits(g), 2 (run start, the low S bits of bits(r):
 * the rest of r is the run's sort key) */
__global__ void k_fix_keys(const double *__restrict__ T, uint64_t n,
                           const uint32_t *__restrict__ rstart, const uint32_t *__restrict__ perm,
                           uint64_t m, int c, int S, uint64_t *out) {
    const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (q >= m) return;
    const uint32_t j = perm[q];
    out[q] = c == 2 ? ((uint64_t)rstart[j] << S) | (dbits(T[j]) & ((1ull << S) - 1ull))
                    : dbits(T[(2 - c) * n + j]);
}

/* apply the permutation: the terms at positions perm[q] move to positions pos[q] (both lists
 * hold the same positions) */
__global__ void k_fix_take(const double *__restrict__ T, uint64_t n, const uint32_t *__restrict__ perm,
                           uint64_t m, double *tmp) {
    const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (q >= m) return;
    const uint32_t j = perm[q];
    tmp[q] = T[j];
    tmp[m + q] = T[n + j];
    tmp[2 * m + q] = T[2 * n + j];
}

__global__ void k_fix_put(const double *__restrict__ tmp, const uint32_t *__restrict__ pos,
                          uint64_t m, double *T, uint64_t n) {
    const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (q >= m) return;
    const uint32_t j = pos[q];
    T[j] = tmp[q];
    T[n + j] = tmp[m + q];
    T[2 * n + j] = tmp[2 * m + q];
}

#define SLOT_FOLD_WARP 32 /* slots with more value calls than this are folded by a warp */

__device__ __forceinline__ double4 *slot_acc(const Stores4 &st, uint64_t key, int capl) {
    const int S = capl + 2;
    const uint64_t sk = key >> (64 - S);
    return acc_ptr(st.s[sk >> capl], sk & ((1ull << capl) - 1ull));
}

/* short slots, one thread each: acc += v (weight 1.0, field.cpp:168-170) in the sorted order */
__global__ void k_slot_fold(const double *__restrict__ T, uint64_t n,
                            const uint64_t *__restrict__ key, const uint32_t *__restrict__ start,
                            const uint32_t *__restrict__ nseg, int capl, Stores4 st) {
    const uint32_t ns = *nseg;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < ns;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q0 = start[g], q1 = start[g + 1];
        if (q1 - q0 > SLOT_FOLD_WARP) continue;
        double4 *dst = slot_acc(st, key[q0], capl);
        double4 acc = *dst;
        for (uint32_t q = q0; q < q1; ++q) {
            acc.x += T[q];
            acc.y += T[n + q];
            acc.z += T[2 * n + q];
        }
        *dst = acc;
    }
}

/* the slots folded by a warp (more than SLOT_FOLD_WARP calls), the longest first: the ones of
 * at least SFL_HUGE calls go to list H, the rest to list M (sizes in cnt[0], cnt[1]) */
#define SFL_HUGE 2048
__global__ void k_seg_lists(const uint32_t *__restrict__ start, const uint32_t *__restrict__ nseg,
                            uint32_t *lh, uint32_t *lm, unsigned int *cnt) {
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint32_t ns = *nseg;
    const uint32_t len = g < ns ? start[g + 1] - start[g] : 0u;
    const bool h = len >= SFL_HUGE, m = len > SLOT_FOLD_WARP && len < SFL_HUGE;
    const unsigned lane = lane_id(), lt = (1u << lane) - 1u;
    const unsigned bh = __ballot_sync(0xffffffffu, h), bm = __ballot_sync(0xffffffffu, m);
    unsigned baseh = 0, basem = 0;
    if (lane == 0) {
        if (bh) baseh = atomicAdd(&cnt[0], (unsigned)__popc(bh));
        if (bm) basem = atomicAdd(&cnt[1], (unsigned)__popc(bm));
    }
    baseh = __shfl_sync(0xffffffffu, baseh, 0);
    basem = __shfl_sync(0xffffffffu, basem, 0);
    if (h) lh[baseh + __popc(bh & lt)] = (uint32_t)g;
    if (m) lm[basem + __popc(bm & lt)] = (uint32_t)g;
}

/* long slots, one warp each, taken dynamically from H then M (the longest sequential chains
 * start first); the warp loads the next 8 x 32 terms of each component (coalesced, in flight
 * while the current ones are summed) and lanes 0, 1, 2 add the r, g, b components in order
 * from shared memory */
#define SFL_G 7 /* 7 x 32 terms per component in flight (the padded rows fit 48 KB) */
__global__ void __launch_bounds__(256) k_slot_fold_long(const double *__restrict__ T, uint64_t n,
                                                        const uint64_t *__restrict__ key,
                                                        const uint32_t *__restrict__ start,
                                                        const uint32_t *__restrict__ lh,
                                                        const uint32_t *__restrict__ lm,
                                                        unsigned int *cnt, int capl, Stores4 st) {
    __shared__ double sv[8][3][SFL_G * 32 + 1]; /* +1: the three lanes' rows in different banks */
    const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    const uint32_t nh = cnt[0], nl = nh + cnt[1];
    for (;;) {
        uint32_t item = 0;
        if (lane == 0) item = atomicAdd(&cnt[2], 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= nl) break;
        const uint32_t g = item < nh ? lh[item] : lm[item - nh];
        const uint32_t q0 = start[g], q1 = start[g + 1];
        double4 *dst = slot_acc(st, key[q0], capl);
        const unsigned c = lane < 3 ? lane : 0;
        double acc = (&dst->x)[c];
        double nx[3][SFL_G];
        const auto fetch = [&](uint32_t q) {
#pragma unroll
            for (int k = 0; k < SFL_G; ++k) {
                const uint32_t e = q + k * 32 + lane;
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) nx[cc][k] = e < q1 ? T[cc * n + e] : 0.0;
            }
        };
        fetch(q0);
        for (uint32_t q = q0; q < q1; q += SFL_G * 32) {
            __syncwarp();
#pragma unroll
            for (int k = 0; k < SFL_G; ++k)
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) sv[w][cc][k * 32 + lane] = nx[cc][k];
            __syncwarp();
            if (q + SFL_G * 32 < q1) fetch(q + SFL_G * 32);
            const uint32_t cnt2 = min((uint32_t)(SFL_G * 32), q1 - q);
            if (lane < 3) {
                const double *v = sv[w][c];
                if (cnt2 == SFL_G * 32) {
                    /* 32 terms into registers first, then the dependent adds: the shared loads
                     * stay off the add chain */
#pragma unroll 1
                    for (int ch = 0; ch < SFL_G; ++ch) {
                        double t[32];
#pragma unroll
                        for (int k = 0; k < 32; ++k) t[k] = v[ch * 32 + k];
#pragma unroll
                        for (int k = 0; k < 32; ++k) acc += t[k];
                    }
                } else {
                    for (uint32_t k = 0; k < cnt2; ++k) acc += v[k];
                }
            }
        }
        if (lane < 3) (&dst->x)[c] = acc;
    }
}

/* returns through *fallback whether the records must take the general path instead */
static int fold_slot_records(Scratch &sc, pstf_field *const *fs, int nf, uint64_t nr,
                             uint64_t n, bool *fallback, cudaStream_t st) {
    *fallback = false;
    int capl = 0;
    for (int i = 0; i < nf; ++i)
        if (fs[i]) capl = std::max<int>(capl, (int)fs[i]->cfg.capacity_log2);
    if (capl > 30 || nr >= (1ull << 31)) {
        *fallback = true;
        return PSTF_OK;
    }
    /* nr entries, n real calls: the holes (key ~0) sort behind every call and are dropped */
    const int S = capl + 2;
    const double4 *val = sc.pend2_val.as<double4>();
    const Stores4 S4 = stores4(fs, nf);
    const uint64_t nw = (n + 31) / 32;
    ENSURE(sc.o_key2, nr * 8);
    ENSURE(sc.o_idx, nr * 4);
    ENSURE(sc.o_idx2, nr * 4);
    ENSURE(sc.o_flag, 32); /* [0] flags, [3] calls in over-long runs, [1] [2] [4] [7] [5] lists */
    ENSURE(sc.head, n * 4);
    ENSURE(sc.uid, n * 4);
    ENSURE(sc.rank, n * 4);       /* run lengths (at run starts) */
    ENSURE(sc.o_tgt, nw * 8);     /* run-mark bitmaps: marked, over-long */
    ENSURE(sc.o_fp, (n / 2 + n / 9 + n / 17 + n / (FIX_THREAD + 1) + n / (FIX_WARP + 1) + 5) * 8);
    ENSURE(sc.fterms, n * 24);    /* the terms r | g | b in the sorted order */
    ENSURE(sc.fstart, (n + 1) * 4);
    ENSURE(sc.fnruns, 8);
    const uint64_t *key = sc.pend2_key.as<uint64_t>();
    uint64_t *key2 = sc.o_key2.as<uint64_t>();
    uint32_t *idx0 = sc.o_idx.as<uint32_t>(), *idx = sc.o_idx2.as<uint32_t>();
    unsigned int *flag = sc.o_flag.as<unsigned int>();
    uint32_t *hp = sc.head.as<uint32_t>(), *rstart = sc.uid.as<uint32_t>();
    uint32_t *claim = sc.o_tgt.as<uint32_t>(), *claim2 = claim + nw;
    uint2 *lst_t = sc.o_fp.as<uint2>();
    double *T = sc.fterms.as<double>();
    CK(cudaMemsetAsync(sc.o_flag.p, 0, 32, st));
    CK(cudaMemsetAsync(sc.o_tgt.p, 0, nw * 8, st));
    if (sc.iota_n < nr) { /* the sort's input indices, written once per size */
        ENSURE(sc.iota, nr * 4);
        sc.iota_n = sc.iota.bytes / 4;
        LAUNCH(k_iota32, grid_for(sc.iota_n, 256), 256, 0, st, sc.iota.as<uint32_t>(), sc.iota_n);
    }
    const uint32_t *iota = sc.iota.as<uint32_t>();
    const auto cub_call = [&](const char *name, int nlaunch, auto &&fn) -> int {
        size_t bytes = 0;
        CK(fn((void *)nullptr, bytes));
        ENSURE(sc.cub, bytes);
        bytes = sc.cub.bytes;
        ProfScope ps_(name, st);
        CK(fn(sc.cub.p, bytes));
        g_launches.fetch_add(nlaunch, std::memory_order_relaxed);
        return PSTF_OK;
    };
    int rc = cub_call("cub::DeviceRadixSort", 4, [&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortPairs(t, b, key, key2, iota, idx, (int64_t)nr, 0, 64, st);
    });
    if (rc) return rc;
    /* runs of equal sort keys holding an out-of-order pair, re-sorted in place by length class */
    uint32_t *sh = idx0; /* slot-segment heads */
    LAUNCH(k_run_heads, grid_for(n, 256), 256, 0, st, key2, n, S, hp, sh);
    rc = cub_call("cub::DeviceScan", 2, [&](void *t, size_t &b) {
        return cub::DeviceScan::InclusiveScan(t, b, hp, rstart, cub::Max(), (int64_t)n, st);
    });
    if (rc) return rc;
    LAUNCH(k_slot_terms, grid_for(n, 256), 256, 0, st, val, idx, n, T);
    LAUNCH(k_run_check, grid_for(n, 256), 256, 0, st, T, key2, rstart, n, claim,
           sc.rank.as<uint32_t>());
    /* at most n/2 marked runs (each holds two calls or more), n/9 longer than 8, ... */
    uint2 *lst8 = lst_t, *lst16 = lst8 + n / 2 + 1, *lst32 = lst16 + n / 9 + 1,
          *lst_w = lst32 + n / 17 + 1, *lst_b = lst_w + n / (FIX_THREAD + 1) + 1;
    LAUNCH(k_marked_lists, grid_for(nw, 256), 256, 0, st, claim, nw, sc.rank.as<uint32_t>(), lst8,
           lst16, lst32, lst_w, lst_b, flag, claim2);
    const unsigned grid = (unsigned)sm_count() * 8;
    LAUNCH(k_fix_small<8>, grid, 256, 0, st, T, n, lst8, flag + 1);
    LAUNCH(k_fix_small<16>, grid, 256, 0, st, T, n, lst16, flag + 2);
    LAUNCH(k_fix_small<32>, grid, 256, 0, st, T, n, lst32, flag + 4);
    LAUNCH(k_fix_warp, grid, 256, 0, st, T, n, lst_w, flag);
    const size_t fsm = 3 * FIX_BLOCK * 8;
    SMEM_ATTR(k_fix_block, fsm);
    LAUNCH(k_fix_block, (unsigned)sm_count() * 2, 512, fsm, st, T, n, lst_b, flag);
    rc = read_small(sc, sc.o_flag.p, 32, st); /* the pass's one host read */
    if (rc) return rc;
    const uint32_t *h = (const uint32_t *)sc.h_small;
    const uint32_t fl = h[0];
    const uint64_t m = h[3];
    if (getenv("PSTF_ORDERED_DEBUG"))
        fprintf(stderr, "[ordered] %llu value calls of existing slots, flag %u, marked runs %u "
                "(thread) %u (warp) %u (block), %llu calls in longer marked runs\n",
                (unsigned long long)n, fl, h[1] + h[2] + h[4], h[7], h[5], (unsigned long long)m);
    if (m) { /* the runs too long for a block: b, g, then (run start, r) (stable, LSD) */
        ENSURE(sc.fisc, n);
        LAUNCH(k_run_marked, grid_for(n, 256), 256, 0, st, rstart, claim2, n, sc.fisc.as<uint8_t>());
        uint32_t *F = sc.fstart.as<uint32_t>(); /* their positions, ascending */
        rc = cub_call("cub::DeviceSelect", 2, [&](void *t, size_t &b) {
            return cub::DeviceSelect::Flagged(t, b, cub::CountingInputIterator<uint32_t>(0),
                                              sc.fisc.as<uint8_t>(), F, flag + 6, (int64_t)n, st);
        });
        if (rc) return rc;
        ENSURE(sc.o_fk, m * 40);
        uint32_t *P0 = reinterpret_cast<uint32_t *>(sc.o_fk.as<uint64_t>() + 4 * m), *P1 = P0 + m;
        uint64_t *K0 = sc.o_fk.as<uint64_t>(), *K1 = K0 + m;
        CK(cudaMemcpyAsync(P0, F, m * 4, cudaMemcpyDeviceToDevice, st));
        int nbits = 1;
        while ((1ull << nbits) < n) ++nbits;
        for (int c = 0; c < 3; ++c) {
            LAUNCH(k_fix_keys, grid_for(m, 256), 256, 0, st, T, n, rstart, P0, m, c, S, K0);
            rc = cub_call("cub::DeviceRadixSort", 4, [&](void *t, size_t &b) {
                return cub::DeviceRadixSort::SortPairs(t, b, K0, K1, P0, P1, (int64_t)m, 0,
                                                       c == 2 ? nbits + S : 64, st);
            });
            if (rc) return rc;
            std::swap(P0, P1);
        }
        double *tmp = reinterpret_cast<double *>(K0); /* 3m doubles: K0, K1 and the next m */
        LAUNCH(k_fix_take, grid_for(m, 256), 256, 0, st, T, n, P0, m, tmp);
        LAUNCH(k_fix_put, grid_for(m, 256), 256, 0, st, tmp, F, m, T, n);
    }
    /* one segment per slot, folded in that order */
    rc = cub_call("cub::DeviceScan", 2, [&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, sh, rstart, (int64_t)n, st);
    });
    if (rc) return rc;
    uint32_t *seg = sc.fstart.as<uint32_t>(); /* segment starts (+ the end sentinel) */
    LAUNCH(k_fold_starts, grid_for(n, 256), 256, 0, st, sh, rstart, n, seg);
    LAUNCH(k_fold_nruns, 1, 1, 0, st, sh, rstart, n, sc.fnruns.as<uint32_t>());
    LAUNCH(k_slot_fold, grid, 256, 0, st, T, n, key2, seg, sc.fnruns.as<uint32_t>(), capl, S4);
    /* the warp-folded slots, longest first, taken dynamically (lists reuse the run-list space) */
    uint32_t *lh = reinterpret_cast<uint32_t *>(lst_t), *lm = lh + n / SFL_HUGE + 1;
    CK(cudaMemsetAsync(flag, 0, 12, st));
    LAUNCH(k_seg_lists, grid_for(n, 256), 256, 0, st, seg, sc.fnruns.as<uint32_t>(), lh, lm, flag);
    LAUNCH(k_slot_fold_long, grid, 256, 0, st, T, n, key2, seg, lh, lm, flag, capl, S4);
    return PSTF_OK;
}

/* ORDERED vertex pass, phase 2: the slot-grouped fold of existing slots' value calls, then the
 * general path (sort, placement, fold) for the new keys' calls */
static int resolve_ordered(Scratch &sc, pstf_field *const *fs, int nf, cudaStream_t st) {
    int rc = read_small(sc, sc.pend_count.p, 8, st);
    if (rc) return rc;
    uint64_t n1 = sc.h_small[0];
    rc = read_small(sc, sc.pend2_count.p, 24, st);
    if (rc) return rc;
    if (sc.h_small[0] > sc.pend2_key.bytes / 8)
        return set_err(PSTF_E_NOMEM, "slot-grouped call buffer overflow");
    const uint64_t n2r = sc.h_small[0], n2 = n2r - sc.h_small[2]; /* reserved, real calls */
    const bool alias = sc.h_small[1] != 0;
    if (n2) {
        bool fallback = alias;
        const bool force = getenv("PSTF_ORDERED_GENERAL") != nullptr; /* parity tests */
        if (!force && !alias) {
            rc = fold_slot_records(sc, fs, nf, n2r, n2, &fallback, st);
            if (rc) return rc;
        }
        if (force || fallback) { /* as full records, appended to the general path's */
            if (n1 + n2 > sc.pend.bytes / sizeof(PendRec)) {
                /* grow, keeping the n1 records already there */
                DBuf nb;
                CK(nb.ensure((n1 + n2) * sizeof(PendRec)));
                CK(cudaMemcpyAsync(nb.p, sc.pend.p, n1 * sizeof(PendRec), cudaMemcpyDeviceToDevice,
                                   st));
                CK(cudaStreamSynchronize(st));
                std::swap(nb.p, sc.pend.p);
                std::swap(nb.bytes, sc.pend.bytes);
            }
            int capl = 0;
            for (int i = 0; i < nf; ++i)
                if (fs[i]) capl = std::max<int>(capl, (int)fs[i]->cfg.capacity_log2);
            ENSURE(sc.o_flag, 32);
            CK(cudaMemsetAsync(sc.o_flag.p, 0, 8, st));
            LAUNCH(k_slot_expand, grid_for(n2r, 256), 256, 0, st, sc.pend2_key.as<uint64_t>(),
                   sc.pend2_val.as<double4>(), n2r, capl, stores4(fs, nf),
                   sc.pend.as<PendRec>() + n1, sc.o_flag.as<unsigned long long>());
            n1 += n2;
            LAUNCH(k_set_u64, 1, 1, 0, st, sc.pend_count.as<unsigned long long>(),
                   (unsigned long long)n1);
        }
    }
    return resolve_pending(sc, fs, nf, PSTF_MODE_ORDERED, n1, st);
}

/* Completes the deferred vertex pass (if any) that involves store cf: waits for its pending
 * count and places the new keys (phase 2). */
static int settle(const pstf_field *cf) {
    pstf_field *o = cf ? cf->owed_by : nullptr;
    if (!o || !o->dp.active) return PSTF_OK;
    DeferredPass &d = o->dp;
    d.active = false;
    for (int i = 0; i < 4; ++i)
        if (d.fs[i]) d.fs[i]->owed_by = nullptr;
    CK(cudaSetDevice(o->device));
    CK(cudaEventSynchronize(d.ev));
    const uint64_t n = *d.h_count;
    if (n == 0) return PSTF_OK;
    return resolve_pending(o->sc, d.fs, d.nf, d.mode, n, d.st);
}

#define SETTLE(f)                                                                                  \
    do {                                                                                           \
        int rc_ = settle(f);                                                                       \
        if (rc_) return rc_;                                                                       \
    } while (0)

/* Ends a vertex pass: phase 2 now (PSTF_NO_DEFER), or deferred (see DeferredPass). */
static int finish_vertex_pass(pstf_field *const fs[4], int mode, cudaStream_t st) {
    pstf_field *lo = fs[0];
    const int nf = fs[3] ? 4 : 3;
    if (mode == PSTF_MODE_ORDERED) return resolve_ordered(lo->sc, fs, nf, st);
    static const bool no_defer = getenv("PSTF_NO_DEFER") != nullptr;
    if (no_defer) return resolve_pending(lo->sc, fs, nf, mode, (uint64_t)-1, st);
    DeferredPass &d = lo->dp;
    if (!d.ev) CK(cudaEventCreateWithFlags(&d.ev, cudaEventDisableTiming));
    if (!d.h_count) CK(cudaMallocHost(&d.h_count, 8));
    CK(cudaMemcpyAsync(d.h_count, lo->sc.pend_count.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(d.ev, st));
    for (int i = 0; i < 4; ++i) {
        d.fs[i] = fs[i];
        if (fs[i]) fs[i]->owed_by = lo;
    }
    d.nf = nf;
    d.mode = mode;
    d.st = st;
    d.active = true;
    return PSTF_OK;
}

static int ensure_pending(Scratch &sc, uint64_t cap, bool with_seq, cudaStream_t st) {
    ENSURE(sc.pend, cap * sizeof(PendRec));
    ENSURE(sc.pend_count, 8);
    if (with_seq) ENSURE(sc.pend_seq, cap * 8);
    CK(cudaMemsetAsync(sc.pend_count.p, 0, 8, st));
    ENSURE(sc.pend2_count, 32); /* calls (incl. holes), alias flag, holes */
    CK(cudaMemsetAsync(sc.pend2_count.p, 0, 32, st));
    return PSTF_OK;
}

/* ORDERED vertex passes: room for every value call of an existing slot (<= 7 per vertex) */
static int ensure_pending2(Scratch &sc, uint64_t calls, uint64_t launches = 1) {
    /* every value call (<= 7 per vertex) plus the tiled kernel's unused chunk tails (at most
     * one chunk per warp of its persistent grid, per launch) */
    const uint64_t cap =
        calls + launches * (uint64_t)sm_count() * VT_MINB * (VT / 32) * PAIR_CHUNK;
    ENSURE(sc.pend2_key, cap * 8);
    ENSURE(sc.pend2_val, cap * 32);
    return PSTF_OK;
}

static bool same_quant(const pstf_field_config &a, const pstf_field_config &b) {
    return a.base_cell_size == b.base_cell_size && a.level_select_k == b.level_select_k &&
           a.max_level == b.max_level;
}

static void twin_break(pstf_field *f) {
    if (!f) return;
    if (f->twin) f->twin->twin = nullptr;
    f->twin = nullptr;
    f->pristine = false;
}

/* a batch operation on stores fs[0..n): a store whose twin is not in the batch loses it */
static void twin_batch(pstf_field *const *fs, int n) {
    for (int i = 0; i < n; ++i) {
        if (!fs[i]) continue;
        bool in = false;
        for (int j = 0; j < n; ++j) in = in || (fs[j] && fs[j] == fs[i]->twin);
        if (fs[i]->twin && !in) twin_break(fs[i]);
        fs[i]->pristine = false;
    }
}

/* the twin relation of (lo, loe) for a vertex pass: kept, established (both fresh and alike),
 * or ended; the other stores of the pass lose theirs */
static bool twin_for_pass(pstf_field *lo, pstf_field *loe, pstf_field *fli, pstf_field *li) {
    bool twin = lo->twin == loe && loe->twin == lo;
    if (!twin) {
        const pstf_field_config &a = lo->cfg, &b = loe->cfg;
        if (lo->pristine && loe->pristine && lo != loe && a.capacity_log2 == b.capacity_log2 &&
            a.probe_window == b.probe_window && a.evict_age_frames == b.evict_age_frames &&
            same_quant(a, b) && lo->frame == loe->frame && !getenv("PSTF_NO_TWIN")) {
            twin_break(lo);
            twin_break(loe);
            lo->twin = loe;
            loe->twin = lo;
            twin = true;
        } else {
            twin_break(lo);
            twin_break(loe);
        }
    }
    if (fli != lo && fli != loe) twin_break(fli);
    if (li && li != lo && li != loe) twin_break(li);
    lo->pristine = loe->pristine = false;
    return twin;
}


static int check_config(const pstf_field_config *c) {
    if (!c) return set_err(PSTF_E_INVALID, "config is NULL");
    if (c->capacity_log2 < 1 || c->capacity_log2 > 30)
        return set_err(PSTF_E_INVALID, "capacity_log2 must be in [1, 30]");
    if (c->max_level < 0 || c->max_level > 62)
        return set_err(PSTF_E_INVALID, "max_level must be in [0, 62]");
    if (c->probe_window < 1) return set_err(PSTF_E_INVALID, "probe_window must be >= 1");
    if (c->kind > 3) return set_err(PSTF_E_INVALID, "unknown field kind");
    return PSTF_OK;
}

/* ========================================================================================== */
/* C ABI                                                                                       */

extern "C" {

int pstf_abi_version(void) { return PSTF_ABI_VERSION; }
const char *pstf_last_error(void) { return g_last_error.c_str(); }
uint64_t pstf_kernel_launch_count(void) { return g_launches.load(); }

int pstf_profile_enable(int on) {
    g_prof.store(on ? 1 : 0);
    return PSTF_OK;
}

/* Synchronises on the recorded events, aggregates per kernel name, clears the record.
 * names: n_max entries of 64 chars; ms / counts: n_max entries. */
int pstf_profile_collect(char *names, double *ms, uint64_t *counts, int n_max, int *n_out) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    std::vector<std::string> nm;
    std::vector<double> tot;
    std::vector<uint64_t> cnt;
    for (auto &r : g_prof_recs) {
        float t = 0.f;
        cudaEventSynchronize(r.b);
        cudaEventElapsedTime(&t, r.a, r.b);
        size_t k = 0;
        while (k < nm.size() && nm[k] != r.name) ++k;
        if (k == nm.size()) {
            nm.push_back(r.name);
            tot.push_back(0.0);
            cnt.push_back(0);
        }
        tot[k] += t;
        cnt[k] += 1;
        g_prof_pool.push_back(r.a);
        g_prof_pool.push_back(r.b);
    }
    g_prof_recs.clear();
    int n = (int)std::min<size_t>(nm.size(), (size_t)std::max(n_max, 0));
    for (int i = 0; i < n; ++i) {
        if (names) {
            strncpy(names + 64 * i, nm[i].c_str(), 63);
            names[64 * i + 63] = 0;
        }
        if (ms) ms[i] = tot[i];
        if (counts) counts[i] = cnt[i];
    }
    if (n_out) *n_out = n;
    return PSTF_OK;
}

int pstf_field_create(const pstf_field_config *config, int device, pstf_field **out) {
    if (!out) return set_err(PSTF_E_INVALID, "out is NULL");
    *out = nullptr;
    int rc = check_config(config);
    if (rc) return rc;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0)
        return set_err(PSTF_E_CUDA, "no CUDA device available (the field cache has no CPU path)");
    if (device < 0 || device >= ndev) return set_err(PSTF_E_INVALID, "bad device ordinal");
    CK(cudaSetDevice(device));
    pstf_field *f = new (std::nothrow) pstf_field();
    if (!f) return set_err(PSTF_E_NOMEM, "host allocation failed");
    f->cfg = *config;
    f->device = device;
    const uint64_t cap = 1ull << config->capacity_log2;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~(size_t)255;
        return o;
    };
    size_t o_meta = take(cap * 8), o_com = take(cap * 32), o_acc = take(cap * 32),
           o_keyf = take(cap * sizeof(KeyFields)), o_h0 = take(cap * 4), o_h1 = take(cap * 4),
           o_tbits = take(((cap + 31) / 32) * 4), o_lbits = take(((cap + 31) / 32) * 4),
           o_tlist = take(cap * 4), o_ctr = take(C_NUM * 8),
           o_sum = take(8);
    cudaError_t e = cudaMalloc(&f->arena, off);
    if (e != cudaSuccess) {
        delete f;
        return set_err(PSTF_E_NOMEM, std::string("device allocation failed: ") + cudaGetErrorString(e));
    }
    char *base = (char *)f->arena;
    DevStore &d = f->d;
    memset(&d, 0, sizeof(d));
    d.meta = (uint2 *)(base + o_meta);
    d.com = (double4 *)(base + o_com);
    d.acc = (double4 *)(base + o_acc);
    d.keyf = (KeyFields *)(base + o_keyf);
    d.tbits = (uint32_t *)(base + o_tbits);
    d.lbits = (uint32_t *)(base + o_lbits);
    d.tlist = (uint32_t *)(base + o_tlist);
    d.hold0 = (uint32_t *)(base + o_h0);
    d.hold1 = (uint32_t *)(base + o_h1);
    d.ctr = (unsigned long long *)(base + o_ctr);
    d.cn_sum = (double *)(base + o_sum);
    d.mask = (uint32_t)(cap - 1);
    d.window = config->probe_window;
    d.kp.base_cell_size = config->base_cell_size;
    d.kp.level_select_k = config->level_select_k;
    d.kp.max_level = config->max_level;
    d.t_max = config->t_max;
    d.blend = config->blend;
    d.evict_age = config->evict_age_frames;
    d.rank = 0;
    /* value-initialised slots (field.cpp:232: make_unique<Slot[]>) */
    e = cudaMemset(f->arena, 0, off);
    if (e == cudaSuccess) e = cudaMemset(d.hold0, 0xff, cap * 4);
    if (e == cudaSuccess) e = cudaMemset(d.hold1, 0xff, cap * 4);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(f->arena);
        delete f;
        return set_err(PSTF_E_CUDA, cudaGetErrorString(e));
    }
    *out = f;
    return PSTF_OK;
}

int pstf_field_destroy(pstf_field *f) {
    if (!f) return PSTF_OK;
    twin_break(f); /* the partner must not keep a pointer to it */
    cudaSetDevice(f->device);
    settle(f); /* no dangling deferred pass may reference this store */
    cudaDeviceSynchronize();
    if (f->arena) cudaFree(f->arena);
    delete f;
    return PSTF_OK;
}

int pstf_field_get_config(const pstf_field *f, pstf_field_config *out) {
    if (!f || !out) return set_err(PSTF_E_INVALID, "NULL argument");
    *out = f->cfg;
    return PSTF_OK;
}

int pstf_select_level(const pstf_field *f, const double *footprint, int32_t *level, uint64_t n,
                      void *stream) {
    if (!f || (!footprint && n) || (!level && n)) return set_err(PSTF_E_INVALID, "NULL argument");
    if (!n) return PSTF_OK;
    CK(cudaSetDevice(f->device));
    LAUNCH(k_select_level, grid_for(n, 256), 256, 0, (cudaStream_t)stream, f->d.kp, footprint,
           level, n);
    return PSTF_OK;
}

int pstf_key_for(const pstf_field *f, const pstf_vec3_soa *pos, const pstf_vec3_soa *dir,
                 const int32_t *level, uint64_t n, pstf_key *keys, void *stream) {
    if (!f || !pos || !dir || (n && (!level || !keys))) return set_err(PSTF_E_INVALID, "NULL argument");
    if (!n) return PSTF_OK;
    CK(cudaSetDevice(f->device));
    LAUNCH(k_key_for, grid_for(n, 256), 256, 0, (cudaStream_t)stream, f->d.kp, *pos, *dir, level,
           n, keys);
    return PSTF_OK;
}

int pstf_field_apply(pstf_field *f, const pstf_key *keys, const pstf_vec3_soa *value,
                     const double *w, const uint8_t *is_counter, uint64_t n, int mode,
                     void *stream) {
    if (f) f->unit_frame = false; /* arbitrary weights: endFrame's reduce pass */
    twin_break(f);                /* an update of this store alone */
    if (!f || (n && (!keys || !w))) return set_err(PSTF_E_INVALID, "NULL argument");
    if (mode < 0 || mode > 2) return set_err(PSTF_E_INVALID, "bad mode");
    if (!n) return PSTF_OK;
    if (n >= 0xffffffffULL) return set_err(PSTF_E_INVALID, "batch too large");
    CK(cudaSetDevice(f->device));
    SETTLE(f);
    cudaStream_t st = (cudaStream_t)stream;
    Scratch &sc = f->sc;
    ApplyArgs a;
    a.s = dev_view(f);
    a.keys = keys;
    a.vr = value ? value->x : nullptr;
    a.vg = value ? value->y : nullptr;
    a.vb = value ? value->z : nullptr;
    a.w = w;
    a.isc = is_counter;
    a.n = n;
    int rc = ensure_pending(sc, n, mode == PSTF_MODE_SEQUENTIAL, st);
    if (rc) return rc;
    if (is_counter && !getenv("PSTF_CN_PARALLEL")) { /* the env: experiment / test switch */
        LAUNCH(k_cn_flag, grid_for(n, 256), 256, 0, st, w, is_counter, n, f->d.ctr);
        f->counted_apply = true;
    }
    uint64_t known = (uint64_t)-1;
    if (mode == PSTF_MODE_ATOMIC) {
        LAUNCH(k_apply_atomic, grid_for(n, 256), 256, 0, st, a, sc.pend.as<PendRec>(),
               sc.pend_count.as<unsigned long long>(), n);
    } else {
        ENSURE(sc.valid, n * 4);
        ENSURE(sc.scan, n * 4);
        LAUNCH(k_apply_flags, grid_for(n, 256), 256, 0, st, a, sc.valid.as<uint32_t>());
        size_t bytes = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, sc.valid.as<uint32_t>(),
                                         sc.scan.as<uint32_t>(), (int64_t)n, st));
        ENSURE(sc.cub, bytes);
        bytes = sc.cub.bytes;
        { ProfScope ps_("cub::DeviceScan", st);
        CK(cub::DeviceScan::ExclusiveSum(sc.cub.p, bytes, sc.valid.as<uint32_t>(),
                                         sc.scan.as<uint32_t>(), (int64_t)n, st));
        g_launches.fetch_add(2, std::memory_order_relaxed); }
        LAUNCH(k_apply_records, grid_for(n, 256), 256, 0, st, a, sc.valid.as<uint32_t>(),
               sc.scan.as<uint32_t>(), sc.pend.as<PendRec>(),
               mode == PSTF_MODE_SEQUENTIAL ? sc.pend_seq.as<uint64_t>() : nullptr);
        uint32_t last[2];
        rc = read_small(sc, sc.scan.as<uint32_t>() + (n - 1), 4, st);
        if (rc) return rc;
        last[0] = ((uint32_t *)sc.h_small)[0];
        rc = read_small(sc, sc.valid.as<uint32_t>() + (n - 1), 4, st);
        if (rc) return rc;
        last[1] = ((uint32_t *)sc.h_small)[0];
        known = (uint64_t)last[0] + last[1];
    }
    pstf_field *fs[1] = {f};
    return resolve_pending(sc, fs, 1, mode, known, st);
}

/* ---- host-pointer variants (scalar facade): stage through device scratch, synchronise ---- */
static int stage_h2d(Scratch &sc, const std::vector<const void *> &src,
                     const std::vector<size_t> &bytes, std::vector<char *> &dst) {
    size_t tot = 0;
    for (size_t b : bytes) tot += (b + 255) & ~(size_t)255;
    ENSURE(sc.hio, tot + 256);
    char *p = sc.hio.as<char>();
    dst.clear();
    for (size_t k = 0; k < src.size(); ++k) {
        dst.push_back(p);
        if (src[k] && bytes[k]) CK(cudaMemcpy(p, src[k], bytes[k], cudaMemcpyHostToDevice));
        p += (bytes[k] + 255) & ~(size_t)255;
    }
    return PSTF_OK;
}

static void aos_to_soa(const double *aos, uint64_t n, std::vector<double> &soa) {
    soa.resize(3 * n);
    for (uint64_t i = 0; i < n; ++i)
        for (int c = 0; c < 3; ++c) soa[c * n + i] = aos[3 * i + c];
}

int pstf_key_for_host(const pstf_field *f, const double *pos_xyz, const double *dir_xyz,
                      const int32_t *level, uint64_t n, pstf_key *keys) {
    if (!f) return set_err(PSTF_E_INVALID, "NULL store");
    std::lock_guard<std::mutex> lk(const_cast<pstf_field *>(f)->host_mu);
    if (!f || (n && (!pos_xyz || !dir_xyz || !level || !keys)))
        return set_err(PSTF_E_INVALID, "NULL argument");
    if (!n) return PSTF_OK;
    CK(cudaSetDevice(f->device));
    CK(cudaDeviceSynchronize());
    std::vector<double> p, d;
    aos_to_soa(pos_xyz, n, p);
    aos_to_soa(dir_xyz, n, d);
    std::vector<char *> dv;
    Scratch &sc = const_cast<pstf_field *>(f)->sc;
    int rc = stage_h2d(sc, {p.data(), d.data(), level, nullptr},
                       {p.size() * 8, d.size() * 8, n * 4, n * sizeof(pstf_key)}, dv);
    if (rc) return rc;
    const double *dp = (const double *)dv[0], *dd = (const double *)dv[1];
    pstf_vec3_soa ps{dp, dp + n, dp + 2 * n}, ds{dd, dd + n, dd + 2 * n};
    rc = pstf_key_for(f, &ps, &ds, (const int32_t *)dv[2], n, (pstf_key *)dv[3], nullptr);
    if (rc) return rc;
    CK(cudaMemcpy(keys, dv[3], n * sizeof(pstf_key), cudaMemcpyDeviceToHost));
    return PSTF_OK;
}

int pstf_select_level_host(const pstf_field *f, const double *footprint, int32_t *level,
                           uint64_t n) {
    if (!f) return set_err(PSTF_E_INVALID, "NULL store");
    std::lock_guard<std::mutex> lk(const_cast<pstf_field *>(f)->host_mu);
    if (!f || (n && (!footprint || !level))) return set_err(PSTF_E_INVALID, "NULL argument");
    if (!n) return PSTF_OK;
    CK(cudaSetDevice(f->device));
    CK(cudaDeviceSynchronize());
    std::vector<char *> dv;
    Scratch &sc = const_cast<pstf_field *>(f)->sc;
    int rc = stage_h2d(sc, {footprint, nullptr}, {n * 8, n * 4}, dv);
    if (rc) return rc;
    rc = pstf_select_level(f, (const double *)dv[0], (int32_t *)dv[1], n, nullptr);
    if (rc) return rc;
    CK(cudaMemcpy(level, dv[1], n * 4, cudaMemcpyDeviceToHost));
    return PSTF_OK;
}

int pstf_field_apply_host(pstf_field *f, const pstf_key *keys, const double *rgb_xyz,
                          const double *w, const uint8_t *is_counter, uint64_t n, int mode) {
    if (f) f->unit_frame = false; /* arbitrary weights: endFrame's reduce pass */
    if (!f) return set_err(PSTF_E_INVALID, "NULL store");
    std::lock_guard<std::mutex> lk(const_cast<pstf_field *>(f)->host_mu);
    if (!f || (n && (!keys || !w))) return set_err(PSTF_E_INVALID, "NULL argument");
    if (!n) return PSTF_OK;
    CK(cudaSetDevice(f->device));
    SETTLE(f);
    CK(cudaDeviceSynchronize());
    std::vector<double> v;
    if (rgb_xyz) aos_to_soa(rgb_xyz, n, v);
    std::vector<char *> dv;
    /* staging lives in its own buffer: pstf_field_apply reuses the store scratch */
    static thread_local DBuf io;
    size_t sz[4] = {n * sizeof(pstf_key), rgb_xyz ? 3 * n * 8 : 0, n * 8, is_counter ? n : 0};
    size_t tot = 0;
    for (size_t b : sz) tot += (b + 255) & ~(size_t)255;
    ENSURE(io, tot + 256);
    char *p = io.as<char>();
    const void *src[4] = {keys, rgb_xyz ? (const void *)v.data() : nullptr, w, is_counter};
    for (int k = 0; k < 4; ++k) {
        dv.push_back(p);
        if (src[k] && sz[k]) CK(cudaMemcpy(p, src[k], sz[k], cudaMemcpyHostToDevice));
        p += (sz[k] + 255) & ~(size_t)255;
    }
    const double *dvv = (const double *)dv[1];
    pstf_vec3_soa vs{dvv, dvv + n, dvv + 2 * n};
    int rc = pstf_field_apply(f, (const pstf_key *)dv[0], rgb_xyz ? &vs : nullptr,
                              (const double *)dv[2], is_counter ? (const uint8_t *)dv[3] : nullptr,
                              n, mode, nullptr);
    if (rc) return rc;
    CK(cudaDeviceSynchronize());
    return PSTF_OK;
}

int pstf_field_query_host(const pstf_field *f, const double *pos_xyz, const double *dir_xyz,
                          const double *footprint, const int32_t *level, uint64_t n,
                          double *value_rgb, uint8_t *valid, uint8_t *fallback,
                          int32_t *out_level) {
    if (!f) return set_err(PSTF_E_INVALID, "NULL store");
    std::lock_guard<std::mutex> lk(const_cast<pstf_field *>(f)->host_mu);
    if (!f || (n && (!pos_xyz || !dir_xyz))) return set_err(PSTF_E_INVALID, "NULL argument");
    if ((footprint == nullptr) == (level == nullptr))
        return set_err(PSTF_E_INVALID, "exactly one of footprint / level must be given");
    if (!n) return PSTF_OK;
    CK(cudaSetDevice(f->device));
    SETTLE(f);
    CK(cudaDeviceSynchronize());
    std::vector<double> p, d;
    aos_to_soa(pos_xyz, n, p);
    aos_to_soa(dir_xyz, n, d);
    std::vector<char *> dv;
    Scratch &sc = const_cast<pstf_field *>(f)->sc;
    int rc = stage_h2d(sc, {p.data(), d.data(), footprint ? (const void *)footprint : level,
                            nullptr, nullptr, nullptr, nullptr},
                       {3 * n * 8, 3 * n * 8, footprint ? n * 8 : n * 4, 3 * n * 8, n, n, n * 4},
                       dv);
    if (rc) return rc;
    const double *dp = (const double *)dv[0], *dd = (const double *)dv[1];
    pstf_vec3_soa ps{dp, dp + n, dp + 2 * n}, ds{dd, dd + n, dd + 2 * n};
    double *val = (double *)dv[3];
    rc = pstf_field_query(f, &ps, &ds, footprint ? (const double *)dv[2] : nullptr,
                          footprint ? nullptr : (const int32_t *)dv[2], n, val, val + n,
                          val + 2 * n, (uint8_t *)dv[4], (uint8_t *)dv[5], (int32_t *)dv[6],
                          nullptr);
    if (rc) return rc;
    std::vector<double> hv(3 * n);
    CK(cudaMemcpy(hv.data(), val, 3 * n * 8, cudaMemcpyDeviceToHost));
    if (value_rgb)
        for (uint64_t i = 0; i < n; ++i)
            for (int c = 0; c < 3; ++c) value_rgb[3 * i + c] = hv[c * n + i];
    if (valid) CK(cudaMemcpy(valid, dv[4], n, cudaMemcpyDeviceToHost));
    if (fallback) CK(cudaMemcpy(fallback, dv[5], n, cudaMemcpyDeviceToHost));
    if (out_level) CK(cudaMemcpy(out_level, dv[6], n * 4, cudaMemcpyDeviceToHost));
    return PSTF_OK;
}

int pstf_field_query(const pstf_field *f, const pstf_vec3_soa *pos, const pstf_vec3_soa *dir,
                     const double *footprint, const int32_t *level, uint64_t n, double *value_r,
                     double *value_g, double *value_b, uint8_t *valid, uint8_t *fallback,
                     int32_t *out_level, void *stream) {
    if (!f || !pos || !dir) return set_err(PSTF_E_INVALID, "NULL argument");
    if ((footprint == nullptr) == (level == nullptr))
        return set_err(PSTF_E_INVALID, "exactly one of footprint / level must be given");
    if (!n) return PSTF_OK;
    CK(cudaSetDevice(f->device));
    SETTLE(f);
    LAUNCH(k_query, grid_for(n, 256), 256, 0, (cudaStream_t)stream, dev_view(f), *pos, *dir,
           footprint, level, n, value_r, value_g, value_b, valid, fallback, out_level);
    return PSTF_OK;
}

int pstf_fields_end_frame(pstf_field *const *fs, int n, void *stream) {
    if (!fs || n < 1 || n > 4) return set_err(PSTF_E_INVALID, "1..4 stores per batch");
    for (int i = 0; i < n; ++i) {
        if (!fs[i]) return set_err(PSTF_E_INVALID, "NULL store");
        if (fs[i]->device != fs[0]->device)
            return set_err(PSTF_E_INVALID, "all stores must live on one device");
        for (int j = 0; j < i; ++j)
            if (fs[j] == fs[i]) return set_err(PSTF_E_INVALID, "store listed twice");
    }
    CK(cudaSetDevice(fs[0]->device));
    twin_batch(fs, n); /* twins are end-framed together or not at all */
    cudaStream_t st = (cudaStream_t)stream;
    /* a deferred vertex pass of these stores on this stream: enqueue endFrame guarded by its
     * device-side pending count, then look at the count; other deferred passes settle first */
    pstf_field *owner = nullptr;
    for (int i = 0; i < n; ++i) {
        pstf_field *o = fs[i]->owed_by;
        if (o && o->dp.active && o->dp.st == st && (!owner || owner == o)) owner = o;
        else SETTLE(fs[i]);
    }
    Stores4 S = stores4(fs, n);
    uint64_t maxcap = 0;
    for (int i = 0; i < n; ++i) maxcap = std::max<uint64_t>(maxcap, (uint64_t)fs[i]->d.mask + 1);
    const unsigned g = std::min<unsigned>(grid_for(maxcap, EF_BLOCK), (unsigned)sm_count() * 8);
    const unsigned long long *guard =
        owner ? owner->sc.pend_count.as<const unsigned long long>() : nullptr;
    static int fused_blocks = -1; /* co-resident blocks per SM of the cooperative kernel */
    if (fused_blocks < 0) {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fused_blocks, k_ef_fused, EF_BLOCK, 0));
        if (getenv("PSTF_NO_FUSED_EF")) fused_blocks = 0;
    }
    static const bool no_onepass = getenv("PSTF_NO_ONEPASS_EF") != nullptr;
    bool unit = !no_onepass;
    for (int i = 0; i < n; ++i) unit = unit && fs[i]->unit_frame;
    /* the Lo store of this frame's tiled vertex pass: the tail reports its RED density */
    int rd_lo = -1;
    unsigned long long *rd_dev = nullptr;
    for (int i = 0; i < n && rd_lo < 0; ++i)
        if (fs[i]->rd_probe && unit) {
            pstf_field *f = fs[i];
            if (!f->rd_host) {
                CK(cudaHostAlloc(&f->rd_host, 16, cudaHostAllocMapped));
                f->rd_host[0] = f->rd_host[1] = 0;
            }
            if (!f->rd_ev) CK(cudaEventCreateWithFlags(&f->rd_ev, cudaEventDisableTiming));
            CK(cudaHostGetDevicePointer((void **)&rd_dev, f->rd_host, 0));
            rd_lo = i;
        }
    auto launch = [&](const unsigned long long *gd) -> int {
        if (unit) { /* counted frame: one pass over the touched slots, then the tail */
            Scratch &sc0 = fs[0]->sc;
            if (!sc0.ef_done.p) {
                ENSURE(sc0.ef_done, 4);
                CK(cudaMemsetAsync(sc0.ef_done.p, 0, 4, st));
            }
            LAUNCH(k_ef_onepass, g, EF_BLOCK, 0, st, S, n, gd);
            /* one block per SM: the deferred list is short, eviction rarely runs */
            LAUNCH(k_ef_tail, std::min<unsigned>(g, (unsigned)sm_count()), EF_BLOCK, 0, st, S, n, gd,
                   sc0.ef_done.as<unsigned int>(), rd_lo, rd_dev);
            return PSTF_OK;
        }
        for (int i = 0; i < n; ++i) { /* Σc_new in slot order, inexact frames only */
            if (!fs[i]->counted_apply) continue; /* no counter weight but vertex passes' 1 */
            Scratch &sc = fs[i]->sc;
            const uint64_t nw = ((uint64_t)fs[i]->d.mask + 32) / 32;
            ENSURE(sc.cn_cnt, nw * 8);
            ENSURE(sc.cn_vals, ((uint64_t)fs[i]->d.mask + 1) * 8);
            uint32_t *cnt = sc.cn_cnt.as<uint32_t>(), *pos = cnt + nw;
            LAUNCH(k_cn_words, grid_for(nw, 256), 256, 0, st, fs[i]->d, gd, cnt);
            size_t bytes = 0;
            CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt, pos, (int64_t)nw, st));
            ENSURE(sc.cub, bytes);
            bytes = sc.cub.bytes;
            {
                ProfScope ps_("cub::DeviceScan", st);
                CK(cub::DeviceScan::ExclusiveSum(sc.cub.p, bytes, cnt, pos, (int64_t)nw, st));
                g_launches.fetch_add(2, std::memory_order_relaxed);
            }
            LAUNCH(k_cn_scatter, grid_for(nw, 256), 256, 0, st, fs[i]->d, gd, pos,
                   sc.cn_vals.as<double>());
            LAUNCH(k_cn_seq, 1, 1, 0, st, fs[i]->d, gd, pos, cnt, sc.cn_vals.as<double>());
        }
        if (fused_blocks > 0) { /* one cooperative launch: reduce | blend | evict */
            unsigned gf = std::min<unsigned>(g, (unsigned)(sm_count() * fused_blocks));
            int nn = n;
            void *args[] = {&S, &nn, &gd};
            ProfScope ps_("k_ef_fused", st);
            CK(cudaLaunchCooperativeKernel((const void *)k_ef_fused, gf, EF_BLOCK, args, 0, st));
            g_launches.fetch_add(1, std::memory_order_relaxed);
            return PSTF_OK;
        }
        LAUNCH(k_ef_reduce, g, EF_BLOCK, 0, st, S, n, gd);
        LAUNCH(k_ef_blend, g, EF_BLOCK, 0, st, S, n, gd);
        LAUNCH(k_ef_evict, g, EF_BLOCK, 0, st, S, n, 1, gd); /* + the per-frame scratch roll */
        return PSTF_OK;
    };
    int rc = launch(guard);
    if (rc) return rc;
    if (owner) {
        CK(cudaEventSynchronize(owner->dp.ev));
        if (*owner->dp.h_count) { /* the guarded sweeps did nothing: place, then sweep */
            SETTLE(owner);
            rc = launch(nullptr);
            if (rc) return rc;
        } else {
            SETTLE(owner); /* nothing pending: just retire the deferred pass */
        }
    }
    if (rd_lo >= 0) { /* the density is readable once this event completes */
        CK(cudaEventRecord(fs[rd_lo]->rd_ev, st));
        fs[rd_lo]->rd_pending = true;
    }
    for (int i = 0; i < n; ++i) fs[i]->rd_probe = false;
    for (int i = 0; i < n; ++i) {
        fs[i]->frame += 1;
        fs[i]->unit_frame = true;
        fs[i]->counted_apply = false;
    }
    return PSTF_OK;
}

int pstf_field_end_frame(pstf_field *f, void *stream) {
    if (!f) return set_err(PSTF_E_INVALID, "NULL argument");
    return pstf_fields_end_frame(&f, 1, stream);
}

int pstf_field_invalidate(pstf_field *f, const double *aabb, void *stream) {
    if (!f) return set_err(PSTF_E_INVALID, "NULL argument");
    twin_break(f);
    CK(cudaSetDevice(f->device));
    SETTLE(f);
    const uint64_t cap = (uint64_t)f->d.mask + 1;
    unsigned g = std::min<unsigned>(grid_for(cap, 256), (unsigned)sm_count() * 8);
    if (aabb)
        LAUNCH(k_invalidate, g, 256, 0, (cudaStream_t)stream, f->d, 1, aabb[0], aabb[1], aabb[2],
               aabb[3], aabb[4], aabb[5]);
    else
        LAUNCH(k_invalidate, g, 256, 0, (cudaStream_t)stream, f->d, 0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0);
    return PSTF_OK;
}

int pstf_field_get_stats(pstf_field *f, pstf_field_stats *out) {
    if (!f || !out) return set_err(PSTF_E_INVALID, "NULL argument");
    CK(cudaSetDevice(f->device));
    SETTLE(f);
    CK(cudaDeviceSynchronize());
    unsigned long long c[C_NUM];
    CK(cudaMemcpy(c, f->d.ctr, sizeof(c), cudaMemcpyDeviceToHost));
    out->frame = f->frame;
    out->rejected = c[C_REJECTED];
    out->dropped = c[C_DROPPED];
    out->internal_errors = c[C_INTERNAL];
    out->live = c[C_LIVE];
    out->touched_last = c[C_TOUCHED_LAST];
    out->new_keys_last = c[C_NEW_KEYS];
    out->evicted_last = c[C_EVICTED];
    out->placement_rounds_last = c[C_ROUNDS];
    out->touched_total = c[C_TOUCHED_TOTAL];
    out->reds_total = c[C_REDS];
    return PSTF_OK;
}

__global__ void k_probe_hist(DevStore s, unsigned long long *hist) {
    __shared__ unsigned h[33];
    for (int i = threadIdx.x; i < 33; i += blockDim.x) h[i] = 0u;
    __syncthreads();
    const uint64_t cap = (uint64_t)s.mask + 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (s.meta[i].x == 0u) continue;
        const KeyFields k = s.keyf[i];
        const uint32_t home = (uint32_t)pack_key_fields(k.level, k.c0, k.c1, k.c2, k.d0, k.d1) &
                              s.mask;
        const uint32_t d = ((uint32_t)i - home) & s.mask;
        atomicAdd(&h[d < 32u ? d : 32u], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 33; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], (unsigned long long)h[i]);
}

int pstf_field_probe_histogram(pstf_field *f, uint64_t hist[33]) {
    if (!f || !hist) return set_err(PSTF_E_INVALID, "NULL argument");
    CK(cudaSetDevice(f->device));
    SETTLE(f);
    Scratch &sc = f->sc;
    ENSURE(sc.ranges, 33 * 8);
    CK(cudaMemset(sc.ranges.p, 0, 33 * 8));
    const uint64_t cap = (uint64_t)f->d.mask + 1;
    unsigned g = std::min<unsigned>(grid_for(cap, 256), (unsigned)sm_count() * 8);
    LAUNCH(k_probe_hist, g, 256, 0, (cudaStream_t)0, f->d, sc.ranges.as<unsigned long long>());
    CK(cudaMemcpy(hist, sc.ranges.p, 33 * 8, cudaMemcpyDeviceToHost));
    return PSTF_OK;
}

/* RED peak: lane -> cell 8k + lane/4 (k = instruction), component lane%4, cells spread over an
 * L2-resident array so the updates of one instruction hit 8 distinct sectors */
__global__ void k_red_peak(double4 *cells, uint32_t mask, int iters) {
    const unsigned lane = threadIdx.x & 31u;
    uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int it = 0; it < iters; ++it) {
        h = h * 1664525u + 1013904223u; /* per-warp LCG: warp-uniform */
        const uint32_t cell = ((h >> 8) * 8u + (lane >> 2)) & mask;
        atomicAdd(reinterpret_cast<double *>(&cells[cell]) + (lane & 3u), 1.0);
    }
}

int pstf_diag_red_peak(int device, double *ops_per_second) {
    if (!ops_per_second) return set_err(PSTF_E_INVALID, "NULL argument");
    CK(cudaSetDevice(device));
    const uint32_t ncell = 1u << 21; /* 64 MiB of double4: L2-resident (126 MB L2) */
    double4 *cells = nullptr;
    CK(cudaMalloc(&cells, (size_t)ncell * sizeof(double4)));
    CK(cudaMemset(cells, 0, (size_t)ncell * sizeof(double4)));
    const unsigned grid = (unsigned)sm_count() * 8, block = 256;
    const int iters = 256;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    k_red_peak<<<grid, block>>>(cells, ncell - 1, iters); /* warm-up */
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 4; ++r) k_red_peak<<<grid, block>>>(cells, ncell - 1, iters);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    *ops_per_second = 4.0 * grid * block * (double)iters / (ms * 1e-3);
    CK(cudaEventDestroy(e0));
    CK(cudaEventDestroy(e1));
    CK(cudaFree(cells));
    return PSTF_OK;
}

int pstf_field_weighted_mean(pstf_field *f, double out[3]) {
    if (!f || !out) return set_err(PSTF_E_INVALID, "NULL argument");
    CK(cudaSetDevice(f->device));
    SETTLE(f);
    Scratch &sc = f->sc;
    ENSURE(sc.ranges, 64);
    CK(cudaMemset(sc.ranges.p, 0, 32));
    const uint64_t cap = (uint64_t)f->d.mask + 1;
    unsigned g = std::min<unsigned>(grid_for(cap, 256), (unsigned)sm_count() * 8);
    LAUNCH(k_weighted_mean, g, 256, 0, (cudaStream_t)0, f->d, sc.ranges.as<double>());
    double h[4];
    CK(cudaMemcpy(h, sc.ranges.p, 32, cudaMemcpyDeviceToHost));
    for (int c = 0; c < 3; ++c) out[c] = h[3] > 0.0 ? h[c] / h[3] : 0.0;
    return PSTF_OK;
}

static int snapshot_device(pstf_field *f, uint64_t *count, pstf_snapshot_record **dev_sorted) {
    Scratch &sc = f->sc;
    const uint64_t cap = (uint64_t)f->d.mask + 1;
    CK(cudaDeviceSynchronize());
    unsigned long long live = 0;
    CK(cudaMemcpy(&live, &f->d.ctr[C_LIVE], 8, cudaMemcpyDeviceToHost));
    ENSURE(sc.snap, (live + 1) * 2 * sizeof(pstf_snapshot_record));
    ENSURE(sc.pend_count, 8);
    CK(cudaMemset(sc.pend_count.p, 0, 8));
    pstf_snapshot_record *tmp = sc.snap.as<pstf_snapshot_record>();
    pstf_snapshot_record *sorted = tmp + (live + 1);
    LAUNCH(k_snap_gather, grid_for(cap, 256), 256, 0, (cudaStream_t)0, f->d, tmp,
           sc.pend_count.as<unsigned long long>());
    unsigned long long n = 0;
    CK(cudaMemcpy(&n, sc.pend_count.p, 8, cudaMemcpyDeviceToHost));
    if (n != live) return set_err(PSTF_E_CUDA, "live counter disagrees with the table");
    if (n) {
        ENSURE(sc.words, n * 3 * 8);
        LAUNCH(k_snap_words, grid_for(n, 256), 256, 0, (cudaStream_t)0, tmp, n,
               sc.words.as<uint64_t>());
        int bb[3] = {0, 0, 0};
        uint32_t *perm = nullptr;
        int rc = sort_multiword(sc, sc.words.as<uint64_t>(), bb, 3, n, &perm, 0);
        if (rc) return rc;
        LAUNCH(k_snap_permute, grid_for(n, 256), 256, 0, (cudaStream_t)0, tmp, perm, n, sorted);
    }
    *count = n;
    *dev_sorted = sorted;
    return PSTF_OK;
}

int pstf_field_snapshot(pstf_field *f, pstf_snapshot_record *records, uint64_t cap,
                        uint64_t *count) {
    if (!f || !count || (cap && !records)) return set_err(PSTF_E_INVALID, "NULL argument");
    CK(cudaSetDevice(f->device));
    SETTLE(f);
    uint64_t n = 0;
    pstf_snapshot_record *d = nullptr;
    int rc = snapshot_device(f, &n, &d);
    if (rc) return rc;
    *count = n;
    uint64_t m = std::min(n, cap);
    if (m) CK(cudaMemcpy(records, d, m * sizeof(pstf_snapshot_record), cudaMemcpyDeviceToHost));
    return PSTF_OK;
}

int pstf_field_dump_snapshot(pstf_field *f, const char *path) {
    if (!f || !path) return set_err(PSTF_E_INVALID, "NULL argument");
    CK(cudaSetDevice(f->device));
    SETTLE(f);
    uint64_t n = 0;
    pstf_snapshot_record *d = nullptr;
    int rc = snapshot_device(f, &n, &d);
    if (rc) return rc;
    std::vector<pstf_snapshot_record> h(n);
    if (n) CK(cudaMemcpy(h.data(), d, n * sizeof(pstf_snapshot_record), cudaMemcpyDeviceToHost));
    FILE *fp = fopen(path, "wb");
    if (!fp) /* field.cpp:340-341 */
        return set_err(PSTF_E_IO, std::string("cannot open snapshot file '") + path + "' for writing");
    const char magic[8] = {'P', 'S', 'T', 'F', 'S', 'N', 'A', 'P'};
    uint32_t version = 1, kind = f->cfg.kind;
    uint64_t cnt = n;
    bool ok = fwrite(magic, 1, 8, fp) == 8 && fwrite(&version, 4, 1, fp) == 1 &&
              fwrite(&kind, 4, 1, fp) == 1 && fwrite(&cnt, 8, 1, fp) == 1;
    for (uint64_t i = 0; ok && i < n; ++i) { /* 60-byte packed records, field.cpp:348-355 */
        const pstf_snapshot_record &r = h[i];
        ok = fwrite(&r.level, 4, 1, fp) == 1 && fwrite(r.cell, 4, 3, fp) == 3 &&
             fwrite(r.dir_cell, 4, 2, fp) == 2 && fwrite(&r.checksum, 4, 1, fp) == 1 &&
             fwrite(r.value, 8, 3, fp) == 3 && fwrite(&r.c_old, 8, 1, fp) == 1;
    }
    if (fclose(fp) != 0) ok = false;
    if (!ok) return set_err(PSTF_E_IO, std::string("write failed: ") + path);
    return PSTF_OK;
}

int pstf_read_snapshot(const char *path, pstf_snapshot_record *records, uint64_t cap,
                       uint64_t *count, uint32_t *kind_out) {
    if (!path || !count) return set_err(PSTF_E_INVALID, "NULL argument");
    FILE *fp = fopen(path, "rb");
    if (!fp) return set_err(PSTF_E_IO, std::string("cannot open snapshot file '") + path + "'");
    char magic[8];
    uint32_t version = 0, kind = 0;
    uint64_t n = 0;
    if (fread(magic, 1, 8, fp) != 8 || memcmp(magic, "PSTFSNAP", 8) != 0) {
        fclose(fp);
        return set_err(PSTF_E_FORMAT, std::string("'") + path + "': not a field snapshot");
    }
    if (fread(&version, 4, 1, fp) != 1 || fread(&kind, 4, 1, fp) != 1 || fread(&n, 8, 1, fp) != 1) {
        fclose(fp);
        return set_err(PSTF_E_FORMAT, std::string("'") + path + "': truncated snapshot");
    }
    if (version != 1) {
        fclose(fp);
        return set_err(PSTF_E_FORMAT, std::string("'") + path + "': unsupported snapshot version");
    }
    bool ok = true;
    for (uint64_t i = 0; i < n; ++i) {
        pstf_snapshot_record r;
        memset(&r, 0, sizeof(r));
        ok = fread(&r.level, 4, 1, fp) == 1 && fread(r.cell, 4, 3, fp) == 3 &&
             fread(r.dir_cell, 4, 2, fp) == 2 && fread(&r.checksum, 4, 1, fp) == 1 &&
             fread(r.value, 8, 3, fp) == 3 && fread(&r.c_old, 8, 1, fp) == 1;
        if (!ok) break;
        if (i < cap && records) records[i] = r;
    }
    fclose(fp);
    if (!ok) return set_err(PSTF_E_FORMAT, std::string("'") + path + "': truncated snapshot");
    *count = n;
    if (kind_out) *kind_out = kind;
    return PSTF_OK;
}

/* ---- snapshot restore (the reference writes snapshots but has no restore) */

__device__ __forceinline__ uint32_t snap_home(const pstf_snapshot_record &q, uint32_t mask) {
    return (uint32_t)pack_key_fields(q.level, q.cell[0], q.cell[1], q.cell[2], q.dir_cell[0],
                                     q.dir_cell[1]) & mask;
}

/* record i -> a zero-weight counter update of its key: phase 2 (ORDERED) then inserts the keys
 * exactly as findOrInsertSlot in ascending key order would (field.cpp:116-146, 402-419) */
__global__ void k_restore_records(const pstf_snapshot_record *r, uint64_t n, PendRec *pend) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const pstf_snapshot_record q = r[i];
    Key k;
    k.level = q.level;
    k.cell[0] = q.cell[0];
    k.cell[1] = q.cell[1];
    k.cell[2] = q.cell[2];
    k.dir[0] = q.dir_cell[0];
    k.dir[1] = q.dir_cell[1];
    k.checksum = q.checksum;
    put_record(&pend[i], k, PSTF_META(0, 1, 1), 0.0, 0.0, 0.0, 0.0);
}

/* the slot a record's key resolves to after the inserts (findSlot, field.cpp:103-114; no slot
 * empties during a restore, so it is the slot findOrInsertSlot returned); the last record in
 * key order that resolves to a slot owns its committed value */
__global__ void k_restore_claim(DevStore s, const pstf_snapshot_record *r, uint64_t n,
                                uint32_t *winner) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int slot = probe_find(s, snap_home(r[i], s.mask), r[i].checksum);
    if (slot >= 0) atomicMax(&winner[slot], (uint32_t)i + 1u);
}

__global__ void k_restore_write(DevStore s, const pstf_snapshot_record *r, uint64_t n,
                                const uint32_t *winner) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const pstf_snapshot_record q = r[i];
    const int slot = probe_find(s, snap_home(q, s.mask), q.checksum);
    if (slot >= 0 && winner[slot] == (uint32_t)i + 1u)
        *com_ptr(s, slot) = make_double4(q.value[0], q.value[1], q.value[2], q.c_old);
}

static bool snap_key_less(const pstf_snapshot_record &a, const pstf_snapshot_record &b) {
    const int32_t ka[6] = {a.level, a.cell[0], a.cell[1], a.cell[2], a.dir_cell[0], a.dir_cell[1]};
    const int32_t kb[6] = {b.level, b.cell[0], b.cell[1], b.cell[2], b.dir_cell[0], b.dir_cell[1]};
    return std::lexicographical_compare(ka, ka + 6, kb, kb + 6); /* field.cpp:334-337 */
}

extern "C" int pstf_field_restore(pstf_field *f, const pstf_snapshot_record *records, uint64_t n) {
    if (f) f->unit_frame = false; /* arbitrary weights: endFrame's reduce pass */
    twin_break(f);
    if (!f || (n && !records)) return set_err(PSTF_E_INVALID, "NULL argument");
    if (n >= 0xffffffffULL) return set_err(PSTF_E_INVALID, "too many records");
    for (uint64_t i = 0; i < n; ++i) { /* keyFor's checksum (field.cpp:98-99) */
        const pstf_snapshot_record &q = records[i];
        const uint32_t cs = checksum_of(pack_key_fields(q.level, q.cell[0], q.cell[1], q.cell[2],
                                                        q.dir_cell[0], q.dir_cell[1]));
        if (cs != q.checksum)
            return set_err(PSTF_E_FORMAT, "snapshot record " + std::to_string(i) +
                                              ": checksum does not match its key");
    }
    CK(cudaSetDevice(f->device));
    SETTLE(f);
    if (!n) return PSTF_OK;
    /* ascending key order, stable (snapshots are written sorted: usually nothing to do) */
    std::vector<pstf_snapshot_record> sorted;
    const pstf_snapshot_record *src = records;
    if (!std::is_sorted(records, records + n, snap_key_less)) {
        sorted.assign(records, records + n);
        std::stable_sort(sorted.begin(), sorted.end(), snap_key_less);
        src = sorted.data();
    }
    Scratch &sc = f->sc;
    const cudaStream_t st = 0;
    const uint64_t cap = (uint64_t)f->d.mask + 1;
    ENSURE(sc.snap, n * sizeof(pstf_snapshot_record));
    ENSURE(sc.winner, cap * 4);
    pstf_snapshot_record *d = sc.snap.as<pstf_snapshot_record>();
    CK(cudaMemcpy(d, src, n * sizeof(pstf_snapshot_record), cudaMemcpyHostToDevice));
    int rc = ensure_pending(sc, n, false, st);
    if (rc) return rc;
    LAUNCH(k_restore_records, grid_for(n, 256), 256, 0, st, d, n, sc.pend.as<PendRec>());
    const unsigned long long cnt = n;
    CK(cudaMemcpyAsync(sc.pend_count.p, &cnt, 8, cudaMemcpyHostToDevice, st));
    pstf_field *fs[1] = {f};
    rc = resolve_pending(sc, fs, 1, PSTF_MODE_ORDERED, n, st);
    if (rc) return rc;
    const DevStore ds = dev_view(f);
    CK(cudaMemsetAsync(sc.winner.p, 0, cap * 4, st));
    LAUNCH(k_restore_claim, grid_for(n, 256), 256, 0, st, ds, d, n, sc.winner.as<uint32_t>());
    LAUNCH(k_restore_write, grid_for(n, 256), 256, 0, st, ds, d, n, sc.winner.as<uint32_t>());
    CK(cudaStreamSynchronize(st));
    return PSTF_OK;
}

extern "C" int pstf_field_load_snapshot(pstf_field *f, const char *path) {
    if (!f || !path) return set_err(PSTF_E_INVALID, "NULL argument");
    uint64_t n = 0;
    uint32_t kind = 0;
    int rc = pstf_read_snapshot(path, nullptr, 0, &n, &kind);
    if (rc) return rc;
    if (kind != f->cfg.kind)
        return set_err(PSTF_E_FORMAT, std::string("'") + path + "': snapshot of field kind " +
                                          std::to_string(kind) + ", store is kind " +
                                          std::to_string(f->cfg.kind));
    std::vector<pstf_snapshot_record> h(n);
    rc = pstf_read_snapshot(path, h.data(), n, &n, nullptr);
    if (rc) return rc;
    return pstf_field_restore(f, h.data(), n);
}

int pstf_field_slots(pstf_field *f, uint64_t begin, uint64_t count, pstf_slot_record *out) {
    if (!f || (count && !out)) return set_err(PSTF_E_INVALID, "NULL argument");
    const uint64_t cap = (uint64_t)f->d.mask + 1;
    if (begin > cap || count > cap - begin) return set_err(PSTF_E_INVALID, "slot range out of bounds");
    if (!count) return PSTF_OK;
    CK(cudaSetDevice(f->device));
    SETTLE(f);
    CK(cudaDeviceSynchronize());
    std::vector<uint2> meta(count);
    std::vector<double4> com(count), acc(count);
    std::vector<KeyFields> kf(count);
    CK(cudaMemcpy(meta.data(), f->d.meta + begin, count * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(com.data(), f->d.com + begin, count * 32, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(acc.data(), f->d.acc + begin, count * 32, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(kf.data(), f->d.keyf + begin, count * sizeof(KeyFields), cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < count; ++i) {
        pstf_slot_record &r = out[i];
        memset(&r, 0, sizeof(r));
        r.checksum = meta[i].x;
        r.level = kf[i].level;
        r.cell[0] = kf[i].c0;
        r.cell[1] = kf[i].c1;
        r.cell[2] = kf[i].c2;
        r.dir_cell[0] = kf[i].d0;
        r.dir_cell[1] = kf[i].d1;
        r.value_old[0] = com[i].x;
        r.value_old[1] = com[i].y;
        r.value_old[2] = com[i].z;
        r.c_old = com[i].w;
        r.accum[0] = acc[i].x;
        r.accum[1] = acc[i].y;
        r.accum[2] = acc[i].z;
        r.c_new = acc[i].w;
        r.last_touched = meta[i].y == 0 ? 0u : meta[i].y - 1u; /* stored biased by +1 */
    }
    return PSTF_OK;
}

__global__ void k_checksums(const uint2 *meta, uint64_t n, uint32_t *out) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = meta[i].x;
}

int pstf_field_committed_host(pstf_field *f, uint32_t *checksum, double *com4) {
    if (!f || !checksum || !com4) return set_err(PSTF_E_INVALID, "NULL argument");
    CK(cudaSetDevice(f->device));
    SETTLE(f);
    std::lock_guard<std::mutex> lk(f->host_mu);
    const uint64_t cap = (uint64_t)f->d.mask + 1;
    Scratch &sc = f->sc;
    ENSURE(sc.hio, cap * 4);
    LAUNCH(k_checksums, grid_for(cap, 256), 256, 0, (cudaStream_t)0, f->d.meta, cap,
           sc.hio.as<uint32_t>());
    CK(cudaMemcpy(checksum, sc.hio.p, cap * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(com4, f->d.com, cap * 32, cudaMemcpyDeviceToHost));
    return PSTF_OK;
}

struct CvOut { /* fused CV-lookup outputs (pstf_vertex_pass_cv) */
    double *r, *g, *b;
    uint8_t *valid;
};

static int vertex_phase1(pstf_field *lo, pstf_field *loe, pstf_field *fli, pstf_field *li,
                         const pstf_vertex_soa *v, uint64_t n, uint32_t loe_mask,
                         uint32_t fli_mask, int mode, cudaStream_t st,
                         const CvOut *cv = nullptr) {
    const bool twin = twin_for_pass(lo, loe, fli, li);
    VPArgs a;
    memset(&a, 0, sizeof(a));
    pstf_field *fs[4] = {lo, loe, fli, li};
    a.st = stores4(fs, 4);
    a.has_li = li != nullptr;
    a.same_lo_loe = same_quant(lo->cfg, loe->cfg);
    a.same_fli_lo = same_quant(fli->cfg, lo->cfg);
    a.same_li_fli = li ? same_quant(li->cfg, fli->cfg) : 1;
    a.loe_mask = loe_mask;
    a.fli_mask = fli_mask;
    a.v = *v;
    a.n = n;
    a.pend = lo->sc.pend.as<PendRec>();
    a.pend_count = lo->sc.pend_count.as<unsigned long long>();
    a.pend_cap = lo->sc.pend.bytes / sizeof(PendRec);
    if (mode == PSTF_MODE_ORDERED) {
        a.pend2_key = lo->sc.pend2_key.as<uint64_t>();
        a.pend2_val = lo->sc.pend2_val.as<double4>();
        a.pend2_count = lo->sc.pend2_count.as<unsigned long long>();
        a.pend2_cap = std::min(lo->sc.pend2_key.bytes / 8, lo->sc.pend2_val.bytes / 32);
        int capl = 0;
        for (int i = 0; i < 4; ++i)
            if (fs[i]) capl = std::max<int>(capl, (int)fs[i]->cfg.capacity_log2);
        a.pend2_capl = capl;
    }
    const bool shared_quant = a.same_lo_loe && a.same_fli_lo && a.same_li_fli;
    /* TMA path: every SoA segment must be 16 B aligned for cp.async.bulk */
    const void *ptrs[35] = {v->position.x, v->position.y, v->position.z, v->wo.x, v->wo.y,
                            v->wo.z, v->wi.x, v->wi.y, v->wi.z, v->next_position.x,
                            v->next_position.y, v->next_position.z, v->nee_dir.x, v->nee_dir.y,
                            v->nee_dir.z, v->footprint, v->next_footprint, v->ratio,
                            v->next_emis_mis_weight, v->emission_here.x, v->emission_here.y,
                            v->emission_here.z, v->f.x, v->f.y, v->f.z, v->next_emission.x,
                            v->next_emission.y, v->next_emission.z, v->nee_loe.x, v->nee_loe.y,
                            v->nee_loe.z, v->nee_fli.x, v->nee_fli.y, v->nee_fli.z, v->flags};
    bool aligned = true;
    for (int k = 0; k < 35; ++k) aligned = aligned && ((uintptr_t)ptrs[k] % 16 == 0);
    const bool ord_tiled = mode == PSTF_MODE_ORDERED && !cv && !getenv("PSTF_ORDERED_PERTHREAD");
    if ((mode == PSTF_MODE_ATOMIC || ord_tiled) && shared_quant && aligned &&
        !getenv("PSTF_NO_TMA")) {
        VPArgs2 b;
        memset(&b, 0, sizeof(b));
        b.st = a.st;
        b.fp = make_fast_params(lo->d.kp);
        b.pf = getenv("PSTF_VP_PF") ? std::max(0, atoi(getenv("PSTF_VP_PF"))) : 1;
        b.has_li = a.has_li;
        b.loe_mask = loe_mask;
        b.fli_mask = fli_mask;
        for (int k = 0; k < PS_NUM_F64; ++k) b.fld[k] = (const double *)ptrs[k];
        b.flags = v->flags;
        b.n = n;
        b.pend = a.pend;
        b.pend_count = a.pend_count;
        b.pend_cap = a.pend_cap;
        /* (stages, CTAs/SM): 1x4 (cfg 1, default, 0.84 ms) measured fastest on config 2; 2x3
         * (cfg 0, double buffering), 1x5 (cfg 2, 93 registers, no spills: 0.95 ms) and 1x3
         * (cfg 3: 0.97 ms) are slower (fewer warps, or less L1 next to the stages), as were
         * VT = 64 / 96,
         * L2-prefetch-only loads without staging, refilling the stage before the
         * contributions (mid-tile barrier, or last-warp refill without one), and two stage
         * groups refilled at different points of the tile. */
        const char *cfgs = getenv("PSTF_TILED_CFG");
        const int cfg = cfgs ? std::min(std::max(atoi(cfgs), 0), 3) : 1;
        const uint64_t tiles = (n + VT - 1) / VT;
        /* one 2-D tensor map over the 34 f64 fields when they sit at a uniform stride */
        CUtensorMap tm;
        memset(&tm, 0, sizeof(tm));
        bool tmap = false;
        if (cfg >= 1 && !getenv("PSTF_NO_TMAP")) {
            const long long stride = (const char *)ptrs[1] - (const char *)ptrs[0];
            bool uniform = stride > 0 && stride % 16 == 0 && (uint64_t)stride >= n * 8 &&
                           n < (1ull << 31);
            for (int k = 2; k < PS_NUM_F64 && uniform; ++k)
                uniform = (const char *)ptrs[k] - (const char *)ptrs[0] == k * stride;
            PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
            if (uniform && enc) {
                const cuuint64_t gdim[2] = {(cuuint64_t)n, (cuuint64_t)PS_NUM_F64};
                const cuuint64_t gstride[1] = {(cuuint64_t)stride};
                const cuuint32_t box[2] = {VT, PS_NUM_F64};
                const cuuint32_t es[2] = {1, 1};
                tmap = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void *>(ptrs[0]),
                           gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
            }
        }
        if (mode == PSTF_MODE_ORDERED) { /* the default tiled kernel, ORDERED instantiation */
            if (!tmap || cfg != 1) goto per_thread;
            b.pend2_key = a.pend2_key;
            b.pend2_val = a.pend2_val;
            b.pend2_count = a.pend2_count;
            b.pend2_cap = a.pend2_cap;
            b.pend2_capl = a.pend2_capl;
            for (pstf_field *f : fs)
                if (f) f->unit_frame = false; /* counters are not counted (k_ef_onepass) */
            const size_t smem1 = sizeof(TileStage) + 64;
            const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)sm_count() * VT_MINB);
            const uint32_t used = PSTF_TECH_CONTINUATION | PSTF_TECH_NEE;
            if (twin && !li && (loe_mask & used) == used && (fli_mask & used) == used) {
                SMEM_ATTR((k_vertex_pass_tiled<1, VT_MINB, true, false, true, false, true>), smem1);
                LAUNCH((k_vertex_pass_tiled<1, VT_MINB, true, false, true, false, true>), grid, VT,
                       smem1, st, b, tm);
                return PSTF_OK;
            }
            SMEM_ATTR((k_vertex_pass_tiled<1, VT_MINB, true, false, true>), smem1);
            LAUNCH((k_vertex_pass_tiled<1, VT_MINB, true, false, true>), grid, VT, smem1, st, b, tm);
            return PSTF_OK;
        }
        const int stages = cfg == 0 ? 2 : 1;
        const int minb = cfg == 0 ? 3 : cfg == 1 ? VT_MINB : cfg == 2 ? 5 : 3;
        const size_t smem = stages * sizeof(TileStage) + 64;
        const bool cvf = cv && cfg == 1; /* the CV lookup fused into the default kernel */
        if (cv && !cvf)
            LAUNCH(k_cv_lookup, grid_for(n, 256), 256, 0, st, loe->d, *v, n, cv->r, cv->g, cv->b,
                   cv->valid);
        if (cvf) {
            b.cv[0] = cv->r;
            b.cv[1] = cv->g;
            b.cv[2] = cv->b;
            b.cv_valid = cv->valid;
        }
        const int fi = cfg == 0 ? 0 : cfg == 2 ? (tmap ? 6 : 1) : cfg == 3 ? 7
                     : (tmap ? 3 : 2) + (cvf ? 2 : 0);
        const uint32_t used = PSTF_TECH_CONTINUATION | PSTF_TECH_NEE; /* the bits onVertex reads */
        const bool all_tech = (loe_mask & used) == used && (fli_mask & used) == used;
        if (fi == 5 && twin && !li && all_tech) { /* fused CV lookup, Lo\E probes from Lo's */
            SMEM_ATTR((k_vertex_pass_tiled<1, VT_MINB, true, true, false, false, true>), smem);
            const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)sm_count() * minb);
            LAUNCH((k_vertex_pass_tiled<1, VT_MINB, true, true, false, false, true>), grid, VT, smem,
                   st, b, tm);
            return PSTF_OK;
        }
        if (fi == 3) { /* hot slots: the warp-aggregating instantiation (RED density > 1000) */
            bool agg = lo->agg;
            if (lo->rd_pending && cudaEventQuery(lo->rd_ev) == cudaSuccess) {
                const volatile unsigned long long *h = lo->rd_host;
                const unsigned long long reds = h[0], touched = h[1]; /* of one frame */
                if (touched) agg = (double)reds / (double)touched > 1000.0;
                lo->rd_pending = false;
                lo->agg = agg;
            }
            if (const char *e = getenv("PSTF_RED_AGG")) agg = atoi(e) != 0; /* force on / off */
            /* measured on the first frames (the first one inserts: few REDs), then every 4th */
            lo->rd_probe = lo->frame < 4 || (lo->frame & 3) == 0;
            if (agg) {
                SMEM_ATTR((k_vertex_pass_tiled<1, VT_MINB, true, false, false, true>), smem);
                const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)sm_count() * minb);
                LAUNCH((k_vertex_pass_tiled<1, VT_MINB, true, false, false, true>), grid, VT, smem, st,
                       b, tm);
                return PSTF_OK;
            }
            if (twin && !li && all_tech) { /* Lo\E's probes from Lo's (pstf_field::twin) */
                SMEM_ATTR((k_vertex_pass_tiled<1, VT_MINB, true, false, false, false, true>), smem);
                const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)sm_count() * minb);
                LAUNCH((k_vertex_pass_tiled<1, VT_MINB, true, false, false, false, true>), grid, VT,
                       smem, st, b, tm);
                return PSTF_OK;
            }
        }
        {
            const void *fns[8] = {(const void *)k_vertex_pass_tiled<2, 3, false>,
                                  (const void *)k_vertex_pass_tiled<1, 5, false>,
                                  (const void *)k_vertex_pass_tiled<1, VT_MINB, false>,
                                  (const void *)k_vertex_pass_tiled<1, VT_MINB, true>,
                                  (const void *)k_vertex_pass_tiled<1, VT_MINB, false, true>,
                                  (const void *)k_vertex_pass_tiled<1, VT_MINB, true, true>,
                                  (const void *)k_vertex_pass_tiled<1, 5, true>,
                                  (const void *)k_vertex_pass_tiled<1, 3, true>};
            SMEM_ATTR(fns[fi], smem);
            if (getenv("PSTF_CARVEOUT")) /* experiment: the L1 / shared-memory split */
                CK(cudaFuncSetAttribute(fns[fi], cudaFuncAttributePreferredSharedMemoryCarveout,
                                        atoi(getenv("PSTF_CARVEOUT"))));
        }
        const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)sm_count() * minb);
        switch (fi) {
        case 0: LAUNCH((k_vertex_pass_tiled<2, 3, false>), grid, VT, smem, st, b, tm); break;
        case 1: LAUNCH((k_vertex_pass_tiled<1, 5, false>), grid, VT, smem, st, b, tm); break;
        case 2: LAUNCH((k_vertex_pass_tiled<1, VT_MINB, false>), grid, VT, smem, st, b, tm); break;
        case 3: LAUNCH((k_vertex_pass_tiled<1, VT_MINB, true>), grid, VT, smem, st, b, tm); break;
        case 4: LAUNCH((k_vertex_pass_tiled<1, VT_MINB, false, true>), grid, VT, smem, st, b, tm); break;
        case 6: LAUNCH((k_vertex_pass_tiled<1, 5, true>), grid, VT, smem, st, b, tm); break;
        case 7: LAUNCH((k_vertex_pass_tiled<1, 3, true>), grid, VT, smem, st, b, tm); break;
        default: LAUNCH((k_vertex_pass_tiled<1, VT_MINB, true, true>), grid, VT, smem, st, b, tm);
        }
        return PSTF_OK;
    }
per_thread:
    for (pstf_field *f : fs)
        if (f) f->unit_frame = false; /* the per-thread kernels do not count (k_ef_onepass) */
    if (cv)
        LAUNCH(k_cv_lookup, grid_for(n, 256), 256, 0, st, loe->d, *v, n, cv->r, cv->g, cv->b,
               cv->valid);
    if (mode == PSTF_MODE_ATOMIC)
        LAUNCH(k_vertex_pass<PSTF_MODE_ATOMIC>, grid_for(n, VP_BLOCK), VP_BLOCK, 0, st, a);
    else
        LAUNCH(k_vertex_pass<PSTF_MODE_ORDERED>, grid_for(n, VP_BLOCK), VP_BLOCK, 0, st, a);
    return PSTF_OK;
}

static int vertex_checks(pstf_field *lo, pstf_field *loe, pstf_field *fli, pstf_field *li, int mode) {
    if (!lo || !loe || !fli) return set_err(PSTF_E_INVALID, "lo, loe and fli stores are required");
    if (mode != PSTF_MODE_ATOMIC && mode != PSTF_MODE_ORDERED)
        return set_err(PSTF_E_INVALID, "vertex pass supports ATOMIC and ORDERED modes");
    if (loe->device != lo->device || fli->device != lo->device || (li && li->device != lo->device))
        return set_err(PSTF_E_INVALID, "all stores must live on one device");
    return PSTF_OK;
}

static uint64_t records_per_vertex(int mode, bool li) {
    return mode == PSTF_MODE_ATOMIC ? (li ? 5 : 4) : (li ? 12 : 10);
}

int pstf_vertex_pass(pstf_field *lo, pstf_field *loe, pstf_field *fli, pstf_field *li,
                     const pstf_vertex_soa *v, uint64_t n, uint32_t loe_mask, uint32_t fli_mask,
                     int mode, void *stream) {
    int rc = vertex_checks(lo, loe, fli, li, mode);
    if (rc) return rc;
    if (!v) return set_err(PSTF_E_INVALID, "NULL vertex record");
    CK(cudaSetDevice(lo->device));
    SETTLE(lo);
    SETTLE(loe);
    SETTLE(fli);
    SETTLE(li);
    cudaStream_t st = (cudaStream_t)stream;
    rc = ensure_pending(lo->sc, std::max<uint64_t>(1, n * records_per_vertex(mode, li)), false, st);
    if (rc) return rc;
    if (mode == PSTF_MODE_ORDERED) {
        rc = ensure_pending2(lo->sc, std::max<uint64_t>(1, n * 7));
        if (rc) return rc;
    }
    if (n) {
        rc = vertex_phase1(lo, loe, fli, li, v, n, loe_mask, fli_mask, mode, st);
        if (rc) return rc;
    }
    pstf_field *fs[4] = {lo, loe, fli, li};
    for (int i = 0; i < 4; ++i) /* "new keys / rounds of the last pass" start at 0 */
        if (fs[i]) CK(cudaMemsetAsync(&fs[i]->d.ctr[C_NEW_KEYS], 0, 8, st));
    for (int i = 0; i < 4; ++i)
        if (fs[i]) CK(cudaMemsetAsync(&fs[i]->d.ctr[C_ROUNDS], 0, 8, st));
    return finish_vertex_pass(fs, mode, st);
}

int pstf_vertex_pass_cv(pstf_field *lo, pstf_field *loe, pstf_field *fli, pstf_field *li,
                        const pstf_vertex_soa *v, uint64_t n, uint32_t loe_mask,
                        uint32_t fli_mask, int mode, double *cv_r, double *cv_g, double *cv_b,
                        uint8_t *cv_valid, void *stream) {
    int rc = vertex_checks(lo, loe, fli, li, mode);
    if (rc) return rc;
    if (!v) return set_err(PSTF_E_INVALID, "NULL vertex record");
    if (n && (!cv_r || !cv_g || !cv_b || !cv_valid))
        return set_err(PSTF_E_INVALID, "CV outputs required");
    CK(cudaSetDevice(lo->device));
    SETTLE(lo);
    SETTLE(loe);
    SETTLE(fli);
    SETTLE(li);
    cudaStream_t st = (cudaStream_t)stream;
    rc = ensure_pending(lo->sc, std::max<uint64_t>(1, n * records_per_vertex(mode, li)), false, st);
    if (rc) return rc;
    if (mode == PSTF_MODE_ORDERED) {
        rc = ensure_pending2(lo->sc, std::max<uint64_t>(1, n * 7));
        if (rc) return rc;
    }
    if (n) {
        const CvOut cv{cv_r, cv_g, cv_b, cv_valid};
        rc = vertex_phase1(lo, loe, fli, li, v, n, loe_mask, fli_mask, mode, st, &cv);
        if (rc) return rc;
    }
    pstf_field *fs[4] = {lo, loe, fli, li};
    for (int i = 0; i < 4; ++i) /* "new keys / rounds of the last pass" start at 0 */
        if (fs[i]) CK(cudaMemsetAsync(&fs[i]->d.ctr[C_NEW_KEYS], 0, 8, st));
    for (int i = 0; i < 4; ++i)
        if (fs[i]) CK(cudaMemsetAsync(&fs[i]->d.ctr[C_ROUNDS], 0, 8, st));
    return finish_vertex_pass(fs, mode, st);
}

void pstf_vertex_soa_from_buffer(const double *b, uint64_t n, pstf_vertex_soa *o) {
    auto v3 = [&](int k) {
        pstf_vec3_soa s;
        s.x = b + (uint64_t)k * n;
        s.y = b + (uint64_t)(k + 1) * n;
        s.z = b + (uint64_t)(k + 2) * n;
        return s;
    };
    o->position = v3(PS_POS);
    o->wo = v3(PS_WO);
    o->wi = v3(PS_WI);
    o->next_position = v3(PS_NPOS);
    o->nee_dir = v3(PS_NDIR);
    o->footprint = b + (uint64_t)PS_FP * n;
    o->next_footprint = b + (uint64_t)PS_NFP * n;
    o->ratio = b + (uint64_t)PS_RATIO * n;
    o->next_emis_mis_weight = b + (uint64_t)PS_NMIS * n;
    o->emission_here = v3(PS_EMIS);
    o->f = v3(PS_F);
    o->next_emission = v3(PS_NEMIS);
    o->nee_loe = v3(PS_NEELOE);
    o->nee_fli = v3(PS_NEEFLI);
    o->flags = (const uint32_t *)(b + (uint64_t)PS_NUM_F64 * n);
}

/* Host-resident vertex arrays: chunked H2D on a copy stream (double-buffered staging) overlapped
 * with phase 1 of the previous chunk on the compute stream; phase 2 runs once at the end so
 * every lookup sees the frame-start table (Jacobi). */
int pstf_vertex_pass_host(pstf_field *lo, pstf_field *loe, pstf_field *fli, pstf_field *li,
                          const pstf_vertex_soa *hv, uint64_t n, uint32_t loe_mask,
                          uint32_t fli_mask, int mode, void *stream) {
    int rc = vertex_checks(lo, loe, fli, li, mode);
    if (rc) return rc;
    if (!hv) return set_err(PSTF_E_INVALID, "NULL vertex record");
    CK(cudaSetDevice(lo->device));
    SETTLE(lo);
    SETTLE(loe);
    SETTLE(fli);
    SETTLE(li);
    cudaStream_t st = (cudaStream_t)stream;
    rc = ensure_pending(lo->sc, std::max<uint64_t>(1, n * records_per_vertex(mode, li)), false, st);
    if (rc) return rc;
    const uint64_t chunk = std::min<uint64_t>(n, 1ull << 21);
    if (mode == PSTF_MODE_ORDERED) { /* one phase-1 launch per chunk */
        rc = ensure_pending2(lo->sc, std::max<uint64_t>(1, n * 7),
                             chunk ? (n + chunk - 1) / chunk : 1);
        if (rc) return rc;
    }
    static thread_local cudaStream_t cs = nullptr;
    static thread_local cudaEvent_t ev_copy[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr};
    static thread_local DBuf stage[2];
    if (!cs) {
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            CK(cudaEventCreateWithFlags(&ev_copy[b], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ev_done[b], cudaEventDisableTiming));
        }
    }
    const size_t per = PS_BYTES_PER_VERTEX;
    for (int b = 0; b < 2; ++b) ENSURE(stage[b], chunk * per + 64);
    /* the copy stream must not run ahead of earlier work on the compute stream */
    CK(cudaEventRecord(ev_done[0], st));
    CK(cudaStreamWaitEvent(cs, ev_done[0], 0));
    CK(cudaEventRecord(ev_done[1], st));
    for (uint64_t off = 0, k = 0; off < n; off += chunk, ++k) {
        const int b = (int)(k & 1);
        const uint64_t m = std::min(chunk, n - off);
        CK(cudaStreamWaitEvent(cs, ev_done[b], 0));
        double *d = stage[b].as<double>();
        const pstf_vec3_soa *v3s[10] = {&hv->position, &hv->wo, &hv->wi, &hv->next_position,
                                        &hv->nee_dir, &hv->emission_here, &hv->f,
                                        &hv->next_emission, &hv->nee_loe, &hv->nee_fli};
        const int v3f[10] = {PS_POS, PS_WO, PS_WI, PS_NPOS, PS_NDIR, PS_EMIS, PS_F, PS_NEMIS,
                             PS_NEELOE, PS_NEEFLI};
        for (int q = 0; q < 10; ++q) {
            const double *c[3] = {v3s[q]->x, v3s[q]->y, v3s[q]->z};
            for (int j = 0; j < 3; ++j)
                CK(cudaMemcpyAsync(d + (uint64_t)(v3f[q] + j) * m, c[j] + off, m * 8,
                                   cudaMemcpyHostToDevice, cs));
        }
        const double *sc1[4] = {hv->footprint, hv->next_footprint, hv->ratio, hv->next_emis_mis_weight};
        const int sf[4] = {PS_FP, PS_NFP, PS_RATIO, PS_NMIS};
        for (int q = 0; q < 4; ++q)
            CK(cudaMemcpyAsync(d + (uint64_t)sf[q] * m, sc1[q] + off, m * 8, cudaMemcpyHostToDevice, cs));
        CK(cudaMemcpyAsync(d + (uint64_t)PS_NUM_F64 * m, hv->flags + off, m * 4,
                           cudaMemcpyHostToDevice, cs));
        CK(cudaEventRecord(ev_copy[b], cs));
        CK(cudaStreamWaitEvent(st, ev_copy[b], 0));
        pstf_vertex_soa dv;
        pstf_vertex_soa_from_buffer(d, m, &dv);
        rc = vertex_phase1(lo, loe, fli, li, &dv, m, loe_mask, fli_mask, mode, st);
        if (rc) return rc;
        CK(cudaEventRecord(ev_done[b], st));
    }
    pstf_field *fs[4] = {lo, loe, fli, li};
    if (mode == PSTF_MODE_ORDERED) return resolve_ordered(lo->sc, fs, li ? 4 : 3, st);
    return resolve_pending(lo->sc, fs, li ? 4 : 3, mode, (uint64_t)-1, st);
}

int pstf_cv_lookup(const pstf_field *loe, const pstf_vertex_soa *v, uint64_t n, double *value_r,
                   double *value_g, double *value_b, uint8_t *valid, void *stream) {
    if (!loe || !v) return set_err(PSTF_E_INVALID, "NULL argument");
    if (!n) return PSTF_OK;
    CK(cudaSetDevice(loe->device));
    SETTLE(loe);
    LAUNCH(k_cv_lookup, grid_for(n, 256), 256, 0, (cudaStream_t)stream, dev_view(loe), *v, n,
           value_r, value_g, value_b, valid);
    return PSTF_OK;
}

int pstf_synth_generate_stripe(int width, int height, int bounces, uint64_t seed,
                               uint64_t iteration, double cam_shift_x, uint64_t path0,
                               uint64_t npaths, double *buffer, void *stream) {
    return pstf_synth_generate_scene(0, width, height, bounces, seed, iteration, cam_shift_x,
                                     path0, npaths, buffer, stream);
}

int pstf_synth_generate_scene(int scene, int width, int height, int bounces, uint64_t seed,
                              uint64_t iteration, double cam_shift_x, uint64_t path0,
                              uint64_t npaths, double *buffer, void *stream) {
    const uint64_t total = (uint64_t)width * (uint64_t)height;
    if (scene != 0 && scene != 1) return set_err(PSTF_E_INVALID, "scene must be 0 or 1");
    if (width <= 0 || height <= 0 || bounces <= 0 || !buffer || path0 + npaths > total)
        return set_err(PSTF_E_INVALID, "bad synthetic stream arguments");
    ps_params P;
    P.width = width;
    P.height = height;
    P.bounces = bounces;
    P.seed = seed;
    P.iter = iteration;
    P.cam_shift_x = cam_shift_x;
    P.path0 = path0;
    P.n_local = npaths == total && path0 == 0 ? 0 : npaths;
    P.glossy = scene;
    LAUNCH(k_synth, grid_for(npaths, 128), 128, 0, (cudaStream_t)stream, P, buffer,
           npaths * (uint64_t)bounces);
    return PSTF_OK;
}

int pstf_synth_generate(int width, int height, int bounces, uint64_t seed, uint64_t iteration,
                        double cam_shift_x, double *buffer, void *stream) {
    return pstf_synth_generate_stripe(width, height, bounces, seed, iteration, cam_shift_x, 0,
                                      (uint64_t)width * (uint64_t)height, buffer, stream);
}

/* ---------------- key-owner sharding (multi-GPU) ---------------- */
static int shard_checks(pstf_field *const *fs, int n) {
    if (!fs || n < 1 || n > 4) return set_err(PSTF_E_INVALID, "1..4 stores per batch");
    for (int i = 0; i < n; ++i) {
        if (!fs[i]) return set_err(PSTF_E_INVALID, "NULL store");
        if (fs[i]->device != fs[0]->device || fs[i]->world != fs[0]->world ||
            fs[i]->d.rank != fs[0]->d.rank)
            return set_err(PSTF_E_INVALID, "stores must share device and shard layout");
    }
    return PSTF_OK;
}

int pstf_shard_set(pstf_field *f, int rank, int world) {
    if (!f) return set_err(PSTF_E_INVALID, "NULL store");
    SETTLE(f);
    if (world < 1 || world > 32) return set_err(PSTF_E_INVALID, "world must be in [1, 32]");
    if (rank < 0 || rank >= world) return set_err(PSTF_E_INVALID, "bad rank");
    f->d.rank = rank; /* origin tag of this rank's pending records */
    f->world = world;
    return PSTF_OK;
}

int pstf_vertex_pass_local(pstf_field *lo, pstf_field *loe, pstf_field *fli, pstf_field *li,
                           const pstf_vertex_soa *v, uint64_t n, uint32_t loe_mask,
                           uint32_t fli_mask, void *stream) {
    int rc = vertex_checks(lo, loe, fli, li, PSTF_MODE_ATOMIC);
    if (rc) return rc;
    if (!v) return set_err(PSTF_E_INVALID, "NULL vertex record");
    CK(cudaSetDevice(lo->device));
    SETTLE(lo);
    SETTLE(loe);
    SETTLE(fli);
    SETTLE(li);
    cudaStream_t st = (cudaStream_t)stream;
    rc = ensure_pending(lo->sc, std::max<uint64_t>(1, n * records_per_vertex(PSTF_MODE_ATOMIC, li)),
                        false, st);
    if (rc) return rc;
    if (n) return vertex_phase1(lo, loe, fli, li, v, n, loe_mask, fli_mask, PSTF_MODE_ATOMIC, st);
    return PSTF_OK;
}

int pstf_pending_count(pstf_field *lo, uint64_t *n) {
    if (!lo || !n) return set_err(PSTF_E_INVALID, "NULL argument");
    CK(cudaSetDevice(lo->device));
    SETTLE(lo);
    CK(cudaDeviceSynchronize());
    unsigned long long c = 0;
    if (lo->sc.pend_count.p) CK(cudaMemcpy(&c, lo->sc.pend_count.p, 8, cudaMemcpyDeviceToHost));
    *n = std::min<uint64_t>(c, lo->sc.pend.bytes / sizeof(PendRec));
    return PSTF_OK;
}

__global__ void k_count_out(const unsigned long long *src, uint64_t cap, long long *dst) {
    if (threadIdx.x == 0) dst[0] = (long long)(src ? (*src < cap ? *src : cap) : 0ull);
}

int pstf_pending_count_dev(pstf_field *lo, int64_t *dev_count, void *stream) {
    if (!lo || !dev_count) return set_err(PSTF_E_INVALID, "NULL argument");
    CK(cudaSetDevice(lo->device));
    SETTLE(lo);
    LAUNCH(k_count_out, 1, 32, 0, (cudaStream_t)stream,
           lo->sc.pend_count.as<unsigned long long>(), lo->sc.pend.bytes / sizeof(PendRec),
           reinterpret_cast<long long *>(dev_count));
    return PSTF_OK;
}

int pstf_pending_copy(pstf_field *lo, void *dst, uint64_t n, void *stream) {
    if (!lo || (n && !dst)) return set_err(PSTF_E_INVALID, "NULL argument");
    if (!n) return PSTF_OK;
    CK(cudaSetDevice(lo->device));
    SETTLE(lo);
    CK(cudaMemcpyAsync(dst, lo->sc.pend.p, n * sizeof(PendRec), cudaMemcpyDeviceToDevice,
                       (cudaStream_t)stream));
    return PSTF_OK;
}

int pstf_resolve_records(pstf_field *const *stores, int nst, const void *recs, uint64_t n,
                         void *stream) {
    int rc = shard_checks(stores, nst);
    if (rc) return rc;
    twin_batch(stores, nst);
    CK(cudaSetDevice(stores[0]->device));
    for (int i_ = 0; i_ < nst; ++i_) SETTLE(stores[i_]);
    cudaStream_t st = (cudaStream_t)stream;
    Scratch &sc = stores[0]->sc;
    rc = ensure_pending(sc, std::max<uint64_t>(n, 1), false, st);
    if (rc) return rc;
    if (n) CK(cudaMemcpyAsync(sc.pend.p, recs, n * sizeof(PendRec), cudaMemcpyDeviceToDevice, st));
    /* the device count too: phase 2's key-range pass reads it (an empty range would force the
     * multi-word sort path instead of the sort-free one) */
    LAUNCH(k_set_u64, 1, 1, 0, st, sc.pend_count.as<unsigned long long>(),
           (unsigned long long)n); /* stream-ordered, no host staging (capture-safe) */
    return resolve_pending(sc, stores, nst, PSTF_MODE_ATOMIC, n, st, stores[0]->d.rank);
}

static WSeg live_word_segments(pstf_field *const *stores, int nst) {
    WSeg w;
    uint64_t t = 0;
    for (int j = 0; j < nst; ++j) {
        w.o[j] = (uint32_t)t;
        t += ((uint64_t)stores[j]->d.mask + 1) / 32;
    }
    for (int j = nst; j < 5; ++j) w.o[j] = (uint32_t)t;
    return w;
}

int pstf_shard_live_pack(pstf_field *const *stores, int nst, double *packed, uint64_t bound,
                         int64_t *dev_live_total, void *stream) {
    int rc = shard_checks(stores, nst);
    if (rc) return rc;
    if ((bound && !packed) || !dev_live_total) return set_err(PSTF_E_INVALID, "NULL argument");
    for (int j = 0; j < nst; ++j)
        if ((uint64_t)stores[j]->d.mask + 1 < 32)
            return set_err(PSTF_E_INVALID, "sharding needs capacity >= 32");
    CK(cudaSetDevice(stores[0]->device));
    for (int i_ = 0; i_ < nst; ++i_) SETTLE(stores[i_]);
    cudaStream_t st = (cudaStream_t)stream;
    Scratch &sc = stores[0]->sc;
    const WSeg wseg = live_word_segments(stores, nst);
    const uint64_t words = wseg.o[nst];
    ENSURE(sc.head, (words + 1) * 4);   /* word counts */
    ENSURE(sc.scan, (words + 1) * 4);   /* their exclusive scan */
    ENSURE(sc.ulist, std::max<uint64_t>(bound, 1) * 8);
    ENSURE(sc.overflow, 8);
    if (!sc.overflow_zeroed) {
        CK(cudaMemsetAsync(sc.overflow.p, 0, 8, st));
        sc.overflow_zeroed = true;
    }
    uint32_t *cnt = sc.head.as<uint32_t>(), *scan = sc.scan.as<uint32_t>();
    const Stores4 S = stores4(stores, nst);
    LAUNCH(k_live_count, grid_for(words + 1, 256), 256, 0, st, S, nst, wseg, cnt);
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, scan, (int64_t)(words + 1), st));
    ENSURE(sc.cub, tmp);
    CK(cub::DeviceScan::ExclusiveSum(sc.cub.p, tmp, cnt, scan, (int64_t)(words + 1), st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const unsigned g = std::min<unsigned>(grid_for(std::max(words, bound), 256),
                                          (unsigned)sm_count() * 8);
    LAUNCH(k_live_pack, g, 256, 0, st, S, nst, wseg, scan, bound,
           sc.ulist.as<unsigned long long>(), reinterpret_cast<double4 *>(packed),
           reinterpret_cast<long long *>(dev_live_total), sc.overflow.as<unsigned long long>());
    sc.live_bound = bound;
    sc.live_total_dev = reinterpret_cast<long long *>(dev_live_total);
    return PSTF_OK;
}

int pstf_shard_live_unpack(pstf_field *const *stores, int nst, const double *packed,
                           void *stream) {
    int rc = shard_checks(stores, nst);
    if (rc) return rc;
    twin_batch(stores, nst);
    Scratch &sc = stores[0]->sc;
    if (!sc.live_total_dev) return set_err(PSTF_E_INVALID, "pstf_shard_live_pack first");
    if (sc.live_bound && !packed) return set_err(PSTF_E_INVALID, "NULL packed");
    for (int i_ = 0; i_ < nst; ++i_) stores[i_]->unit_frame = false; /* remote sums */
    CK(cudaSetDevice(stores[0]->device));
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g = std::min<unsigned>(grid_for(sc.live_bound, 256), (unsigned)sm_count() * 8);
    if (sc.live_bound)
        LAUNCH(k_live_unpack, g, 256, 0, st, stores4(stores, nst),
               sc.ulist.as<unsigned long long>(), reinterpret_cast<const double4 *>(packed),
               sc.live_total_dev, sc.live_bound);
    return PSTF_OK;
}

int pstf_shard_end_frame(pstf_field *const *stores, int nst, const double *packed,
                         void *stream) {
    int rc = shard_checks(stores, nst);
    if (rc) return rc;
    twin_batch(stores, nst);
    for (int i = 0; i < nst; ++i)
        for (int j = 0; j < i; ++j)
            if (stores[j] == stores[i]) return set_err(PSTF_E_INVALID, "store listed twice");
    Scratch &sc = stores[0]->sc;
    if (!sc.live_total_dev) return set_err(PSTF_E_INVALID, "pstf_shard_live_pack first");
    if (sc.live_bound && !packed) return set_err(PSTF_E_INVALID, "NULL packed");
    CK(cudaSetDevice(stores[0]->device));
    for (int i_ = 0; i_ < nst; ++i_) SETTLE(stores[i_]);
    cudaStream_t st = (cudaStream_t)stream;
    static int blocks = -1; /* co-resident blocks per SM of the cooperative kernel */
    if (blocks < 0)
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_ef_packed, EF_BLOCK, 0));
    uint64_t maxcap = 0;
    for (int i = 0; i < nst; ++i) maxcap = std::max<uint64_t>(maxcap, (uint64_t)stores[i]->d.mask + 1);
    const unsigned gf = std::min<unsigned>(grid_for(std::max(maxcap, sc.live_bound), EF_BLOCK),
                                           (unsigned)(sm_count() * std::max(blocks, 1)));
    Stores4 S = stores4(stores, nst);
    int nn = nst;
    const unsigned long long *list = sc.ulist.as<const unsigned long long>();
    const double4 *pk = reinterpret_cast<const double4 *>(packed);
    const long long *lt = sc.live_total_dev;
    uint64_t bound = sc.live_bound;
    void *args[] = {&S, &nn, &list, &pk, &lt, &bound};
    {
        ProfScope ps_("k_ef_packed", st);
        CK(cudaLaunchCooperativeKernel((const void *)k_ef_packed, gf, EF_BLOCK, args, 0, st));
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    for (int i = 0; i < nst; ++i) { /* the phase-1 touch marks of this replica */
        CK(cudaMemsetAsync(stores[i]->d.tbits, 0, (((uint64_t)stores[i]->d.mask + 32) / 32) * 4, st));
        stores[i]->frame += 1;
        stores[i]->unit_frame = true;
    }
    return PSTF_OK;
}

int pstf_shard_info(pstf_field *const *stores, int nst, int64_t *dev_out3, void *stream) {
    int rc = shard_checks(stores, nst);
    if (rc) return rc;
    if (!dev_out3) return set_err(PSTF_E_INVALID, "NULL argument");
    CK(cudaSetDevice(stores[0]->device));
    for (int i_ = 0; i_ < nst; ++i_) SETTLE(stores[i_]);
    Scratch &sc = stores[0]->sc;
    ENSURE(sc.overflow, 8);
    if (!sc.overflow_zeroed) {
        CK(cudaMemsetAsync(sc.overflow.p, 0, 8, (cudaStream_t)stream));
        sc.overflow_zeroed = true;
    }
    LAUNCH(k_shard_info, 1, 32, 0, (cudaStream_t)stream, stores4(stores, nst), nst,
           sc.pend_count.as<unsigned long long>(), sc.pend.bytes / sizeof(PendRec),
           sc.overflow.as<unsigned long long>(), reinterpret_cast<long long *>(dev_out3));
    return PSTF_OK;
}

uint64_t pstf_pending_record_bytes(void) { return sizeof(PendRec); }

} // extern "C"


/* CV-profile / guiding model store: same translation unit */
#include "model_store.cuh"
