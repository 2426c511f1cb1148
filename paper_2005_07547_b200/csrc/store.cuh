/*
 * store.cuh — HBM layout of one B200 field store and the device-side probe/touch helpers.
 *
 * One pstf::FieldStore (reference: proj/core/src/field.cpp:48-58, an AoS of 104 B slots) becomes
 * slot-indexed arrays so each kernel streams only what it needs:
 *
 *   meta  uint2[cap]    {checksum (0 = empty), lastTouched + 1 (0 = never touched)}
 *                       one 8 B probe load gives identity and "already touched this frame"
 *   com   double4[cap]  {valueOld.rgb, cOld}  committed     (lookup reads one 32 B sector)
 *   acc   double4[cap]  {accum.rgb, cNew}     this frame    (fp64 RED target, one sector)
 *   keyf  KeyFields[cap] level, cell[3], dirCell[2]         (written on insert; snapshot/invalidate)
 *   tbits u32[cap/32]    touched-this-frame bitmap: a slot's first touch in a frame (seen via
 *                       meta.y != frame + 1) sets its bit with a fire-and-forget RED.OR
 *   tlist u32[cap]       endFrame compacts the bitmap into this list and blends only those slots
 *   lbits u32[cap/32]    live bitmap (checksum != 0), kept by placement and eviction: the
 *                       multi-GPU path packs the live slots from it
 *   hold  u32[2][cap]   deterministic-placement scratch (rank of the proposing key, ~0 = none)
 */
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "pstf_keys.cuh"

namespace pstf_b200 {

/* 32-byte records moved with one 256-bit access (LDG/STG.E.256 on sm_100) instead of two
 * 128-bit halves: one L1 request and one L2 sector transaction per record.
 *   ld4_ro  read-only data of the running kernel (committed values in the vertex pass)
 *   ld4/st4 ordered with the thread's other memory accesses (endFrame read-modify-write) */
/* L1 policy of the probe and committed-record loads: keeping them L1-resident over the other
 * traffic measured 0.5% faster on config 2 (0.808 vs 0.812 ms, 3 interleaved A/B rounds).
 * The meta probes live off L1 (L1::no_allocate on them: 0.877 ms); the committed records do
 * not (no_allocate on them: unchanged).  Experiment builds: PSTF_L1_COM 0 plain volatile,
 * 1 non-volatile, 2 + L1::evict_last, 3 + L1::evict_first, 4 + L1::no_allocate; PSTF_L1_META
 * 0 plain, 1 L1::evict_last, 2 L1::no_allocate */
#ifndef PSTF_L1_COM
#define PSTF_L1_COM 2
#endif
#ifndef PSTF_L1_META
#define PSTF_L1_META 1
#endif
__device__ __forceinline__ double4 ld4_ro(const double4 *p) {
    double4 v;
#if PSTF_L1_COM == 1
    asm("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
        : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
#elif PSTF_L1_COM == 2
    asm("ld.global.L1::evict_last.v4.f64 {%0, %1, %2, %3}, [%4];"
        : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
#elif PSTF_L1_COM == 3
    asm("ld.global.L1::evict_first.v4.f64 {%0, %1, %2, %3}, [%4];"
        : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
#elif PSTF_L1_COM == 4
    asm("ld.global.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
        : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
#else
    asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "l"(p));
#endif
    return v;
}
/* a slot's meta word as the vertex pass's probes read it */
__device__ __forceinline__ uint2 ld_meta(const uint2 *p) {
#if PSTF_L1_META == 1
    uint2 v;
    asm volatile("ld.global.L1::evict_last.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
#elif PSTF_L1_META == 2
    uint2 v;
    asm volatile("ld.global.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
#else
    return *p;
#endif
}
__device__ __forceinline__ double4 ld4(const double4 *p) {
    double4 v;
    asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ void st4(double4 *p, double4 v) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.x), "d"(v.y),
                 "d"(v.z), "d"(v.w)
                 : "memory");
}

struct KeyFields {
    int32_t level, c0, c1, c2, d0, d1;
};

enum Ctr : int {
    C_REJECTED = 0,
    C_DROPPED,
    C_INTERNAL,
    C_LIVE,
    C_TOUCHED_N,    // entries in tlist (endFrame of the current frame)
    C_NEW_KEYS,     // keys placed by the last pass
    C_EVICTED,      // evicted by the last endFrame
    C_CN_COUNT,     // endFrame: live slots with cNew > 0
    C_LIVE_SNAP,    // endFrame: live count before eviction (field.cpp:205-212)
    C_TOUCHED_LAST, // touched slots of the last committed frame
    C_TOUCHED_TOTAL, // touched slots summed over all committed frames
    C_REDS,          // fp64 RED element updates of the fused vertex passes' contributions, before
                     // any warp aggregation (Lo store)
    C_ROUNDS,        // deterministic-placement rounds of the last update pass
    C_F_CN,          // this frame: sum of counter weights into existing/placed slots (unit-
                     // weight frames: an exact integer, = field.cpp:205-212's sum of c_new)
    C_F_DEFER,       // one-pass endFrame: touched slots deferred to k_ef_tail (may be capped)
    C_REDS_MARK,     // C_REDS at the start of the frame (the hot-slot measure's per-frame REDs)
    C_CN_INEXACT,    // this frame: a counter weight that is not a whole number <= 2^20 (then
                     // Σc_new is summed sequentially in slot order, field.cpp:201-213)
    C_NUM
};

struct DevStore {
    uint2 *meta;
    double4 *com;
    double4 *acc;
    KeyFields *keyf;
    uint32_t *tbits;
    uint32_t *lbits; // live bitmap (meta.x != 0): set at placement, cleared at eviction
    uint32_t *tlist;
    uint32_t *hold0, *hold1;
    unsigned long long *hold64_0, *hold64_1; /* 64-bit priority holds (sort-free ATOMIC phase 2),
                                                allocated on first use, ~0 = none */
    unsigned long long *ctr; // C_NUM counters
    double *cn_sum;          // endFrame scratch
    uint32_t mask;
    uint32_t window;
    KeyParams kp;
    double t_max;
    uint32_t blend;
    uint32_t evict_age;
    uint32_t frame;       // uint32_t(m_frame) for this launch
    int32_t rank;         // multi-GPU: this rank (origin tag of pending records; 0 unsharded)
};

/* the accumulator / committed record of a slot */
__device__ __forceinline__ double4 *acc_ptr(const DevStore &s, uint64_t slot) {
    return s.acc + slot;
}
__device__ __forceinline__ double4 *com_ptr(const DevStore &s, uint64_t slot) {
    return s.com + slot;
}

/* the members of a store that a contribution touches, selectable per loop iteration */
struct StoreRef {
    uint2 *meta;
    double4 *acc;
    uint32_t *tbits;
    unsigned long long *ctr;
    uint32_t frame;
    int32_t rank;
};

__device__ __forceinline__ StoreRef store_ref(const DevStore &s) {
    return StoreRef{s.meta, s.acc, s.tbits, s.ctr, s.frame, s.rank};
}


#define PSTF_HOLD_NONE 0xffffffffu

__device__ __forceinline__ uint32_t ld_chk(const DevStore &s, uint32_t idx) {
    return s.meta[idx].x;
}

/* findSlot (field.cpp:103-114): slot index, or -1 */
__device__ __forceinline__ int probe_find(const DevStore &s, uint32_t home, uint32_t cs) {
    for (uint32_t i = 0; i < s.window; ++i) {
        uint32_t idx = (home + i) & s.mask;
        uint32_t c = ld_chk(s, idx);
        if (c == cs) return (int)idx;
        if (c == 0) return -1;
    }
    return -1;
}

/* findOrInsertSlot's search over the frame-start table (field.cpp:116-146):
 * >= 0 existing slot, -1 an empty slot comes first (new key -> deterministic placement),
 * -2 window exhausted with no empty slot and no match (dropped; new keys cannot change that).
 * *touched_mark receives the slot's lastTouched+1 word. */
__device__ __forceinline__ int probe_existing(const DevStore &s, uint32_t home, uint32_t cs,
                                              uint32_t *touched_mark) {
    for (uint32_t i = 0; i < s.window; ++i) {
        uint32_t idx = (home + i) & s.mask;
        uint2 m = ld_meta(&s.meta[idx]);
        if (m.x == cs) {
            *touched_mark = m.y;
            return (int)idx;
        }
        if (m.x == 0) return -1;
    }
    return -2;
}

/* lastTouched = frame (field.cpp:123,133,137); mark = the meta.y word seen by the probe, so an
 * already-touched slot costs no store */
template <class Store>
__device__ __forceinline__ void touch_slot(const Store &s, uint32_t slot, uint32_t mark) {
    const uint32_t m = s.frame + 1u;
    if (mark != m) {
        s.meta[slot].y = m;
        atomicOr(&s.tbits[slot >> 5], 1u << (slot & 31u)); /* RED.OR, idempotent */
    }
}

template <class Store>
__device__ __forceinline__ void touch_slot(const Store &s, uint32_t slot) {
    s.meta[slot].y = s.frame + 1u;
    atomicOr(&s.tbits[slot >> 5], 1u << (slot & 31u));
}

/* finish a probe whose home-slot word m0 was already loaded (findOrInsertSlot's search) */
__device__ __forceinline__ int resolve_probe(const DevStore &s, uint32_t home, uint32_t cs,
                                             uint2 m0, uint32_t *mark) {
    if (m0.x == cs) {
        *mark = m0.y;
        return (int)home;
    }
    if (m0.x == 0) return -1;
    for (uint32_t i = 1; i < s.window; ++i) {
        uint32_t idx = (home + i) & s.mask;
        uint2 m = ld_meta(&s.meta[idx]);
        if (m.x == cs) {
            *mark = m.y;
            return (int)idx;
        }
        if (m.x == 0) return -1;
    }
    return -2;
}

/* same with the word after home also preloaded (one round trip settles a single collision) */
__device__ __forceinline__ int resolve_probe2(const DevStore &s, uint32_t home, uint32_t cs,
                                              uint2 m0, uint2 m1, uint32_t *mark) {
    if (m0.x == cs) {
        *mark = m0.y;
        return (int)home;
    }
    if (m0.x == 0) return -1;
    if (s.window < 2) return -2;
    if (m1.x == cs) {
        *mark = m1.y;
        return (int)((home + 1) & s.mask);
    }
    if (m1.x == 0) return -1;
    for (uint32_t i = 2; i < s.window; ++i) {
        uint32_t idx = (home + i) & s.mask;
        uint2 m = ld_meta(&s.meta[idx]);
        if (m.x == cs) {
            *mark = m.y;
            return (int)idx;
        }
        if (m.x == 0) return -1;
    }
    return -2;
}

/* finish a findSlot (lookup) whose home word was already loaded: slot or -1 */
__device__ __forceinline__ int resolve_find(const DevStore &s, uint32_t home, uint32_t cs,
                                            uint32_t c0) {
    if (c0 == cs) return (int)home;
    if (c0 == 0) return -1;
    for (uint32_t i = 1; i < s.window; ++i) {
        uint32_t idx = (home + i) & s.mask;
        uint32_t c = s.meta[idx].x;
        if (c == cs) return (int)idx;
        if (c == 0) return -1;
    }
    return -1;
}

} // namespace pstf_b200
