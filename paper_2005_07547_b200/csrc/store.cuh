/*
 * store.cuh — HBM layout of one B200 field store and the device-side probe/touch helpers.
 *
 * One pstf::FieldStore (reference: proj/core/src/field.cpp:48-58, an AoS of 104 B slots) becomes
 * a set of slot-indexed SoA arrays so each kernel streams only what it needs:
 *
 *   chk   u32[cap]      checksum, 0 = empty                 (probe path, L2-resident: 4 B/slot)
 *   com   double4[cap]  {valueOld.rgb, cOld}  committed     (lookup reads one 32 B sector)
 *   acc   double4[cap]  {accum.rgb, cNew}     this frame    (fp64 RED target, one sector)
 *   keyf  KeyFields[cap] level, cell[3], dirCell[2]         (written on insert; snapshot/invalidate)
 *   last  u32[cap]      lastTouched                          (eviction age, field.cpp:123-137)
 *   tmark u32[cap]      frame+1 when the slot was first touched this frame (touched-list dedupe)
 *   touched u32[cap]    list of slots touched this frame -> endFrame works on touched cells only
 *   hold  u32[2][cap]   deterministic-placement scratch (rank of the proposing key, ~0 = none)
 */
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "pstf_keys.cuh"

namespace pstf_b200 {

struct KeyFields {
    int32_t level, c0, c1, c2, d0, d1;
};

enum Ctr : int {
    C_REJECTED = 0,
    C_DROPPED,
    C_INTERNAL,
    C_LIVE,
    C_TOUCHED_N,   // entries in the touched list
    C_NEW_KEYS,    // keys placed by the last pass
    C_EVICTED,     // evicted by the last endFrame
    C_CN_COUNT,    // endFrame: live slots with cNew > 0
    C_LIVE_SNAP,   // endFrame: live count before eviction (field.cpp:205-212)
    C_TOUCHED_LAST, // touched slots of the last committed frame
    C_NUM
};

struct DevStore {
    uint32_t *chk;
    double4 *com;
    double4 *acc;
    KeyFields *keyf;
    uint32_t *last;
    uint32_t *tmark;
    uint32_t *touched;
    uint32_t *hold0, *hold1;
    unsigned long long *ctr; // C_NUM counters
    double *cn_sum;          // endFrame scratch
    uint32_t mask;
    uint32_t window;
    KeyParams kp;
    double t_max;
    uint32_t blend;
    uint32_t evict_age;
    uint32_t frame; // uint32_t(m_frame) for this launch
};

#define PSTF_HOLD_NONE 0xffffffffu

/* findSlot (field.cpp:103-114): slot index, or -1 */
__device__ __forceinline__ int probe_find(const DevStore &s, uint32_t home, uint32_t cs) {
    for (uint32_t i = 0; i < s.window; ++i) {
        uint32_t idx = (home + i) & s.mask;
        uint32_t c = __ldg(&s.chk[idx]);
        if (c == cs) return (int)idx;
        if (c == 0) return -1;
    }
    return -1;
}

/* findOrInsertSlot's search over the frame-start table (field.cpp:116-146):
 * >= 0 existing slot, -1 an empty slot comes first (new key -> deterministic placement),
 * -2 window exhausted with no empty slot and no match (dropped; new keys cannot change that). */
__device__ __forceinline__ int probe_existing(const DevStore &s, uint32_t home, uint32_t cs) {
    for (uint32_t i = 0; i < s.window; ++i) {
        uint32_t idx = (home + i) & s.mask;
        uint32_t c = s.chk[idx];
        if (c == cs) return (int)idx;
        if (c == 0) return -1;
    }
    return -2;
}

/* lastTouched = frame (field.cpp:123,133,137) + append to the touched list once per frame */
__device__ __forceinline__ void touch_slot(const DevStore &s, uint32_t slot) {
    if (s.last[slot] != s.frame) s.last[slot] = s.frame;
    uint32_t m = s.frame + 1u;
    if (s.tmark[slot] != m && atomicExch(&s.tmark[slot], m) != m) {
        unsigned long long pos = atomicAdd(&s.ctr[C_TOUCHED_N], 1ull);
        s.touched[pos] = slot;
    }
}

} // namespace pstf_b200
