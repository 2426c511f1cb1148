/*
 * kernels.cuh — device kernels of the B200 field cache (declarations shared by field.cu).
 *
 * K1 keygen/select_level   field.cpp:68-101            (batch API)
 * K2 insert/accumulate     field.cpp:116-172           (vertex pass phase 1 + apply + placement)
 * K3 blend/evict           field.cpp:197-263           (endFrame on the touched list)
 * K4 lookup                field.cpp:174-195           (batch query + inside the vertex pass)
 * K5 fused vertex pass     estimators.cpp:194-262      (onVertex for a wavefront of vertices)
 */
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pstf_field.h"
#include "store.cuh"

namespace pstf_b200 {

/* One pending update record (new-key path, or every call in ORDERED/SEQUENTIAL mode). */
struct PendRec {
    int32_t k[6];  // level, cell[3], dirCell[2]
    uint32_t cs;   // checksum
    uint32_t meta; // bits 0-1 store id, bit 2 is_counter, bits 3-7 origin rank, 8-31 calls
    double v[4];   // ATOMIC: {r,g,b,c} aggregated; ORDERED/SEQUENTIAL: {r,g,b,w} of one call
};
static_assert(sizeof(PendRec) == 64, "PendRec must be 64 B");

#define PSTF_META(sid, is_counter, ncalls) \
    ((uint32_t)(sid) | ((uint32_t)(is_counter) << 2) | ((uint32_t)(ncalls) << 8))
#define PSTF_META_SID(m) ((m)&3u)
#define PSTF_META_ISC(m) (((m) >> 2) & 1u)
#define PSTF_META_CALLS(m) ((m) >> 8)
#define PSTF_META_ORIGIN(m) (((m) >> 3) & 31u) /* producing rank (key-owner sharding) */

struct Stores4 {
    DevStore s[4];
};

/* placement result encoding (int64): type << 32 | slot */
enum : uint32_t { R_NONE = 0, R_FIXED = 1, R_MERGE = 2, R_PROPOSE = 3, R_DROP = 4 };
#define PSTF_RES(t, slot) (((unsigned long long)(t) << 32) | (unsigned long long)(uint32_t)(slot))
#define PSTF_RES_T(r) ((uint32_t)((r) >> 32))
#define PSTF_RES_SLOT(r) ((uint32_t)(r))

} // namespace pstf_b200
