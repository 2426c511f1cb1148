// capture_shim.cpp — extern "C" access to the UNMODIFIED reference renderer for parity tests
// (TEST INFRASTRUCTURE ONLY; built into oracle/_ref/libpstf_capture.so by oracle/Makefile).
//
// Two things the GPU parity tests need from the reference itself:
//   1. real vertex streams: the reference path tracer (pathtracer.cpp:80-206 tracePath, fired
//      through renderFrame pathtracer.cpp:208-239) renders a scene with a PathHooks collector
//      attached (the pattern of VertexCollector, tests/unit/test_pathtracer.cpp:14-17); every
//      VertexRecord (pathtracer.h:59-90) is converted to the canonical 276 B SoA record the B200
//      vertex pass consumes: transportRatio() (pathtracer.h:86-89),
//      nee.value() (pathtracer.h:42-46) and nee.f * nee.radiance * nee.misWeight
//      (estimators.cpp:251) are evaluated here with the reference's own operators;
//   2. the reference estimator run on the same scene: EstimatorRun (estimators.cpp:308-343,
//      560-655) with its own field stores, whose per-frame snapshots and slot arrays are the
//      ground truth the replayed GPU stores are compared against.  `#define private public`
//      exposes FieldStore::m_slots without editing any reference file.
// All reference sources are compiled in place from /root/reference (never copied).
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <functional>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <unordered_map>
#include <vector>

#define private public
#include "pstf/field.h"
#include PSTF_REF_FIELD_CPP
#include "pstf/estimators.h"
#undef private
#include "pstf/pathtracer.h"
#include "pstf/scene.h"

using namespace pstf;

namespace {

struct Collector : PathHooks { // test_pathtracer.cpp:14-17, made safe for concurrent workers
    std::mutex mu;
    std::vector<VertexRecord> records;
    void onVertex(const VertexRecord &rec) override {
        std::lock_guard<std::mutex> lk(mu);
        records.push_back(rec);
    }
};

struct Capture {
    std::vector<VertexRecord> records;
};

thread_local std::string g_err;

} // namespace

extern "C" {

struct pc_slot { // == pr_slot (ref_shim.cpp) / po_slot
    uint32_t checksum;
    int32_t level, cell[3], dir[2];
    double value_old[3];
    double c_old;
    double accum[3];
    double c_new;
    uint32_t last_touched;
};

struct pc_stats {
    uint64_t frame, rejected, dropped, internal_errors, live;
};

const char *pc_last_error() { return g_err.c_str(); }

/* loadScene (scene.cpp:646) with the camera resolution overridden the way the acceptance suite
 * does it (acceptance_main.cpp:60-61); NULL on a parse error */
void *pc_scene_load(const char *path, int width, int height) {
    try {
        auto *s = new Scene(loadScene(path));
        if (width > 0) s->camera.width = width;
        if (height > 0) s->camera.height = height;
        return s;
    } catch (const std::exception &e) {
        g_err = e.what();
        return nullptr;
    }
}
void pc_scene_free(void *s) { delete static_cast<Scene *>(s); }
double pc_scene_diameter(void *s) { return static_cast<Scene *>(s)->diameter(); }

/* one frame of the reference tracer (renderFrame, pathtracer.cpp:208-239) with the default
 * TraceConfig (pathtracer.h:14-20: NEE, RR from depth 3, maxDepth 64), as EstimatorRun drives it
 * for PT_NEE (estimators.cpp:592-595): the same Rng(seed, streamId(frame*spp+s, pixel)) streams */
void *pc_capture(void *scene, uint64_t frame, uint64_t seed, int spp, int threads, int max_depth,
                 int64_t *n_out) {
    const Scene &sc = *static_cast<Scene *>(scene);
    TraceConfig tc;
    if (max_depth > 0) tc.maxDepth = max_depth;
    Collector col;
    ImageBuffer buf(sc.camera.width, sc.camera.height);
    renderFrame(sc, tc, buf, frame, seed, spp, threads, &col);
    auto *c = new Capture{std::move(col.records)};
    *n_out = int64_t(c->records.size());
    return c;
}

/* The canonical SoA record (34 fp64 arrays of n, then u32 flags[n]; field order of
 * paper_2005_07547_b200/csrc/pstf_synth.h PS_*), values computed with the reference's operators */
void pc_capture_soa(void *cap, double *buf) {
    const auto &R = static_cast<Capture *>(cap)->records;
    const size_t n = R.size();
    auto put3 = [&](int k, size_t i, double x, double y, double z) {
        buf[size_t(k) * n + i] = x;
        buf[size_t(k + 1) * n + i] = y;
        buf[size_t(k + 2) * n + i] = z;
    };
    uint32_t *flags = reinterpret_cast<uint32_t *>(buf + size_t(34) * n);
    for (size_t i = 0; i < n; ++i) {
        const VertexRecord &r = R[i];
        put3(0, i, r.position.x, r.position.y, r.position.z);
        put3(3, i, r.wo.x, r.wo.y, r.wo.z);
        put3(6, i, r.wi.x, r.wi.y, r.wi.z);
        put3(9, i, r.nextPosition.x, r.nextPosition.y, r.nextPosition.z);
        put3(12, i, r.nee.dir.x, r.nee.dir.y, r.nee.dir.z);
        buf[15 * n + i] = r.footprint;
        buf[16 * n + i] = r.nextFootprint;
        buf[17 * n + i] = r.transportRatio();
        buf[18 * n + i] = r.nextEmisMisWeight;
        put3(19, i, r.emissionHere.r, r.emissionHere.g, r.emissionHere.b);
        put3(22, i, r.f.r, r.f.g, r.f.b);
        put3(25, i, r.nextEmission.r, r.nextEmission.g, r.nextEmission.b);
        const RGB nv = r.nee.value();
        put3(28, i, nv.r, nv.g, nv.b);
        const RGB nf = r.nee.f * r.nee.radiance * r.nee.misWeight;
        put3(31, i, nf.r, nf.g, nf.b);
        flags[i] = (r.contExtended ? 1u : 0u) | (r.nextIsSurface ? 2u : 0u) |
                   (r.nee.sampled ? 4u : 0u);
    }
}

/* path depth of every captured vertex (VertexRecord::depth), for stream statistics */
void pc_capture_depths(void *cap, int32_t *depth) {
    const auto &R = static_cast<Capture *>(cap)->records;
    for (size_t i = 0; i < R.size(); ++i) depth[i] = R[i].depth;
}

void pc_capture_free(void *cap) { delete static_cast<Capture *>(cap); }

/* EstimatorRun with the reference's field stores (estimators.cpp:308-343).  kind: EstimatorKind
 * ordinal (PT=0, PT_NEE=1, IS, CV, IS_CV, B); the stores use EstimatorConfig's field knobs */
void *pc_run_create(void *scene, int kind, int deterministic, int threads, uint64_t seed,
                    uint32_t capacity_log2, int track_li, uint32_t loe_mask, uint32_t fli_mask) {
    EstimatorConfig c;
    c.kind = EstimatorKind(kind);
    c.deterministic = deterministic != 0;
    c.threads = threads;
    c.seed = seed;
    c.hashCapacityLog2 = capacity_log2;
    c.trackLi = track_li != 0;
    c.loeTechniqueMask = loe_mask;
    c.fliTechniqueMask = fli_mask;
    return new EstimatorRun(*static_cast<Scene *>(scene), c);
}
void pc_run_free(void *run) { delete static_cast<EstimatorRun *>(run); }
void pc_run_frame(void *run) { static_cast<EstimatorRun *>(run)->renderFrame(nullptr); }

static FieldStore *store_of(void *run, int which) {
    auto *r = static_cast<EstimatorRun *>(run);
    switch (which) {
    case 0: return &r->loStore();
    case 1: return &r->loeStore();
    case 2: return &r->fliStore();
    default: return r->liStore();
    }
}

/* the store's configuration as the EstimatorRun built it: base cell, K, max level, capacity,
 * tMax (doubles {base, K, tMax}, ints {capacity_log2, max_level, probe_window, evict_age}) */
void pc_run_store_config(void *run, int which, double *d3, int32_t *i4) {
    const FieldStoreConfig &c = store_of(run, which)->config();
    d3[0] = c.baseCellSize;
    d3[1] = c.levelSelectK;
    d3[2] = c.tMax;
    i4[0] = int32_t(c.capacityLog2);
    i4[1] = c.maxLevel;
    i4[2] = int32_t(c.probeWindow);
    i4[3] = int32_t(c.evictAgeFrames);
}

int pc_run_dump_snapshot(void *run, int which, const char *path) {
    try {
        store_of(run, which)->dumpSnapshot(path);
        return 0;
    } catch (const std::exception &e) {
        g_err = e.what();
        return -1;
    }
}

void pc_run_stats(void *run, int which, pc_stats *o) {
    FieldStore *s = store_of(run, which);
    o->frame = s->frameIndex();
    o->rejected = s->rejectedUpdates();
    o->dropped = s->droppedInserts();
    o->internal_errors = s->internalErrors();
    o->live = s->liveCellCount();
}

/* the whole slot array (field.cpp:48-58) of one store, index = slot */
void pc_run_slots(void *run, int which, pc_slot *out) {
    FieldStore *s = store_of(run, which);
    const size_t cap = size_t(s->m_mask) + 1;
    for (size_t i = 0; i < cap; ++i) {
        const auto &sl = s->m_slots[i];
        pc_slot &o = out[i];
        o.checksum = sl.checksum.load(std::memory_order_relaxed);
        o.level = sl.level;
        std::copy(sl.cell, sl.cell + 3, o.cell);
        std::copy(sl.dirCell, sl.dirCell + 2, o.dir);
        o.value_old[0] = sl.valueOld.r;
        o.value_old[1] = sl.valueOld.g;
        o.value_old[2] = sl.valueOld.b;
        o.c_old = sl.cOld;
        for (int c = 0; c < 3; ++c) o.accum[c] = sl.accum[c].load(std::memory_order_relaxed);
        o.c_new = sl.cNew.load(std::memory_order_relaxed);
        o.last_touched = sl.lastTouched.load(std::memory_order_relaxed);
    }
}

} // extern "C"
