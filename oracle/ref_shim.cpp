// ref_shim.cpp — extern "C" wrapper around the UNMODIFIED reference field engine
// (TEST INFRASTRUCTURE ONLY; built into oracle/_ref/ by oracle/Makefile).
//
// The reference translation unit /root/reference/proj/core/src/field.cpp is compiled in
// place (#included, never copied).  `#define private public` exposes FieldStore::m_slots so
// slot occupancy and probe distances are observable (SURVEY.md §8c, Appendix B probe 4).
// The vertex driver below restates FieldRecorder::onVertex (estimators.cpp:194-262, which is
// file-local in the reference) over the reference's PUBLIC FieldStore/FieldUpdateQueue API;
// threading follows EstimatorRun::renderFrame (estimators.cpp:566-623): row-interleaved
// std::thread workers writing straight into the stores (non-deterministic mode) or into
// per-worker FieldUpdateQueues merged and applied at the barrier (deterministic mode).
#include <algorithm>
#include <chrono>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#define private public
#include "pstf/field.h"
#include PSTF_REF_FIELD_CPP
#undef private

using namespace pstf;

extern "C" {

struct pr_config {
    uint32_t kind, capacity_log2;
    int32_t max_level;
    double base_cell_size, level_select_k, t_max;
    uint32_t blend, technique_mask, probe_window, evict_age_frames;
};

struct pr_key {
    int32_t level, cell[3], dir[2];
    uint32_t checksum;
};

struct pr_slot {
    uint32_t checksum;
    int32_t level, cell[3], dir[2];
    double value_old[3];
    double c_old;
    double accum[3];
    double c_new;
    uint32_t last_touched;
};

struct pr_stats {
    uint64_t frame, rejected, dropped, internal_errors, live;
};

static FieldStoreConfig toCfg(const pr_config *c) {
    FieldStoreConfig f;
    f.kind = FieldKind(c->kind);
    f.capacityLog2 = c->capacity_log2;
    f.maxLevel = c->max_level;
    f.baseCellSize = c->base_cell_size;
    f.levelSelectK = c->level_select_k;
    f.tMax = c->t_max;
    f.blend = c->blend == 0 ? FieldStoreConfig::Blend::Sqrt : FieldStoreConfig::Blend::Linear;
    f.techniqueMask = c->technique_mask;
    f.probeWindow = c->probe_window;
    f.evictAgeFrames = c->evict_age_frames;
    return f;
}

static SpatioDirectionalKey toKey(const pr_key *k) {
    SpatioDirectionalKey s;
    s.level = k->level;
    std::copy(k->cell, k->cell + 3, s.cell);
    std::copy(k->dir, k->dir + 2, s.dirCell);
    s.checksum = k->checksum;
    return s;
}

static void fromKey(const SpatioDirectionalKey &s, pr_key *k) {
    k->level = s.level;
    std::copy(s.cell, s.cell + 3, k->cell);
    std::copy(s.dirCell, s.dirCell + 2, k->dir);
    k->checksum = s.checksum;
}

void *pr_store_create(const pr_config *c) { return new FieldStore(toCfg(c)); }
void pr_store_destroy(void *s) { delete static_cast<FieldStore *>(s); }

int pr_select_level(void *s, double footprint) {
    return static_cast<FieldStore *>(s)->selectLevel(footprint);
}

void pr_key_for(void *s, const double *pos, const double *dir, int level, pr_key *out) {
    fromKey(static_cast<FieldStore *>(s)->keyFor(Vec3(pos[0], pos[1], pos[2]),
                                                 Vec3(dir[0], dir[1], dir[2]), level),
            out);
}

// batched key generation: pos/dir are SoA (x[n], y[n], z[n])
void pr_key_for_batch(void *s, const double *pos, const double *dir, const int32_t *level,
                      int64_t n, pr_key *out) {
    FieldStore *st = static_cast<FieldStore *>(s);
    for (int64_t i = 0; i < n; ++i)
        fromKey(st->keyFor(Vec3(pos[i], pos[n + i], pos[2 * n + i]),
                           Vec3(dir[i], dir[n + i], dir[2 * n + i]), level[i]),
                &out[i]);
}

void pr_select_level_batch(void *s, const double *fp, int64_t n, int32_t *out) {
    FieldStore *st = static_cast<FieldStore *>(s);
    for (int64_t i = 0; i < n; ++i) out[i] = st->selectLevel(fp[i]);
}

void pr_sphere_to_square_batch(const double *dir, int64_t n, double *uv) {
    for (int64_t i = 0; i < n; ++i) {
        Vec2 p = sphereToSquare(Vec3(dir[i], dir[n + i], dir[2 * n + i]));
        uv[i] = p.x;
        uv[n + i] = p.y;
    }
}

uint64_t pr_home_slot(void *s, const pr_key *k) {
    FieldStore *st = static_cast<FieldStore *>(s);
    return uint32_t(packKeyFields(toKey(k))) & st->m_mask;
}

void pr_increment(void *s, const pr_key *k, double w) {
    static_cast<FieldStore *>(s)->incrementCounter(toKey(k), w);
}

void pr_accumulate(void *s, const pr_key *k, const double *v, double w) {
    static_cast<FieldStore *>(s)->accumulate(toKey(k), RGB(v[0], v[1], v[2]), w);
}

// out: value[3], valid, fallback, level as doubles/ints
void pr_query_from_level(void *s, const double *pos, const double *dir, int level, double *value,
                         int32_t *flags3) {
    auto r = static_cast<FieldStore *>(s)->queryFromLevel(Vec3(pos[0], pos[1], pos[2]),
                                                          Vec3(dir[0], dir[1], dir[2]), level);
    value[0] = r.value.r;
    value[1] = r.value.g;
    value[2] = r.value.b;
    flags3[0] = r.valid;
    flags3[1] = r.fallback;
    flags3[2] = r.level;
}

void pr_query(void *s, const double *pos, const double *dir, double footprint, double *value,
              int32_t *flags3) {
    auto r = static_cast<FieldStore *>(s)->query(Vec3(pos[0], pos[1], pos[2]),
                                                 Vec3(dir[0], dir[1], dir[2]), footprint);
    value[0] = r.value.r;
    value[1] = r.value.g;
    value[2] = r.value.b;
    flags3[0] = r.valid;
    flags3[1] = r.fallback;
    flags3[2] = r.level;
}

// batched query (SoA pos/dir), footprint or (if level != NULL) explicit level
void pr_query_batch(void *s, const double *pos, const double *dir, const double *fp,
                    const int32_t *level, int64_t n, double *value, int32_t *flags3) {
    FieldStore *st = static_cast<FieldStore *>(s);
    for (int64_t i = 0; i < n; ++i) {
        Vec3 p(pos[i], pos[n + i], pos[2 * n + i]), d(dir[i], dir[n + i], dir[2 * n + i]);
        auto r = level ? st->queryFromLevel(p, d, level[i]) : st->query(p, d, fp[i]);
        value[i] = r.value.r;
        value[n + i] = r.value.g;
        value[2 * n + i] = r.value.b;
        flags3[i] = r.valid;
        flags3[n + i] = r.fallback;
        flags3[2 * n + i] = r.level;
    }
}

void pr_end_frame(void *s) { static_cast<FieldStore *>(s)->endFrame(); }
void pr_invalidate_all(void *s) { static_cast<FieldStore *>(s)->invalidate(); }
void pr_invalidate_box(void *s, const double *lo, const double *hi) {
    Aabb b;
    b.lo = Vec3(lo[0], lo[1], lo[2]);
    b.hi = Vec3(hi[0], hi[1], hi[2]);
    static_cast<FieldStore *>(s)->invalidate(b);
}

void pr_stats_get(void *s, pr_stats *out) {
    FieldStore *st = static_cast<FieldStore *>(s);
    out->frame = st->frameIndex();
    out->rejected = st->rejectedUpdates();
    out->dropped = st->droppedInserts();
    out->internal_errors = st->internalErrors();
    out->live = st->liveCellCount();
}

void pr_weighted_mean(void *s, double *out) {
    RGB m = static_cast<FieldStore *>(s)->weightedMeanValue();
    out[0] = m.r;
    out[1] = m.g;
    out[2] = m.b;
}

int pr_dump_snapshot(void *s, const char *path) {
    try {
        static_cast<FieldStore *>(s)->dumpSnapshot(path);
        return 0;
    } catch (...) {
        return -1;
    }
}

// Snapshot restore over the reference's own insert (the reference has no restore API; this is
// the restore a maintainer would add to FieldStore): records in ascending key order (stable),
// FieldStore::findOrInsertSlot (field.cpp:116-146), then valueOld/cOld at the returned slot.
struct pr_snap {
    int32_t level, cell[3], dir[2];
    uint32_t checksum;
    double value[3];
    double c_old;
};

void pr_restore(void *s, const pr_snap *recs, int64_t n) {
    FieldStore *st = static_cast<FieldStore *>(s);
    std::vector<const pr_snap *> ord(size_t(n > 0 ? n : 0));
    for (int64_t i = 0; i < n; ++i) ord[size_t(i)] = &recs[i];
    std::stable_sort(ord.begin(), ord.end(), [](const pr_snap *a, const pr_snap *b) {
        return std::tie(a->level, a->cell[0], a->cell[1], a->cell[2], a->dir[0], a->dir[1]) <
               std::tie(b->level, b->cell[0], b->cell[1], b->cell[2], b->dir[0], b->dir[1]);
    });
    for (const pr_snap *r : ord) {
        SpatioDirectionalKey k;
        k.level = r->level;
        std::copy(r->cell, r->cell + 3, k.cell);
        std::copy(r->dir, r->dir + 2, k.dirCell);
        k.checksum = r->checksum;
        int idx = st->findOrInsertSlot(k);
        if (idx < 0) continue;
        st->m_slots[idx].valueOld = RGB{r->value[0], r->value[1], r->value[2]};
        st->m_slots[idx].cOld = r->c_old;
    }
}

// slot array (private state, exposed by `#define private public`)
void pr_slots(void *s, pr_slot *out) {
    FieldStore *st = static_cast<FieldStore *>(s);
    size_t cap = size_t(st->m_mask) + 1;
    for (size_t i = 0; i < cap; ++i) {
        auto &sl = st->m_slots[i];
        pr_slot &o = out[i];
        o.checksum = sl.checksum.load();
        o.level = sl.level;
        std::copy(sl.cell, sl.cell + 3, o.cell);
        std::copy(sl.dirCell, sl.dirCell + 2, o.dir);
        o.value_old[0] = sl.valueOld.r;
        o.value_old[1] = sl.valueOld.g;
        o.value_old[2] = sl.valueOld.b;
        o.c_old = sl.cOld;
        for (int c = 0; c < 3; ++c) o.accum[c] = sl.accum[c].load();
        o.c_new = sl.cNew.load();
        o.last_touched = sl.lastTouched.load();
    }
}

// ---- deterministic queue ----
void *pr_queue_create() { return new FieldUpdateQueue(); }
void pr_queue_destroy(void *q) { delete static_cast<FieldUpdateQueue *>(q); }
void pr_queue_push_counter(void *q, const pr_key *k, double w) {
    static_cast<FieldUpdateQueue *>(q)->pushCounter(toKey(k), w);
}
void pr_queue_push_value(void *q, const pr_key *k, const double *v, double w) {
    static_cast<FieldUpdateQueue *>(q)->pushValue(toKey(k), RGB(v[0], v[1], v[2]), w);
}
void pr_queue_apply(void *q, void *s) {
    static_cast<FieldUpdateQueue *>(q)->apply(*static_cast<FieldStore *>(s));
}

// ---- FieldRecorder::onVertex restated over the public API (estimators.cpp:160-262) ----
struct Sink { // EstimatorRun::WorkerSink estimators.cpp:160-179
    bool queued = false;
    FieldUpdateQueue qLo, qLoe, qFli, qLi;
    void increment(FieldStore *s, FieldUpdateQueue &q, const SpatioDirectionalKey &k, double w) {
        if (queued) q.pushCounter(k, w);
        else s->incrementCounter(k, w);
    }
    void accumulate(FieldStore *s, FieldUpdateQueue &q, const SpatioDirectionalKey &k,
                    const RGB &v, double w) {
        if (queued) q.pushValue(k, v, w);
        else s->accumulate(k, v, w);
    }
};

static void onVertex(Sink &sink, FieldStore *lo, FieldStore *loe, FieldStore *fli, FieldStore *li,
                     uint32_t loeMask, uint32_t fliMask, const double *const *F,
                     const uint32_t *flags, size_t i) {
    auto v3 = [&](int k) { return Vec3(F[k][i], F[k + 1][i], F[k + 2][i]); };
    auto rgb = [&](int k) { return RGB(F[k][i], F[k + 1][i], F[k + 2][i]); };
    Vec3 position = v3(0), wo = v3(3), wi = v3(6), nextPosition = v3(9), neeDir = v3(12);
    double footprint = F[15][i], nextFootprint = F[16][i], ratio = F[17][i];
    double nextEmisMisWeight = F[18][i];
    RGB emissionHere = rgb(19), f = rgb(22), nextEmission = rgb(25), neeValue = rgb(28),
        neeFliValue = rgb(31);
    bool contExtended = flags[i] & 1u, nextIsSurface = flags[i] & 2u, neeSampled = flags[i] & 4u;

    int level = lo->selectLevel(footprint);
    RGB loNext(0.0), loeNext(0.0);
    if (contExtended) {
        if (nextIsSurface) {
            Vec3 woNext = -wi;
            auto qLo = lo->query(nextPosition, woNext, nextFootprint);
            if (qLo.valid) loNext = qLo.value;
            auto qLoe = loe->query(nextPosition, woNext, nextFootprint);
            if (qLoe.valid) loeNext = qLoe.value;
        } else {
            loNext = nextEmission;
        }
    }
    SpatioDirectionalKey loKey = lo->keyFor(position, wo, level);
    sink.increment(lo, sink.qLo, loKey, 1.0);
    sink.accumulate(lo, sink.qLo, loKey, emissionHere, 1.0);
    if (contExtended && ratio > 0.0) {
        RGB update = computeUpdateValue(FieldKind::Lo, loNext, RGB(0.0), f, ratio);
        sink.accumulate(lo, sink.qLo, loKey, update, 1.0);
    }
    SpatioDirectionalKey loeKey = loe->keyFor(position, wo, level);
    sink.increment(loe, sink.qLoe, loeKey, 1.0);
    if (contExtended && ratio > 0.0 && (loeMask & TechContinuation)) {
        RGB update = computeUpdateValue(FieldKind::LoMinusE, loeNext,
                                        nextEmission * nextEmisMisWeight, f, ratio);
        sink.accumulate(loe, sink.qLoe, loeKey, update, 1.0);
    }
    if (neeSampled && (loeMask & TechNee)) sink.accumulate(loe, sink.qLoe, loeKey, neeValue, 1.0);
    RGB lIncoming = nextEmission * nextEmisMisWeight + loeNext;
    if (contExtended) {
        SpatioDirectionalKey k = fli->keyFor(position, wi, level);
        sink.increment(fli, sink.qFli, k, 1.0);
        if (fliMask & TechContinuation) sink.accumulate(fli, sink.qFli, k, f * lIncoming, 1.0);
    }
    if (neeSampled) {
        SpatioDirectionalKey k = fli->keyFor(position, neeDir, level);
        sink.increment(fli, sink.qFli, k, 1.0);
        if (fliMask & TechNee) sink.accumulate(fli, sink.qFli, k, neeFliValue, 1.0);
    }
    if (li && contExtended) {
        SpatioDirectionalKey k = li->keyFor(position, wi, level);
        sink.increment(li, sink.qLi, k, 1.0);
        RGB update = computeUpdateValue(FieldKind::Li, lIncoming, RGB(0.0), f, 1.0);
        sink.accumulate(li, sink.qLi, k, update, 1.0);
    }
}

// Replays n vertices (contiguous SoA buffer: 34 fp64 arrays then u32 flags) with `threads`
// workers; vertex i goes to worker (i / chunk) % threads in contiguous chunks of `chunk`
// vertices (row interleaving, estimators.cpp:578-597).
void pr_vertex_pass(void *lo, void *loe, void *fli, void *li, const double *buf, int64_t n,
                    uint32_t loeMask, uint32_t fliMask, int deterministic, int threads,
                    int64_t chunk) {
    const double *F[34];
    for (int k = 0; k < 34; ++k) F[k] = buf + size_t(k) * size_t(n);
    const uint32_t *flags = reinterpret_cast<const uint32_t *>(buf + size_t(34) * size_t(n));
    if (threads < 1) threads = 1;
    if (chunk < 1) chunk = 1;
    std::vector<Sink> sinks(threads);
    for (auto &s : sinks) s.queued = deterministic != 0;
    auto worker = [&](int t) {
        for (int64_t start = int64_t(t) * chunk; start < n; start += int64_t(threads) * chunk) {
            int64_t end = std::min(n, start + chunk);
            for (int64_t i = start; i < end; ++i)
                onVertex(sinks[t], static_cast<FieldStore *>(lo), static_cast<FieldStore *>(loe),
                         static_cast<FieldStore *>(fli), static_cast<FieldStore *>(li), loeMask,
                         fliMask, F, flags, size_t(i));
        }
    };
    if (threads == 1) {
        worker(0);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) pool.emplace_back(worker, t);
        for (auto &th : pool) th.join();
    }
    if (deterministic) { // estimators.cpp:610-623
        FieldUpdateQueue qLo, qLoe, qFli, qLi;
        for (auto &s : sinks) {
            qLo.append(std::move(s.qLo));
            qLoe.append(std::move(s.qLoe));
            qFli.append(std::move(s.qFli));
            qLi.append(std::move(s.qLi));
        }
        qLo.apply(*static_cast<FieldStore *>(lo));
        qLoe.apply(*static_cast<FieldStore *>(loe));
        qFli.apply(*static_cast<FieldStore *>(fli));
        if (li) qLi.apply(*static_cast<FieldStore *>(li));
    }
}

// The same replay timed by phase (SURVEY.md §8(d) CPU protocol, Appendix B probe 2): all
// workers run keygen (selectLevel + keyFor of every key of their vertices), then the next-vertex
// queries, then the counter/accumulate calls with the precomputed keys and values, with a join
// between phases.  Queries read committed state only (field.h:73-75), so the phase order does
// not change what they see.  ms_out = {keygen, lookup, insert} wall milliseconds.
void pr_vertex_pass_phases(void *lo_, void *loe_, void *fli_, const double *buf, int64_t n,
                           uint32_t loeMask, uint32_t fliMask, int threads, double *ms_out) {
    FieldStore *lo = static_cast<FieldStore *>(lo_), *loe = static_cast<FieldStore *>(loe_),
               *fli = static_cast<FieldStore *>(fli_);
    const double *F[34];
    for (int k = 0; k < 34; ++k) F[k] = buf + size_t(k) * size_t(n);
    const uint32_t *flags = reinterpret_cast<const uint32_t *>(buf + size_t(34) * size_t(n));
    if (threads < 1) threads = 1;
    struct Keys {
        SpatioDirectionalKey lo, loe, fc, fn;
    };
    std::vector<Keys> keys(static_cast<size_t>(n));
    std::vector<RGB> loNext(static_cast<size_t>(n)), loeNext(static_cast<size_t>(n));
    auto run = [&](auto &&body) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t)
            pool.emplace_back([&, t] {
                for (int64_t i = int64_t(t); i < n; i += threads) body(size_t(i));
            });
        for (auto &th : pool) th.join();
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
            .count();
    };
    auto v3 = [&](int k, size_t i) { return Vec3(F[k][i], F[k + 1][i], F[k + 2][i]); };
    auto rgb = [&](int k, size_t i) { return RGB(F[k][i], F[k + 1][i], F[k + 2][i]); };
    ms_out[0] = run([&](size_t i) { // keygen (estimators.cpp:205, 218, 226, 242, 248)
        const int level = lo->selectLevel(F[15][i]);
        Keys &k = keys[i];
        k.lo = lo->keyFor(v3(0, i), v3(3, i), level);
        k.loe = loe->keyFor(v3(0, i), v3(3, i), level);
        if (flags[i] & 1u) k.fc = fli->keyFor(v3(0, i), v3(6, i), level);
        if (flags[i] & 4u) k.fn = fli->keyFor(v3(0, i), v3(12, i), level);
    });
    ms_out[1] = run([&](size_t i) { // next-vertex lookups (estimators.cpp:207-216)
        RGB a(0.0), b(0.0);
        if ((flags[i] & 1u) && (flags[i] & 2u)) {
            const Vec3 woNext = -v3(6, i);
            auto qa = lo->query(v3(9, i), woNext, F[16][i]);
            if (qa.valid) a = qa.value;
            auto qb = loe->query(v3(9, i), woNext, F[16][i]);
            if (qb.valid) b = qb.value;
        } else if (flags[i] & 1u) {
            a = rgb(25, i);
        }
        loNext[i] = a;
        loeNext[i] = b;
    });
    ms_out[2] = run([&](size_t i) { // inserts (estimators.cpp:218-254)
        const Keys &k = keys[i];
        const bool cont = flags[i] & 1u, nee = flags[i] & 4u;
        const double ratio = F[17][i], emis = F[18][i];
        const RGB f = rgb(22, i), nextEmission = rgb(25, i);
        lo->incrementCounter(k.lo, 1.0);
        lo->accumulate(k.lo, rgb(19, i), 1.0);
        if (cont && ratio > 0.0)
            lo->accumulate(k.lo, computeUpdateValue(FieldKind::Lo, loNext[i], RGB(0.0), f, ratio),
                           1.0);
        loe->incrementCounter(k.loe, 1.0);
        if (cont && ratio > 0.0 && (loeMask & TechContinuation))
            loe->accumulate(k.loe, computeUpdateValue(FieldKind::LoMinusE, loeNext[i],
                                                      nextEmission * emis, f, ratio), 1.0);
        if (nee && (loeMask & TechNee)) loe->accumulate(k.loe, rgb(28, i), 1.0);
        const RGB lIncoming = nextEmission * emis + loeNext[i];
        if (cont) {
            fli->incrementCounter(k.fc, 1.0);
            if (fliMask & TechContinuation) fli->accumulate(k.fc, f * lIncoming, 1.0);
        }
        if (nee) {
            fli->incrementCounter(k.fn, 1.0);
            if (fliMask & TechNee) fli->accumulate(k.fn, rgb(31, i), 1.0);
        }
    });
}

int pr_hardware_concurrency() { return int(std::thread::hardware_concurrency()); }

} // extern "C"
