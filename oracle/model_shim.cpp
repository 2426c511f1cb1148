// model_shim.cpp — extern "C" wrapper around the UNMODIFIED reference ModelStore with DirGrid /
// SphericalKdTree models
// (TEST INFRASTRUCTURE ONLY; built into oracle/_ref/libpstf_model_ref.so by oracle/Makefile).
//
// /root/reference/proj/core/src/estimators.cpp (ModelStore, estimators.cpp:104-144) and
// models.cpp (DirGrid, models.cpp:16-94) are compiled in place (#included, never copied) with
// `#define private public`, so the store's map and each DirGrid's weights/accumulators are
// observable.  The rest of the core (tracer, scene, image, field) is linked as separate
// translation units compiled in place.  Records are applied exactly as
// EstimatorRun::renderFrame does in deterministic mode (estimators.cpp:625-645): sorted by
// (key fields, uv.x, uv.y, contribution), then applyRecord in that order.
#include <algorithm>
#include <array>
#include <atomic>
#include <cassert>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <functional>
#include <memory>
#include <mutex>
#include <optional>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <unordered_map>
#include <variant>
#include <vector>

#define private public
#include PSTF_REF_MODELS_CPP
#include PSTF_REF_ESTIMATORS_CPP
#undef private

using namespace pstf;

extern "C" {

struct pm_key {
    int32_t level, cell[3], dir[2];
    uint32_t checksum;
};

struct pm_entry { // == po_model_entry / pstf_model_entry
    int32_t level, cell[3], dir[2];
    uint32_t warm;
    double c_old, c_new;
    uint64_t records, record_count;
    double total;
};

static SpatioDirectionalKey toKey(const pm_key &k) {
    SpatioDirectionalKey s;
    s.level = k.level;
    std::copy(k.cell, k.cell + 3, s.cell);
    std::copy(k.dir, k.dir + 2, s.dirCell);
    s.checksum = k.checksum;
    return s;
}

void *pm_create(int kind, int res, int leaves, double tsplit, int comps, double alpha_em,
                double smin, double smax, double reseed_frac, double t_max, int min_samples) {
    ModelConfig cfg;
    cfg.kind = kind == 1 ? ModelKind::KdTree : kind == 2 ? ModelKind::Gmm : ModelKind::Grid;
    cfg.gridResolution = res;
    cfg.kdLeafCount = leaves;
    cfg.kdSplitThreshold = tsplit;
    cfg.gmm.components = comps;
    cfg.gmm.alphaEm = alpha_em;
    cfg.gmm.sigmaMinSq = smin;
    cfg.gmm.sigmaMaxSq = smax;
    cfg.gmm.reseedFraction = reseed_frac;
    return new ModelStore(cfg, t_max, min_samples);
}

void pm_destroy(void *m) { delete static_cast<ModelStore *>(m); }

void pm_apply(void *m, const pm_key *keys, const double *u, const double *v, const double *c,
              int64_t n) {
    std::vector<ModelRecord> records;
    records.reserve(size_t(n));
    for (int64_t i = 0; i < n; ++i) {
        ModelRecord r{};
        r.key = toKey(keys[i]);
        r.uv = Vec2{u[i], v[i]};
        r.contribution = c[i];
        r.profile = true;
        records.push_back(r);
    }
    // estimators.cpp:633-637, restated over the file-local ModelRecord
    std::sort(records.begin(), records.end(), [](const ModelRecord &a, const ModelRecord &b) {
        return std::tie(a.profile, a.key.level, a.key.cell[0], a.key.cell[1], a.key.cell[2],
                        a.key.dirCell[0], a.key.dirCell[1], a.uv.x, a.uv.y, a.contribution) <
               std::tie(b.profile, b.key.level, b.key.cell[0], b.key.cell[1], b.key.cell[2],
                        b.key.dirCell[0], b.key.dirCell[1], b.uv.x, b.uv.y, b.contribution);
    });
    ModelStore *st = static_cast<ModelStore *>(m);
    for (const ModelRecord &r : records) st->applyRecord(r.key, r.uv, r.contribution);
}

void pm_end_frame(void *m) { static_cast<ModelStore *>(m)->endFrame(); }

// lookupWarm + DirGrid::pdf; *found = 0 and 1.0 without a warm model
double pm_pdf(void *m, const pm_key *k, double u, double v, int *found) {
    const DirectionalModel *d = static_cast<ModelStore *>(m)->lookupWarm(toKey(*k));
    *found = d != nullptr;
    return d ? d->pdf(Vec2{u, v}) : 1.0;
}

// lookupWarm + DirGrid::sample(u)
void pm_sample(void *m, const pm_key *k, double u1, double u2, double usel, double *su,
               double *sv, double *pdf, int *found) {
    const DirectionalModel *d = static_cast<ModelStore *>(m)->lookupWarm(toKey(*k));
    *found = d != nullptr;
    if (!d) {
        *su = u1;
        *sv = u2;
        *pdf = 1.0;
        return;
    }
    Sample2D s;
    if (const DirGrid *g = std::get_if<DirGrid>(&d->m_impl))
        s = g->sample(Vec2{u1, u2});
    else if (const Gmm *gm = std::get_if<Gmm>(&d->m_impl))
        s = gm->sample(usel, Vec2{u1, u2}); // DirectionalModel::sample draws uSelect first
    else
        s = std::get<SphericalKdTree>(d->m_impl).sample(Vec2{u1, u2});
    *su = s.uv.x;
    *sv = s.uv.y;
    *pdf = s.pdf;
}

// every entry sorted by key, with its DirGrid state (private members)
int64_t pm_dump(void *m, pm_entry *out, double *weights, double *accum, int64_t cap) {
    ModelStore *st = static_cast<ModelStore *>(m);
    std::vector<const std::pair<const SpatioDirectionalKey, ModelStore::Entry> *> ord;
    for (const auto &kv : st->m_map) ord.push_back(&kv);
    std::sort(ord.begin(), ord.end(), [](auto *a, auto *b) {
        const SpatioDirectionalKey &x = a->first, &y = b->first;
        return std::tie(x.level, x.cell[0], x.cell[1], x.cell[2], x.dirCell[0], x.dirCell[1]) <
               std::tie(y.level, y.cell[0], y.cell[1], y.cell[2], y.dirCell[0], y.dirCell[1]);
    });
    const int64_t n = int64_t(ord.size()), k = std::min(n, cap);
    for (int64_t i = 0; i < k; ++i) {
        const SpatioDirectionalKey &key = ord[size_t(i)]->first;
        const ModelStore::Entry &e = ord[size_t(i)]->second;
        pm_entry &o = out[i];
        std::memset(&o, 0, sizeof(o));
        o.level = key.level;
        std::copy(key.cell, key.cell + 3, o.cell);
        std::copy(key.dirCell, key.dirCell + 2, o.dir);
        o.warm = e.warm;
        o.c_old = e.cOld;
        o.c_new = e.cNew;
        o.records = e.records;
        if (const DirGrid *g = std::get_if<DirGrid>(&e.model->m_impl)) {
            o.record_count = g->m_recordCount;
            o.total = g->m_total;
            const size_t r2 = g->m_weights.size();
            if (weights) std::copy(g->m_weights.begin(), g->m_weights.end(), weights + size_t(i) * r2);
            if (accum) std::copy(g->m_accum.begin(), g->m_accum.end(), accum + size_t(i) * r2);
        } else if (const Gmm *gm = std::get_if<Gmm>(&e.model->m_impl)) {
            // Gmm: the state vector {W, M, V, U, cache, i, underflows, reseed counter}
            o.record_count = gm->m_recordCount;
            o.total = 0.0;
            const size_t C = gm->m_weights.size(), ns = 21 * C + 3;
            if (weights) {
                double *S = weights + size_t(i) * ns;
                for (size_t c = 0; c < C; ++c) {
                    S[c] = gm->m_weights[c];
                    S[C + 2 * c] = gm->m_means[c].x;
                    S[C + 2 * c + 1] = gm->m_means[c].y;
                    for (int q = 0; q < 3; ++q) S[3 * C + 3 * c + q] = gm->m_cov[c][q];
                    for (int q = 0; q < 8; ++q) S[6 * C + 8 * c + q] = gm->m_u[c][q];
                    const auto &k = gm->m_cache[c];
                    double *K = S + 14 * C + 7 * c;
                    K[0] = k.inv[0];
                    K[1] = k.inv[1];
                    K[2] = k.inv[2];
                    K[3] = k.norm;
                    K[4] = k.chol[0];
                    K[5] = k.chol[1];
                    K[6] = k.chol[2];
                }
                S[21 * C] = double(gm->m_i);
                S[21 * C + 1] = double(gm->m_underflows);
                S[21 * C + 2] = double(gm->m_reseedCounter);
            }
            if (accum) std::fill(accum + size_t(i) * ns, accum + size_t(i + 1) * ns, 0.0);
        } else { // SphericalKdTree: per node prob / accum in node order
            const SphericalKdTree &t = std::get<SphericalKdTree>(e.model->m_impl);
            o.record_count = t.m_recordCount;
            o.total = 0.0;
            const size_t nn = t.m_nodes.size();
            for (size_t j = 0; j < nn; ++j) {
                if (weights) weights[size_t(i) * nn + j] = t.m_nodes[j].prob;
                if (accum) accum[size_t(i) * nn + j] = t.m_nodes[j].accum;
            }
        }
    }
    return n;
}

// k-d tree topology (SphericalKdTree::Node, models.h:91-99), same entry order as pm_dump
int64_t pm_dump_tree(void *m, int32_t *node_i32, double *node_f64, int64_t cap) {
    ModelStore *st = static_cast<ModelStore *>(m);
    std::vector<const std::pair<const SpatioDirectionalKey, ModelStore::Entry> *> ord;
    for (const auto &kv : st->m_map) ord.push_back(&kv);
    std::sort(ord.begin(), ord.end(), [](auto *a, auto *b) {
        const SpatioDirectionalKey &x = a->first, &y = b->first;
        return std::tie(x.level, x.cell[0], x.cell[1], x.cell[2], x.dirCell[0], x.dirCell[1]) <
               std::tie(y.level, y.cell[0], y.cell[1], y.cell[2], y.dirCell[0], y.dirCell[1]);
    });
    const int64_t n = int64_t(ord.size()), k = std::min(n, cap);
    for (int64_t i = 0; i < k; ++i) {
        const SphericalKdTree &t = std::get<SphericalKdTree>(ord[size_t(i)]->second.model->m_impl);
        const size_t nn = t.m_nodes.size();
        for (size_t j = 0; j < nn; ++j) {
            const auto &nd = t.m_nodes[j];
            int32_t *o = node_i32 + (size_t(i) * nn + j) * 5;
            o[0] = nd.leaf;
            o[1] = nd.axis;
            o[2] = nd.left;
            o[3] = nd.right;
            o[4] = nd.parent;
            node_f64[(size_t(i) * nn + j) * 2] = nd.split;
            node_f64[(size_t(i) * nn + j) * 2 + 1] = nd.mass;
        }
    }
    return n;
}

} // extern "C"
