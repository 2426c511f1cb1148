// C++ drop-in facade: pstf::FieldStore / FieldUpdateQueue (reference field.h) implemented over
// the B200 C ABI (include/pstf_field.h).  Every key, lookup, update, blend and snapshot runs in
// the sm_100a library; this file only marshals arguments and stages scalar calls.
#include "pstf/field.h"

#include <cstring>
#include <stdexcept>

#include "../../include/pstf_field.h"

namespace pstf {

namespace {

[[noreturn]] void fail(const char *what) {
    throw std::runtime_error(std::string(what) + ": " + pstf_last_error());
}

void check(int rc, const char *what) {
    if (rc != PSTF_OK) fail(what);
}

pstf_key toC(const SpatioDirectionalKey &k) {
    pstf_key o;
    o.level = k.level;
    for (int i = 0; i < 3; ++i) o.cell[i] = k.cell[i];
    o.dir_cell[0] = k.dirCell[0];
    o.dir_cell[1] = k.dirCell[1];
    o.checksum = k.checksum;
    return o;
}

SpatioDirectionalKey fromC(const pstf_key &k) {
    SpatioDirectionalKey o;
    o.level = k.level;
    for (int i = 0; i < 3; ++i) o.cell[i] = k.cell[i];
    o.dirCell[0] = k.dir_cell[0];
    o.dirCell[1] = k.dir_cell[1];
    o.checksum = k.checksum;
    return o;
}

} // namespace

// (lENext + lTildeNext) * f * ratio etc., same association as the reference (field.cpp:13-25)
RGB computeUpdateValue(FieldKind kind, const RGB &lTildeNext, const RGB &lENext, const RGB &f,
                       double ratio) {
    switch (kind) {
    case FieldKind::Lo:
    case FieldKind::LoMinusE:
        return (lENext + lTildeNext) * f * ratio;
    case FieldKind::Li:
        return lTildeNext * ratio;
    case FieldKind::FLi:
        return lTildeNext * f * ratio;
    }
    throw std::runtime_error("computeUpdateValue: unknown field kind");
}

struct FieldStore::Impl {
    pstf_field *h = nullptr;
    std::mutex mu;
    std::vector<pstf_key> keys;
    std::vector<double> rgb, w;
    std::vector<uint8_t> isCounter;
};

FieldStore::FieldStore(const FieldStoreConfig &config) : m_config(config), m_impl(new Impl) {
    pstf_field_config c;
    std::memset(&c, 0, sizeof(c));
    c.kind = uint32_t(config.kind);
    c.capacity_log2 = config.capacityLog2;
    c.max_level = config.maxLevel;
    c.base_cell_size = config.baseCellSize;
    c.level_select_k = config.levelSelectK;
    c.t_max = config.tMax;
    c.blend = config.blend == FieldStoreConfig::Blend::Sqrt ? PSTF_BLEND_SQRT : PSTF_BLEND_LINEAR;
    c.technique_mask = config.techniqueMask;
    c.probe_window = config.probeWindow;
    c.evict_age_frames = config.evictAgeFrames;
    check(pstf_field_create(&c, 0, &m_impl->h), "pstf_field_create");
}

FieldStore::~FieldStore() {
    if (m_impl && m_impl->h) pstf_field_destroy(m_impl->h);
}

void *FieldStore::nativeHandle() const {
    flush();
    return m_impl->h;
}

void FieldStore::flush() const {
    Impl &s = *m_impl;
    std::lock_guard<std::mutex> lk(s.mu);
    if (s.keys.empty()) return;
    check(pstf_field_apply_host(s.h, s.keys.data(), s.rgb.data(), s.w.data(), s.isCounter.data(),
                                s.keys.size(), PSTF_MODE_SEQUENTIAL),
          "pstf_field_apply_host");
    s.keys.clear();
    s.rgb.clear();
    s.w.clear();
    s.isCounter.clear();
}

int FieldStore::selectLevel(double footprint) const {
    int32_t l = 0;
    check(pstf_select_level_host(m_impl->h, &footprint, &l, 1), "pstf_select_level_host");
    return l;
}

double FieldStore::cellSize(int level) const {
    return m_config.baseCellSize * double(uint64_t(1) << level);
}

int FieldStore::dirResolution(int level) const { return 8 >> (level < 2 ? level : 2); }

SpatioDirectionalKey FieldStore::keyFor(const Vec3 &position, const Vec3 &direction,
                                        int level) const {
    const double p[3] = {position.x, position.y, position.z};
    const double d[3] = {direction.x, direction.y, direction.z};
    const int32_t l = level;
    pstf_key k;
    check(pstf_key_for_host(m_impl->h, p, d, &l, 1, &k), "pstf_key_for_host");
    return fromC(k);
}

void FieldStore::incrementCounter(const SpatioDirectionalKey &key, double w) {
    Impl &s = *m_impl;
    std::lock_guard<std::mutex> lk(s.mu);
    s.keys.push_back(toC(key));
    s.rgb.insert(s.rgb.end(), {0.0, 0.0, 0.0});
    s.w.push_back(w);
    s.isCounter.push_back(1);
}

void FieldStore::accumulate(const SpatioDirectionalKey &key, const RGB &value, double w) {
    Impl &s = *m_impl;
    std::lock_guard<std::mutex> lk(s.mu);
    s.keys.push_back(toC(key));
    s.rgb.insert(s.rgb.end(), {value.r, value.g, value.b});
    s.w.push_back(w);
    s.isCounter.push_back(0);
}

static FieldQueryResult query_impl(pstf_field *h, const Vec3 &position, const Vec3 &direction,
                                   const double *fp, const int32_t *level) {
    const double p[3] = {position.x, position.y, position.z};
    const double d[3] = {direction.x, direction.y, direction.z};
    double v[3];
    uint8_t valid = 0, fb = 0;
    int32_t lv = 0;
    check(pstf_field_query_host(h, p, d, fp, level, 1, v, &valid, &fb, &lv),
          "pstf_field_query_host");
    FieldQueryResult r;
    r.value = RGB(v[0], v[1], v[2]);
    r.valid = valid != 0;
    r.fallback = fb != 0;
    r.level = lv;
    return r;
}

FieldQueryResult FieldStore::query(const Vec3 &position, const Vec3 &direction,
                                   double footprint) const {
    flush();
    return query_impl(m_impl->h, position, direction, &footprint, nullptr);
}

FieldQueryResult FieldStore::queryFromLevel(const Vec3 &position, const Vec3 &direction,
                                            int level) const {
    flush();
    const int32_t l = level;
    return query_impl(m_impl->h, position, direction, nullptr, &l);
}

void FieldStore::endFrame() {
    flush();
    check(pstf_field_end_frame(m_impl->h, nullptr), "pstf_field_end_frame");
}

void FieldStore::invalidate() {
    flush();
    check(pstf_field_invalidate(m_impl->h, nullptr, nullptr), "pstf_field_invalidate");
}

void FieldStore::invalidate(const Aabb &region) {
    flush();
    const double box[6] = {region.lo.x, region.lo.y, region.lo.z,
                           region.hi.x, region.hi.y, region.hi.z};
    check(pstf_field_invalidate(m_impl->h, box, nullptr), "pstf_field_invalidate");
}

static pstf_field_stats stats_of(pstf_field *h) {
    pstf_field_stats st;
    check(pstf_field_get_stats(h, &st), "pstf_field_get_stats");
    return st;
}

uint64_t FieldStore::frameIndex() const {
    flush();
    return stats_of(m_impl->h).frame;
}
uint64_t FieldStore::rejectedUpdates() const {
    flush();
    return stats_of(m_impl->h).rejected;
}
uint64_t FieldStore::droppedInserts() const {
    flush();
    return stats_of(m_impl->h).dropped;
}
uint64_t FieldStore::internalErrors() const {
    flush();
    return stats_of(m_impl->h).internal_errors;
}
size_t FieldStore::liveCellCount() const {
    flush();
    return size_t(stats_of(m_impl->h).live);
}

RGB FieldStore::weightedMeanValue() const {
    flush();
    double out[3];
    check(pstf_field_weighted_mean(m_impl->h, out), "pstf_field_weighted_mean");
    return RGB(out[0], out[1], out[2]);
}

void FieldStore::dumpSnapshot(const std::string &path) const {
    flush();
    check(pstf_field_dump_snapshot(m_impl->h, path.c_str()), "dumpSnapshot");
}

void FieldStore::loadSnapshot(const std::string &path) {
    flush();
    check(pstf_field_load_snapshot(m_impl->h, path.c_str()), "loadSnapshot");
}

std::vector<FieldStore::SnapshotRecord> FieldStore::readSnapshot(const std::string &path) {
    uint64_t n = 0;
    check(pstf_read_snapshot(path.c_str(), nullptr, 0, &n, nullptr), "readSnapshot");
    std::vector<pstf_snapshot_record> raw(n);
    check(pstf_read_snapshot(path.c_str(), raw.data(), n, &n, nullptr), "readSnapshot");
    std::vector<SnapshotRecord> out(n);
    for (uint64_t i = 0; i < n; ++i) {
        SnapshotRecord &r = out[i];
        r.level = raw[i].level;
        for (int c = 0; c < 3; ++c) {
            r.cell[c] = raw[i].cell[c];
            r.value[c] = raw[i].value[c];
        }
        r.dirCell[0] = raw[i].dir_cell[0];
        r.dirCell[1] = raw[i].dir_cell[1];
        r.checksum = raw[i].checksum;
        r.cOld = raw[i].c_old;
    }
    return out;
}

void FieldUpdateQueue::append(FieldUpdateQueue &&other) {
    m_items.insert(m_items.end(), other.m_items.begin(), other.m_items.end());
    other.m_items.clear();
}

void FieldUpdateQueue::apply(FieldStore &store) {
    store.flush();
    const size_t n = m_items.size();
    if (n) {
        std::vector<pstf_key> keys(n);
        std::vector<double> rgb(3 * n), w(n);
        std::vector<uint8_t> isc(n);
        for (size_t i = 0; i < n; ++i) {
            keys[i] = toC(m_items[i].key);
            rgb[3 * i] = m_items[i].value.r;
            rgb[3 * i + 1] = m_items[i].value.g;
            rgb[3 * i + 2] = m_items[i].value.b;
            w[i] = m_items[i].w;
            isc[i] = m_items[i].isCounter ? 1 : 0;
        }
        check(pstf_field_apply_host(store.m_impl->h, keys.data(), rgb.data(), w.data(), isc.data(),
                                    n, PSTF_MODE_ORDERED),
              "FieldUpdateQueue::apply");
    }
    m_items.clear();
}

} // namespace pstf
