// C++ drop-in facade: pstf::FieldStore / FieldUpdateQueue (reference field.h) implemented over
// the B200 C ABI (include/pstf_field.h).  Updates, placement, blends, invalidation, statistics
// and snapshots run in the sm_100a library.  The per-vertex scalar calls of unmodified reference
// callers (estimators.cpp:165-206) are served without a device round trip each:
//   * keyFor / selectLevel evaluate the library's key math (csrc/pstf_keys.cuh, the exact path:
//     bitwise the reference's, tests/test_keys_host.py) on the calling thread;
//   * incrementCounter / accumulate are staged and applied in submission order (SEQUENTIAL
//     mode) before anything observes the store;
//   * query / queryFromLevel read a host mirror of the committed state, refreshed once after
//     each endFrame / invalidate / loadSnapshot: queries see committed state only
//     (field.h:73-75), which changes nowhere else.
#include "pstf/field.h"

#include <cstring>
#include <stdexcept>

#include "../../include/pstf_field.h"
#include "../csrc/pstf_keys.cuh"

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
    pstf_b200::KeyParams kp;
    uint32_t mask = 0, window = 32;
    /* committed-state mirror */
    std::mutex mirror_mu;
    std::atomic<bool> mirror_ok{false};
    std::vector<uint32_t> chk;
    std::vector<double> com; /* 4 per slot */
    void refresh() {
        if (mirror_ok.load(std::memory_order_acquire)) return;
        std::lock_guard<std::mutex> lk(mirror_mu);
        if (mirror_ok.load(std::memory_order_relaxed)) return;
        chk.resize(size_t(mask) + 1);
        com.resize(4 * (size_t(mask) + 1));
        check(pstf_field_committed_host(h, chk.data(), com.data()), "pstf_field_committed_host");
        mirror_ok.store(true, std::memory_order_release);
    }
    void invalidate_mirror() { mirror_ok.store(false, std::memory_order_release); }
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
    m_impl->kp.base_cell_size = config.baseCellSize;
    m_impl->kp.level_select_k = config.levelSelectK;
    m_impl->kp.max_level = config.maxLevel;
    m_impl->mask = uint32_t((uint64_t(1) << config.capacityLog2) - 1);
    m_impl->window = config.probeWindow;
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

int FieldStore::selectLevel(double footprint) const { /* field.cpp:68-76 */
    return pstf_b200::select_level(m_impl->kp, footprint);
}

double FieldStore::cellSize(int level) const {
    return m_config.baseCellSize * double(uint64_t(1) << level);
}

int FieldStore::dirResolution(int level) const { return 8 >> (level < 2 ? level : 2); }

SpatioDirectionalKey FieldStore::keyFor(const Vec3 &position, const Vec3 &direction,
                                        int level) const { /* field.cpp:86-101 */
    const pstf_b200::Key k = pstf_b200::key_for(m_impl->kp, position.x, position.y, position.z,
                                                direction.x, direction.y, direction.z, level);
    SpatioDirectionalKey o;
    o.level = k.level;
    for (int i = 0; i < 3; ++i) o.cell[i] = k.cell[i];
    o.dirCell[0] = k.dir[0];
    o.dirCell[1] = k.dir[1];
    o.checksum = k.checksum;
    return o;
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

/* queryFromLevel (field.cpp:179-195) on the committed-state mirror: findSlot's linear probe
 * (checksum identity, stop at an empty slot) at each level up to maxLevel */
static FieldQueryResult query_mirror(FieldStore::Impl &s, int maxLevel, const Vec3 &position,
                                     const Vec3 &direction, int level) {
    s.refresh();
    FieldQueryResult r;
    r.level = level;
    for (int l = level; l <= maxLevel; ++l) {
        const pstf_b200::Key k = pstf_b200::key_for(s.kp, position.x, position.y, position.z,
                                                    direction.x, direction.y, direction.z, l);
        const uint32_t home = k.pack_lo & s.mask;
        for (uint32_t i = 0; i < s.window; ++i) {
            const uint32_t idx = (home + i) & s.mask;
            const uint32_t c = s.chk[idx];
            if (c == 0) break;
            if (c != k.checksum) continue;
            const double *cv = &s.com[4 * size_t(idx)];
            if (cv[3] > 0.0) {
                r.value = RGB(cv[0], cv[1], cv[2]);
                r.valid = true;
                r.fallback = l != level;
                r.level = l;
                return r;
            }
            break;
        }
    }
    return r;
}

FieldQueryResult FieldStore::query(const Vec3 &position, const Vec3 &direction,
                                   double footprint) const {
    return query_mirror(*m_impl, m_config.maxLevel, position, direction, selectLevel(footprint));
}

FieldQueryResult FieldStore::queryFromLevel(const Vec3 &position, const Vec3 &direction,
                                            int level) const {
    return query_mirror(*m_impl, m_config.maxLevel, position, direction, level);
}

void FieldStore::endFrame() {
    flush();
    check(pstf_field_end_frame(m_impl->h, nullptr), "pstf_field_end_frame");
    m_impl->invalidate_mirror();
}

void FieldStore::invalidate() {
    flush();
    check(pstf_field_invalidate(m_impl->h, nullptr, nullptr), "pstf_field_invalidate");
    m_impl->invalidate_mirror();
}

void FieldStore::invalidate(const Aabb &region) {
    flush();
    const double box[6] = {region.lo.x, region.lo.y, region.lo.z,
                           region.hi.x, region.hi.y, region.hi.z};
    check(pstf_field_invalidate(m_impl->h, box, nullptr), "pstf_field_invalidate");
    m_impl->invalidate_mirror();
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
    m_impl->invalidate_mirror();
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
