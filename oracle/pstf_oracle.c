/*
 * pstf_oracle.c — CPU restatement of the PSTF field cache (TEST INFRASTRUCTURE ONLY).
 * See pstf_oracle.h for the scope and the rule that the product never uses this file.
 * Compiled with -O2 -ffp-contract=off and no -march, like the reference build
 * (proj/CMakeLists.txt:1-8), so no FMA contraction changes the arithmetic.
 */
#define _GNU_SOURCE
#include "pstf_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "../paper_2005_07547_b200/csrc/pstf_synth.h"

#define PO_PI 3.14159265358979323846 /* vecmath.h:11 kPi */

struct po_store {
    po_config cfg;
    uint32_t mask;
    po_slot *slots;
    uint64_t frame, rejected, dropped, internal_errors;
};

/* x86-64 cvttsd2si semantics of the reference's int32_t(double) casts: NaN and out-of-range
 * give INT32_MIN (the "integer indefinite" value). field.cpp:74,91-97 */
static int32_t po_i32(double x) {
    if (!(x >= -2147483648.0 && x < 2147483648.0))
        return INT32_MIN;
    return (int32_t)x;
}

/* rng.h:61-68 */
uint64_t po_mix_bits(uint64_t v) {
    v ^= v >> 30;
    v *= 0xbf58476d1ce4e5b9ULL;
    v ^= v >> 27;
    v *= 0x94d049bb133111ebULL;
    v ^= v >> 31;
    return v;
}

/* field.cpp:38-44 */
uint64_t po_pack_key_fields(const po_key *k) {
    uint64_t h = (uint64_t)(uint32_t)k->level;
    h = po_mix_bits(h ^ (((uint64_t)(uint32_t)k->cell[0] << 32) | (uint32_t)k->cell[1]));
    h = po_mix_bits(h ^ (((uint64_t)(uint32_t)k->cell[2] << 32) | (uint32_t)k->dir[0]));
    h = po_mix_bits(h ^ (uint64_t)(uint32_t)k->dir[1]);
    return h;
}

/* field.cpp:68-76 */
int po_select_level(const po_config *c, double footprint) {
    if (!(footprint > 0.0))
        return 0;
    double scaled = footprint * c->level_select_k / c->base_cell_size;
    if (scaled <= 1.0)
        return 0;
    int level = po_i32(floor(log2(scaled)));
    if (level < 0) level = 0;               /* std::max(level, 0) */
    return level < c->max_level ? level : c->max_level; /* std::min(.., maxLevel) */
}

/* field.cpp:78-80 */
double po_cell_size(const po_config *c, int level) {
    return c->base_cell_size * (double)((uint64_t)1 << level);
}

/* field.cpp:82-84 */
int po_dir_resolution(int level) { return 8 >> (level < 2 ? level : 2); }

/* mappings.h:33-51 */
void po_sphere_to_square(const double dir[3], double uv[2]) {
    double x = fabs(dir[0]), y = fabs(dir[1]), z = fabs(dir[2]);
    double omz = 1.0 - z;
    double r = sqrt((0.0 < omz) ? omz : 0.0); /* safeSqrt = sqrt(std::max(0.0, x)) vecmath.h:22 */
    double phi = (x == 0.0 && y == 0.0) ? 0.0 : atan2(y, x) * (2.0 / PO_PI);
    double v = phi * r;
    double u = r - v;
    if (dir[2] < 0.0) {
        double t = u;
        u = v;
        v = t;
        u = 1.0 - u;
        v = 1.0 - v;
    }
    u = copysign(u, dir[0]);
    v = copysign(v, dir[1]);
    uv[0] = 0.5 * (u + 1.0);
    uv[1] = 0.5 * (v + 1.0);
}

/* field.cpp:86-101 */
po_key po_key_for(const po_config *c, const double pos[3], const double dir[3], int level) {
    po_key k;
    k.level = level;
    double cs = po_cell_size(c, level);
    for (int i = 0; i < 3; ++i)
        k.cell[i] = po_i32(floor(pos[i] / cs));
    int d = po_dir_resolution(level);
    double uv[2];
    po_sphere_to_square(dir, uv);
    for (int i = 0; i < 2; ++i) {
        int32_t q = po_i32(uv[i] * d);
        k.dir[i] = q < d - 1 ? q : d - 1; /* std::min(int32(uv*d), d-1) */
    }
    uint32_t sum = (uint32_t)po_mix_bits(po_pack_key_fields(&k) ^ 0x5bf03635ULL);
    k.checksum = sum == 0 ? 1u : sum;
    return k;
}

uint32_t po_home_slot(const po_key *k, uint32_t mask) {
    return (uint32_t)po_pack_key_fields(k) & mask; /* field.cpp:104,117 */
}

/* field.cpp:229-233 */
po_store *po_store_create(const po_config *c) {
    po_store *s = (po_store *)calloc(1, sizeof(po_store));
    s->cfg = *c;
    size_t cap = (size_t)1 << c->capacity_log2;
    s->mask = (uint32_t)(cap - 1);
    s->slots = (po_slot *)calloc(cap, sizeof(po_slot));
    return s;
}

void po_store_destroy(po_store *s) {
    if (!s) return;
    free(s->slots);
    free(s);
}

const po_config *po_store_config(const po_store *s) { return &s->cfg; }

/* field.cpp:103-114 */
static int po_find_slot(const po_store *s, const po_key *k) {
    uint32_t start = (uint32_t)po_pack_key_fields(k) & s->mask;
    for (uint32_t i = 0; i < s->cfg.probe_window; ++i) {
        uint32_t idx = (start + i) & s->mask;
        uint32_t sum = s->slots[idx].checksum;
        if (sum == k->checksum) return (int)idx;
        if (sum == 0) return -1;
    }
    return -1;
}

/* field.cpp:116-146 (single-threaded: the CAS always succeeds on an empty slot) */
static int po_find_or_insert(po_store *s, const po_key *k) {
    uint32_t start = (uint32_t)po_pack_key_fields(k) & s->mask;
    for (uint32_t i = 0; i < s->cfg.probe_window; ++i) {
        uint32_t idx = (start + i) & s->mask;
        po_slot *sl = &s->slots[idx];
        if (sl->checksum == k->checksum) {
            sl->last_touched = (uint32_t)s->frame;
            return (int)idx;
        }
        if (sl->checksum == 0) {
            sl->checksum = k->checksum;
            sl->level = k->level;
            memcpy(sl->cell, k->cell, sizeof(sl->cell));
            memcpy(sl->dir, k->dir, sizeof(sl->dir));
            sl->last_touched = (uint32_t)s->frame;
            return (int)idx;
        }
    }
    s->dropped++;
    return -1;
}

/* field.cpp:148-158 */
void po_increment_counter(po_store *s, const po_key *k, double w) {
    if (!(w >= 0.0) || !isfinite(w)) {
        s->rejected++;
        return;
    }
    int idx = po_find_or_insert(s, k);
    if (idx < 0) return;
    if (w > 0.0) s->slots[idx].c_new += w;
}

/* field.cpp:160-172 */
void po_accumulate(po_store *s, const po_key *k, const double value[3], double w) {
    if (!(isfinite(value[0]) && isfinite(value[1]) && isfinite(value[2])) || !isfinite(w) ||
        w < 0.0) {
        s->rejected++;
        return;
    }
    int idx = po_find_or_insert(s, k);
    if (idx < 0) return;
    po_slot *sl = &s->slots[idx];
    sl->accum[0] += value[0] * w;
    sl->accum[1] += value[1] * w;
    sl->accum[2] += value[2] * w;
}

/* field.cpp:179-195 */
po_query_result po_query_from_level(const po_store *s, const double pos[3], const double dir[3],
                                    int level) {
    po_query_result r;
    memset(&r, 0, sizeof(r));
    for (int l = level; l <= s->cfg.max_level; ++l) {
        po_key k = po_key_for(&s->cfg, pos, dir, l);
        int idx = po_find_slot(s, &k);
        if (idx >= 0 && s->slots[idx].c_old > 0.0) {
            memcpy(r.value, s->slots[idx].value_old, sizeof(r.value));
            r.valid = 1;
            r.fallback = l != level;
            r.level = l;
            return r;
        }
    }
    r.level = level;
    return r;
}

/* field.cpp:174-177 */
po_query_result po_query(const po_store *s, const double pos[3], const double dir[3],
                         double footprint) {
    return po_query_from_level(s, pos, dir, po_select_level(&s->cfg, footprint));
}

/* field.cpp:197-263 */
void po_end_frame(po_store *s) {
    size_t capacity = (size_t)s->mask + 1;
    double cNewSum = 0.0;
    size_t touched = 0, live = 0;
    for (size_t i = 0; i < capacity; ++i) {
        po_slot *sl = &s->slots[i];
        if (sl->checksum == 0) continue;
        ++live;
        double cn = sl->c_new;
        if (cn > 0.0) {
            cNewSum += cn;
            ++touched;
        }
    }
    double meanCNew = touched > 0 ? cNewSum / (double)touched : 0.0;
    int limited = s->cfg.t_max > 0.0 && isfinite(s->cfg.t_max);
    double tMax = s->cfg.t_max;
    double cOldCap = limited ? (tMax * tMax - tMax) * meanCNew : 0.0;

    for (size_t i = 0; i < capacity; ++i) {
        po_slot *sl = &s->slots[i];
        if (sl->checksum == 0) continue;
        double cn = sl->c_new;
        double a0 = sl->accum[0], a1 = sl->accum[1], a2 = sl->accum[2];
        if (cn > 0.0) {
            double cand[3] = {a0 / cn, a1 / cn, a2 / cn};
            double alpha = s->cfg.blend == 0 ? sqrt(cn / (sl->c_old + cn)) : cn / (sl->c_old + cn);
            if (limited) {
                double fl = 1.0 / tMax;
                alpha = (alpha < fl) ? fl : alpha; /* std::max(alpha, 1/tMax) */
            }
            for (int c = 0; c < 3; ++c)
                sl->value_old[c] = sl->value_old[c] * (1.0 - alpha) + cand[c] * alpha;
            sl->c_old += cn;
            if (limited) sl->c_old = (cOldCap < sl->c_old) ? cOldCap : sl->c_old; /* std::min */
        } else if (!(a0 == 0.0 && a1 == 0.0 && a2 == 0.0)) {
            s->internal_errors++;
        }
        sl->c_new = 0.0;
        sl->accum[0] = sl->accum[1] = sl->accum[2] = 0.0;
    }

    if (live * 4 > capacity * 3) {
        for (size_t i = 0; i < capacity; ++i) {
            po_slot *sl = &s->slots[i];
            if (sl->checksum == 0) continue;
            uint32_t age = (uint32_t)s->frame - sl->last_touched;
            if (age >= s->cfg.evict_age_frames) {
                sl->checksum = 0;
                sl->value_old[0] = sl->value_old[1] = sl->value_old[2] = 0.0;
                sl->c_old = 0.0;
            }
        }
    }
    ++s->frame;
}

/* field.cpp:265-270 */
void po_invalidate_all(po_store *s) {
    size_t capacity = (size_t)s->mask + 1;
    for (size_t i = 0; i < capacity; ++i)
        if (s->slots[i].checksum != 0) s->slots[i].c_old = 0.0;
}

/* field.cpp:272-284, Aabb::contains vecmath.h:107-109 */
void po_invalidate_box(po_store *s, const double lo[3], const double hi[3]) {
    size_t capacity = (size_t)s->mask + 1;
    for (size_t i = 0; i < capacity; ++i) {
        po_slot *sl = &s->slots[i];
        if (sl->checksum == 0) continue;
        double cs = po_cell_size(&s->cfg, sl->level);
        double c[3];
        for (int k = 0; k < 3; ++k) c[k] = (sl->cell[k] + 0.5) * cs;
        if (c[0] >= lo[0] && c[0] <= hi[0] && c[1] >= lo[1] && c[1] <= hi[1] && c[2] >= lo[2] &&
            c[2] <= hi[2])
            sl->c_old = 0.0;
    }
}

void po_stats_get(const po_store *s, po_stats *out) {
    size_t capacity = (size_t)s->mask + 1, live = 0;
    for (size_t i = 0; i < capacity; ++i) /* field.cpp:286-291 liveCellCount */
        if (s->slots[i].checksum != 0) ++live;
    out->frame = s->frame;
    out->rejected = s->rejected;
    out->dropped = s->dropped;
    out->internal_errors = s->internal_errors;
    out->live = live;
}

/* field.cpp:293-306 */
void po_weighted_mean(const po_store *s, double out[3]) {
    size_t capacity = (size_t)s->mask + 1;
    double sum[3] = {0.0, 0.0, 0.0}, weight = 0.0;
    for (size_t i = 0; i < capacity; ++i) {
        const po_slot *sl = &s->slots[i];
        if (sl->checksum == 0 || sl->c_old <= 0.0) continue;
        for (int c = 0; c < 3; ++c) sum[c] += sl->value_old[c] * sl->c_old;
        weight += sl->c_old;
    }
    for (int c = 0; c < 3; ++c) out[c] = weight > 0.0 ? sum[c] / weight : 0.0;
}

void po_slots(const po_store *s, po_slot *out) {
    memcpy(out, s->slots, ((size_t)s->mask + 1) * sizeof(po_slot));
}

static int po_key_cmp(const int32_t *a, const int32_t *b) {
    /* lexicographic (level, cell0, cell1, cell2, dir0, dir1), signed (field.cpp:334-337) */
    for (int i = 0; i < 6; ++i) {
        if (a[i] < b[i]) return -1;
        if (a[i] > b[i]) return 1;
    }
    return 0;
}

static int po_snap_cmp(const void *pa, const void *pb) {
    const po_snapshot_record *a = (const po_snapshot_record *)pa, *b = (const po_snapshot_record *)pb;
    int32_t ka[6] = {a->level, a->cell[0], a->cell[1], a->cell[2], a->dir[0], a->dir[1]};
    int32_t kb[6] = {b->level, b->cell[0], b->cell[1], b->cell[2], b->dir[0], b->dir[1]};
    return po_key_cmp(ka, kb);
}

/* field.cpp:311-337 (records; the file framing lives in the reference / product writers) */
size_t po_snapshot(const po_store *s, po_snapshot_record *out, size_t cap) {
    size_t capacity = (size_t)s->mask + 1, n = 0;
    for (size_t i = 0; i < capacity; ++i) {
        const po_slot *sl = &s->slots[i];
        if (sl->checksum == 0) continue;
        if (n < cap) {
            po_snapshot_record *r = &out[n];
            r->level = sl->level;
            memcpy(r->cell, sl->cell, sizeof(r->cell));
            memcpy(r->dir, sl->dir, sizeof(r->dir));
            r->checksum = sl->checksum;
            memcpy(r->value, sl->value_old, sizeof(r->value));
            r->c_old = sl->c_old;
        }
        ++n;
    }
    size_t m = n < cap ? n : cap;
    qsort(out, m, sizeof(po_snapshot_record), po_snap_cmp);
    return m;
}

/* Snapshot restore (no reference counterpart: field.cpp:311-386 only writes/reads the file; the
 * semantics are those of include/pstf_field.h pstf_field_restore).  Records in ascending key
 * order (stable: ties keep input order), each inserted by findOrInsertSlot (field.cpp:116-146),
 * then valueOld/cOld set at the slot it returned; later records overwrite earlier ones. */
typedef struct {
    const po_snapshot_record *r;
    size_t i;
} po_snap_ref;

static int po_snap_ref_cmp(const void *pa, const void *pb) {
    const po_snap_ref *a = (const po_snap_ref *)pa, *b = (const po_snap_ref *)pb;
    int c = po_snap_cmp(a->r, b->r);
    if (c) return c;
    return a->i < b->i ? -1 : (a->i > b->i ? 1 : 0);
}

void po_restore(po_store *s, const po_snapshot_record *recs, size_t n) {
    po_snap_ref *ord = (po_snap_ref *)malloc((n ? n : 1) * sizeof(po_snap_ref));
    for (size_t i = 0; i < n; ++i) {
        ord[i].r = &recs[i];
        ord[i].i = i;
    }
    qsort(ord, n, sizeof(po_snap_ref), po_snap_ref_cmp);
    for (size_t j = 0; j < n; ++j) {
        const po_snapshot_record *r = ord[j].r;
        po_key k;
        k.level = r->level;
        memcpy(k.cell, r->cell, sizeof(k.cell));
        memcpy(k.dir, r->dir, sizeof(k.dir));
        k.checksum = r->checksum;
        int idx = po_find_or_insert(s, &k);
        if (idx < 0) continue;
        memcpy(s->slots[idx].value_old, r->value, sizeof(r->value));
        s->slots[idx].c_old = r->c_old;
    }
    free(ord);
}

static uint64_t po_bits(double v) {
    uint64_t b;
    memcpy(&b, &v, sizeof(b));
    return b;
}

/* field.cpp:402-411 comparator */
static int po_update_cmp(const void *pa, const void *pb) {
    const po_update *a = (const po_update *)pa, *b = (const po_update *)pb;
    int32_t ka[6] = {a->key.level, a->key.cell[0], a->key.cell[1], a->key.cell[2], a->key.dir[0],
                     a->key.dir[1]};
    int32_t kb[6] = {b->key.level, b->key.cell[0], b->key.cell[1], b->key.cell[2], b->key.dir[0],
                     b->key.dir[1]};
    int c = po_key_cmp(ka, kb);
    if (c) return c;
    int ia = a->is_counter != 0, ib = b->is_counter != 0;
    if (ia != ib) return ia < ib ? -1 : 1;
    uint64_t xa[4] = {po_bits(a->value[0]), po_bits(a->value[1]), po_bits(a->value[2]), po_bits(a->w)};
    uint64_t xb[4] = {po_bits(b->value[0]), po_bits(b->value[1]), po_bits(b->value[2]), po_bits(b->w)};
    for (int i = 0; i < 4; ++i) {
        if (xa[i] < xb[i]) return -1;
        if (xa[i] > xb[i]) return 1;
    }
    return 0;
}

/* field.cpp:396-420 */
void po_queue_apply(po_store *s, po_update *u, size_t n) {
    qsort(u, n, sizeof(po_update), po_update_cmp);
    for (size_t i = 0; i < n; ++i) {
        if (u[i].is_counter)
            po_increment_counter(s, &u[i].key, u[i].w);
        else
            po_accumulate(s, &u[i].key, u[i].value, u[i].w);
    }
}

/* ---- FieldRecorder::onVertex restatement (estimators.cpp:194-262) ---- */

typedef struct {
    po_update *u;
    size_t n, cap;
} po_queue;

static void po_q_push(po_queue *q, const po_key *k, const double v[3], double w, int is_counter) {
    if (q->n == q->cap) {
        q->cap = q->cap ? q->cap * 2 : 1024;
        q->u = (po_update *)realloc(q->u, q->cap * sizeof(po_update));
    }
    po_update *x = &q->u[q->n++];
    x->key = *k;
    if (v) memcpy(x->value, v, sizeof(x->value));
    else x->value[0] = x->value[1] = x->value[2] = 0.0;
    x->w = w;
    x->is_counter = is_counter;
}

/* WorkerSink::increment/accumulate estimators.cpp:165-178 */
static void po_sink_inc(po_store *s, po_queue *q, const po_key *k, double w) {
    if (q) po_q_push(q, k, NULL, w, 1);
    else po_increment_counter(s, k, w);
}
static void po_sink_acc(po_store *s, po_queue *q, const po_key *k, const double v[3], double w) {
    if (q) po_q_push(q, k, v, w, 0);
    else po_accumulate(s, k, v, w);
}

#define PO_TECH_CONT 2u /* field.h:24 */
#define PO_TECH_NEE 4u  /* field.h:25 */

void po_vertex_pass(po_store *lo, po_store *loe, po_store *fli, po_store *li,
                    const double *const F[34], const uint32_t *flags, size_t n,
                    uint32_t loe_mask, uint32_t fli_mask, int deterministic) {
    po_queue qLo = {0}, qLoe = {0}, qFli = {0}, qLi = {0};
    po_queue *pLo = deterministic ? &qLo : NULL, *pLoe = deterministic ? &qLoe : NULL;
    po_queue *pFli = deterministic ? &qFli : NULL, *pLi = deterministic ? &qLi : NULL;
    for (size_t i = 0; i < n; ++i) {
#define G(k) F[k][i]
        double pos[3] = {G(PS_POS), G(PS_POS + 1), G(PS_POS + 2)};
        double wo[3] = {G(PS_WO), G(PS_WO + 1), G(PS_WO + 2)};
        double wi[3] = {G(PS_WI), G(PS_WI + 1), G(PS_WI + 2)};
        double npos[3] = {G(PS_NPOS), G(PS_NPOS + 1), G(PS_NPOS + 2)};
        double ndir[3] = {G(PS_NDIR), G(PS_NDIR + 1), G(PS_NDIR + 2)};
        double emis[3] = {G(PS_EMIS), G(PS_EMIS + 1), G(PS_EMIS + 2)};
        double f[3] = {G(PS_F), G(PS_F + 1), G(PS_F + 2)};
        double nemis[3] = {G(PS_NEMIS), G(PS_NEMIS + 1), G(PS_NEMIS + 2)};
        double neeLoe[3] = {G(PS_NEELOE), G(PS_NEELOE + 1), G(PS_NEELOE + 2)};
        double neeFli[3] = {G(PS_NEEFLI), G(PS_NEEFLI + 1), G(PS_NEEFLI + 2)};
        double footprint = G(PS_FP), nfp = G(PS_NFP), ratio = G(PS_RATIO), nmis = G(PS_NMIS);
#undef G
        uint32_t fl = flags[i];
        int contExtended = (fl & PS_FLAG_CONT) != 0;
        int nextIsSurface = (fl & PS_FLAG_NEXT_SURF) != 0;
        int neeSampled = (fl & PS_FLAG_NEE) != 0;

        int level = po_select_level(&lo->cfg, footprint); /* 195 */
        double loNext[3] = {0, 0, 0}, loeNext[3] = {0, 0, 0};
        if (contExtended) { /* 198-211 */
            if (nextIsSurface) {
                double woNext[3] = {-wi[0], -wi[1], -wi[2]};
                po_query_result q1 = po_query(lo, npos, woNext, nfp);
                if (q1.valid) memcpy(loNext, q1.value, sizeof(loNext));
                po_query_result q2 = po_query(loe, npos, woNext, nfp);
                if (q2.valid) memcpy(loeNext, q2.value, sizeof(loeNext));
            } else {
                memcpy(loNext, nemis, sizeof(loNext));
            }
        }
        /* ratio = rec.transportRatio() is precomputed in the record (pathtracer.h:86-89) */

        po_key loKey = po_key_for(&lo->cfg, pos, wo, level); /* 215-221 */
        po_sink_inc(lo, pLo, &loKey, 1.0);
        po_sink_acc(lo, pLo, &loKey, emis, 1.0);
        if (contExtended && ratio > 0.0) {
            double upd[3]; /* computeUpdateValue(Lo, loNext, 0, f, ratio) field.cpp:17-18 */
            for (int c = 0; c < 3; ++c) upd[c] = ((0.0 + loNext[c]) * f[c]) * ratio;
            po_sink_acc(lo, pLo, &loKey, upd, 1.0);
        }

        po_key loeKey = po_key_for(&loe->cfg, pos, wo, level); /* 226-234 */
        po_sink_inc(loe, pLoe, &loeKey, 1.0);
        if (contExtended && ratio > 0.0 && (loe_mask & PO_TECH_CONT)) {
            double upd[3];
            for (int c = 0; c < 3; ++c) upd[c] = ((nemis[c] * nmis + loeNext[c]) * f[c]) * ratio;
            po_sink_acc(loe, pLoe, &loeKey, upd, 1.0);
        }
        if (neeSampled && (loe_mask & PO_TECH_NEE)) po_sink_acc(loe, pLoe, &loeKey, neeLoe, 1.0);

        double lIn[3]; /* 237 */
        for (int c = 0; c < 3; ++c) lIn[c] = nemis[c] * nmis + loeNext[c];

        if (contExtended) { /* 241-246 */
            po_key k = po_key_for(&fli->cfg, pos, wi, level);
            po_sink_inc(fli, pFli, &k, 1.0);
            if (fli_mask & PO_TECH_CONT) {
                double v[3] = {f[0] * lIn[0], f[1] * lIn[1], f[2] * lIn[2]};
                po_sink_acc(fli, pFli, &k, v, 1.0);
            }
        }
        if (neeSampled) { /* 247-254 */
            po_key k = po_key_for(&fli->cfg, pos, ndir, level);
            po_sink_inc(fli, pFli, &k, 1.0);
            if (fli_mask & PO_TECH_NEE) po_sink_acc(fli, pFli, &k, neeFli, 1.0);
        }
        if (li && contExtended) { /* 256-261 */
            po_key k = po_key_for(&li->cfg, pos, wi, level);
            po_sink_inc(li, pLi, &k, 1.0);
            double v[3] = {lIn[0] * 1.0, lIn[1] * 1.0, lIn[2] * 1.0};
            po_sink_acc(li, pLi, &k, v, 1.0);
        }
    }
    if (deterministic) { /* estimators.cpp:610-623 */
        po_queue_apply(lo, qLo.u, qLo.n);
        po_queue_apply(loe, qLoe.u, qLoe.n);
        po_queue_apply(fli, qFli.u, qFli.n);
        if (li) po_queue_apply(li, qLi.u, qLi.n);
    }
    free(qLo.u);
    free(qLoe.u);
    free(qFli.u);
    free(qLi.u);
}

void po_vertex_pass_contig(po_store *lo, po_store *loe, po_store *fli, po_store *li,
                           const double *buf, size_t n, uint32_t loe_mask, uint32_t fli_mask,
                           int deterministic) {
    const double *F[34];
    for (int k = 0; k < 34; ++k) F[k] = buf + (size_t)k * n;
    const uint32_t *flags = (const uint32_t *)(buf + (size_t)34 * n);
    po_vertex_pass(lo, loe, fli, li, F, flags, n, loe_mask, fli_mask, deterministic);
}

/* ---- host synthetic generator (threads over paths) ---- */
typedef struct {
    ps_params P;
    double *buf;
    uint64_t n_total, p0, p1;
} po_gen_job;

static void *po_gen_worker(void *arg) {
    po_gen_job *j = (po_gen_job *)arg;
    uint32_t *flags = (uint32_t *)(j->buf + (size_t)34 * j->n_total);
    for (uint64_t p = j->p0; p < j->p1; ++p) ps_gen_path(&j->P, p, j->buf, flags, j->n_total);
    return NULL;
}

void po_synth_generate_scene(int scene, int width, int height, int bounces, uint64_t seed,
                             uint64_t iter, double cam_shift_x, double *buf, int threads);

void po_synth_generate(int width, int height, int bounces, uint64_t seed, uint64_t iter,
                       double cam_shift_x, double *buf, int threads) {
    po_synth_generate_scene(0, width, height, bounces, seed, iter, cam_shift_x, buf, threads);
}

void po_synth_generate_scene(int scene, int width, int height, int bounces, uint64_t seed,
                             uint64_t iter, double cam_shift_x, double *buf, int threads) {
    ps_params P;
    P.glossy = scene;
    P.width = width;
    P.height = height;
    P.bounces = bounces;
    P.seed = seed;
    P.iter = iter;
    P.cam_shift_x = cam_shift_x;
    P.path0 = 0;
    P.n_local = 0;
    uint64_t n_paths = (uint64_t)width * (uint64_t)height;
    uint64_t n_total = n_paths * (uint64_t)bounces;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    po_gen_job jobs[256];
    for (int t = 0; t < threads; ++t) {
        jobs[t].P = P;
        jobs[t].buf = buf;
        jobs[t].n_total = n_total;
        jobs[t].p0 = n_paths * (uint64_t)t / (uint64_t)threads;
        jobs[t].p1 = n_paths * (uint64_t)(t + 1) / (uint64_t)threads;
        pthread_create(&th[t], NULL, po_gen_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

/* ---- batch helpers for the test harness (SoA: x[n], y[n], z[n]) ---- */
void po_key_for_batch(const po_config *c, const double *pos, const double *dir,
                      const int32_t *level, size_t n, po_key *out) {
    for (size_t i = 0; i < n; ++i) {
        double p[3] = {pos[i], pos[n + i], pos[2 * n + i]};
        double d[3] = {dir[i], dir[n + i], dir[2 * n + i]};
        out[i] = po_key_for(c, p, d, level[i]);
    }
}

void po_select_level_batch(const po_config *c, const double *fp, size_t n, int32_t *out) {
    for (size_t i = 0; i < n; ++i) out[i] = po_select_level(c, fp[i]);
}

/* value SoA [3][n]; flags SoA [3][n] = valid, fallback, level. level==NULL -> footprint */
void po_query_batch(const po_store *s, const double *pos, const double *dir, const double *fp,
                    const int32_t *level, size_t n, double *value, int32_t *flags) {
    for (size_t i = 0; i < n; ++i) {
        double p[3] = {pos[i], pos[n + i], pos[2 * n + i]};
        double d[3] = {dir[i], dir[n + i], dir[2 * n + i]};
        po_query_result r = level ? po_query_from_level(s, p, d, level[i]) : po_query(s, p, d, fp[i]);
        for (int c = 0; c < 3; ++c) value[(size_t)c * n + i] = r.value[c];
        flags[i] = r.valid;
        flags[n + i] = r.fallback;
        flags[2 * n + i] = r.level;
    }
}
