/* pstf_model_oracle.c — CPU restatement of the reference's ModelStore with DirGrid models
 * and SphericalKdTree models (TEST INFRASTRUCTURE ONLY: the checker of the B200 model store,
 * never the product path).
 *
 *   ModelStore      estimators.h:124-150, estimators.cpp:104-144
 *   DirGrid         models.h:30-52, models.cpp:16-94
 *   SphericalKdTree models.h:59-109, models.cpp:96-298
 *   Gmm             models.h:113-177, models.cpp:427-702 (state vector as the device's:
 *                   W[C], M[2C], V[3C], U[8C], cache[7C], i, underflows, reseed counter)
 *   record order    estimators.cpp:625-645 (deterministic mode: sorted, then applied in order)
 *
 * Pinned bitwise against the reference's own ModelStore compiled in place
 * (oracle/model_shim.cpp -> oracle/_ref/libpstf_model_ref.so, tests/test_oracle_pin.py).
 * The map is an open-addressing table that doubles when half full: unbounded like the
 * reference's std::unordered_map; iteration order is never observable (dumps sort by key). */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "pstf_oracle.h"

/* SphericalKdTree::Node (models.h:91-99) */
typedef struct {
    int leaf, axis;
    double split;
    int32_t left, right, parent;
    double prob, accum, mass;
} pm_node;

typedef struct {
    po_key key; /* checksum ignored: equality on the key fields (field.h:38-41) */
    double *w, *acc; /* DirGrid; Gmm: w = the state vector */
    pm_node *nodes;  /* SphericalKdTree: 2L-1 nodes */
    double *fs;      /* Gmm::m_frameSamples: (u, v, contribution) triples */
    size_t nfs, cfs;
    double total, c_old, c_new;
    uint64_t records, rec_count;
    int warm, used;
} pm_entry;

struct po_model {
    int kind; /* 0 DirGrid, 1 SphericalKdTree, 2 Gmm (ModelKind, models.h:183) */
    int comps; /* GmmConfig (models.h:113-119) */
    double alpha_em, smin, smax, reseed_frac;
    double *gtmpl; /* Gmm's constructor state */
    int leaves;
    double tsplit;
    pm_node *tmpl; /* the constructor's uniform tree */
    int res;
    double t_max;
    int min_samples;
    size_t cap, size;
    pm_entry *tab;
};

static uint64_t pm_hash(const po_key *k) { return po_pack_key_fields(k); }

static int pm_eq(const po_key *a, const po_key *b) {
    return a->level == b->level && a->cell[0] == b->cell[0] && a->cell[1] == b->cell[1] &&
           a->cell[2] == b->cell[2] && a->dir[0] == b->dir[0] && a->dir[1] == b->dir[1];
}

/* SphericalKdTree(leafCount) (models.cpp:96-127): children are appended when their parent is
 * visited, the left subtree is built first, axes alternate with depth, splits at the midpoint */
static int pm_kd_add(pm_node *t, int *n) {
    pm_node *z = &t[*n];
    memset(z, 0, sizeof(*z));
    z->leaf = 1;
    z->split = 0.5;
    z->left = z->right = z->parent = -1;
    return (*n)++;
}

static void pm_kd_build(pm_node *t, int *n, int node, int depth, int below, int leaves) {
    if (below == 1) {
        t[node].leaf = 1;
        t[node].prob = 1.0 / leaves;
        return;
    }
    int l = pm_kd_add(t, n), r = pm_kd_add(t, n);
    t[node].leaf = 0;
    t[node].axis = depth & 1;
    t[node].split = 0.5;
    t[node].left = l;
    t[node].right = r;
    t[l].parent = node;
    t[r].parent = node;
    pm_kd_build(t, n, l, depth + 1, below / 2, leaves);
    pm_kd_build(t, n, r, depth + 1, below / 2, leaves);
}

/* refreshMass (models.cpp:129-138) */
static double pm_kd_mass(pm_node *t, int n) {
    t[n].mass = t[n].leaf ? t[n].prob : pm_kd_mass(t, t[n].left) + pm_kd_mass(t, t[n].right);
    return t[n].mass;
}

#define GMM_TWO_PI (2.0 * 3.14159265358979323846) /* kTwoPi, vecmath.h:13-14 */
#define GW(S) (S)
#define GM(S, C) ((S) + (C))
#define GV(S, C) ((S) + 3 * (C))
#define GU(S, C) ((S) + 6 * (C))
#define GK(S, C) ((S) + 14 * (C))
#define GT(S, C) ((S) + 21 * (C))

/* Gmm::rebuildCache (models.cpp:449-463) */
static void pm_gmm_cache(double *S, int C, int c) {
    double a = GV(S, C)[3 * c], b = GV(S, C)[3 * c + 1], d = GV(S, C)[3 * c + 2];
    double det = a * d - b * b;
    double *k = GK(S, C) + 7 * c;
    k[0] = d / det;
    k[1] = -b / det;
    k[2] = a / det;
    k[3] = 1.0 / (GMM_TWO_PI * sqrt(det));
    k[4] = sqrt(a);
    k[5] = b / k[4];
    double r = d - k[5] * k[5];
    k[6] = sqrt(r < 0.0 ? 0.0 : r);
}

po_model *po_model_create(int kind, int res, int leaves, double tsplit, int comps,
                          double alpha_em, double smin, double smax, double reseed_frac,
                          double t_max, int min_samples) {
    po_model *m = (po_model *)calloc(1, sizeof(po_model));
    m->kind = kind;
    m->comps = comps;
    m->alpha_em = alpha_em;
    m->smin = smin;
    m->smax = smax;
    m->reseed_frac = reseed_frac;
    if (kind == 2) { /* Gmm::Gmm (models.cpp:427-447) */
        int C = comps, grid = 1;
        m->gtmpl = (double *)calloc((size_t)(21 * C + 3), sizeof(double));
        while (grid * grid < C) ++grid;
        for (int c = 0; c < C; ++c) {
            GW(m->gtmpl)[c] = 1.0 / C;
            GV(m->gtmpl, C)[3 * c] = 0.02;
            GV(m->gtmpl, C)[3 * c + 2] = 0.02;
            GM(m->gtmpl, C)[2 * c] = ((c % grid) + 0.5) / grid;
            GM(m->gtmpl, C)[2 * c + 1] = ((c / grid) + 0.5) / grid;
            pm_gmm_cache(m->gtmpl, C, c);
        }
    }
    m->res = res;
    m->leaves = leaves;
    m->tsplit = tsplit;
    m->t_max = t_max;
    m->min_samples = min_samples;
    m->cap = 1024;
    m->tab = (pm_entry *)calloc(m->cap, sizeof(pm_entry));
    if (kind == 1) {
        int n = 0;
        m->tmpl = (pm_node *)calloc((size_t)(2 * leaves - 1), sizeof(pm_node));
        pm_kd_add(m->tmpl, &n);
        pm_kd_build(m->tmpl, &n, 0, 0, leaves, leaves);
        pm_kd_mass(m->tmpl, 0);
    }
    return m;
}

static size_t pm_slots(const po_model *m) {
    return m->kind == 1   ? (size_t)(2 * m->leaves - 1)
           : m->kind == 2 ? (size_t)(21 * m->comps + 3)
                          : (size_t)m->res * m->res;
}

void po_model_destroy(po_model *m) {
    for (size_t i = 0; i < m->cap; ++i)
        if (m->tab[i].used) {
            free(m->tab[i].w);
            free(m->tab[i].acc);
            free(m->tab[i].nodes);
            free(m->tab[i].fs);
        }
    free(m->tab);
    free(m->tmpl);
    free(m->gtmpl);
    free(m);
}

static pm_entry *pm_find(const po_model *m, const po_key *k) {
    size_t i = (size_t)(pm_hash(k) & (m->cap - 1));
    for (;;) {
        pm_entry *e = &m->tab[i];
        if (!e->used) return NULL;
        if (pm_eq(&e->key, k)) return e;
        i = (i + 1) & (m->cap - 1);
    }
}

static pm_entry *pm_slot_for_insert(pm_entry *tab, size_t cap, const po_key *k) {
    size_t i = (size_t)(pm_hash(k) & (cap - 1));
    while (tab[i].used && !pm_eq(&tab[i].key, k)) i = (i + 1) & (cap - 1);
    return &tab[i];
}

/* m_map[key] (estimators.cpp:111) + the DirGrid constructor (models.cpp:16-22) */
static pm_entry *pm_get_or_create(po_model *m, const po_key *k) {
    pm_entry *e = pm_find(m, k);
    if (e) return e;
    if (2 * (m->size + 1) > m->cap) {
        size_t nc = m->cap * 2;
        pm_entry *nt = (pm_entry *)calloc(nc, sizeof(pm_entry));
        for (size_t i = 0; i < m->cap; ++i)
            if (m->tab[i].used) *pm_slot_for_insert(nt, nc, &m->tab[i].key) = m->tab[i];
        free(m->tab);
        m->tab = nt;
        m->cap = nc;
    }
    e = pm_slot_for_insert(m->tab, m->cap, k);
    memset(e, 0, sizeof(*e));
    e->used = 1;
    e->key = *k;
    if (m->kind == 1) {
        size_t nn = pm_slots(m);
        e->nodes = (pm_node *)malloc(nn * sizeof(pm_node));
        memcpy(e->nodes, m->tmpl, nn * sizeof(pm_node));
    } else if (m->kind == 2) {
        size_t ns = pm_slots(m);
        e->w = (double *)malloc(ns * sizeof(double));
        memcpy(e->w, m->gtmpl, ns * sizeof(double));
    } else {
        size_t r2 = (size_t)m->res * m->res;
        e->w = (double *)malloc(r2 * sizeof(double));
        e->acc = (double *)calloc(r2, sizeof(double));
        for (size_t j = 0; j < r2; ++j) e->w[j] = 1.0 / ((double)m->res * m->res);
        e->total = 1.0;
    }
    m->size++;
    return e;
}

/* DirGrid::cellIndex (models.cpp:24-28); int(double) with x86 truncation, uv < 0 clamped as on
 * the device (the reference indexes outside the grid there) */
static int pm_cell(int res, double u, double v) {
    double fx = u * res, fy = v * res;
    int ix = (fx >= -2147483648.0 && fx < 2147483648.0) ? (int)fx : INT32_MIN;
    int iy = (fy >= -2147483648.0 && fy < 2147483648.0) ? (int)fy : INT32_MIN;
    if (ix > res - 1) ix = res - 1;
    if (iy > res - 1) iy = res - 1;
    if (ix < 0) ix = 0;
    if (iy < 0) iy = 0;
    return iy * res + ix;
}

typedef struct {
    const po_key *k;
    double u, v, c;
} pm_rec;

static int pm_cmp_d(double a, double b) { return a < b ? -1 : (b < a ? 1 : 0); }

/* std::tie(level, cell..., dirCell..., uv.x, uv.y, contribution) < (estimators.cpp:633-637) */
static int pm_rec_cmp(const void *pa, const void *pb) {
    const pm_rec *a = (const pm_rec *)pa, *b = (const pm_rec *)pb;
    const int32_t ka[6] = {a->k->level, a->k->cell[0], a->k->cell[1], a->k->cell[2], a->k->dir[0],
                           a->k->dir[1]};
    const int32_t kb[6] = {b->k->level, b->k->cell[0], b->k->cell[1], b->k->cell[2], b->k->dir[0],
                           b->k->dir[1]};
    for (int i = 0; i < 6; ++i)
        if (ka[i] != kb[i]) return ka[i] < kb[i] ? -1 : 1;
    int c = pm_cmp_d(a->u, b->u);
    if (c) return c;
    c = pm_cmp_d(a->v, b->v);
    if (c) return c;
    return pm_cmp_d(a->c, b->c);
}

static double pm_lerp(double a, double b, double t) { return a + (b - a) * t; } /* vecmath.h:22 */

/* findLeaf (models.cpp:140-159) */
static int pm_kd_find(const pm_node *t, double u, double v, double lo[2], double hi[2]) {
    lo[0] = lo[1] = 0.0;
    hi[0] = hi[1] = 1.0;
    int node = 0;
    while (!t[node].leaf) {
        const pm_node *n = &t[node];
        double split_abs = pm_lerp(lo[n->axis], hi[n->axis], n->split);
        double coord = n->axis == 0 ? u : v;
        if (coord <= split_abs) {
            hi[n->axis] = split_abs;
            node = n->left;
        } else {
            lo[n->axis] = split_abs;
            node = n->right;
        }
    }
    return node;
}

static double pm_max(double a, double b) { return a < b ? b : a; } /* std::max */

/* SphericalKdTree::endFrame (models.cpp:202-298) */
static void pm_kd_end_frame(po_model *m, pm_node *t, double blend) {
    int nn = 2 * m->leaves - 1;
    double total = 0.0;
    for (int i = 0; i < nn; ++i)
        if (t[i].leaf) total += t[i].accum;
    if (total > 0.0) {
        double floor_prob = 1e-4 / m->leaves, norm_sum = 0.0;
        for (int i = 0; i < nn; ++i)
            if (t[i].leaf) norm_sum += pm_max(t[i].accum / total, floor_prob);
        for (int i = 0; i < nn; ++i) {
            if (!t[i].leaf) continue;
            double target = pm_max(t[i].accum / total, floor_prob) / norm_sum;
            t[i].prob = (1.0 - blend) * t[i].prob + blend * target;
        }
        double prob_sum = 0.0;
        for (int i = 0; i < nn; ++i)
            if (t[i].leaf) prob_sum += t[i].prob;
        for (int i = 0; i < nn; ++i)
            if (t[i].leaf) t[i].prob /= prob_sum;
    }
    int l_max = -1, p_min = -1;
    double p_max = -1.0, p_min_mass = 2.0;
    for (int i = 0; i < nn; ++i)
        if (t[i].leaf && t[i].prob > p_max) {
            p_max = t[i].prob;
            l_max = i;
        }
    for (int i = 0; i < nn; ++i) {
        const pm_node *n = &t[i];
        if (n->leaf || !t[n->left].leaf || !t[n->right].leaf) continue;
        double mass = t[n->left].prob + t[n->right].prob;
        if (mass < p_min_mass) {
            p_min_mass = mass;
            p_min = i;
        }
    }
    if (l_max >= 0 && p_min >= 0 && t[l_max].parent != p_min && p_max > m->tsplit * p_min_mass) {
        int fl = t[p_min].left, fr = t[p_min].right;
        t[p_min].leaf = 1;
        t[p_min].prob = p_min_mass;
        t[p_min].accum = 0.0;
        t[p_min].left = t[p_min].right = -1;
        int chain[1024], nc = 0;
        for (int n = l_max; n != -1; n = t[n].parent) chain[nc++] = n;
        double lo[2] = {0.0, 0.0}, hi[2] = {1.0, 1.0};
        for (int i = nc - 1; i >= 1; --i) {
            const pm_node *n = &t[chain[i]];
            double split_abs = pm_lerp(lo[n->axis], hi[n->axis], n->split);
            if (chain[i - 1] == n->left)
                hi[n->axis] = split_abs;
            else
                lo[n->axis] = split_abs;
        }
        pm_node *hot = &t[l_max];
        hot->leaf = 0;
        hot->axis = (hi[0] - lo[0]) >= (hi[1] - lo[1]) ? 0 : 1;
        hot->split = 0.5;
        hot->left = fl;
        hot->right = fr;
        int kids[2] = {fl, fr};
        for (int c = 0; c < 2; ++c) {
            pm_node *z = &t[kids[c]];
            memset(z, 0, sizeof(*z));
            z->split = 0.5;
            z->left = z->right = -1;
            z->leaf = 1;
            z->prob = p_max * 0.5;
            z->parent = l_max;
        }
        hot->prob = 0.0;
    }
    for (int i = 0; i < nn; ++i) t[i].accum = 0.0;
    pm_kd_mass(t, 0);
}

/* componentPdf (models.cpp:465-480) */
static double pm_gmm_cpdf(const double *S, int C, int c, double x, double y) {
    const double *k = GK(S, C) + 7 * c;
    double sum = 0.0;
    for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
            double ex = x + dx - GM(S, C)[2 * c], ey = y + dy - GM(S, C)[2 * c + 1];
            double q = k[0] * ex * ex + 2.0 * k[1] * ex * ey + k[2] * ey * ey;
            sum += k[3] * exp(-0.5 * q);
        }
    return sum;
}

static double pm_gmm_pdf(const double *S, int C, double x, double y) { /* models.cpp:657-662 */
    double p = 0.0;
    for (int c = 0; c < C; ++c) p += GW(S)[c] * pm_gmm_cpdf(S, C, c, x, y);
    return p;
}

/* responsibilities (models.cpp:482-497) */
static void pm_gmm_resp(double *S, int C, double x, double y, double *gamma) {
    double total = 0.0;
    for (int c = 0; c < C; ++c) {
        gamma[c] = GW(S)[c] * pm_gmm_cpdf(S, C, c, x, y);
        total += gamma[c];
    }
    if (total <= 0.0 || !isfinite(total)) {
        GT(S, C)[1] += 1.0;
        for (int c = 0; c < C; ++c) gamma[c] = 1.0 / C;
        return;
    }
    for (int c = 0; c < C; ++c) gamma[c] /= total;
}

/* estepBatch (models.cpp:525-585), sequential as in the reference */
static void pm_gmm_estep(po_model *m, double *S, const double *fs, size_t n) {
    int C = m->comps;
    uint64_t i0 = (uint64_t)GT(S, C)[0];
    double *gamma = (double *)malloc(n * C * sizeof(double) + 1);
    for (size_t j = 0; j < n; ++j) pm_gmm_resp(S, C, fs[3 * j], fs[3 * j + 1], gamma + j * C);
    double *lp = (double *)calloc(n + 1, sizeof(double));
    size_t last_zero = 0;
    for (size_t k = 1; k <= n; ++k) {
        double factor = 1.0 - pow((double)(i0 + k), -m->alpha_em);
        if (factor <= 0.0) {
            last_zero = k;
            lp[k] = 0.0;
        } else {
            lp[k] = lp[k - 1] + log(factor);
        }
    }
#define GOF(j) ((j) < last_zero ? 0.0 : exp(lp[n] - lp[(j)]))
    double g_total = GOF(0);
    for (int q = 0; q < 8 * C; ++q) GU(S, C)[q] *= g_total;
    for (size_t j = 1; j <= n; ++j) {
        double sx = fs[3 * (j - 1)], sy = fs[3 * (j - 1) + 1], w = fs[3 * (j - 1) + 2];
        double g = GOF(j);
        if (g == 0.0) continue;
        double step = pow((double)(i0 + j), -m->alpha_em);
        for (int c = 0; c < C; ++c) {
            double b = step * w * gamma[(j - 1) * C + c];
            if (b <= 0.0) continue;
            double bg = b * g, *u = GU(S, C) + 8 * c;
            u[0] += bg;
            u[1] += bg * sx;
            u[2] += bg * sy;
            u[3] += bg * sx * sx;
            u[4] += bg * sy * sy;
            u[5] += bg * sx * sy;
            u[6] += g * step * w;
            u[7] += g;
        }
    }
#undef GOF
    GT(S, C)[0] = (double)(i0 + n);
    free(gamma);
    free(lp);
}

static double pm_clamp3(double x, double lo, double hi) { /* vecmath.h:19 */
    double a = x < lo ? lo : x;
    return hi < a ? hi : a;
}

/* Gmm::mstep (models.cpp:587-655) */
static void pm_gmm_mstep(po_model *m, double *S) {
    int C = m->comps;
    double total = 0.0;
    for (int c = 0; c < C; ++c) total += GU(S, C)[8 * c];
    if (total <= 0.0) return;
    int heaviest = 0;
    for (int c = 1; c < C; ++c)
        if (GU(S, C)[8 * c] > GU(S, C)[8 * heaviest]) heaviest = c;
    for (int c = 0; c < C; ++c) {
        const double *u = GU(S, C) + 8 * c;
        double mass = u[0];
        if (mass <= m->reseed_frac * total) {
            const double *h = GU(S, C) + 8 * heaviest;
            double sx = h[1] / h[0], sy = h[2] / h[0];
            uint32_t rc = (uint32_t)GT(S, C)[2];
            GT(S, C)[2] = (double)(uint32_t)(rc + 1u);
            double jitter = 0.05 * (1.0 + (double)(rc % 7u));
            double mx = sx + jitter * 0.01, my = sy - jitter * 0.01;
            mx -= floor(mx);
            my -= floor(my);
            GM(S, C)[2 * c] = mx;
            GM(S, C)[2 * c + 1] = my;
            GW(S)[c] = 1e-3;
            GV(S, C)[3 * c] = 0.01;
            GV(S, C)[3 * c + 1] = 0.0;
            GV(S, C)[3 * c + 2] = 0.01;
            continue;
        }
        GW(S)[c] = mass / total;
        double mx = u[1] / mass, my = u[2] / mass;
        double exx = u[3] / mass, eyy = u[4] / mass, exy = u[5] / mass;
        double cxx = exx - mx * mx, cyy = eyy - my * my, cxy = exy - mx * my;
        double tr = cxx + cyy, diff = cxx - cyy;
        double dd = diff * diff + 4.0 * cxy * cxy;
        double disc = sqrt(dd < 0.0 ? 0.0 : dd);
        double l1 = 0.5 * (tr + disc), l2 = 0.5 * (tr - disc);
        double c1 = pm_clamp3(l1, m->smin, m->smax), c2 = pm_clamp3(l2, m->smin, m->smax);
        double vx, vy;
        if (fabs(cxy) > 1e-30) {
            vx = l1 - cyy;
            vy = cxy;
        } else {
            vx = cxx >= cyy ? 1.0 : 0.0;
            vy = cxx >= cyy ? 0.0 : 1.0;
        }
        double len = sqrt(vx * vx + vy * vy);
        if (len > 0.0) {
            vx /= len;
            vy /= len;
        }
        GV(S, C)[3 * c] = c1 * vx * vx + c2 * vy * vy;
        GV(S, C)[3 * c + 1] = (c1 - c2) * vx * vy;
        GV(S, C)[3 * c + 2] = c1 * vy * vy + c2 * vx * vx;
        GM(S, C)[2 * c] = mx;
        GM(S, C)[2 * c + 1] = my;
    }
    double wsum = 0.0;
    for (int c = 0; c < C; ++c) wsum += GW(S)[c];
    for (int c = 0; c < C; ++c) GW(S)[c] /= wsum;
    for (int c = 0; c < C; ++c) pm_gmm_cache(S, C, c);
}

/* applyRecord (estimators.cpp:109-117) with DirGrid::record (models.cpp:30-35) */
static void pm_apply_one(po_model *m, const po_key *k, double u, double v, double c) {
    pm_entry *e = pm_get_or_create(m, k);
    if (c >= 0.0 && isfinite(c)) { /* DirGrid::record / SphericalKdTree::record (models.cpp:161-167) */
        if (m->kind == 1) {
            double lo[2], hi[2];
            e->nodes[pm_kd_find(e->nodes, u, v, lo, hi)].accum += c;
        } else if (m->kind == 2) { /* Gmm::record (models.cpp:689-694) */
            if (e->nfs == e->cfs) {
                e->cfs = e->cfs ? 2 * e->cfs : 16;
                e->fs = (double *)realloc(e->fs, e->cfs * 3 * sizeof(double));
            }
            e->fs[3 * e->nfs] = u;
            e->fs[3 * e->nfs + 1] = v;
            e->fs[3 * e->nfs + 2] = c;
            e->nfs++;
        } else {
            e->acc[pm_cell(m->res, u, v)] += c;
        }
        e->rec_count++;
    }
    e->c_new += 1.0;
    e->records++;
}

void po_model_apply(po_model *m, const po_key *keys, const double *u, const double *v,
                    const double *c, size_t n) {
    pm_rec *r = (pm_rec *)malloc((n ? n : 1) * sizeof(pm_rec));
    for (size_t i = 0; i < n; ++i) {
        r[i].k = &keys[i];
        r[i].u = u[i];
        r[i].v = v[i];
        r[i].c = c[i];
    }
    qsort(r, n, sizeof(pm_rec), pm_rec_cmp);
    for (size_t i = 0; i < n; ++i) pm_apply_one(m, r[i].k, r[i].u, r[i].v, r[i].c);
    free(r);
}

/* ModelStore::endFrame (estimators.cpp:119-144) with DirGrid::endFrame (models.cpp:37-50) */
void po_model_end_frame(po_model *m) {
    int limited = m->t_max > 0.0 && isfinite(m->t_max);
    double sum_c = 0.0;
    size_t touched = 0;
    for (size_t i = 0; i < m->cap; ++i)
        if (m->tab[i].used && m->tab[i].c_new > 0.0) {
            sum_c += m->tab[i].c_new;
            ++touched;
        }
    double cap = limited && touched ? (m->t_max * m->t_max - m->t_max) * (sum_c / (double)touched)
                                    : 0.0;
    size_t r2 = (size_t)m->res * m->res;
    for (size_t i = 0; i < m->cap; ++i) {
        pm_entry *e = &m->tab[i];
        if (!e->used || e->c_new <= 0.0) continue;
        double alpha = sqrt(e->c_new / (e->c_old + e->c_new));
        if (limited && alpha < 1.0 / m->t_max) alpha = 1.0 / m->t_max;
        if (m->kind == 1) {
            pm_kd_end_frame(m, e->nodes, alpha);
            goto close;
        }
        if (m->kind == 2) { /* Gmm::endFrame (models.cpp:696-702) */
            if (e->nfs) {
                pm_gmm_estep(m, e->w, e->fs, e->nfs);
                e->nfs = 0;
                pm_gmm_mstep(m, e->w);
            }
            goto close;
        }
        double s = 0.0;
        for (size_t j = 0; j < r2; ++j) s += e->acc[j];
        if (s > 0.0) {
            for (size_t j = 0; j < r2; ++j)
                e->w[j] = (1.0 - alpha) * e->w[j] + alpha * (e->acc[j] / s);
            e->total = 0.0;
            for (size_t j = 0; j < r2; ++j) e->total += e->w[j];
        }
        memset(e->acc, 0, r2 * sizeof(double));
    close:
        e->c_old += e->c_new;
        if (limited && cap < e->c_old) e->c_old = cap;
        e->c_new = 0.0;
        e->warm = e->records >= (uint64_t)(int64_t)m->min_samples;
    }
}

/* lookupWarm (estimators.cpp:104-107) + DirGrid::pdf (models.cpp:52-56); no warm model -> 1.0
 * with *found = 0 */
double po_model_pdf(const po_model *m, const po_key *k, double u, double v, int *found) {
    const pm_entry *e = pm_find(m, k);
    *found = e && e->warm;
    if (*found && m->kind == 2) return pm_gmm_pdf(e->w, m->comps, u, v);
    if (*found && m->kind == 1) { /* SphericalKdTree::pdf (models.cpp:169-174) */
        double lo[2], hi[2];
        int leaf = pm_kd_find(e->nodes, u, v, lo, hi);
        double area = (hi[0] - lo[0]) * (hi[1] - lo[1]);
        return area > 0.0 ? e->nodes[leaf].prob / area : 0.0;
    }
    if (!*found || e->total <= 0.0) return 1.0;
    return e->w[pm_cell(m->res, u, v)] / e->total * (double)m->res * m->res;
}

static double pm_clamp(double x, double lo, double hi) { /* vecmath.h:19 */
    double a = x < lo ? lo : x;
    return hi < a ? hi : a;
}

/* lookupWarm + DirGrid::sample (models.cpp:58-92); no warm model -> (u, 1.0), *found = 0 */
void po_model_sample(const po_model *m, const po_key *k, double u1, double u2, double usel,
                     double *su, double *sv, double *pdf, int *found) {
    const pm_entry *e = pm_find(m, k);
    *found = e && e->warm;
    if (*found && m->kind == 2) { /* Gmm::sample (models.cpp:664-687) */
        int C = m->comps, comp = 0;
        const double *S = e->w;
        double acc = 0.0;
        for (int c = 0; c < C; ++c) {
            acc += GW(S)[c];
            if (usel < acc || c == C - 1) {
                comp = c;
                break;
            }
        }
        double om = 1.0 - u1;
        double r = sqrt(-2.0 * log(om < 1e-300 ? 1e-300 : om));
        double z0 = r * cos(GMM_TWO_PI * u2), z1 = r * sin(GMM_TWO_PI * u2);
        const double *kk = GK(S, C) + 7 * comp;
        double px = GM(S, C)[2 * comp] + kk[4] * z0;
        double py = GM(S, C)[2 * comp + 1] + kk[5] * z0 + kk[6] * z1;
        px -= floor(px);
        py -= floor(py);
        *su = px;
        *sv = py;
        *pdf = pm_gmm_pdf(S, C, px, py);
        return;
    }
    if (*found && m->kind == 1) { /* SphericalKdTree::sample (models.cpp:176-200) */
        const pm_node *t = e->nodes;
        const double below_one = nextafter(1.0, 0.0);
        double r[2] = {u1, u2}, lo[2] = {0.0, 0.0}, hi[2] = {1.0, 1.0};
        int node = 0;
        while (!t[node].leaf) {
            const pm_node *n = &t[node];
            double mass = n->mass;
            double left_frac = mass > 0.0 ? t[n->left].mass / mass : 0.5;
            double split_abs = pm_lerp(lo[n->axis], hi[n->axis], n->split);
            double *coord = &r[n->axis];
            if (left_frac > 0.0 && (*coord < left_frac || left_frac >= 1.0)) {
                double q = *coord / left_frac;
                *coord = below_one < q ? below_one : q;
                hi[n->axis] = split_abs;
                node = n->left;
            } else {
                double q = (*coord - left_frac) / (1.0 - left_frac);
                *coord = below_one < q ? below_one : q;
                lo[n->axis] = split_abs;
                node = n->right;
            }
        }
        *su = pm_lerp(lo[0], hi[0], r[0]);
        *sv = pm_lerp(lo[1], hi[1], r[1]);
        double area = (hi[0] - lo[0]) * (hi[1] - lo[1]);
        *pdf = area > 0.0 ? t[node].prob / area : 0.0;
        return;
    }
    if (!*found || e->total <= 0.0) {
        *su = u1;
        *sv = u2;
        *pdf = 1.0;
        return;
    }
    const int R = m->res;
    double target = u2 * e->total;
    int row = 0;
    double row_sum = 0.0, acc = 0.0;
    for (; row < R; ++row) {
        row_sum = 0.0;
        for (int x = 0; x < R; ++x) row_sum += e->w[(size_t)row * R + x];
        if (acc + row_sum > target || row == R - 1) break;
        acc += row_sum;
    }
    double vin = row_sum > 0.0 ? pm_clamp((target - acc) / row_sum, 0.0, 1.0) : u2;
    double col_target = u1 * row_sum;
    int col = 0;
    double col_acc = 0.0, w = 0.0;
    for (; col < R; ++col) {
        w = e->w[(size_t)row * R + col];
        if (col_acc + w > col_target || col == R - 1) break;
        col_acc += w;
    }
    double uin = w > 0.0 ? pm_clamp((col_target - col_acc) / w, 0.0, 1.0) : u1;
    double x = (col + uin) / R, y = (row + vin) / R;
    const double below_one = nextafter(1.0, 0.0);
    if (below_one < x) x = below_one;
    if (below_one < y) y = below_one;
    *su = x;
    *sv = y;
    *pdf = e->w[pm_cell(R, x, y)] / e->total * (double)R * R;
}

static int pm_entry_cmp(const void *pa, const void *pb) {
    const pm_entry *a = *(const pm_entry *const *)pa, *b = *(const pm_entry *const *)pb;
    const int32_t ka[6] = {a->key.level, a->key.cell[0], a->key.cell[1], a->key.cell[2],
                           a->key.dir[0], a->key.dir[1]};
    const int32_t kb[6] = {b->key.level, b->key.cell[0], b->key.cell[1], b->key.cell[2],
                           b->key.dir[0], b->key.dir[1]};
    for (int i = 0; i < 6; ++i)
        if (ka[i] != kb[i]) return ka[i] < kb[i] ? -1 : 1;
    return 0;
}

/* every entry sorted by key; weights/accum: res^2 doubles per entry (may be NULL) */
size_t po_model_dump(const po_model *m, po_model_entry *out, double *weights, double *accum,
                     size_t cap) {
    const pm_entry **ord = (const pm_entry **)malloc((m->size ? m->size : 1) * sizeof(void *));
    size_t n = 0;
    for (size_t i = 0; i < m->cap; ++i)
        if (m->tab[i].used) ord[n++] = &m->tab[i];
    qsort(ord, n, sizeof(void *), pm_entry_cmp);
    size_t r2 = pm_slots(m), k = n < cap ? n : cap;
    for (size_t i = 0; i < k; ++i) {
        const pm_entry *e = ord[i];
        po_model_entry *o = &out[i];
        memset(o, 0, sizeof(*o));
        o->level = e->key.level;
        memcpy(o->cell, e->key.cell, sizeof(o->cell));
        memcpy(o->dir, e->key.dir, sizeof(o->dir));
        o->warm = (uint32_t)e->warm;
        o->c_old = e->c_old;
        o->c_new = e->c_new;
        o->records = e->records;
        o->record_count = e->rec_count;
        o->total = m->kind == 0 ? e->total : 0.0;
        for (size_t j = 0; j < r2; ++j) {
            if (weights) weights[i * r2 + j] = m->kind == 1 ? e->nodes[j].prob : e->w[j];
            if (accum) accum[i * r2 + j] = m->kind == 1 ? e->nodes[j].accum
                                           : m->kind == 2 ? 0.0 : e->acc[j];
        }
    }
    free(ord);
    return n;
}

/* k-d tree topology, same entry order: {leaf, axis, left, right, parent}, {split, mass} */
size_t po_model_dump_tree(const po_model *m, int32_t *node_i32, double *node_f64, size_t cap) {
    const pm_entry **ord = (const pm_entry **)malloc((m->size ? m->size : 1) * sizeof(void *));
    size_t n = 0;
    for (size_t i = 0; i < m->cap; ++i)
        if (m->tab[i].used) ord[n++] = &m->tab[i];
    qsort(ord, n, sizeof(void *), pm_entry_cmp);
    size_t nn = pm_slots(m), k = n < cap ? n : cap;
    for (size_t i = 0; i < k && m->kind == 1; ++i)
        for (size_t j = 0; j < nn; ++j) {
            const pm_node *t = &ord[i]->nodes[j];
            int32_t *o = node_i32 + (i * nn + j) * 5;
            o[0] = t->leaf;
            o[1] = t->axis;
            o[2] = t->left;
            o[3] = t->right;
            o[4] = t->parent;
            node_f64[(i * nn + j) * 2] = t->split;
            node_f64[(i * nn + j) * 2 + 1] = t->mass;
        }
    free(ord);
    return n;
}
