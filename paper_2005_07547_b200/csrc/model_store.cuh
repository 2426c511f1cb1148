/* CV-profile / guiding model store on the device.
 *
 * ModelStore (estimators.h:124-150, estimators.cpp:104-144) holding DirGrid (models.h:30-52,
 * models.cpp:16-94), SphericalKdTree (models.h:59-109, models.cpp:96-298) or Gmm models
 * (models.h:113-177, models.cpp:427-702).  Included at the end of field.cu (one translation
 * unit: it shares the scratch buffers, the multi-word radix sort and the exact key functions).
 *
 * Layout (per entry e of a 2^k open-addressing table, home = packKeyFields(key) & mask):
 *   state[e]   u32   0 empty, 1 being written, 2 ready (entries are never removed, as in the
 *                    reference's unordered_map)
 *   keyf[e]    6 x i32 key fields (equality ignores the checksum, field.h:38-41)
 *   ent[e]     {total, cOld, cNew, records, recordCount, warm, touched}
 *   w[e][ns], acc[e][ns]  f64: DirGrid weights / accumulators (row-major, ns = R^2); k-d tree
 *                    node prob / accum (ns = 2L-1, topology in kn[e][ns]); Gmm state vector
 *   entry 2^k        the template a new k-d tree / Gmm entry is copied from
 *
 * apply:  every record finds (or inserts, CAS on state) its key's entry; the records are then
 *         radix-sorted by (entry, slot, uv.x, uv.y, contribution) (slot = grid cell or tree
 *         leaf, 0 for Gmm), which within one key is the canonical order of
 *         estimators.cpp:633-637; one thread per (entry, slot) run folds it in a register, so
 *         each accumulator sum has the reference's order (Gmm: the samples are appended in that
 *         order instead).  ATOMIC: no sort, fp64 atomics.  No host round trip.
 * endFrame: the touched entries only (a list built by apply): Σ cNew (integer-valued, exact in
 *         any order), then per entry: one warp blends a grid (sums in index order); one warp
 *         runs a staged k-d tree update; Gmm runs a chunked, sample-parallel E-step, then the
 *         M-step per entry. */

struct ModelEnt {
    double total, c_old, c_new;
    unsigned long long records, rec_count;
    uint32_t warm, touched;
};

/* SphericalKdTree::Node (models.h:91-99) minus prob/accum, which live in w/acc */
struct KdNode {
    double split, mass;
    int32_t left, right, parent;
    uint8_t leaf, axis;
};

struct MdlDev {
    uint32_t *state;
    KeyFields *keyf;
    ModelEnt *ent;
    double *w, *acc; /* ns per entry: Grid weights / accumulators, or KdTree node prob / accum */
    KdNode *kn;      /* KdTree: ns nodes per entry; entry `mask + 1` holds the initial tree */
    unsigned long long *ctr; /* [0] entries, [1] dropped records, [2] touched-list length */
    uint32_t *tlist;
    uint32_t mask;
    int kind, res, ns, leaves; /* ns: slots per entry (R^2, 2L-1 nodes, or 21C+3 GMM state) */
    double tsplit;
    int comps; /* GMM: components, alphaEm, eigenvalue floor / cap, reseed fraction */
    double alpha_em, smin, smax, reseed_frac;
    /* GMM frame samples (Gmm::m_frameSamples, in applyRecord order): entry, uv, contribution;
     * count in ctr[MC_SAMPLES]; per-entry segments of the entry-sorted samples */
    uint32_t *fs_entry;
    double *fs_u, *fs_v, *fs_c;
    uint32_t *seg_begin, *seg_end;
};

enum { MC_ENTRIES = 0, MC_DROPPED = 1, MC_TOUCHED = 2, MC_SAMPLES = 3, MC_N = 4 };

struct pstf_model_store {
    pstf_model_config cfg;
    int device = 0;
    uint32_t mask = 0;
    int ns = 0;
    DBuf state, keyf, ent, w, acc, kn, ctr, tlist, sums;
    DBuf fs_entry, fs_u, fs_v, fs_c, seg, fs_key, fs_pos; /* GMM frame samples */
    DBuf gch_n, gch_f;                                     /* GMM E-step chunks */
    uint64_t fs_bound = 0; /* host upper bound of the samples appended this frame */
    Scratch sc;
    DBuf words;
    MdlDev dev() const {
        MdlDev d;
        d.state = state.as<uint32_t>();
        d.keyf = keyf.as<KeyFields>();
        d.ent = ent.as<ModelEnt>();
        d.w = w.as<double>();
        d.acc = acc.as<double>();
        d.kn = kn.as<KdNode>();
        d.ctr = ctr.as<unsigned long long>();
        d.tlist = tlist.as<uint32_t>();
        d.mask = mask;
        d.kind = cfg.kind;
        d.res = cfg.grid_resolution;
        d.ns = ns;
        d.leaves = cfg.kd_leaf_count;
        d.tsplit = cfg.kd_split_threshold;
        d.comps = cfg.gmm_components;
        d.alpha_em = cfg.gmm_alpha_em;
        d.smin = cfg.gmm_sigma_min_sq;
        d.smax = cfg.gmm_sigma_max_sq;
        d.reseed_frac = cfg.gmm_reseed_fraction;
        d.fs_entry = fs_entry.as<uint32_t>();
        d.fs_u = fs_u.as<double>();
        d.fs_v = fs_v.as<double>();
        d.fs_c = fs_c.as<double>();
        d.seg_begin = seg.as<uint32_t>();
        d.seg_end = seg.as<uint32_t>() + (mask + 1ull);
        return d;
    }
};

__device__ __forceinline__ uint32_t mdl_home(const KeyFields &k, uint32_t mask) {
    return (uint32_t)pack_key_fields(k.level, k.c0, k.c1, k.c2, k.d0, k.d1) & mask;
}

__device__ __forceinline__ bool kf_equal(const KeyFields &a, const KeyFields &b) {
    return a.level == b.level && a.c0 == b.c0 && a.c1 == b.c1 && a.c2 == b.c2 && a.d0 == b.d0 &&
           a.d1 == b.d1;
}

__device__ __forceinline__ KeyFields kf_of(const pstf_key &k) {
    return KeyFields{k.level, k.cell[0], k.cell[1], k.cell[2], k.dir_cell[0], k.dir_cell[1]};
}

__device__ __forceinline__ uint32_t ld_state(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

/* DirGrid::cellIndex (models.cpp:24-28): min(int(uv * R), R - 1) per axis; the reference
 * indexes outside the grid for uv < 0 (undefined), here that clamps to 0 */
__device__ __forceinline__ int mdl_cell(double u, double v, int res) {
    int ix = min(i32_x86(u * (double)res), res - 1);
    int iy = min(i32_x86(v * (double)res), res - 1);
    return max(iy, 0) * res + max(ix, 0);
}

/* order-preserving u64 of a double; -0.0 sorts as +0.0 (std::tie compares them equal) */
__device__ __forceinline__ uint64_t ord_f64(double d) {
    uint64_t b = dbits(d == 0.0 ? 0.0 : d);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

/* ---- SphericalKdTree (models.cpp:96-298) on one entry's node arrays ---- */
__device__ __forceinline__ double lerp_ref(double a, double b, double t) { /* vecmath.h:22 */
    return a + (b - a) * t;
}

__device__ __forceinline__ double min_ref(double a, double b) { return b < a ? b : a; } /* std::min */
__device__ __forceinline__ double clamp_ref(double x, double lo, double hi) { /* vecmath.h:19 */
    const double a = x < lo ? lo : x;
    return hi < a ? hi : a;
}

__device__ __forceinline__ double max_ref(double a, double b) { return a < b ? b : a; } /* std::max */

/* findLeaf (models.cpp:140-159): boundary ties go to the lower child */
__device__ int kd_find_leaf(const KdNode *K, double u, double v, double2 *lo_out, double2 *hi_out) {
    double2 lo = make_double2(0.0, 0.0), hi = make_double2(1.0, 1.0);
    int node = 0; /* m_root */
    while (!K[node].leaf) {
        const KdNode n = K[node];
        const double split_abs = n.axis == 0 ? lerp_ref(lo.x, hi.x, n.split)
                                             : lerp_ref(lo.y, hi.y, n.split);
        const double coord = n.axis == 0 ? u : v;
        if (coord <= split_abs) {
            if (n.axis == 0) hi.x = split_abs; else hi.y = split_abs;
            node = n.left;
        } else {
            if (n.axis == 0) lo.x = split_abs; else lo.y = split_abs;
            node = n.right;
        }
    }
    if (lo_out) *lo_out = lo;
    if (hi_out) *hi_out = hi;
    return node;
}

/* refreshMass (models.cpp:129-138): mass = prob at leaves, left + right above; computed in
 * reverse breadth-first order (children before parents), each sum being the same single add */
__device__ void kd_refresh_mass(KdNode *K, const double *P, int nn, int *order) {
    int head = 0, tail = 0;
    order[tail++] = 0;
    while (head < tail) {
        const int n = order[head++];
        if (!K[n].leaf) {
            order[tail++] = K[n].left;
            order[tail++] = K[n].right;
        }
    }
    for (int i = tail - 1; i >= 0; --i) {
        const int n = order[i];
        K[n].mass = K[n].leaf ? P[n] : K[K[n].left].mass + K[K[n].right].mass;
    }
}

/* sum over i in [0, n) of f(i) in index order, by one warp (every lane gets the same value):
 * lanes evaluate 32 consecutive terms, every lane adds them in order via broadcasts.  Terms
 * that the reference skips are +0.0 here, which leaves a non-negative sum unchanged. */
template <class F>
__device__ __forceinline__ double warp_ordered_sum_f(int n, unsigned lane, F f) {
    double s = 0.0;
    for (int b = 0; b < n; b += 32) {
        const double mine = b + (int)lane < n ? f(b + (int)lane) : 0.0;
        const int k = min(32, n - b);
        for (int l = 0; l < k; ++l) s += __shfl_sync(0xffffffffu, mine, l);
    }
    return s;
}

/* first index of the extreme value (strict comparison, as the reference's loops): best = lowest
 * (sign -1) or highest (sign +1) value, ties to the lower index; idx -1 when no candidate */
__device__ __forceinline__ void warp_first_extreme(double &val, int &idx, double sign) {
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, val, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        const bool better = oi >= 0 && (idx < 0 || sign * ov > sign * val ||
                                        (ov == val && oi < idx));
        if (better) {
            val = ov;
            idx = oi;
        }
    }
}

/* SphericalKdTree::endFrame (models.cpp:202-298), one warp per tree: the node loops run across
 * lanes (sums in node order, first-index extremes), the split-collapse step on lane 0 */
__device__ void kd_end_frame_warp(KdNode *K, double *P, double *A, int nn, int leaves,
                                  double blend, double tsplit, unsigned lane, int *scratch) {
    const double total = warp_ordered_sum_f(nn, lane, [&](int i) { return K[i].leaf ? A[i] : 0.0; });
    if (total > 0.0) {
        const double floor_prob = 1e-4 / leaves;
        const double norm_sum = warp_ordered_sum_f(nn, lane, [&](int i) {
            return K[i].leaf ? max_ref(A[i] / total, floor_prob) : 0.0;
        });
        for (int i = lane; i < nn; i += 32)
            if (K[i].leaf) {
                const double target = max_ref(A[i] / total, floor_prob) / norm_sum;
                P[i] = (1.0 - blend) * P[i] + blend * target;
            }
        __syncwarp();
        const double prob_sum =
            warp_ordered_sum_f(nn, lane, [&](int i) { return K[i].leaf ? P[i] : 0.0; });
        __syncwarp();
        for (int i = lane; i < nn; i += 32)
            if (K[i].leaf) P[i] /= prob_sum;
        __syncwarp();
    }
    /* l_max: first leaf of highest prob (the reference starts from pMax = -1: every leaf
     * qualifies); p_min: first internal node over two leaves of lowest pair mass below 2 */
    double p_max = -1.0, p_min_mass = 2.0;
    int l_max = -1, p_min = -1;
    for (int i = lane; i < nn; i += 32) {
        const KdNode n = K[i];
        if (n.leaf) {
            if (P[i] > p_max) {
                p_max = P[i];
                l_max = i;
            }
        } else if (K[n.left].leaf && K[n.right].leaf) {
            const double mass = P[n.left] + P[n.right];
            if (mass < p_min_mass) {
                p_min_mass = mass;
                p_min = i;
            }
        }
    }
    warp_first_extreme(p_max, l_max, 1.0);
    warp_first_extreme(p_min_mass, p_min, -1.0);
    if (lane == 0 && l_max >= 0 && p_min >= 0 && K[l_max].parent != p_min &&
        p_max > tsplit * p_min_mass) {
        const int freed_l = K[p_min].left, freed_r = K[p_min].right;
        K[p_min].leaf = 1; /* the coldest leaf pair collapses into its parent */
        P[p_min] = p_min_mass;
        A[p_min] = 0.0;
        K[p_min].left = K[p_min].right = -1;
        /* the hot leaf's rectangle, from the root down its ancestor chain */
        int *chain = scratch;
        int nc = 0;
        for (int n = l_max; n != -1; n = K[n].parent) chain[nc++] = n;
        double2 lo = make_double2(0.0, 0.0), hi = make_double2(1.0, 1.0);
        for (int i = nc - 1; i >= 1; --i) {
            const KdNode &n = K[chain[i]];
            const double split_abs = n.axis == 0 ? lerp_ref(lo.x, hi.x, n.split)
                                                 : lerp_ref(lo.y, hi.y, n.split);
            const bool to_left = chain[i - 1] == n.left;
            if (n.axis == 0) {
                if (to_left) hi.x = split_abs; else lo.x = split_abs;
            } else {
                if (to_left) hi.y = split_abs; else lo.y = split_abs;
            }
        }
        KdNode &hot = K[l_max]; /* splits at the midpoint of its longer axis */
        hot.leaf = 0;
        hot.axis = (hi.x - lo.x) >= (hi.y - lo.y) ? 0 : 1;
        hot.split = 0.5;
        hot.left = freed_l;
        hot.right = freed_r;
        const int kids[2] = {freed_l, freed_r};
        for (int c : kids) {
            KdNode z;
            z.split = 0.5;
            z.mass = 0.0;
            z.left = z.right = -1;
            z.parent = l_max;
            z.leaf = 1;
            z.axis = 0;
            K[c] = z;
            P[c] = p_max * 0.5;
        }
        P[l_max] = 0.0;
    }
    __syncwarp();
    for (int i = lane; i < nn; i += 32) A[i] = 0.0;
    __syncwarp();
    if (lane == 0) kd_refresh_mass(K, P, nn, scratch);
    __syncwarp();
}

/* ---- Gmm (models.cpp:427-702) on one entry's state vector ----
 * layout (C components): W[C] weights, M[2C] means, V[3C] cov (cxx, cxy, cyy), U[8C] stepwise
 * statistics, K[7C] cache (inv[3], norm, chol[3]), then i, underflows, reseed counter */
#define GMM_TWO_PI (2.0 * 3.14159265358979323846) /* kTwoPi, vecmath.h:13-14 */
#define GMM_MAX_COMPS 8

struct GmmView {
    double *W, *M, *V, *U, *K, *tail;
    int C;
};

__host__ __device__ inline GmmView gmm_view(double *S, int C) {
    return GmmView{S, S + C, S + 3 * C, S + 6 * C, S + 14 * C, S + 21 * C, C};
}

/* Gmm::rebuildCache (models.cpp:449-463) for component c */
__host__ __device__ inline void gmm_cache(GmmView g, int c) {
    const double a = g.V[3 * c], b = g.V[3 * c + 1], d = g.V[3 * c + 2];
    const double det = a * d - b * b;
    double *k = g.K + 7 * c;
    k[0] = d / det;
    k[1] = -b / det;
    k[2] = a / det;
    k[3] = 1.0 / (GMM_TWO_PI * sqrt(det));
    k[4] = sqrt(a);
    k[5] = b / k[4];
    const double r = d - k[5] * k[5];
    k[6] = sqrt(r < 0.0 ? 0.0 : r); /* std::max(., 0.0) */
}

/* componentPdf (models.cpp:465-480): the Gaussian wrapped over the 3x3 torus replicas */
__device__ inline double gmm_component_pdf(const GmmView &g, int c, double x, double y) {
    const double *k = g.K + 7 * c;
    double sum = 0.0;
    for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
            const double ex = x + dx - g.M[2 * c], ey = y + dy - g.M[2 * c + 1];
            const double q = k[0] * ex * ex + 2.0 * k[1] * ex * ey + k[2] * ey * ey;
            sum += k[3] * exp(-0.5 * q);
        }
    return sum;
}

/* Gmm::pdf (models.cpp:657-662) */
__device__ inline double gmm_pdf(const GmmView &g, double x, double y) {
    double p = 0.0;
    for (int c = 0; c < g.C; ++c) p += g.W[c] * gmm_component_pdf(g, c, x, y);
    return p;
}

/* responsibilities (models.cpp:482-497); returns 1 when the mixture underflowed */
__device__ inline int gmm_resp(const GmmView &g, double x, double y, double *gamma) {
    double total = 0.0;
    for (int c = 0; c < g.C; ++c) {
        gamma[c] = g.W[c] * gmm_component_pdf(g, c, x, y);
        total += gamma[c];
    }
    if (total <= 0.0 || !isfinite(total)) {
        for (int c = 0; c < g.C; ++c) gamma[c] = 1.0 / g.C;
        return 1;
    }
    for (int c = 0; c < g.C; ++c) gamma[c] /= total;
    return 0;
}

/* Gmm::mstep (models.cpp:587-655), sequential (lane 0) */
__device__ void gmm_mstep(GmmView g, const MdlDev &m) {
    const int C = g.C;
    double total = 0.0;
    for (int c = 0; c < C; ++c) total += g.U[8 * c];
    if (total <= 0.0) return;
    int heaviest = 0;
    for (int c = 1; c < C; ++c)
        if (g.U[8 * c] > g.U[8 * heaviest]) heaviest = c;
    for (int c = 0; c < C; ++c) {
        const double *u = g.U + 8 * c;
        const double mass = u[0];
        if (mass <= m.reseed_frac * total) { /* reseed next to the heaviest component */
            const double *h = g.U + 8 * heaviest;
            const double sx = h[1] / h[0], sy = h[2] / h[0];
            const uint32_t rc = (uint32_t)g.tail[2];
            g.tail[2] = (double)(uint32_t)(rc + 1u);
            const double jitter = 0.05 * (1.0 + (double)(rc % 7u));
            double mx = sx + jitter * 0.01, my = sy - jitter * 0.01;
            mx -= floor(mx);
            my -= floor(my);
            g.M[2 * c] = mx;
            g.M[2 * c + 1] = my;
            g.W[c] = 1e-3;
            g.V[3 * c] = 0.01;
            g.V[3 * c + 1] = 0.0;
            g.V[3 * c + 2] = 0.01;
            continue;
        }
        g.W[c] = mass / total;
        const double mx = u[1] / mass, my = u[2] / mass;
        const double exx = u[3] / mass, eyy = u[4] / mass, exy = u[5] / mass;
        const double cxx = exx - mx * mx, cyy = eyy - my * my, cxy = exy - mx * my;
        const double tr = cxx + cyy, diff = cxx - cyy;
        const double dd = diff * diff + 4.0 * cxy * cxy;
        const double disc = sqrt(dd < 0.0 ? 0.0 : dd);
        const double l1 = 0.5 * (tr + disc), l2 = 0.5 * (tr - disc);
        const double c1 = clamp_ref(l1, m.smin, m.smax), c2 = clamp_ref(l2, m.smin, m.smax);
        double vx, vy;
        if (fabs(cxy) > 1e-30) {
            vx = l1 - cyy;
            vy = cxy;
        } else {
            vx = cxx >= cyy ? 1.0 : 0.0;
            vy = cxx >= cyy ? 0.0 : 1.0;
        }
        const double len = sqrt(vx * vx + vy * vy);
        if (len > 0.0) {
            vx /= len;
            vy /= len;
        }
        g.V[3 * c] = c1 * vx * vx + c2 * vy * vy;
        g.V[3 * c + 1] = (c1 - c2) * vx * vy;
        g.V[3 * c + 2] = c1 * vy * vy + c2 * vx * vx;
        g.M[2 * c] = mx;
        g.M[2 * c + 1] = my;
    }
    double wsum = 0.0;
    for (int c = 0; c < C; ++c) wsum += g.W[c];
    for (int c = 0; c < C; ++c) g.W[c] /= wsum;
    for (int c = 0; c < C; ++c) gmm_cache(g, c);
}

/* Gmm::estepBatch (models.cpp:525-585), sample-parallel.  An entry's n frame samples are cut
 * into chunks of GMM_CHUNK; every chunk is one warp in each of two passes:
 *   A  the chunk's sum of log(1 - (i0+k)^-alpha) (the factor of index k; zero up to the
 *      restart at i0 + k == 1, as the reference's lastZero);
 *   (per entry, sequential over its chunks: the chunk offsets of logPrefix and logPrefix[n])
 *   C  per sample: responsibilities at the pre-batch mixture, g(j) = exp(logPrefix[n] -
 *      logPrefix[j]), the stepScale-weighted terms, summed per chunk in lane order;
 * then per entry: U = U * g(0) + the chunk partials in chunk order, i += n, mstep.  The sums
 * associate differently from the reference's sequential loops: agreement to rounding. */
#define GMM_CHUNK 256

struct GmmChunks {
    const uint32_t *chbase; /* exclusive scan of the chunk counts over the touched list */
    double *lsum, *off, *ln; /* per chunk: log-factor sum, logPrefix at its start; per entry: total */
    double *part;            /* per chunk: 8C partial statistics */
    unsigned long long *uflow;
    const uint32_t *pos;     /* frame samples in entry order */
};

__device__ __forceinline__ double gmm_lfac(uint64_t i0, uint32_t k, double alpha) {
    if (i0 + k <= 1) return 0.0; /* factor 0 at i0 + k == 1: logPrefix restarts there */
    return log(1.0 - pow((double)(i0 + k), -alpha));
}

/* chunk q -> (touched index t, chunk k of that entry); chbase[t] <= q < chbase[t + 1] */
__device__ __forceinline__ uint32_t gmm_chunk_owner(const uint32_t *chbase, uint32_t nt,
                                                    uint32_t q) {
    uint32_t lo = 0, hi = nt; /* chbase[lo] <= q < chbase[hi] */
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (chbase[mid] <= q) lo = mid; else hi = mid;
    }
    return lo;
}

/* accumulator slot of a record: the DirGrid cell or the k-d tree leaf */
__device__ __forceinline__ int mdl_slot(const MdlDev &m, uint32_t e, double u, double v) {
    if (m.kind == PSTF_MODEL_GRID) return mdl_cell(u, v, m.res);
    if (m.kind == PSTF_MODEL_GMM) return 0; /* one run per entry: its samples in canonical order */
    return kd_find_leaf(m.kn + (uint64_t)e * m.ns, u, v, nullptr, nullptr);
}

/* find-or-insert a key (field.h:38-41 equality); -1 when the table is full.  Threads carrying
 * the same new key meet at the entry the first of them claims (same probe sequence; a claimed
 * entry is waited for until published).  A new entry is a fresh DirGrid: uniform weights
 * 1/R^2, total 1 (models.cpp:16-22), zero counters (estimators.cpp:111-113). */
__device__ int32_t mdl_find_or_insert(const MdlDev &m, const KeyFields &k) {
    const uint32_t home = mdl_home(k, m.mask);
    for (uint32_t i = 0; i <= m.mask; ++i) {
        const uint32_t e = (home + i) & m.mask;
        uint32_t s = ld_state(&m.state[e]);
        if (s == 0) {
            s = atomicCAS(&m.state[e], 0u, 1u);
            if (s == 0) { /* claimed: write the entry, then publish it */
                m.keyf[e] = k;
                ModelEnt z;
                z.total = 1.0;
                z.c_old = z.c_new = 0.0;
                z.records = z.rec_count = 0;
                z.warm = z.touched = 0;
                m.ent[e] = z;
                if (m.kind == PSTF_MODEL_GRID) {
                    const double w0 = 1.0 / ((double)m.res * m.res);
                    for (int j = 0; j < m.ns; ++j) {
                        m.w[(uint64_t)e * m.ns + j] = w0;
                        m.acc[(uint64_t)e * m.ns + j] = 0.0;
                    }
                } else { /* the initial tree / mixture (models.cpp:96-127, 427-447), built
                          * once on the host into the template entry */
                    const uint64_t t = (uint64_t)(m.mask + 1ull) * m.ns;
                    for (int j = 0; j < m.ns; ++j) {
                        m.w[(uint64_t)e * m.ns + j] = m.w[t + j];
                        m.acc[(uint64_t)e * m.ns + j] = 0.0;
                        if (m.kind == PSTF_MODEL_KDTREE) m.kn[(uint64_t)e * m.ns + j] = m.kn[t + j];
                    }
                }
                __threadfence();
                atomicExch(&m.state[e], 2u);
                atomicAdd(&m.ctr[MC_ENTRIES], 1ull);
                return (int32_t)e;
            }
        }
        while (s == 1) s = ld_state(&m.state[e]); /* another key is being written here */
        if (kf_equal(m.keyf[e], k)) return (int32_t)e;
    }
    return -1;
}

/* per record: its entry (inserting new keys) and the sort words, most significant first:
 * (entry, grid cell) in the top bits of word 0, then uv.x, uv.y, contribution.  Sorting on them
 * puts each (entry, cell)'s records in the canonical order of estimators.cpp:633-637 (only the
 * order within one key matters: records of different keys never share an accumulator).
 * Records of keys without an entry (table full) sort last and are counted as dropped. */
__global__ void k_mdl_records(MdlDev m, const pstf_key *keys, const double *u, const double *v,
                              const double *c, uint64_t n, int shift, uint64_t *words) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t e = mdl_find_or_insert(m, kf_of(keys[i]));
    uint64_t w0 = ~0ull;
    if (e >= 0)
        w0 = ((uint64_t)e << 16 | (uint32_t)mdl_slot(m, (uint32_t)e, u[i], v[i])) << shift;
    else
        atomicAdd(&m.ctr[MC_DROPPED], 1ull);
    words[0 * n + i] = w0;
    words[1 * n + i] = ord_f64(u[i]);
    words[2 * n + i] = ord_f64(v[i]);
    words[3 * n + i] = ord_f64(c[i]);
}

/* one thread per (entry, cell) run of the sorted records: DirGrid::record (models.cpp:30-35)
 * folded in a register in the canonical order, and applyRecord's counters (estimators.cpp:
 * 114-116; cNew += 1 per record is integer-valued, so adding the run length is exact) */
__global__ void k_mdl_fold(MdlDev m, const uint64_t *words, const uint32_t *perm, uint64_t n,
                           int shift, const double *c) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t w = words[perm[i]];
    if (w == ~0ull || (i > 0 && words[perm[i - 1]] == w)) return; /* dropped, or not a run head */
    const uint64_t ec = w >> shift;
    const uint32_t e = (uint32_t)(ec >> 16);
    double *acc = m.acc + (uint64_t)e * m.ns + (uint32_t)(ec & 0xffffu);
    double s = *acc;
    unsigned long long cnt = 0, len = 0;
    for (uint64_t j = i; j < n; ++j) {
        const uint32_t r = perm[j];
        if (words[r] != w) break;
        const double cv = c[r];
        if (cv >= 0.0 && isfinite(cv)) {
            s += cv;
            ++cnt;
        }
        ++len;
    }
    *acc = s;
    ModelEnt &x = m.ent[e];
    if (cnt) atomicAdd(&x.rec_count, cnt);
    atomicAdd(&x.records, len);
    atomicAdd(&x.c_new, (double)len);
    if (atomicExch(&x.touched, 1u) == 0u) m.tlist[atomicAdd(&m.ctr[MC_TOUCHED], 1ull)] = e;
}

/* GMM apply: Gmm::record keeps the accepted samples in applyRecord order (models.cpp:689-694),
 * so each accepted record, in the call's canonical order, goes to position count + rank of the
 * frame-sample list (rank = exclusive scan of the accepted flags); ModelStore's counters are
 * added per warp-run of equal entries (integer-valued: any order is exact) */
__global__ void k_gmm_flags(const uint64_t *words, const uint32_t *perm, uint64_t n,
                            const double *c, uint32_t *flag) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t r = perm[i];
    const double cv = c[r];
    flag[i] = words[r] != ~0ull && cv >= 0.0 && isfinite(cv);
}

__global__ void k_gmm_append(MdlDev m, const uint64_t *words, const uint32_t *perm, uint64_t n,
                             int shift, const uint32_t *flag, const uint32_t *rank,
                             const double *u, const double *v, const double *c) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const bool live = i < n;
    int64_t e = -1;
    bool ok = false;
    if (live) {
        const uint32_t r = perm[i];
        const uint64_t w = words[r];
        if (w != ~0ull) {
            e = (int64_t)((w >> shift) >> 16);
            ok = flag[i] != 0;
            if (ok) {
                const uint64_t o = m.ctr[MC_SAMPLES] + rank[i];
                m.fs_entry[o] = (uint32_t)e;
                m.fs_u[o] = u[r];
                m.fs_v[o] = v[r];
                m.fs_c[o] = c[r];
            }
        }
    }
    const unsigned grp = __match_any_sync(0xffffffffu, (long long)e);
    const unsigned okm = __ballot_sync(0xffffffffu, ok);
    if (e < 0 || lane_id() != (unsigned)(__ffs(grp) - 1)) return;
    const unsigned len = __popc(grp), acc_n = __popc(okm & grp);
    ModelEnt &x = m.ent[e];
    if (acc_n) atomicAdd(&x.rec_count, (unsigned long long)acc_n);
    atomicAdd(&x.records, (unsigned long long)len);
    atomicAdd(&x.c_new, (double)len);
    if (atomicExch(&x.touched, 1u) == 0u) m.tlist[atomicAdd(&m.ctr[MC_TOUCHED], 1ull)] = (uint32_t)e;
}

__global__ void k_gmm_count(MdlDev m, const uint32_t *flag, const uint32_t *rank, uint64_t n) {
    m.ctr[MC_SAMPLES] += rank[n - 1] + flag[n - 1];
}

/* ATOMIC mode: records applied straight into the entries, no sort.  Accumulator sums then
 * depend on the atomic order (within 1e-12 relative of the canonical order); entries, counts,
 * warm flags and every integer-valued field stay exact.  Counters are aggregated over the lanes
 * of a warp that share an entry. */
__global__ void k_mdl_atomic(MdlDev m, const pstf_key *keys, const double *u, const double *v,
                             const double *c, uint64_t n) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const bool live = i < n;
    int32_t e = -2;
    bool ok = false;
    if (live) {
        e = mdl_find_or_insert(m, kf_of(keys[i]));
        if (e >= 0) {
            const double cv = c[i];
            ok = cv >= 0.0 && isfinite(cv);
            if (ok) atomicAdd(m.acc + (uint64_t)e * m.ns + mdl_slot(m, (uint32_t)e, u[i], v[i]), cv);
        }
    }
    const unsigned grp = __match_any_sync(0xffffffffu, e);
    const unsigned okm = __ballot_sync(0xffffffffu, ok);
    const unsigned lane = lane_id();
    if (e == -2 || lane != (unsigned)(__ffs(grp) - 1)) return;
    const unsigned len = __popc(grp), acc_n = __popc(okm & grp);
    if (e < 0) {
        atomicAdd(&m.ctr[MC_DROPPED], (unsigned long long)len);
        return;
    }
    ModelEnt &x = m.ent[e];
    if (acc_n) atomicAdd(&x.rec_count, (unsigned long long)acc_n);
    atomicAdd(&x.records, (unsigned long long)len);
    atomicAdd(&x.c_new, (double)len);
    if (atomicExch(&x.touched, 1u) == 0u) m.tlist[atomicAdd(&m.ctr[MC_TOUCHED], 1ull)] = (uint32_t)e;
}

/* endFrame pass 1: Σ cNew over touched entries and their number (estimators.cpp:122-128) */
__global__ void k_mdl_sums(MdlDev m, double *sums) {
    const uint64_t nt = m.ctr[MC_TOUCHED];
    double s = 0.0, t = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nt;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double cn = m.ent[m.tlist[i]].c_new;
        if (cn > 0.0) {
            s += cn;
            t += 1.0;
        }
    }
    s = warp_sum_d(s);
    t = warp_sum_d(t);
    if (lane_id() == 0 && t > 0.0) { /* integer-valued: exact in any order */
        atomicAdd(&sums[0], s);
        atomicAdd(&sums[1], t);
    }
}

/* sum of x[0..n) in index order (the reference's sequential loop), by one warp: lanes load
 * 32 consecutive values, every lane adds them in order via broadcasts (identical results) */
__device__ __forceinline__ double warp_ordered_sum(const double *x, int n, unsigned lane) {
    double s = 0.0;
    for (int b = 0; b < n; b += 32) {
        const double mine = b + (int)lane < n ? x[b + lane] : 0.0;
        const int k = min(32, n - b);
        for (int l = 0; l < k; ++l) s += __shfl_sync(0xffffffffu, mine, l);
    }
    return s;
}

/* endFrame pass 2 (estimators.cpp:129-143) with DirGrid::endFrame (models.cpp:37-50), one warp
 * per touched entry: elementwise blend across lanes, the two grid sums in index order */
/* ModelStore::endFrame's per-entry step (estimators.cpp:133-142) around the model's own
 * endFrame: the blend weight first, then cOld, the cap, cNew and warm */
__device__ __forceinline__ double mdl_alpha(const ModelEnt &x, double t_max, int limited) {
    double alpha = sqrt(x.c_new / (x.c_old + x.c_new));
    if (limited) alpha = max_ref(alpha, 1.0 / t_max);
    return alpha;
}

__device__ __forceinline__ void mdl_close(ModelEnt &x, const double *sums, double t_max,
                                          int limited, int min_samples) {
    const double touched = sums[1];
    const double cap = limited && touched > 0.0 ? (t_max * t_max - t_max) * (sums[0] / touched)
                                                : 0.0;
    x.c_old += x.c_new;
    if (limited) x.c_old = min_ref(x.c_old, cap);
    x.c_new = 0.0;
    x.warm = x.records >= (unsigned long long)(long long)min_samples;
}

__global__ void k_mdl_blend(MdlDev m, const double *sums, double t_max, int limited,
                            int min_samples) {
    const uint64_t nt = m.ctr[MC_TOUCHED];
    const unsigned lane = lane_id();
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < nt;
         i += nwarps) { /* persistent: the touched count is known only on the device */
        const uint32_t e = m.tlist[i];
        ModelEnt x = m.ent[e];
        x.touched = 0;
        if (x.c_new > 0.0) {
            double *w = m.w + (uint64_t)e * m.ns, *acc = m.acc + (uint64_t)e * m.ns;
            const double alpha = mdl_alpha(x, t_max, limited);
            const double sum = warp_ordered_sum(acc, m.ns, lane);
            __syncwarp();
            if (sum > 0.0) {
                for (int j = lane; j < m.ns; j += 32)
                    w[j] = (1.0 - alpha) * w[j] + alpha * (acc[j] / sum);
                __syncwarp();
                x.total = warp_ordered_sum(w, m.ns, lane);
            }
            for (int j = lane; j < m.ns; j += 32) acc[j] = 0.0;
            mdl_close(x, sums, t_max, limited, min_samples);
        }
        __syncwarp();
        if (lane == 0) m.ent[e] = x;
    }
}

/* the same for k-d tree entries, one warp per touched entry; the tree (nodes, prob, accum) is
 * staged in the warp's slice of shared memory, so the sequential steps (split-collapse,
 * refreshMass) run at shared-memory rather than L2 latency */
#define KD_WARPS 4
#define KD_SMEM_PER_NODE 56 /* node 32 + prob 8 + accum 8 + scratch int 4, 8-aligned */
__global__ void __launch_bounds__(KD_WARPS * 32) k_mdl_blend_kd(MdlDev m, const double *sums,
                                                                double t_max, int limited,
                                                                int min_samples) {
    extern __shared__ __align__(16) unsigned char kd_smem[];
    const uint64_t nt = m.ctr[MC_TOUCHED];
    const unsigned lane = lane_id();
    const int nn = m.ns;
    unsigned char *mine = kd_smem + (size_t)(threadIdx.x >> 5) * nn * KD_SMEM_PER_NODE;
    KdNode *Ks = reinterpret_cast<KdNode *>(mine);
    double *Ps = reinterpret_cast<double *>(mine + (size_t)nn * 32);
    double *As = Ps + nn;
    int *scratch = reinterpret_cast<int *>(As + nn); /* ancestor chain, then the BFS order */
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < nt;
         i += nwarps) {
        const uint32_t e = m.tlist[i];
        ModelEnt x = m.ent[e];
        x.touched = 0;
        if (x.c_new > 0.0) {
            const uint64_t b = (uint64_t)e * nn;
            for (int j = lane; j < nn; j += 32) {
                Ks[j] = m.kn[b + j];
                Ps[j] = m.w[b + j];
                As[j] = m.acc[b + j];
            }
            __syncwarp();
            kd_end_frame_warp(Ks, Ps, As, nn, m.leaves, mdl_alpha(x, t_max, limited), m.tsplit,
                              lane, scratch);
            for (int j = lane; j < nn; j += 32) {
                m.kn[b + j] = Ks[j];
                m.w[b + j] = Ps[j];
                m.acc[b + j] = 0.0;
            }
            __syncwarp();
            mdl_close(x, sums, t_max, limited, min_samples);
        }
        if (lane == 0) m.ent[e] = x;
    }
}

/* GMM endFrame: frame samples sorted by entry (stable: each entry keeps applyRecord order) */
__global__ void k_gmm_keys(MdlDev m, uint64_t bound, uint32_t *key, uint32_t *pos) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= bound) return;
    key[i] = i < m.ctr[MC_SAMPLES] ? m.fs_entry[i] : 0xffffffffu; /* unused tail sorts last */
    pos[i] = (uint32_t)i;
}

__global__ void k_gmm_segs(MdlDev m, const uint32_t *key, uint64_t bound) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= bound) return;
    const uint32_t e = key[i];
    if (e == 0xffffffffu) return;
    if (i == 0 || key[i - 1] != e) m.seg_begin[e] = (uint32_t)i;
    if (i + 1 == bound || key[i + 1] != e) m.seg_end[e] = (uint32_t)i + 1;
}

/* chunk counts per touched entry (0 without samples or past the touched list) */
__global__ void k_gmm_nchunks(MdlDev m, uint64_t cap, uint32_t *nch) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t > cap) return;
    uint32_t c = 0;
    if (t < m.ctr[MC_TOUCHED]) {
        const uint32_t e = m.tlist[t];
        const uint32_t n = m.seg_end[e] - m.seg_begin[e];
        c = (n + GMM_CHUNK - 1) / GMM_CHUNK;
    }
    nch[t] = c;
}

/* pass A: log-factor sum of each chunk */
__global__ void k_gmm_chunk_logs(MdlDev m, GmmChunks ch) {
    const uint32_t nt = (uint32_t)m.ctr[MC_TOUCHED];
    const uint32_t total = ch.chbase[nt];
    const unsigned lane = lane_id();
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < total; q += nwarps) {
        const uint32_t t = gmm_chunk_owner(ch.chbase, nt, q), e = m.tlist[t];
        const uint32_t n = m.seg_end[e] - m.seg_begin[e];
        const uint64_t i0 = (uint64_t)gmm_view(m.w + (uint64_t)e * m.ns, m.comps).tail[0];
        const uint32_t j0 = (q - ch.chbase[t]) * GMM_CHUNK; /* samples j0+1 .. */
        double x = 0.0;
        for (uint32_t j = j0 + lane + 1; j <= min(n, j0 + GMM_CHUNK); j += 32)
            x += gmm_lfac(i0, j, m.alpha_em);
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) ch.lsum[q] = x;
    }
}

/* per entry: logPrefix at each chunk start and logPrefix[n] */
__global__ void k_gmm_chunk_offsets(MdlDev m, GmmChunks ch) {
    const uint32_t nt = (uint32_t)m.ctr[MC_TOUCHED];
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    double run = 0.0;
    for (uint32_t q = ch.chbase[t]; q < ch.chbase[t + 1]; ++q) {
        ch.off[q] = run;
        run += ch.lsum[q];
    }
    ch.ln[t] = run;
}

/* pass C: each chunk's statistics at the pre-batch mixture */
#define GMM_WARPS 2
__global__ void __launch_bounds__(GMM_WARPS * 32) k_gmm_chunk_stats(MdlDev m, GmmChunks ch) {
    extern __shared__ __align__(16) unsigned char gmm_smem[];
    const int C = m.comps, Q = 8 * C;
    double *red = reinterpret_cast<double *>(gmm_smem) + (size_t)(threadIdx.x >> 5) * 32 * Q;
    const uint32_t nt = (uint32_t)m.ctr[MC_TOUCHED];
    const uint32_t total = ch.chbase[nt];
    const unsigned lane = lane_id();
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < total; q += nwarps) {
        const uint32_t t = gmm_chunk_owner(ch.chbase, nt, q), e = m.tlist[t];
        const uint32_t b = m.seg_begin[e], n = m.seg_end[e] - b;
        const GmmView g = gmm_view(m.w + (uint64_t)e * m.ns, C);
        const uint64_t i0 = (uint64_t)g.tail[0];
        const uint32_t j0 = (q - ch.chbase[t]) * GMM_CHUNK, j1 = min(n, j0 + GMM_CHUNK);
        const double ln = ch.ln[t];
        for (int k = 0; k < Q; ++k) red[lane * Q + k] = 0.0;
        unsigned long long uflow = 0;
        double carry = ch.off[q];
        for (uint32_t jb = j0; jb < j1; jb += 32) {
            const uint32_t j = jb + lane + 1; /* sample index 1..n */
            double x = j <= j1 ? gmm_lfac(i0, j, m.alpha_em) : 0.0;
            for (int o = 1; o < 32; o <<= 1) { /* inclusive scan */
                const double y = __shfl_up_sync(0xffffffffu, x, o);
                if ((int)lane >= o) x += y;
            }
            const double lp = carry + x; /* logPrefix[j] */
            carry += __shfl_sync(0xffffffffu, x, 31);
            if (j > j1) continue;
            const uint32_t p = ch.pos[b + j - 1];
            const double sx = m.fs_u[p], sy = m.fs_v[p], w = m.fs_c[p];
            double gamma[GMM_MAX_COMPS];
            uflow += gmm_resp(g, sx, sy, gamma);
            const double gj = exp(ln - lp); /* gOf(j): j >= 1 >= lastZero */
            if (gj == 0.0) continue;
            const double step = pow((double)(i0 + j), -m.alpha_em);
            for (int c = 0; c < C; ++c) {
                const double bb = step * w * gamma[c];
                if (bb <= 0.0) continue;
                const double bg = bb * gj;
                double *r = red + lane * Q + 8 * c;
                r[0] += bg;
                r[1] += bg * sx;
                r[2] += bg * sy;
                r[3] += bg * sx * sx;
                r[4] += bg * sy * sy;
                r[5] += bg * sx * sy;
                r[6] += gj * step * w;
                r[7] += gj;
            }
        }
        for (int o = 16; o > 0; o >>= 1) uflow += __shfl_xor_sync(0xffffffffu, uflow, o);
        __syncwarp();
        for (int k = lane; k < Q; k += 32) { /* lanes in order */
            double acc = 0.0;
            for (int l = 0; l < 32; ++l) acc += red[l * Q + k];
            ch.part[(uint64_t)q * Q + k] = acc;
        }
        if (lane == 0) ch.uflow[q] = uflow;
        __syncwarp();
    }
}

/* per touched entry: U = U * g(0) + the chunk partials (chunk order), i += n, mstep, then
 * ModelStore's bookkeeping (estimators.cpp:129-143) */
__global__ void k_mdl_blend_gmm(MdlDev m, const double *sums, double t_max, int limited,
                                int min_samples, GmmChunks ch) {
    const uint64_t nt = m.ctr[MC_TOUCHED];
    const unsigned lane = lane_id();
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < nt;
         i += nwarps) {
        const uint32_t e = m.tlist[i];
        ModelEnt x = m.ent[e];
        x.touched = 0;
        if (x.c_new > 0.0) {
            const uint32_t n = m.seg_end[e] - m.seg_begin[e];
            if (n) { /* Gmm::endFrame (models.cpp:696-702): nothing without samples */
                GmmView g = gmm_view(m.w + (uint64_t)e * m.ns, m.comps);
                const int Q = 8 * m.comps;
                const uint64_t i0 = (uint64_t)g.tail[0];
                const double g0 = i0 == 0 ? 0.0 : exp(ch.ln[i]); /* gOf(0) */
                const uint32_t q0 = ch.chbase[i], q1 = ch.chbase[i + 1];
                for (int k = lane; k < Q; k += 32) {
                    double acc = g.U[k] * g0;
                    for (uint32_t q = q0; q < q1; ++q) acc += ch.part[(uint64_t)q * Q + k];
                    g.U[k] = acc;
                }
                unsigned long long uf = 0;
                for (uint32_t q = q0 + lane; q < q1; q += 32) uf += ch.uflow[q];
                for (int o = 16; o > 0; o >>= 1) uf += __shfl_xor_sync(0xffffffffu, uf, o);
                __syncwarp();
                if (lane == 0) {
                    g.tail[0] = (double)(i0 + n);
                    g.tail[1] += (double)uf;
                    gmm_mstep(g, m);
                }
                __syncwarp();
            }
            mdl_close(x, sums, t_max, limited, min_samples);
        }
        if (lane == 0) m.ent[e] = x;
    }
}

__device__ __forceinline__ int32_t mdl_find_warm(const MdlDev &m, const KeyFields &k) {
    const uint32_t home = mdl_home(k, m.mask);
    for (uint32_t i = 0; i <= m.mask; ++i) {
        const uint32_t e = (home + i) & m.mask;
        const uint32_t s = m.state[e];
        if (s == 0) return -1;
        if (kf_equal(m.keyf[e], k)) return m.ent[e].warm ? (int32_t)e : -1;
    }
    return -1;
}

__global__ void k_mdl_lookup(MdlDev m, const pstf_key *keys, uint64_t n, int32_t *out) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = mdl_find_warm(m, kf_of(keys[i]));
}

__global__ void k_mdl_lookup_levels(MdlDev m, KeyParams kp, pstf_vec3_soa pos, pstf_vec3_soa dir,
                                    const double *fp, uint64_t n, int32_t *out) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t e = -1;
    for (int l = select_level(kp, fp[i]); l <= kp.max_level && e < 0; ++l) {
        const Key k = key_for(kp, pos.x[i], pos.y[i], pos.z[i], dir.x[i], dir.y[i], dir.z[i], l);
        e = mdl_find_warm(m, KeyFields{k.level, k.cell[0], k.cell[1], k.cell[2], k.dir[0], k.dir[1]});
    }
    out[i] = e;
}

/* SphericalKdTree::pdf (models.cpp:169-174) */
__device__ __forceinline__ double kd_pdf(const MdlDev &m, int32_t e, double u, double v) {
    const uint64_t b = (uint64_t)e * m.ns;
    double2 lo, hi;
    const int leaf = kd_find_leaf(m.kn + b, u, v, &lo, &hi);
    const double area = (hi.x - lo.x) * (hi.y - lo.y);
    return area > 0.0 ? m.w[b + leaf] / area : 0.0;
}

/* SphericalKdTree::sample (models.cpp:176-200): hierarchical warping by subtree mass */
__device__ void kd_sample(const MdlDev &m, int32_t e, double ux, double uy, double *su,
                          double *sv, double *spdf) {
    const uint64_t b = (uint64_t)e * m.ns;
    const KdNode *K = m.kn + b;
    const double below_one = 0x1.fffffffffffffp-1; /* nexttoward(1.0, 0.0) */
    double rx = ux, ry = uy;
    double2 lo = make_double2(0.0, 0.0), hi = make_double2(1.0, 1.0);
    int node = 0;
    while (!K[node].leaf) {
        const KdNode n = K[node];
        const double mass = n.mass;
        const double left_frac = mass > 0.0 ? K[n.left].mass / mass : 0.5;
        double &coord = n.axis == 0 ? rx : ry;
        const double split_abs = n.axis == 0 ? lerp_ref(lo.x, hi.x, n.split)
                                             : lerp_ref(lo.y, hi.y, n.split);
        if (left_frac > 0.0 && (coord < left_frac || left_frac >= 1.0)) {
            coord = min_ref(coord / left_frac, below_one);
            if (n.axis == 0) hi.x = split_abs; else hi.y = split_abs;
            node = n.left;
        } else {
            coord = min_ref((coord - left_frac) / (1.0 - left_frac), below_one);
            if (n.axis == 0) lo.x = split_abs; else lo.y = split_abs;
            node = n.right;
        }
    }
    *su = lerp_ref(lo.x, hi.x, rx);
    *sv = lerp_ref(lo.y, hi.y, ry);
    const double area = (hi.x - lo.x) * (hi.y - lo.y);
    *spdf = area > 0.0 ? m.w[b + node] / area : 0.0;
}

/* DirGrid::pdf (models.cpp:52-56) / SphericalKdTree::pdf */
__device__ __forceinline__ double mdl_pdf(const MdlDev &m, int32_t e, double u, double v) {
    if (e < 0) return 1.0;
    if (m.kind == PSTF_MODEL_GMM) return gmm_pdf(gmm_view(m.w + (uint64_t)e * m.ns, m.comps), u, v);
    if (m.kind != PSTF_MODEL_GRID) return kd_pdf(m, e, u, v);
    const double tot = m.ent[e].total;
    if (tot <= 0.0) return 1.0;
    return m.w[(uint64_t)e * m.ns + mdl_cell(u, v, m.res)] / tot * (double)m.res * (double)m.res;
}

__global__ void k_mdl_pdf(MdlDev m, const int32_t *ent, const double *u, const double *v,
                          uint64_t n, double *out) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = mdl_pdf(m, ent[i], u[i], v[i]);
}

/* DirGrid::sample (models.cpp:58-92): row by the marginal, then column, residuals remapped */
__global__ void k_mdl_sample(MdlDev m, const int32_t *ent, const double *u1, const double *u2,
                             const double *usel, uint64_t n, double *su, double *sv,
                             double *spdf) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t e = ent[i];
    const double ux = u1[i], uy = u2[i];
    if (e >= 0 && m.kind == PSTF_MODEL_GMM) { /* Gmm::sample (models.cpp:664-687) */
        const GmmView g = gmm_view(m.w + (uint64_t)e * m.ns, m.comps);
        const double us = usel[i];
        int comp = 0;
        double acc = 0.0;
        for (int c = 0; c < g.C; ++c) {
            acc += g.W[c];
            if (us < acc || c == g.C - 1) {
                comp = c;
                break;
            }
        }
        const double om = 1.0 - ux;
        const double r = sqrt(-2.0 * log(om < 1e-300 ? 1e-300 : om)); /* std::max */
        const double z0 = r * cos(GMM_TWO_PI * uy), z1 = r * sin(GMM_TWO_PI * uy);
        const double *k = g.K + 7 * comp;
        double px = g.M[2 * comp] + k[4] * z0;
        double py = g.M[2 * comp + 1] + k[5] * z0 + k[6] * z1;
        px -= floor(px);
        py -= floor(py);
        su[i] = px;
        sv[i] = py;
        spdf[i] = gmm_pdf(g, px, py);
        return;
    }
    if (e >= 0 && m.kind != PSTF_MODEL_GRID) {
        kd_sample(m, e, ux, uy, &su[i], &sv[i], &spdf[i]);
        return;
    }
    if (e < 0 || m.ent[e].total <= 0.0) {
        su[i] = ux;
        sv[i] = uy;
        spdf[i] = 1.0;
        return;
    }
    const int R = m.res;
    const double *w = m.w + (uint64_t)e * m.ns;
    const double target = uy * m.ent[e].total;
    int row = 0;
    double row_sum = 0.0, acc = 0.0;
    for (; row < R; ++row) {
        row_sum = 0.0;
        for (int x = 0; x < R; ++x) row_sum += w[row * R + x];
        if (acc + row_sum > target || row == R - 1) break;
        acc += row_sum;
    }
    const double vin = row_sum > 0.0 ? clamp_ref((target - acc) / row_sum, 0.0, 1.0) : uy;
    const double col_target = ux * row_sum;
    int col = 0;
    double col_acc = 0.0, wc = 0.0;
    for (; col < R; ++col) {
        wc = w[row * R + col];
        if (col_acc + wc > col_target || col == R - 1) break;
        col_acc += wc;
    }
    const double uin = wc > 0.0 ? clamp_ref((col_target - col_acc) / wc, 0.0, 1.0) : ux;
    const double below_one = 0x1.fffffffffffffp-1; /* nexttoward(1.0, 0.0) */
    double x = (col + uin) / R, y = (row + vin) / R;
    x = below_one < x ? below_one : x;
    y = below_one < y ? below_one : y;
    su[i] = x;
    sv[i] = y;
    spdf[i] = mdl_pdf(m, e, x, y);
}

extern "C" {

/* the uniform tree of SphericalKdTree's constructor (models.cpp:96-127): nodes appended in
 * the constructor's order (children allocated when their parent is visited, left subtree
 * first), axis alternating with depth, midpoint splits, leaf prob 1/L, then the masses */
static void kd_initial_tree(int leaves, std::vector<KdNode> &K, std::vector<double> &P) {
    K.clear();
    P.clear();
    auto add = [&]() {
        KdNode z;
        z.split = 0.5;
        z.mass = 0.0;
        z.left = z.right = z.parent = -1;
        z.leaf = 1;
        z.axis = 0;
        K.push_back(z);
        P.push_back(0.0);
        return (int)K.size() - 1;
    };
    add();
    std::function<void(int, int, int)> build = [&](int node, int depth, int below) {
        if (below == 1) {
            K[node].leaf = 1;
            P[node] = 1.0 / leaves;
            return;
        }
        const int l = add(), r = add();
        K[node].leaf = 0;
        K[node].axis = (uint8_t)(depth & 1);
        K[node].split = 0.5;
        K[node].left = l;
        K[node].right = r;
        K[l].parent = node;
        K[r].parent = node;
        build(l, depth + 1, below / 2);
        build(r, depth + 1, below / 2);
    };
    build(0, 0, leaves);
    std::function<double(int)> mass = [&](int n) {
        K[n].mass = K[n].leaf ? P[n] : mass(K[n].left) + mass(K[n].right);
        return K[n].mass;
    };
    mass(0);
}

int pstf_model_create(const pstf_model_config *config, int device, pstf_model_store **out) {
    if (!config || !out) return set_err(PSTF_E_INVALID, "NULL argument");
    *out = nullptr;
    const bool kd = config->kind == PSTF_MODEL_KDTREE;
    if (config->kind < PSTF_MODEL_GRID || config->kind > PSTF_MODEL_GMM)
        return set_err(PSTF_E_INVALID, "kind must be PSTF_MODEL_GRID, _KDTREE or _GMM");
    if (config->kind == PSTF_MODEL_GRID &&
        (config->grid_resolution < 1 || config->grid_resolution > 256))
        return set_err(PSTF_E_INVALID, "grid_resolution must be in [1, 256]"); /* models.cpp:17-18 */
    if (kd && (config->kd_leaf_count < 2 || config->kd_leaf_count > 256 ||
               (config->kd_leaf_count & (config->kd_leaf_count - 1)) != 0)) /* models.cpp:99-101 */
        return set_err(PSTF_E_INVALID, "kd_leaf_count must be a power of two in [2, 256]");
    if (kd && !(config->kd_split_threshold > 1.0)) /* models.cpp:203-204 */
        return set_err(PSTF_E_INVALID, "kd_split_threshold must be > 1");
    const bool gmm = config->kind == PSTF_MODEL_GMM;
    if (gmm && (config->gmm_components < 1 || config->gmm_components > GMM_MAX_COMPS))
        return set_err(PSTF_E_INVALID, "gmm_components must be in [1, 8]"); /* models.cpp:429-430 */
    if (gmm && !(config->gmm_alpha_em > 0.5 && config->gmm_alpha_em <= 1.0))
        return set_err(PSTF_E_INVALID, "gmm_alpha_em must lie in (0.5, 1]"); /* models.cpp:431-432 */
    if (config->capacity_log2 < 1 || config->capacity_log2 > 26)
        return set_err(PSTF_E_INVALID, "capacity_log2 must be in [1, 26]");
    CK(cudaSetDevice(device));
    std::unique_ptr<pstf_model_store> m(new pstf_model_store());
    m->cfg = *config;
    m->device = device;
    const uint64_t cap = 1ull << config->capacity_log2;
    m->mask = (uint32_t)(cap - 1);
    m->ns = kd    ? 2 * config->kd_leaf_count - 1
            : gmm ? 21 * config->gmm_components + 3
                  : config->grid_resolution * config->grid_resolution;
    const uint64_t cells = (cap + 1) * (uint64_t)m->ns; /* + the k-d template entry */
    if (cells * 16 > (64ull << 30)) return set_err(PSTF_E_INVALID, "model table too large");
    ENSURE(m->state, cap * 4);
    ENSURE(m->keyf, cap * sizeof(KeyFields));
    ENSURE(m->ent, cap * sizeof(ModelEnt));
    ENSURE(m->w, cells * 8);
    ENSURE(m->acc, cells * 8);
    ENSURE(m->ctr, MC_N * 8);
    ENSURE(m->tlist, cap * 4);
    ENSURE(m->sums, 16);
    CK(cudaMemset(m->state.p, 0, cap * 4));
    CK(cudaMemset(m->ctr.p, 0, MC_N * 8));
    if (kd) {
        static_assert(sizeof(KdNode) == 32, "KdNode staging assumes 32 B nodes");
        CK(cudaFuncSetAttribute(k_mdl_blend_kd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                KD_WARPS * 511 * KD_SMEM_PER_NODE));
        ENSURE(m->kn, cells * sizeof(KdNode));
        std::vector<KdNode> K;
        std::vector<double> P;
        kd_initial_tree(config->kd_leaf_count, K, P);
        CK(cudaMemcpy(m->kn.as<KdNode>() + cap * m->ns, K.data(), m->ns * sizeof(KdNode),
                      cudaMemcpyHostToDevice));
        CK(cudaMemcpy(m->w.as<double>() + cap * m->ns, P.data(), m->ns * 8, cudaMemcpyHostToDevice));
    }
    if (gmm) { /* Gmm's constructor (models.cpp:427-447) into the template entry */
        const int C = config->gmm_components;
        std::vector<double> S(m->ns, 0.0);
        GmmView g = gmm_view(S.data(), C);
        int grid = 1;
        while (grid * grid < C) ++grid;
        for (int c = 0; c < C; ++c) {
            g.W[c] = 1.0 / C;
            g.V[3 * c] = 0.02;
            g.V[3 * c + 1] = 0.0;
            g.V[3 * c + 2] = 0.02;
            g.M[2 * c] = ((c % grid) + 0.5) / grid;
            g.M[2 * c + 1] = ((c / grid) + 0.5) / grid;
            gmm_cache(g, c);
        }
        CK(cudaMemcpy(m->w.as<double>() + cap * m->ns, S.data(), m->ns * 8, cudaMemcpyHostToDevice));
        ENSURE(m->seg, 2 * cap * 4);
        CK(cudaMemset(m->seg.p, 0, 2 * cap * 4));
        ENSURE(m->fs_entry, 1024 * 4);
        ENSURE(m->fs_u, 1024 * 8);
        ENSURE(m->fs_v, 1024 * 8);
        ENSURE(m->fs_c, 1024 * 8);
        CK(cudaFuncSetAttribute(k_gmm_chunk_stats, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                GMM_WARPS * 32 * 8 * GMM_MAX_COMPS * 8));
    }
    CK(cudaDeviceSynchronize());
    *out = m.release();
    return PSTF_OK;
}

int pstf_model_destroy(pstf_model_store *m) {
    if (!m) return PSTF_OK;
    cudaSetDevice(m->device);
    cudaDeviceSynchronize();
    delete m;
    return PSTF_OK;
}

/* grows b to at least `need` bytes keeping its first `keep` bytes (GMM frame samples) */
static int grow_keep(DBuf &b, size_t need, size_t keep, cudaStream_t st) {
    if (need <= b.bytes) return PSTF_OK;
    DBuf nb;
    ENSURE(nb, need);
    if (keep) CK(cudaMemcpyAsync(nb.p, b.p, keep, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    std::swap(b.p, nb.p);
    std::swap(b.bytes, nb.bytes); /* nb now owns (and frees) the old buffer */
    return PSTF_OK;
}

int pstf_model_apply(pstf_model_store *m, const pstf_key *keys, const double *u, const double *v,
                     const double *contribution, uint64_t n, int mode, void *stream) {
    if (!m || (n && (!keys || !u || !v || !contribution)))
        return set_err(PSTF_E_INVALID, "NULL argument");
    if (mode != PSTF_MODE_ATOMIC && mode != PSTF_MODE_ORDERED)
        return set_err(PSTF_E_INVALID, "mode must be PSTF_MODE_ATOMIC or PSTF_MODE_ORDERED");
    if (!n) return PSTF_OK;
    if (n >= 0xffffffffULL) return set_err(PSTF_E_INVALID, "batch too large");
    CK(cudaSetDevice(m->device));
    const cudaStream_t st = (cudaStream_t)stream;
    if (m->cfg.kind == PSTF_MODEL_GMM) { /* samples kept in canonical order (stepwise EM) */
        mode = PSTF_MODE_ORDERED;
        const uint64_t keep = m->fs_bound, need = keep + n;
        int rc = grow_keep(m->fs_entry, need * 4, keep * 4, st);
        if (!rc) rc = grow_keep(m->fs_u, need * 8, keep * 8, st);
        if (!rc) rc = grow_keep(m->fs_v, need * 8, keep * 8, st);
        if (!rc) rc = grow_keep(m->fs_c, need * 8, keep * 8, st);
        if (rc) return rc;
        m->fs_bound = need;
    }
    if (mode == PSTF_MODE_ATOMIC) {
        LAUNCH(k_mdl_atomic, grid_for(n, 256), 256, 0, st, m->dev(), keys, u, v, contribution, n);
        return PSTF_OK;
    }
    ENSURE(m->words, 4 * n * 8);
    uint64_t *words = m->words.as<uint64_t>();
    const int bits = 16 + (int)m->cfg.capacity_log2 + 1; /* entry index, cell, and the drop tag */
    const int shift = 64 - bits;
    const MdlDev d = m->dev();
    LAUNCH(k_mdl_records, grid_for(n, 256), 256, 0, st, d, keys, u, v, contribution, n, shift,
           words);
    const int bb[4] = {shift, 0, 0, 0};
    uint32_t *perm = nullptr;
    int rc = sort_multiword(m->sc, words, bb, 4, n, &perm, st);
    if (rc) return rc;
    if (m->cfg.kind == PSTF_MODEL_GMM) {
        ENSURE(m->fs_key, 2 * n * 4);
        uint32_t *flag = m->fs_key.as<uint32_t>(), *rank = flag + n;
        LAUNCH(k_gmm_flags, grid_for(n, 256), 256, 0, st, words, perm, n, contribution, flag);
        size_t bytes = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flag, rank, (int64_t)n, st));
        ENSURE(m->sc.cub, bytes);
        bytes = m->sc.cub.bytes;
        {
            ProfScope ps_("cub::DeviceScan", st);
            CK(cub::DeviceScan::ExclusiveSum(m->sc.cub.p, bytes, flag, rank, (int64_t)n, st));
            g_launches.fetch_add(2, std::memory_order_relaxed);
        }
        LAUNCH(k_gmm_append, grid_for(n, 256), 256, 0, st, d, words, perm, n, shift, flag, rank,
               u, v, contribution);
        LAUNCH(k_gmm_count, 1, 1, 0, st, d, flag, rank, n);
        return PSTF_OK;
    }
    LAUNCH(k_mdl_fold, grid_for(n, 256), 256, 0, st, d, words, perm, n, shift, contribution);
    return PSTF_OK;
}

int pstf_model_end_frame(pstf_model_store *m, void *stream) {
    if (!m) return set_err(PSTF_E_INVALID, "NULL argument");
    CK(cudaSetDevice(m->device));
    const cudaStream_t st = (cudaStream_t)stream;
    const MdlDev d = m->dev();
    const double t_max = m->cfg.t_max;
    const int limited = t_max > 0.0 && std::isfinite(t_max);
    CK(cudaMemsetAsync(m->sums.p, 0, 16, st));
    LAUNCH(k_mdl_sums, (unsigned)sm_count() * 2, 256, 0, st, d, m->sums.as<double>());
    if (m->cfg.kind == PSTF_MODEL_GMM) {
        const uint64_t bound = m->fs_bound, cap2 = (uint64_t)m->mask + 1;
        uint32_t *pos_sorted = nullptr;
        CK(cudaMemsetAsync(m->seg.p, 0, 2 * cap2 * 4, st));
        if (bound) { /* the frame's samples grouped by entry, each entry in record order */
            ENSURE(m->fs_key, 2 * bound * 4);
            ENSURE(m->fs_pos, 2 * bound * 4);
            uint32_t *key = m->fs_key.as<uint32_t>(), *pos = m->fs_pos.as<uint32_t>();
            LAUNCH(k_gmm_keys, grid_for(bound, 256), 256, 0, st, d, bound, key, pos);
            size_t bytes = 0;
            CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key, key + bound, pos, pos + bound,
                                               (int64_t)bound, 0, 32, st));
            ENSURE(m->sc.cub, bytes);
            bytes = m->sc.cub.bytes;
            {
                ProfScope ps_("cub::DeviceRadixSort", st);
                CK(cub::DeviceRadixSort::SortPairs(m->sc.cub.p, bytes, key, key + bound, pos,
                                                   pos + bound, (int64_t)bound, 0, 32, st));
                g_launches.fetch_add(4, std::memory_order_relaxed);
            }
            LAUNCH(k_gmm_segs, grid_for(bound, 256), 256, 0, st, d, key + bound, bound);
            pos_sorted = pos + bound;
        }
        /* chunked E-step: chunk counts -> their scan over the touched list -> passes A, C */
        ENSURE(m->gch_n, (cap2 + 2) * 4 * 2);
        uint32_t *nch = m->gch_n.as<uint32_t>(), *chbase = nch + cap2 + 2;
        LAUNCH(k_gmm_nchunks, grid_for(cap2 + 1, 256), 256, 0, st, d, cap2, nch);
        {
            size_t bytes = 0;
            CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, nch, chbase, (int64_t)(cap2 + 1), st));
            ENSURE(m->sc.cub, bytes);
            bytes = m->sc.cub.bytes;
            ProfScope ps_("cub::DeviceScan", st);
            CK(cub::DeviceScan::ExclusiveSum(m->sc.cub.p, bytes, nch, chbase, (int64_t)(cap2 + 1),
                                             st));
            g_launches.fetch_add(2, std::memory_order_relaxed);
        }
        const uint64_t max_chunks = bound / GMM_CHUNK + cap2 + 1;
        const int Q = 8 * m->cfg.gmm_components;
        ENSURE(m->gch_f, (max_chunks * (3 + Q) + cap2 + 1) * 8);
        GmmChunks gc;
        gc.chbase = chbase;
        gc.lsum = m->gch_f.as<double>();
        gc.off = gc.lsum + max_chunks;
        gc.part = gc.off + max_chunks;
        gc.ln = gc.part + max_chunks * Q;
        gc.uflow = reinterpret_cast<unsigned long long *>(gc.ln + cap2 + 1);
        gc.pos = pos_sorted;
        if (bound) {
            LAUNCH(k_gmm_chunk_logs, (unsigned)sm_count() * 8, 256, 0, st, d, gc);
            LAUNCH(k_gmm_chunk_offsets, grid_for(cap2, 128), 128, 0, st, d, gc);
            LAUNCH(k_gmm_chunk_stats, (unsigned)sm_count() * 16, GMM_WARPS * 32,
                   (size_t)GMM_WARPS * 32 * Q * 8, st, d, gc);
        }
        LAUNCH(k_mdl_blend_gmm, (unsigned)sm_count() * 8, 256, 0, st, d, m->sums.as<double>(),
               t_max, limited, m->cfg.min_samples, gc);
        CK(cudaMemsetAsync(&m->ctr.as<unsigned long long>()[MC_SAMPLES], 0, 8, st));
        m->fs_bound = 0;
    } else if (m->cfg.kind == PSTF_MODEL_GRID)
        LAUNCH(k_mdl_blend, (unsigned)sm_count() * 8, 256, 0, st, d, m->sums.as<double>(), t_max,
               limited, m->cfg.min_samples);
    else
        LAUNCH(k_mdl_blend_kd, (unsigned)sm_count() * 8, KD_WARPS * 32,
               (size_t)KD_WARPS * m->ns * KD_SMEM_PER_NODE, st, d, m->sums.as<double>(), t_max, limited,
               m->cfg.min_samples);
    CK(cudaMemsetAsync(&m->ctr.as<unsigned long long>()[MC_TOUCHED], 0, 8, st));
    return PSTF_OK;
}

int pstf_model_lookup_warm(const pstf_model_store *m, const pstf_key *keys, uint64_t n,
                           int32_t *entry, void *stream) {
    if (!m || (n && (!keys || !entry))) return set_err(PSTF_E_INVALID, "NULL argument");
    if (!n) return PSTF_OK;
    CK(cudaSetDevice(m->device));
    LAUNCH(k_mdl_lookup, grid_for(n, 256), 256, 0, (cudaStream_t)stream, m->dev(), keys, n, entry);
    return PSTF_OK;
}

int pstf_model_lookup_warm_levels(const pstf_model_store *m, const pstf_field *keyer,
                                  const pstf_vec3_soa *pos, const pstf_vec3_soa *dir,
                                  const double *footprint, uint64_t n, int32_t *entry,
                                  void *stream) {
    if (!m || !keyer || (n && (!pos || !dir || !footprint || !entry)))
        return set_err(PSTF_E_INVALID, "NULL argument");
    if (!n) return PSTF_OK;
    CK(cudaSetDevice(m->device));
    LAUNCH(k_mdl_lookup_levels, grid_for(n, 128), 128, 0, (cudaStream_t)stream, m->dev(),
           keyer->d.kp, *pos, *dir, footprint, n, entry);
    return PSTF_OK;
}

int pstf_model_pdf(const pstf_model_store *m, const int32_t *entry, const double *u,
                   const double *v, uint64_t n, double *pdf, void *stream) {
    if (!m || (n && (!entry || !u || !v || !pdf))) return set_err(PSTF_E_INVALID, "NULL argument");
    if (!n) return PSTF_OK;
    CK(cudaSetDevice(m->device));
    LAUNCH(k_mdl_pdf, grid_for(n, 256), 256, 0, (cudaStream_t)stream, m->dev(), entry, u, v, n, pdf);
    return PSTF_OK;
}

int pstf_model_sample(const pstf_model_store *m, const int32_t *entry, const double *u1,
                      const double *u2, const double *u_select, uint64_t n, double *su,
                      double *sv, double *pdf, void *stream) {
    if (!m || (n && (!entry || !u1 || !u2 || !su || !sv || !pdf)))
        return set_err(PSTF_E_INVALID, "NULL argument");
    if (n && m->cfg.kind == PSTF_MODEL_GMM && !u_select)
        return set_err(PSTF_E_INVALID, "GMM sampling needs u_select");
    if (!n) return PSTF_OK;
    CK(cudaSetDevice(m->device));
    LAUNCH(k_mdl_sample, grid_for(n, 128), 128, 0, (cudaStream_t)stream, m->dev(), entry, u1, u2,
           u_select, n, su, sv, pdf);
    return PSTF_OK;
}

int pstf_model_get_stats(pstf_model_store *m, pstf_model_stats *out) {
    if (!m || !out) return set_err(PSTF_E_INVALID, "NULL argument");
    CK(cudaSetDevice(m->device));
    CK(cudaDeviceSynchronize());
    unsigned long long c[MC_N];
    CK(cudaMemcpy(c, m->ctr.p, sizeof(c), cudaMemcpyDeviceToHost));
    const uint64_t cap = (uint64_t)m->mask + 1;
    std::vector<uint32_t> state(cap);
    std::vector<ModelEnt> ent(cap);
    CK(cudaMemcpy(state.data(), m->state.p, cap * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ent.data(), m->ent.p, cap * sizeof(ModelEnt), cudaMemcpyDeviceToHost));
    uint64_t warm = 0;
    for (uint64_t e = 0; e < cap; ++e) warm += state[e] == 2 && ent[e].warm;
    out->entries = c[MC_ENTRIES];
    out->warm = warm;
    out->dropped_records = c[MC_DROPPED];
    out->capacity = cap;
    return PSTF_OK;
}

int pstf_model_dump(pstf_model_store *m, pstf_model_entry *entries, double *weights,
                    double *accum, uint64_t cap_out, uint64_t *count) {
    if (!m || !count || (cap_out && !entries)) return set_err(PSTF_E_INVALID, "NULL argument");
    CK(cudaSetDevice(m->device));
    CK(cudaDeviceSynchronize());
    const uint64_t cap = (uint64_t)m->mask + 1, ns = (uint64_t)m->ns;
    std::vector<uint32_t> state(cap);
    std::vector<KeyFields> kf(cap);
    std::vector<ModelEnt> ent(cap);
    CK(cudaMemcpy(state.data(), m->state.p, cap * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(kf.data(), m->keyf.p, cap * sizeof(KeyFields), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ent.data(), m->ent.p, cap * sizeof(ModelEnt), cudaMemcpyDeviceToHost));
    std::vector<uint32_t> live;
    for (uint64_t e = 0; e < cap; ++e)
        if (state[e] == 2) live.push_back((uint32_t)e);
    std::sort(live.begin(), live.end(), [&](uint32_t a, uint32_t b) {
        const KeyFields &x = kf[a], &y = kf[b];
        return std::tie(x.level, x.c0, x.c1, x.c2, x.d0, x.d1) <
               std::tie(y.level, y.c0, y.c1, y.c2, y.d0, y.d1);
    });
    *count = live.size();
    const uint64_t k = std::min<uint64_t>(live.size(), cap_out);
    for (uint64_t i = 0; i < k; ++i) {
        const uint32_t e = live[i];
        pstf_model_entry &o = entries[i];
        memset(&o, 0, sizeof(o));
        o.level = kf[e].level;
        o.cell[0] = kf[e].c0;
        o.cell[1] = kf[e].c1;
        o.cell[2] = kf[e].c2;
        o.dir_cell[0] = kf[e].d0;
        o.dir_cell[1] = kf[e].d1;
        o.warm = ent[e].warm;
        o.c_old = ent[e].c_old;
        o.c_new = ent[e].c_new;
        o.records = ent[e].records;
        o.record_count = ent[e].rec_count;
        o.total = m->cfg.kind == PSTF_MODEL_GRID ? ent[e].total : 0.0; /* DirGrid::m_total */
        if (weights) CK(cudaMemcpy(weights + i * ns, m->w.as<double>() + (uint64_t)e * ns, ns * 8,
                                   cudaMemcpyDeviceToHost));
        if (accum) CK(cudaMemcpy(accum + i * ns, m->acc.as<double>() + (uint64_t)e * ns, ns * 8,
                                 cudaMemcpyDeviceToHost));
    }
    return PSTF_OK;
}

int pstf_model_dump_tree(pstf_model_store *m, int32_t *node_i32, double *node_f64, uint64_t cap_out,
                         uint64_t *count) {
    if (!m || !count) return set_err(PSTF_E_INVALID, "NULL argument");
    if (m->cfg.kind != PSTF_MODEL_KDTREE) return set_err(PSTF_E_INVALID, "not a k-d tree store");
    CK(cudaSetDevice(m->device));
    CK(cudaDeviceSynchronize());
    const uint64_t cap = (uint64_t)m->mask + 1, ns = (uint64_t)m->ns;
    std::vector<uint32_t> state(cap);
    std::vector<KeyFields> kf(cap);
    CK(cudaMemcpy(state.data(), m->state.p, cap * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(kf.data(), m->keyf.p, cap * sizeof(KeyFields), cudaMemcpyDeviceToHost));
    std::vector<uint32_t> live;
    for (uint64_t e = 0; e < cap; ++e)
        if (state[e] == 2) live.push_back((uint32_t)e);
    std::sort(live.begin(), live.end(), [&](uint32_t a, uint32_t b) {
        const KeyFields &x = kf[a], &y = kf[b];
        return std::tie(x.level, x.c0, x.c1, x.c2, x.d0, x.d1) <
               std::tie(y.level, y.c0, y.c1, y.c2, y.d0, y.d1);
    });
    *count = live.size();
    std::vector<KdNode> K(ns);
    for (uint64_t i = 0; i < std::min<uint64_t>(live.size(), cap_out); ++i) {
        CK(cudaMemcpy(K.data(), m->kn.as<KdNode>() + (uint64_t)live[i] * ns, ns * sizeof(KdNode),
                      cudaMemcpyDeviceToHost));
        for (uint64_t j = 0; j < ns; ++j) {
            if (node_i32) {
                int32_t *o = node_i32 + (i * ns + j) * 5;
                o[0] = K[j].leaf;
                o[1] = K[j].axis;
                o[2] = K[j].left;
                o[3] = K[j].right;
                o[4] = K[j].parent;
            }
            if (node_f64) {
                node_f64[(i * ns + j) * 2] = K[j].split;
                node_f64[(i * ns + j) * 2 + 1] = K[j].mass;
            }
        }
    }
    return PSTF_OK;
}

} // extern "C"
