/* CV-profile / guiding model store on the device.
 *
 * ModelStore (estimators.h:124-150, estimators.cpp:104-144) holding DirGrid models
 * (models.h:30-52, models.cpp:16-94).  Included at the end of field.cu (one translation unit:
 * it shares the scratch buffers, the multi-word radix sort and the exact key functions).
 *
 * Layout (per entry e of a 2^k open-addressing table, home = packKeyFields(key) & mask):
 *   state[e]   u32   0 empty, 1 being written, 2 ready (entries are never removed, as in the
 *                    reference's unordered_map)
 *   keyf[e]    6 x i32 key fields (equality ignores the checksum, field.h:38-41)
 *   ent[e]     {total, cOld, cNew, records, recordCount, warm, touched}
 *   w[e][R^2], acc[e][R^2]  f64 DirGrid weights / accumulators, row-major (iy * R + ix)
 *
 * apply:  every record finds (or inserts, CAS on state) its key's entry; the records are then
 *         radix-sorted by (entry, grid cell, uv.x, uv.y, contribution), which within one key
 *         is the canonical order of estimators.cpp:633-637, and one thread per (entry, cell)
 *         run folds it in a register: each accumulator sum has the reference's order.  No host
 *         round trip.
 * endFrame: the touched entries only (a list built by apply): Σ cNew (integer-valued, exact in
 *         any order), then one warp per entry blends its grid, the grid sums in index order. */

struct ModelEnt {
    double total, c_old, c_new;
    unsigned long long records, rec_count;
    uint32_t warm, touched;
};

struct MdlDev {
    uint32_t *state;
    KeyFields *keyf;
    ModelEnt *ent;
    double *w, *acc;
    unsigned long long *ctr; /* [0] entries, [1] dropped records, [2] touched-list length */
    uint32_t *tlist;
    uint32_t mask;
    int res, r2;
};

enum { MC_ENTRIES = 0, MC_DROPPED = 1, MC_TOUCHED = 2, MC_N = 4 };

struct pstf_model_store {
    pstf_model_config cfg;
    int device = 0;
    uint32_t mask = 0;
    int r2 = 0;
    DBuf state, keyf, ent, w, acc, ctr, tlist, sums;
    Scratch sc;
    DBuf words;
    MdlDev dev() const {
        MdlDev d;
        d.state = state.as<uint32_t>();
        d.keyf = keyf.as<KeyFields>();
        d.ent = ent.as<ModelEnt>();
        d.w = w.as<double>();
        d.acc = acc.as<double>();
        d.ctr = ctr.as<unsigned long long>();
        d.tlist = tlist.as<uint32_t>();
        d.mask = mask;
        d.res = cfg.grid_resolution;
        d.r2 = r2;
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
                const double w0 = 1.0 / ((double)m.res * m.res);
                for (int j = 0; j < m.r2; ++j) {
                    m.w[(uint64_t)e * m.r2 + j] = w0;
                    m.acc[(uint64_t)e * m.r2 + j] = 0.0;
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
        w0 = ((uint64_t)e << 16 | (uint32_t)mdl_cell(u[i], v[i], m.res)) << shift;
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
    double *acc = m.acc + (uint64_t)e * m.r2 + (uint32_t)(ec & 0xffffu);
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
            if (ok) atomicAdd(m.acc + (uint64_t)e * m.r2 + mdl_cell(u[i], v[i], m.res), cv);
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
            double *w = m.w + (uint64_t)e * m.r2, *acc = m.acc + (uint64_t)e * m.r2;
            double alpha = sqrt(x.c_new / (x.c_old + x.c_new));
            if (limited) {
                const double fl = 1.0 / t_max;
                alpha = alpha < fl ? fl : alpha; /* std::max */
            }
            const double sum = warp_ordered_sum(acc, m.r2, lane);
            __syncwarp();
            if (sum > 0.0) {
                for (int j = lane; j < m.r2; j += 32)
                    w[j] = (1.0 - alpha) * w[j] + alpha * (acc[j] / sum);
                __syncwarp();
                x.total = warp_ordered_sum(w, m.r2, lane);
            }
            for (int j = lane; j < m.r2; j += 32) acc[j] = 0.0;
            const double touched = sums[1];
            const double cap = limited && touched > 0.0
                                   ? (t_max * t_max - t_max) * (sums[0] / touched)
                                   : 0.0;
            x.c_old += x.c_new;
            if (limited) x.c_old = cap < x.c_old ? cap : x.c_old; /* std::min */
            x.c_new = 0.0;
            x.warm = x.records >= (unsigned long long)(long long)min_samples;
        }
        __syncwarp();
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

/* DirGrid::pdf (models.cpp:52-56) */
__device__ __forceinline__ double mdl_pdf(const MdlDev &m, int32_t e, double u, double v) {
    if (e < 0) return 1.0;
    const double tot = m.ent[e].total;
    if (tot <= 0.0) return 1.0;
    return m.w[(uint64_t)e * m.r2 + mdl_cell(u, v, m.res)] / tot * (double)m.res * (double)m.res;
}

__global__ void k_mdl_pdf(MdlDev m, const int32_t *ent, const double *u, const double *v,
                          uint64_t n, double *out) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = mdl_pdf(m, ent[i], u[i], v[i]);
}

__device__ __forceinline__ double clamp_ref(double x, double lo, double hi) { /* vecmath.h:19 */
    const double a = x < lo ? lo : x;
    return hi < a ? hi : a;
}

/* DirGrid::sample (models.cpp:58-92): row by the marginal, then column, residuals remapped */
__global__ void k_mdl_sample(MdlDev m, const int32_t *ent, const double *u1, const double *u2,
                             uint64_t n, double *su, double *sv, double *spdf) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t e = ent[i];
    const double ux = u1[i], uy = u2[i];
    if (e < 0 || m.ent[e].total <= 0.0) {
        su[i] = ux;
        sv[i] = uy;
        spdf[i] = 1.0;
        return;
    }
    const int R = m.res;
    const double *w = m.w + (uint64_t)e * m.r2;
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

int pstf_model_create(const pstf_model_config *config, int device, pstf_model_store **out) {
    if (!config || !out) return set_err(PSTF_E_INVALID, "NULL argument");
    *out = nullptr;
    if (config->grid_resolution < 1 || config->grid_resolution > 256)
        return set_err(PSTF_E_INVALID, "grid_resolution must be in [1, 256]"); /* models.cpp:17-18 */
    if (config->capacity_log2 < 1 || config->capacity_log2 > 26)
        return set_err(PSTF_E_INVALID, "capacity_log2 must be in [1, 26]");
    CK(cudaSetDevice(device));
    std::unique_ptr<pstf_model_store> m(new pstf_model_store());
    m->cfg = *config;
    m->device = device;
    const uint64_t cap = 1ull << config->capacity_log2;
    m->mask = (uint32_t)(cap - 1);
    m->r2 = config->grid_resolution * config->grid_resolution;
    const uint64_t cells = cap * (uint64_t)m->r2;
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
    const uint64_t cap = (uint64_t)m->mask + 1;
    LAUNCH(k_mdl_blend, (unsigned)sm_count() * 8, 256, 0, st, d, m->sums.as<double>(), t_max,
           limited, m->cfg.min_samples);
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
                      const double *u2, uint64_t n, double *su, double *sv, double *pdf,
                      void *stream) {
    if (!m || (n && (!entry || !u1 || !u2 || !su || !sv || !pdf)))
        return set_err(PSTF_E_INVALID, "NULL argument");
    if (!n) return PSTF_OK;
    CK(cudaSetDevice(m->device));
    LAUNCH(k_mdl_sample, grid_for(n, 128), 128, 0, (cudaStream_t)stream, m->dev(), entry, u1, u2,
           n, su, sv, pdf);
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
    const uint64_t cap = (uint64_t)m->mask + 1, r2 = (uint64_t)m->r2;
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
        o.total = ent[e].total;
        if (weights) CK(cudaMemcpy(weights + i * r2, m->w.as<double>() + (uint64_t)e * r2, r2 * 8,
                                   cudaMemcpyDeviceToHost));
        if (accum) CK(cudaMemcpy(accum + i * r2, m->acc.as<double>() + (uint64_t)e * r2, r2 * 8,
                                 cudaMemcpyDeviceToHost));
    }
    return PSTF_OK;
}

} // extern "C"
