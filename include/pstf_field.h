/*
 * pstf_field.h — C ABI of the B200-native PSTF field cache (libpstf_b200.so).
 *
 * Drop-in boundary for the reference's field engine, pstf::FieldStore / FieldUpdateQueue
 * (/root/reference/proj/core/include/pstf/field.h:19-167).  Each entry point below names the
 * reference interface it replaces.  Batch entry points take DEVICE pointers (SoA) and a CUDA
 * stream handle passed as void*; functions that return data to the caller say so.  Every
 * function returns 0 on success and a negative PSTF_E* code on failure; pstf_last_error()
 * gives a thread-local message.  No C++ exception crosses this boundary.
 *
 * There is no CPU implementation behind this ABI: every computing entry point launches
 * sm_100a kernels and fails with PSTF_E_CUDA when no device is usable.
 */
#ifndef PSTF_FIELD_H
#define PSTF_FIELD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSTF_ABI_VERSION 2

enum {
    PSTF_OK = 0,
    PSTF_E_INVALID = -1, /* bad argument */
    PSTF_E_CUDA = -2,    /* CUDA runtime / launch failure (incl. no device) */
    PSTF_E_NOMEM = -3,   /* device or host allocation failed */
    PSTF_E_IO = -4,      /* snapshot file I/O (field.cpp:340-341, 361-384) */
    PSTF_E_FORMAT = -5   /* not a snapshot / bad version / truncated */
};

/* FieldKind (field.h:19) */
enum { PSTF_KIND_LO = 0, PSTF_KIND_LO_MINUS_E = 1, PSTF_KIND_LI = 2, PSTF_KIND_FLI = 3 };
/* Technique (field.h:22-27) */
enum { PSTF_TECH_CAMERA = 1, PSTF_TECH_CONTINUATION = 2, PSTF_TECH_NEE = 4, PSTF_TECH_ALL = 7 };
/* FieldStoreConfig::Blend (field.h:51) */
enum { PSTF_BLEND_SQRT = 0, PSTF_BLEND_LINEAR = 1 };

/* Update application modes.
 * Slot placement is the same in every mode: new keys take slots exactly as sequential
 * insertion in priority order would (field.cpp:116-146).
 *  ATOMIC     : priority = key order (FieldUpdateQueue order, field.cpp:402-406); values are
 *               summed with fp64 atomics (order-free; within 1e-12 relative in practice).
 *  ORDERED    : bit-exact FieldUpdateQueue::apply (field.cpp:396-420): per slot, updates are
 *               folded sequentially in the queue's canonical sort order.
 *  SEQUENTIAL : bit-exact sequence of scalar incrementCounter/accumulate calls in submission
 *               order (priority = first submission of a key; folds in submission order). */
enum { PSTF_MODE_ATOMIC = 0, PSTF_MODE_ORDERED = 1, PSTF_MODE_SEQUENTIAL = 2 };

/* FieldStoreConfig (field.h:44-55), same field order and meaning */
typedef struct pstf_field_config {
    uint32_t kind;
    uint32_t capacity_log2;  /* hash-table entries = 2^capacity_log2 (1..30) */
    int32_t max_level;       /* levels 0..max_level (0..62) */
    double base_cell_size;   /* level-0 spatial cell edge */
    double level_select_k;   /* footprint multiplier for level selection */
    double t_max;            /* temporal window cap; <= 0 or non-finite = unlimited */
    uint32_t blend;          /* PSTF_BLEND_* */
    uint32_t technique_mask; /* carried, not read by the store (as in the reference) */
    uint32_t probe_window;   /* linear-probe window (>= 1) */
    uint32_t evict_age_frames;
} pstf_field_config;

/* SpatioDirectionalKey (field.h:32-42); 28 bytes */
typedef struct pstf_key {
    int32_t level;
    int32_t cell[3];
    int32_t dir_cell[2];
    uint32_t checksum;
} pstf_key;

/* FieldStore::SnapshotRecord (field.h:113-120); 64 bytes in memory */
typedef struct pstf_snapshot_record {
    int32_t level;
    int32_t cell[3];
    int32_t dir_cell[2];
    uint32_t checksum;
    double value[3];
    double c_old;
} pstf_snapshot_record;

/* One table slot (FieldStore::Slot, field.cpp:48-58) for occupancy/parity dumps; 104 bytes */
typedef struct pstf_slot_record {
    uint32_t checksum; /* 0 = empty */
    int32_t level;
    int32_t cell[3];
    int32_t dir_cell[2];
    double value_old[3];
    double c_old;
    double accum[3];
    double c_new;
    uint32_t last_touched;
} pstf_slot_record;

typedef struct pstf_field_stats {
    uint64_t frame;           /* frameIndex()      field.h:105 */
    uint64_t rejected;        /* rejectedUpdates() field.h:106 */
    uint64_t dropped;         /* droppedInserts()  field.h:107 */
    uint64_t internal_errors; /* internalErrors()  field.h:108 */
    uint64_t live;            /* liveCellCount()   field.h:109 */
    uint64_t touched_last;    /* slots touched in the last committed frame */
    uint64_t new_keys_last;   /* keys placed by the last update pass */
    uint64_t evicted_last;    /* slots evicted by the last endFrame */
    uint64_t placement_rounds_last; /* deterministic-placement rounds of the last pass */
    uint64_t touched_total;   /* touched slots summed over all committed frames */
    uint64_t reds_total;      /* fp64 RED element updates issued by fused (ATOMIC, tiled) vertex
                               * passes in which this store was the Lo store, all stores summed */
} pstf_field_stats;

/* Three coordinate arrays of one fp64 vector field (device pointers) */
typedef struct pstf_vec3_soa {
    const double *x, *y, *z;
} pstf_vec3_soa;

/* The canonical per-vertex record FieldRecorder::onVertex reads (estimators.cpp:194-262,
 * VertexRecord pathtracer.h:59-90), SoA.  nee_loe = nee.value() (pathtracer.h:42-46),
 * nee_fli = nee.f * nee.radiance * nee.misWeight (estimators.cpp:251),
 * ratio = transportRatio() (pathtracer.h:86-89), flags bit0 contExtended, bit1 nextIsSurface,
 * bit2 nee.sampled.  276 bytes per vertex. */
typedef struct pstf_vertex_soa {
    pstf_vec3_soa position, wo, wi, next_position, nee_dir;
    const double *footprint, *next_footprint, *ratio, *next_emis_mis_weight;
    pstf_vec3_soa emission_here, f, next_emission, nee_loe, nee_fli;
    const uint32_t *flags;
} pstf_vertex_soa;

#define PSTF_VERTEX_CONT_EXTENDED 1u
#define PSTF_VERTEX_NEXT_IS_SURFACE 2u
#define PSTF_VERTEX_NEE_SAMPLED 4u

typedef struct pstf_field pstf_field;

int pstf_abi_version(void);
const char *pstf_last_error(void);

/* FieldStore(const FieldStoreConfig&) field.h:78 / ~FieldStore() field.h:79 */
int pstf_field_create(const pstf_field_config *config, int device, pstf_field **out);
int pstf_field_destroy(pstf_field *f);
/* config() field.h:81 */
int pstf_field_get_config(const pstf_field *f, pstf_field_config *out);

/* selectLevel(double) field.h:83, batched: level[i] = selectLevel(footprint[i]) */
int pstf_select_level(const pstf_field *f, const double *footprint, int32_t *level, uint64_t n,
                      void *stream);
/* keyFor(pos, dir, level) field.h:86, batched */
int pstf_key_for(const pstf_field *f, const pstf_vec3_soa *pos, const pstf_vec3_soa *dir,
                 const int32_t *level, uint64_t n, pstf_key *keys, void *stream);

/* incrementCounter / accumulate (field.h:89-91) and FieldUpdateQueue::apply (field.h:157),
 * batched.  value = 3 device arrays (r, g, b; ignored where is_counter[i] != 0, may be NULL if
 * all are counters), w[n], is_counter[n] (NULL = all accumulates).  mode = PSTF_MODE_*. */
int pstf_field_apply(pstf_field *f, const pstf_key *keys, const pstf_vec3_soa *value,
                     const double *w, const uint8_t *is_counter, uint64_t n, int mode,
                     void *stream);

/* Host-pointer variants of the small-batch calls (scalar facade use: the C++ drop-in header
 * paper_2005_07547_b200/cxx/include/pstf/field.h).  Inputs/outputs are host arrays, staged
 * through the store's device scratch; the call returns when the result is on the host.
 * pos/dir are AoS xyz triples here (Vec3 layout). */
int pstf_key_for_host(const pstf_field *f, const double *pos_xyz, const double *dir_xyz,
                      const int32_t *level, uint64_t n, pstf_key *keys);
int pstf_select_level_host(const pstf_field *f, const double *footprint, int32_t *level,
                           uint64_t n);
int pstf_field_apply_host(pstf_field *f, const pstf_key *keys, const double *rgb_xyz,
                          const double *w, const uint8_t *is_counter, uint64_t n, int mode);
int pstf_field_query_host(const pstf_field *f, const double *pos_xyz, const double *dir_xyz,
                          const double *footprint, const int32_t *level, uint64_t n,
                          double *value_rgb, uint8_t *valid, uint8_t *fallback,
                          int32_t *out_level);

/* query(pos, dir, footprint) / queryFromLevel(pos, dir, level) field.h:93-94, batched.
 * Exactly one of footprint / level is non-NULL.  Outputs: value (3 arrays), valid, fallback,
 * out_level (any may be NULL). */
int pstf_field_query(const pstf_field *f, const pstf_vec3_soa *pos, const pstf_vec3_soa *dir,
                     const double *footprint, const int32_t *level, uint64_t n, double *value_r,
                     double *value_g, double *value_b, uint8_t *valid, uint8_t *fallback,
                     int32_t *out_level, void *stream);

/* endFrame() field.h:100 */
int pstf_field_end_frame(pstf_field *f, void *stream);
/* endFrame() on n (1..4) stores of one device in a single pair of sweeps (e.g. Lo, LoE, FLi, Li
 * at the frame barrier, estimators.cpp:647-651); same result as n separate calls. */
int pstf_fields_end_frame(pstf_field *const *fields, int n, void *stream);
/* invalidate() / invalidate(const Aabb&) field.h:102-103; aabb = host double[6] {lo, hi} or NULL */
int pstf_field_invalidate(pstf_field *f, const double *aabb, void *stream);

/* frameIndex / rejectedUpdates / droppedInserts / internalErrors / liveCellCount
 * (field.h:105-109); synchronises the store's work. */
int pstf_field_get_stats(pstf_field *f, pstf_field_stats *out);
/* weightedMeanValue() field.h:111 (host out[3]); synchronises. */
int pstf_field_weighted_mean(pstf_field *f, double out[3]);

/* Snapshot records sorted by key, as dumpSnapshot writes them (field.cpp:311-337), into a host
 * buffer.  *count = number of live records; at most cap are written. */
int pstf_field_snapshot(pstf_field *f, pstf_snapshot_record *records, uint64_t cap,
                        uint64_t *count);
/* dumpSnapshot(path) field.h:123: PSTFSNAP v1 file, byte-identical to the reference writer */
int pstf_field_dump_snapshot(pstf_field *f, const char *path);
/* readSnapshot(path) field.h:124; kind may be NULL */
int pstf_read_snapshot(const char *path, pstf_snapshot_record *records, uint64_t cap,
                       uint64_t *count, uint32_t *kind);

/* Snapshot restore (the reference writes snapshots, field.cpp:311-386, but
 * has no restore).  records: host array, any order; each checksum must match its key
 * (field.cpp:98-99), else PSTF_E_FORMAT and the store is unchanged.  Semantics, in ascending key
 * order (stable): findOrInsertSlot(key) (field.cpp:116-146: lastTouched = frame, a full window
 * counts one droppedInserts), then valueOld = value, cOld = c_old at the slot it returned; of
 * several records resolving to one slot the last wins.  accum/cNew are untouched.  Synchronous. */
int pstf_field_restore(pstf_field *f, const pstf_snapshot_record *records, uint64_t n);
/* readSnapshot(path) + pstf_field_restore; PSTF_E_FORMAT when the file's kind is not the store's */
int pstf_field_load_snapshot(pstf_field *f, const char *path);

/* Slot-array dump (host) of slots [begin, begin+count) for occupancy parity. */
int pstf_field_slots(pstf_field *f, uint64_t begin, uint64_t count, pstf_slot_record *out);
/* The committed state (what queries read, field.h:73-75) of every slot, to host memory:
 * checksum[capacity] (0 = empty) and com4[capacity][4] = {valueOld.rgb, cOld}.  The C++ facade
 * mirrors it once per frame and answers scalar query()/queryFromLevel() calls from the mirror
 * (SURVEY.md 8(b)); it changes only at endFrame / invalidate / restore. */
int pstf_field_committed_host(pstf_field *f, uint32_t *checksum, double *com4);

/* Fused per-vertex pass: FieldRecorder::onVertex (estimators.cpp:194-262) for n vertices, i.e.
 * next-vertex Lo/LoE lookups on committed state, key generation, update values, and the
 * counter/accumulate updates into Lo, LoE, FLi (and Li when li != NULL).  Device pointers.
 * mode = PSTF_MODE_ATOMIC (fast) or PSTF_MODE_ORDERED (== EstimatorRun deterministic mode).
 * Returns once phase 1 is enqueued on the stream: the placement of new keys (phase 2) is
 * completed by the next entry point that touches one of these stores, and pstf_fields_end_frame
 * on the same stream needs no host round trip when there are none (PSTF_NO_DEFER=1 places them
 * before returning).  Results are identical either way.  Two behaviours are chosen inside:
 * when lo and loe were created alike and have only ever been updated together (vertex passes,
 * batched end-frames) they hold identical occupancy, and the kernel takes loe's probes from lo's
 * (any other update of either ends that for good: PSTF_NO_TWIN=1 disables it); and when the
 * previous frame issued more than 1000 RED updates per touched slot (hot slots: coarse cells),
 * a warp-aggregating kernel variant runs (PSTF_RED_AGG=0|1 forces it).  ORDERED passes finish before
 * returning: the value calls of keys that already own a slot are put in the queue's order by
 * the slot-grouped path (one radix sort, re-sorted runs, a sequential fold per slot) after one
 * host read of the call counts; a checksum alias sends them through the general path. */
int pstf_vertex_pass(pstf_field *lo, pstf_field *loe, pstf_field *fli, pstf_field *li,
                     const pstf_vertex_soa *v, uint64_t n, uint32_t loe_mask, uint32_t fli_mask,
                     int mode, void *stream);

/* Same with HOST vertex arrays (pinned for overlap): staged to the device in chunks on the
 * stream, overlapping copies with the pass.  Returns after the work is enqueued when the host
 * arrays are pinned, otherwise after the copies complete. */
int pstf_vertex_pass_host(pstf_field *lo, pstf_field *loe, pstf_field *fli, pstf_field *li,
                          const pstf_vertex_soa *host_v, uint64_t n, uint32_t loe_mask,
                          uint32_t fli_mask, int mode, void *stream);

/* pstf_vertex_pass plus the CV lookup of every vertex (the Lo\E query at its position, wo and
 * footprint on the frame-start table, exactly pstf_cv_lookup run before the pass), fused into
 * the vertex kernel: the query's first key is the vertex's Lo key, already probed for the
 * update (config 3 "CV lookup at every vertex", estimators.cpp:453-462 + 194-262). */
int pstf_vertex_pass_cv(pstf_field *lo, pstf_field *loe, pstf_field *fli, pstf_field *li,
                        const pstf_vertex_soa *v, uint64_t n, uint32_t loe_mask,
                        uint32_t fli_mask, int mode, double *cv_r, double *cv_g, double *cv_b,
                        uint8_t *cv_valid, void *stream);

/* Probe-distance histogram of the live slots: hist[d] = number of live slots at distance d =
 * (slot - home) & mask from their key's home slot, d >= 32 counted in hist[32] (SURVEY.md
 * 8(b) stats probe_hist[33]; config 5 reports it per iteration).  Reads the device table. */
int pstf_field_probe_histogram(pstf_field *f, uint64_t hist[33]);

/* Diagnostic: sustained fp64 RED throughput of this GPU (element updates per second) for the
 * vertex pass's access pattern (each warp instruction = 8 distinct 32 B cells x 4 components)
 * on distinct L2-resident addresses: the atomic roofline's peak. */
int pstf_diag_red_peak(int device, double *ops_per_second);

/* CV / guiding lookup at the current vertex (estimators.cpp:438-462): out = Lo\E query at
 * (position, wo, footprint) for every vertex of the record (config 3 "CV lookup"). */
int pstf_cv_lookup(const pstf_field *loe, const pstf_vertex_soa *v, uint64_t n, double *value_r,
                   double *value_g, double *value_b, uint8_t *valid, void *stream);

/* Synthetic Cornell-box vertex stream written on the device into a
 * contiguous buffer of 34*n fp64 followed by n uint32 flags (n = width*height*bounces).
 * Test/bench input, not part of the reference API. */
int pstf_synth_generate(int width, int height, int bounces, uint64_t seed, uint64_t iteration,
                        double cam_shift_x, double *buffer, void *stream);
/* Same for the image stripe of paths [path0, path0 + npaths) (n = npaths*bounces vertices). */
int pstf_synth_generate_stripe(int width, int height, int bounces, uint64_t seed,
                               uint64_t iteration, double cam_shift_x, uint64_t path0,
                               uint64_t npaths, double *buffer, void *stream);
/* ... with a material set: scene 0 = the Lambertian Cornell box (the functions above), scene 1 =
 * the glossy materials of staircase_glossy.scene:11-22 on the same box (BASELINE config 3:
 * floor and back wall diffuse 0.2/0.18/0.15 + Phong lobe albedo 0.6, exponent 48) */
int pstf_synth_generate_scene(int scene, int width, int height, int bounces, uint64_t seed,
                              uint64_t iteration, double cam_shift_x, uint64_t path0,
                              uint64_t npaths, double *buffer, void *stream);
/* Fills a pstf_vertex_soa view of such a contiguous buffer (host or device memory). */
void pstf_vertex_soa_from_buffer(const double *buffer, uint64_t n, pstf_vertex_soa *out);

/* ---- multi-GPU: one field cache over several ranks (one process per GPU) ----
 * Replaces the reference's shared-memory std::thread workers (estimators.cpp:566-623) with one
 * process per GPU, each tracing its own vertices (an image stripe, or its own samples).  Every
 * rank holds a bitwise-identical replica of each store; per frame (collectives are the
 * caller's, e.g. NCCL via torch.distributed):
 *   1. pstf_vertex_pass_local on the rank's vertices: lookups on the replica (committed state,
 *      field.h:73-75), REDs into the replica's accumulators, new keys stay pending
 *   2. the pstf_shard_info vectors (pending sizes, live count) are all-gathered on the device
 *      and read with ONE host synchronisation; all-gather the pending records;
 *      pstf_resolve_records on every rank: identical deterministic placement (the single-GPU
 *      layout), each rank adds only its own records' sums
 *   3. pstf_shard_live_pack: the accumulators of the live slots, packed in slot order (entry i
 *      is the same slot on every rank), zero-padded to `bound` entries -> all-reduce (sum) ->
 *      pstf_shard_live_unpack (sums back, slots touched on any rank marked touched)
 *   4. pstf_fields_end_frame on every rank: identical inputs, identical committed state
 * Slot placement, ages and counts equal the single-GPU run; values differ from it only in fp64
 * summation order.  Only the ATOMIC mode is sharded. */
int pstf_shard_set(pstf_field *f, int rank, int world);
int pstf_vertex_pass_local(pstf_field *lo, pstf_field *loe, pstf_field *fli, pstf_field *li,
                           const pstf_vertex_soa *v, uint64_t n, uint32_t loe_mask,
                           uint32_t fli_mask, void *stream);
int pstf_pending_count(pstf_field *lo, uint64_t *n);
/* the same count written to a device int64 on the stream (no host round trip): the ranks
 * all-gather it on the device and read every size with one synchronisation */
int pstf_pending_count_dev(pstf_field *lo, int64_t *dev_count, void *stream);
int pstf_pending_copy(pstf_field *lo, void *dst, uint64_t n, void *stream);
int pstf_resolve_records(pstf_field *const *stores, int nst, const void *records, uint64_t n,
                         void *stream);
/* dev_out3 (device int64[3]) = {this rank's pending records, live slots over the stores (after
 * the last endFrame: with every rank's pending records an upper bound of the live count after
 * placement), packs whose live count exceeded their bound (must stay 0)} */
int pstf_shard_info(pstf_field *const *stores, int nst, int64_t *dev_out3, void *stream);
/* packed[bound][4] (device f64) <- acc of every live slot of the stores, in (store, slot)
 * order; dev_live_total <- the live count (device int64).  The packed list stays with the
 * stores' scratch until pstf_shard_live_unpack. */
int pstf_shard_live_pack(pstf_field *const *stores, int nst, double *packed, uint64_t bound,
                         int64_t *dev_live_total, void *stream);
int pstf_shard_live_unpack(pstf_field *const *stores, int nst, const double *packed,
                           void *stream);
/* steps 3b + 4 in one: endFrame (field.cpp:197-263) of every store straight from the
 * all-reduced packed accumulators (== pstf_shard_live_unpack then pstf_fields_end_frame) */
int pstf_shard_end_frame(pstf_field *const *stores, int nst, const double *packed, void *stream);
uint64_t pstf_pending_record_bytes(void); /* 64 */

/* Number of kernels this library launched since load (bench evidence). */
uint64_t pstf_kernel_launch_count(void);

/* Per-kernel CUDA-event timing (events recorded on each launch's stream while enabled).
 * pstf_profile_collect synchronises, aggregates by kernel name (names: n_max x 64 chars),
 * total milliseconds and launch counts, then clears the record. */
int pstf_profile_enable(int on);
int pstf_profile_collect(char *names, double *ms, uint64_t *counts, int n_max, int *n_out);

/* ---- CV-profile / guiding model store ------------------------
 * ModelStore (estimators.h:124-150, estimators.cpp:104-144) with DirGrid models
 * (models.h:30-52, models.cpp:16-94; what the CV profiles always use, estimators.cpp:336-339,
 * and the guiding models' default kind, models.h:186) or SphericalKdTree models
 * (models.h:59-109, models.cpp:96-298: the split-collapse learner) or Gmm models
 * (models.h:113-177, models.cpp:427-702: stepwise EM, batch E-step by prefix sums of
 * log(1 - k^-alpha)).  Grid and k-d tree results are bitwise the reference's; the GMM goes
 * through exp/log/pow/sin/cos, so its state agrees to a relative tolerance (1e-9), not bitwise.
 * Keyed by the field's SpatioDirectionalKey with key-field equality (the unordered_map's
 * operator==, field.h:38-41).  The reference map grows without bound; here the table has
 * 2^capacity_log2 entries and records of keys that find no free entry are counted as dropped. */
enum { PSTF_MODEL_GRID = 0, PSTF_MODEL_KDTREE = 1, PSTF_MODEL_GMM = 2 }; /* ModelKind, models.h:183 */

typedef struct pstf_model_config {
    int32_t kind;               /* PSTF_MODEL_GRID (DirGrid), _KDTREE or _GMM */
    int32_t grid_resolution;    /* ModelConfig::gridResolution (models.h:187), >= 1 */
    int32_t kd_leaf_count;      /* ModelConfig::kdLeafCount (models.h:188), power of two >= 2 */
    double kd_split_threshold;  /* ModelConfig::kdSplitThreshold (models.h:189), > 1 */
    int32_t gmm_components;     /* GmmConfig (models.h:113-119): components in [1, 16] */
    double gmm_alpha_em;        /*   step exponent in (0.5, 1] */
    double gmm_sigma_min_sq;    /*   covariance eigenvalue floor */
    double gmm_sigma_max_sq;    /*   covariance eigenvalue cap */
    double gmm_reseed_fraction; /*   mass fraction below which a component is reseeded */
    double t_max;               /* EstimatorConfig::tMax (the blend cap, estimators.cpp:119-144) */
    int32_t min_samples;        /* minModelSamples / profileMinSamples (warm threshold) */
    uint32_t capacity_log2;     /* entries in the device table */
} pstf_model_config;

typedef struct pstf_model_store pstf_model_store;

/* One entry (ModelStore::Entry + its DirGrid), for parity dumps */
typedef struct pstf_model_entry {
    int32_t level;
    int32_t cell[3];
    int32_t dir_cell[2];
    uint32_t warm;         /* Entry::warm */
    double c_old, c_new;   /* Entry::cOld, cNew */
    uint64_t records;      /* Entry::records (applyRecord calls) */
    uint64_t record_count; /* DirGrid::m_recordCount (accepted contributions) */
    double total;          /* DirGrid::m_total */
} pstf_model_entry;

typedef struct pstf_model_stats {
    uint64_t entries;         /* ModelStore::size() */
    uint64_t warm;            /* entries with warm set */
    uint64_t dropped_records; /* records whose key found no free entry (device table full) */
    uint64_t capacity;
} pstf_model_stats;

int pstf_model_create(const pstf_model_config *config, int device, pstf_model_store **out);
int pstf_model_destroy(pstf_model_store *m);
/* applyRecord (estimators.cpp:109-117) for n records, device arrays.
 * PSTF_MODE_ORDERED: applied in the canonical deterministic order of estimators.cpp:633-637
 *   (key fields, uv.x, uv.y, contribution): bitwise the reference's deterministic mode.
 * PSTF_MODE_ATOMIC: no sort, fp64 atomics into the grids; accumulator sums within 1e-12
 *   relative (their order is the atomics'), everything else exact.  GMM stores always take
 *   the canonical order (stepwise EM depends on the sample order, not only on rounding).
 * Precondition of the bitwise claim: ONE apply call per store per frame, carrying all of the
 * frame's records.  The reference sorts the whole frame's records once (estimators.cpp:
 * 625-643); records split over several calls are canonicalised per call, which changes the
 * per-cell accumulation order (and the GMM EM sample order) against the reference. */
int pstf_model_apply(pstf_model_store *m, const pstf_key *keys, const double *u, const double *v,
                     const double *contribution, uint64_t n, int mode, void *stream);
/* ModelStore::endFrame (estimators.cpp:119-144) */
int pstf_model_end_frame(pstf_model_store *m, void *stream);
/* lookupWarm (estimators.cpp:104-107): entry index of a warm model, else -1 */
int pstf_model_lookup_warm(const pstf_model_store *m, const pstf_key *keys, uint64_t n,
                           int32_t *entry, void *stream);
/* The estimator's hierarchical lookup (estimators.cpp:464-469 and 475-480): for
 * l = selectLevel(footprint) .. maxLevel, lookupWarm(keyFor(pos, dir, l)) with the keyer
 * field's quantisation; the first warm entry, else -1. */
int pstf_model_lookup_warm_levels(const pstf_model_store *m, const pstf_field *keyer,
                                  const pstf_vec3_soa *pos, const pstf_vec3_soa *dir,
                                  const double *footprint, uint64_t n, int32_t *entry,
                                  void *stream);
/* DirGrid::pdf (models.cpp:52-56) of entry[i] at (u[i], v[i]); entry < 0 gives 1.0 (the
 * uniform square density the callers use without a model, estimators.cpp:485-487).  uv
 * outside [0,1] indexes outside the grid in the reference (undefined); here it is clamped. */
int pstf_model_pdf(const pstf_model_store *m, const int32_t *entry, const double *u,
                   const double *v, uint64_t n, double *pdf, void *stream);
/* DirGrid / SphericalKdTree::sample(u) (models.cpp:58-92, 176-200) and Gmm::sample(uSelect, u)
 * (models.cpp:664-687; u_select is read only by GMM stores and may be NULL otherwise): square
 * sample + pdf; entry < 0 gives (u, 1.0) */
int pstf_model_sample(const pstf_model_store *m, const int32_t *entry, const double *u1,
                      const double *u2, const double *u_select, uint64_t n, double *su,
                      double *sv, double *pdf, void *stream);
int pstf_model_get_stats(pstf_model_store *m, pstf_model_stats *out);
/* Host dump of every entry, sorted by key.  Per entry, weights and accum (when non-NULL)
 * receive S doubles: Grid: the R^2 weights / accumulators; KdTree: each of the 2L-1 nodes'
 * prob / accum (node order); Gmm: the state {weights[C], means[C][2], cov[C][3] (cxx, cxy,
 * cyy), stats[C][8], cache[C][7] (inv[3], norm, chol[3]), i, underflows, reseed counter} and
 * zeros.  *count = entries; at most cap are written. */
int pstf_model_dump(pstf_model_store *m, pstf_model_entry *entries, double *weights,
                    double *accum, uint64_t cap, uint64_t *count);
/* KdTree topology in the same entry order: per node {leaf, axis, left, right, parent} int32 and
 * {split, mass} double (SphericalKdTree::Node, models.h:91-99). */
int pstf_model_dump_tree(pstf_model_store *m, int32_t *node_i32, double *node_f64, uint64_t cap,
                         uint64_t *count);

#ifdef __cplusplus
}
#endif
#endif /* PSTF_FIELD_H */
