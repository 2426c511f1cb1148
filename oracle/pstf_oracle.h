/*
 * pstf_oracle.h — CPU restatement of the PSTF field cache (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity checker for the B200 field cache.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product path
 * (paper_2005_07547_b200) never links, imports or calls anything in oracle/.
 *
 * It restates, in plain C99 with the host libm (atan2, log2, floor, sqrt) exactly as the
 * reference uses them, the single-threaded semantics of
 *   /root/reference/proj/core/src/field.cpp  (FieldStore, FieldUpdateQueue)
 *   /root/reference/proj/core/src/estimators.cpp:194-262 (FieldRecorder::onVertex, fields part)
 * Every function cites the reference line it follows.  It is pinned against the reference
 * itself compiled from /root/reference into oracle/_ref (see oracle/Makefile and
 * tests/test_oracle_pin.py) and against the reference unit-test vectors
 * (proj/tests/unit/test_field.cpp) in tests/test_oracle_golden.py.
 */
#ifndef PSTF_ORACLE_H
#define PSTF_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t level;
    int32_t cell[3];
    int32_t dir[2];
    uint32_t checksum;
} po_key; /* field.h:32-42 */

typedef struct {
    uint32_t kind;          /* FieldKind field.h:19 */
    uint32_t capacity_log2; /* field.h:46 */
    int32_t max_level;      /* field.h:47 */
    double base_cell_size;  /* field.h:48 */
    double level_select_k;  /* field.h:49 */
    double t_max;           /* field.h:50 */
    uint32_t blend;         /* 0 = Sqrt, 1 = Linear field.h:51 */
    uint32_t technique_mask;
    uint32_t probe_window;  /* field.h:53 */
    uint32_t evict_age_frames; /* field.h:54 */
} po_config;

typedef struct {
    uint32_t checksum;
    int32_t level, cell[3], dir[2];
    double value_old[3];
    double c_old;
    double accum[3];
    double c_new;
    uint32_t last_touched;
} po_slot; /* field.cpp:48-58 */

typedef struct po_store po_store;

typedef struct {
    double value[3];
    int32_t valid, fallback, level;
} po_query_result; /* field.h:57-62 */

typedef struct {
    po_key key;
    double value[3];
    double w;
    int32_t is_counter;
} po_update; /* field.h:160-165 */

typedef struct {
    uint64_t frame, rejected, dropped, internal_errors, live;
} po_stats;

typedef struct {
    int32_t level, cell[3], dir[2];
    uint32_t checksum;
    double value[3];
    double c_old;
} po_snapshot_record; /* field.h:113-120 */

/* key math */
uint64_t po_mix_bits(uint64_t v);
uint64_t po_pack_key_fields(const po_key *k);
int po_select_level(const po_config *c, double footprint);
double po_cell_size(const po_config *c, int level);
int po_dir_resolution(int level);
void po_sphere_to_square(const double dir[3], double uv[2]);
po_key po_key_for(const po_config *c, const double pos[3], const double dir[3], int level);
uint32_t po_home_slot(const po_key *k, uint32_t mask);

/* store */
po_store *po_store_create(const po_config *c);
void po_store_destroy(po_store *s);
const po_config *po_store_config(const po_store *s);
void po_increment_counter(po_store *s, const po_key *k, double w);
void po_accumulate(po_store *s, const po_key *k, const double value[3], double w);
po_query_result po_query_from_level(const po_store *s, const double pos[3], const double dir[3],
                                    int level);
po_query_result po_query(const po_store *s, const double pos[3], const double dir[3],
                         double footprint);
void po_end_frame(po_store *s);
void po_invalidate_all(po_store *s);
void po_invalidate_box(po_store *s, const double lo[3], const double hi[3]);
void po_stats_get(const po_store *s, po_stats *out);
void po_weighted_mean(const po_store *s, double out[3]);
/* copies the slot array (2^capacity_log2 entries) */
void po_slots(const po_store *s, po_slot *out);
/* key-sorted live records (field.cpp:311-337); returns the count written (<= cap) */
size_t po_snapshot(const po_store *s, po_snapshot_record *out, size_t cap);
/* ModelStore<DirGrid> (pstf_model_oracle.c; estimators.cpp:104-144, models.cpp:16-94) */
typedef struct po_model po_model;
typedef struct {
    int32_t level, cell[3], dir[2];
    uint32_t warm;
    double c_old, c_new;
    uint64_t records, record_count;
    double total;
} po_model_entry; /* == pstf_model_entry */
po_model *po_model_create(int kind, int res, int leaves, double tsplit, int comps,
                          double alpha_em, double smin, double smax, double reseed_frac,
                          double t_max, int min_samples); /* kind 0 Grid, 1 KdTree, 2 Gmm */
void po_model_destroy(po_model *m);
void po_model_apply(po_model *m, const po_key *keys, const double *u, const double *v,
                    const double *c, size_t n);
void po_model_end_frame(po_model *m);
double po_model_pdf(const po_model *m, const po_key *k, double u, double v, int *found);
void po_model_sample(const po_model *m, const po_key *k, double u1, double u2, double usel,
                     double *su, double *sv, double *pdf, int *found);
size_t po_model_dump(const po_model *m, po_model_entry *out, double *weights, double *accum,
                     size_t cap);
size_t po_model_dump_tree(const po_model *m, int32_t *node_i32, double *node_f64, size_t cap);
/* snapshot restore, the semantics of pstf_field_restore (include/pstf_field.h) */
void po_restore(po_store *s, const po_snapshot_record *recs, size_t n);

/* FieldUpdateQueue::apply (field.cpp:396-420): sorts in place, then applies sequentially */
void po_queue_apply(po_store *s, po_update *updates, size_t n);

/* FieldRecorder::onVertex (estimators.cpp:194-262) over the SoA record of pstf_synth.h
 * (34 fp64 arrays of n then u32 flags).  deterministic=1 collects per-store queues and
 * applies them with po_queue_apply (EstimatorRun deterministic mode, estimators.cpp:610-623);
 * deterministic=0 calls the store immediately in vertex order.  li may be NULL. */
void po_vertex_pass(po_store *lo, po_store *loe, po_store *fli, po_store *li,
                    const double *const f64[34], const uint32_t *flags, size_t n,
                    uint32_t loe_mask, uint32_t fli_mask, int deterministic);

/* convenience: contiguous SoA buffer */
void po_vertex_pass_contig(po_store *lo, po_store *loe, po_store *fli, po_store *li,
                           const double *buf, size_t n, uint32_t loe_mask, uint32_t fli_mask,
                           int deterministic);

/* batch helpers (SoA x[n], y[n], z[n]) */
void po_key_for_batch(const po_config *c, const double *pos, const double *dir,
                      const int32_t *level, size_t n, po_key *out);
void po_select_level_batch(const po_config *c, const double *fp, size_t n, int32_t *out);
void po_query_batch(const po_store *s, const double *pos, const double *dir, const double *fp,
                    const int32_t *level, size_t n, double *value, int32_t *flags);

/* synthetic stream generator on the host (pstf_synth.h), n = width*height*bounces */
void po_synth_generate(int width, int height, int bounces, uint64_t seed, uint64_t iter,
                       double cam_shift_x, double *buf, int threads);
/* scene 1: the glossy materials (pstf_synth.h glossy mode, BASELINE config 3) */
void po_synth_generate_scene(int scene, int width, int height, int bounces, uint64_t seed,
                             uint64_t iter, double cam_shift_x, double *buf, int threads);

#ifdef __cplusplus
}
#endif
#endif
