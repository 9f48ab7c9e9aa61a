/*
 * gss.h — C ABI of the B200-native survival-scan (Cox / Fine-Gray CCD) engine.
 *
 * This is the drop-in boundary: plain pointers, sizes and int status codes,
 * no C++ or torch types.  It flattens the reference's C++ `survscan::Engine`
 * surface (/root/reference/proj/include/survscan/engine.hpp:33-90) and the
 * CCD driver (include/survscan/ccd.hpp:59-72) so any host language can bind
 * it; the repo's own C++ mirror of the reference API
 * (paper_2204_08183_b200/csrc/host/) and its pybind module sit on top.
 * INTEGRATION.md shows the ctypes / C++ bindings a maintainer would add.
 *
 * Threading: calls on DISTINCT engine handles are thread-safe; one handle
 * must not be used by two threads at once (engine.hpp:29-32).  Each engine
 * owns one CUDA stream.  Errors are returned as status codes (one per
 * reference exception class, include/survscan/errors.hpp:9-65) and the
 * message of the last failure on the calling thread is gss_last_error().
 */
#ifndef GSS_H
#define GSS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: 1:1 with survscan::Error subclasses (errors.hpp) ---- */
enum gss_status {
  GSS_OK = 0,
  GSS_ERR_PARSE = 1,           /* ParseError               errors.hpp:17 */
  GSS_ERR_SCHEMA = 2,          /* SchemaError              errors.hpp:22 */
  GSS_ERR_DOMAIN = 3,          /* DomainError              errors.hpp:27 */
  GSS_ERR_INDEX = 4,           /* IndexError               errors.hpp:32 */
  GSS_ERR_DUPLICATE = 5,       /* DuplicateEntryError      errors.hpp:37 */
  GSS_ERR_INVALID_COLUMN = 6,  /* InvalidColumnError       errors.hpp:42 */
  GSS_ERR_NONPOS_DEN = 7,      /* NonPositiveDenominatorError errors.hpp:49 */
  GSS_ERR_OVERFLOW = 8,        /* OverflowError            errors.hpp:54 */
  GSS_ERR_DEGENERATE = 9,      /* DegenerateCurveError     errors.hpp:59 */
  GSS_ERR_EMPTY_FOLD = 10,     /* EmptyFoldError           errors.hpp:64 */
  GSS_ERR_CUDA = 100,          /* CUDA runtime / driver failure           */
  GSS_ERR_NO_DEVICE = 101,     /* no usable sm_100 device                  */
  GSS_ERR_OOM = 102            /* device allocation failed                 */
};

enum gss_model { GSS_COX = 0, GSS_FINE_GRAY = 1 };            /* engine.hpp:14 */
enum gss_penalty { GSS_PEN_NONE = 0, GSS_PEN_L1 = 1, GSS_PEN_L2 = 2 }; /* ccd.hpp:11 */

/*
 * Host-side dataset in the reference's in-memory layout
 * (include/survscan/dataset.hpp:14-111): rows already sorted by
 * (stratum asc,) time desc, original row id asc (src/dataset.cpp:227-230);
 * CSC columns over sorted positions with strictly ascending row indices.
 */
typedef struct gss_host_dataset {
  int64_t n;                     /* rows (< 2^31)                              */
  int64_t p;                     /* columns                                    */
  const double* times;           /* [n] sorted survival times                 */
  const int32_t* status;         /* [n] 0 censored, 1 event, 2 competing      */
  const int64_t* col_ptr;        /* [p+1] CSC column offsets                  */
  const int32_t* row_idx;        /* [nnz] sorted row positions                */
  const double* vals;            /* [nnz] values, or NULL when all are 1.0    */
  const uint8_t* col_indicator;  /* [p] 1 = indicator column (e*=exp(d) rule,
                                    src/engine.cpp:200-206); NULL = derive:
                                    all-ones and density < 25%               */
  const uint8_t* stratum_start;  /* [n] 1 at the first row of each stratum, or
                                    NULL (one stratum).  New vs the reference
                                    (SPEC.md:174 lists strata as a non-goal). */
} gss_host_dataset;

typedef struct gss_dataset gss_dataset; /* device-resident packed dataset */
typedef struct gss_engine gss_engine;   /* per-fit device state + stream   */

/* Last error message on this thread ("" if none). */
const char* gss_last_error(void);
/* Library/build information (static string). */
const char* gss_version(void);
/* Number of usable devices (0 if none). */
int gss_device_count(void);

/*
 * Pack a host dataset onto `device`: uploads CSC, builds the tile-blocked
 * column pointers, the CSR copy used by load_beta/refresh, per-column max |x|.
 * Replaces sort_and_block's output being handed to Engine
 * (src/dataset.cpp:172-262 -> src/engine.cpp:103-118).
 * The returned handle is reference counted (engines retain it).
 */
int gss_dataset_pack(const gss_host_dataset* host, int device, gss_dataset** out);
void gss_dataset_release(gss_dataset* ds);

/*
 * Device ingestion (sort_and_block / dataset_from_coo, src/dataset.cpp:190-262):
 * orders the rows by (stratum asc,) time desc, row id asc and builds the CSC
 * over sorted positions with CUB radix sorts on `device`.
 *   order_out[n]     sorted position -> input row id
 *   col_ptr_out[p+1], row_pos_out[nnz], vals_out[nnz] (capacity nnz): CSC of
 *                    the nonzero cells (zero values are absent cells)
 *   *nnz_out         stored cells
 *   err_info[2]      on GSS_ERR_INDEX / GSS_ERR_DOMAIN: [0] = first failing
 *                    input entry; on GSS_ERR_DUPLICATE: [0] sorted position,
 *                    [1] column of the first repeated cell
 * strata may be NULL.  n and nnz must be below 2^31 per call.
 */
int gss_coo_sort(int device, int64_t n, const double* times, const int64_t* strata, int64_t nnz,
                 const int64_t* rows, const int64_t* cols, const double* vals, int64_t p,
                 int64_t* order_out, int64_t* col_ptr_out, int32_t* row_pos_out, double* vals_out,
                 int64_t* nnz_out, int64_t* err_info);
/* Bytes of device memory held by the packed dataset. */
int64_t gss_dataset_device_bytes(const gss_dataset* ds);

/*
 * Engine(const SurvivalDataset&, Model, ChunkPlan, recompute_interval)
 * (include/survscan/engine.hpp:38-39, src/engine.cpp:103-118).
 * row_mask: optional [n] 0/1 — the engine sees only rows with mask 1, exactly
 * as if the dataset had been subset_rows()'d (src/dataset.cpp:268-322); used
 * for cross-validation folds without copying the design.
 * Fine-Gray censoring weights are estimated on the visible rows
 * (src/censoring.cpp:39-94).  Cox with competing rows -> GSS_ERR_DOMAIN.
 */
int gss_engine_create(gss_dataset* ds, int model, int64_t recompute_interval,
                      const uint8_t* row_mask, gss_engine** out);
void gss_engine_destroy(gss_engine* e);
/*
 * CTAs of the engine's persistent launches (one per SM by default = the
 * device's co-resident capacity; 0 restores it).  The tile ranges are
 * re-partitioned.  Used by the parity tests to put many tiles on each CTA
 * (the geometry of the full-size fits on small inputs) and by batched
 * multi-fit launches.  The environment variable GSS_MAX_GRID caps it at
 * creation.  No reference counterpart (ChunkPlan, scan.hpp:22-46, is the
 * CPU analogue: it only changes the summation order).
 */
int gss_engine_set_grid(gss_engine* e, int grid);
int gss_engine_grid(gss_engine* e);

/* Engine::load_beta (engine.hpp:46; src/engine.cpp:120-154). */
int gss_engine_load_beta(gss_engine* e, const double* beta, int64_t p);
/* Engine::update_xbeta_sparse (engine.hpp:52; src/engine.cpp:162-218). */
int gss_engine_update(gss_engine* e, int64_t column, double delta);
/* Engine::refresh (engine.hpp:55; src/engine.cpp:156-160). */
int gss_engine_refresh(gss_engine* e);
/* Engine::grad_hessian (engine.hpp:60; src/engine.cpp:220-242). */
int gss_engine_grad_hessian(gss_engine* e, int64_t column, double* gradient,
                            double* hessian, double* fixed_term);
/* Engine::grad_hessian_separated (engine.hpp:61; src/engine.cpp:244-329): the
 * unfused path (materialised lanes, separate prefix / suffix scans, transform);
 * the fusion ablation.  Same results as gss_engine_grad_hessian to ~1e-15. */
int gss_engine_grad_hessian_separated(gss_engine* e, int64_t column, double* gradient,
                                      double* hessian, double* fixed_term);
/* Engine::log_likelihood (engine.hpp:63; src/engine.cpp:331-341). */
int gss_engine_log_likelihood(gss_engine* e, double* out);

/* Accessors (engine.hpp:65-71).  Copy device state to host buffers. */
int gss_engine_get_beta(gss_engine* e, double* out, int64_t p);
int gss_engine_get_xbeta(gss_engine* e, double* out, int64_t n);
int gss_engine_get_exp_xbeta(gss_engine* e, double* out, int64_t n);
int gss_engine_get_fixed_terms(gss_engine* e, double* out, int64_t p);
int gss_engine_get_ipcw(gss_engine* e, double* u, double* g, int64_t n);
int gss_engine_counters(gss_engine* e, int64_t* accepted, int64_t* refreshes);

/* Penalty + fit configuration (ccd.hpp:13-30). */
typedef struct gss_penalty_spec {
  int kind;                  /* gss_penalty */
  double strength;           /* gamma (l1) or tau (l2)                      */
  const uint8_t* exempt;     /* [p] 1 = not penalised, or NULL              */
} gss_penalty_spec;

typedef struct gss_fit_config {
  double tolerance;          /* relative objective change per cycle (1e-6) */
  int64_t max_cycles;        /* 1000 */
  double trust_init;         /* 1.0 */
} gss_fit_config;

typedef struct gss_fit_result {
  double objective;
  int64_t cycles;
  int32_t converged;
  int64_t nonzero_count;
  int64_t skipped_steps;
  int64_t monotonicity_violations;
  double wall_seconds;       /* host wall clock of the whole fit               */
  double device_seconds;     /* CUDA-event time of the coordinate cycles       */
} gss_fit_result;

/*
 * fit_with_engine (src/ccd.cpp:131-184) with the per-coordinate work on the
 * device: each cycle is ONE persistent kernel launch that walks the p
 * coordinates (scan/transform/reduce + coordinate_step + deferred sparse
 * update, one grid-wide exchange per coordinate) and then evaluates the
 * log-likelihood; the host syncs once per cycle to test convergence.
 * beta_out: [p]; trace_out: [max_cycles+1] (may be NULL).
 */
int gss_engine_fit(gss_engine* e, const gss_penalty_spec* pen, const gss_fit_config* cfg,
                   double* beta_out, double* trace_out, gss_fit_result* out);

/*
 * Batched multi-fit ("a single larger
 * kernel to perform many repetitions of k-fold cross-validation"): fits
 * count engines (e.g. the folds x lambda tasks of cross_validate,
 * src/crossval.cpp:153-174, or bootstrap resamples, :218-257), each exactly as
 * gss_engine_fit would (same results), but up to max_active of them (<= 24;
 * <= 0 = 24) advance together: every launch of the cycle kernel runs one CCD
 * cycle of every active fit, each on its own share of the SMs with its own
 * grid barrier, so small-N fits stop paying a whole GPU's exchange latency per
 * coordinate.  A fit that converges (or fails) leaves the batch and the next
 * queued one joins.  All engines must live on one device and share p.
 * pens[count]; cfg shared; beta_out [count][p] (may be NULL); results[count];
 * status[count] (may be NULL): the gss_status of each fit.  Returns the first
 * failing fit's status (GSS_OK if all succeeded); device_seconds (may be NULL)
 * = CUDA-event time of all batched cycle launches.
 */
int gss_fit_batch(gss_engine* const* engines, int64_t count, const gss_penalty_spec* pens,
                  const gss_fit_config* cfg, int max_active, double* beta_out,
                  gss_fit_result* results, int32_t* status, double* device_seconds);

/*
 * Engine::grad_hessian for every column at the engine's current beta in ONE
 * device launch (the batched sweep behind gamma_max, src/crossval.cpp:104-110).
 * Each output is [p] (any may be NULL).
 */
int gss_engine_grad_hessian_all(gss_engine* e, double* gradient, double* hessian,
                                double* fixed_term);
/*
 * gamma_max helper (src/crossval.cpp:104-110): max_j |g'_j| at the engine's
 * current beta, all columns in one batched device sweep.
 */
int gss_engine_max_abs_gradient(gss_engine* e, double* out);

/*
 * Patient sharding (config C5): an engine over one contiguous row shard of the
 * global order (cut at tied-block boundaries; stratum_start[0] = 0 marks a
 * shard whose first row continues a stratum).  Per coordinate every rank
 *   1. gss_shard_aggregate(e, j, agg)  -> agg[0] stratum-start flag,
 *      agg[1..3] fwd tail (sum e, e*x_j, e*x_j^2 from the last stratum start),
 *      agg[4..6] rev head (Fine-Gray u-weighted), agg[7] first row starts a stratum;
 *   2. all-gathers the aggregates and composes its carry (segmented prefix of
 *      the earlier shards' tails / suffix of the later shards' heads);
 *   3. gss_shard_sums(e, j, carry, &s0, &s1) -> this shard's (grad_sum,
 *      hess_sum) of fused_grad_hess (scan_kernels.hpp:74-214), or for j = -1
 *      (sum delta*eta, sum d*log D) of the log-likelihood;
 *   4. all-reduces the sums in rank order, finishes and steps identically.
 * carry8: [0..2] fwd (a, b, c), [4..6] rev (ua, ub, uc), others 0.
 */
int gss_shard_aggregate(gss_engine* e, int64_t column, double* agg8);
int gss_shard_sums(gss_engine* e, int64_t column, const double* carry8, double* s0, double* s1);
/* validate-before-mutate of update_xbeta_sparse (src/engine.cpp:171-190) without mutating */
int gss_engine_update_validate(gss_engine* e, int64_t column, double delta, int32_t* overflow);

/*
 * In-kernel patient sharding (config C5): a communicator gives
 * every shard engine peer-visible exchange buffers; each grid exchange of a
 * shard's cycle kernel is then followed by one exchange of the shard
 * aggregates (slot partials, segmented scan tails/heads, aux flags) over
 * NVLink peer memory, combined in rank order, so every shard computes the
 * identical Engine::finish + coordinate_step.  Cox only (Fine-Gray needs the
 * global censoring KM).  The host CCD loop is gss_engine_fit (one process per
 * GPU; every rank calls it) or gss_sharded_fit_local (all shards in this
 * process, one batched launch per cycle).
 *   gss_comm_unique_id  rank 0 creates the NCCL unique id (128 bytes); the
 *                       caller broadcasts it (e.g. torch.distributed)
 *   gss_comm_init       NCCL bootstrap + CUDA IPC exchange buffers
 *   gss_comm_local      a communicator per shard engine of this process
 *                       (attaches them and makes the fixed terms global)
 *   gss_engine_attach_comm  engine becomes shard `rank`; fixed terms become
 *                       the rank-ordered sums over shards (NCCL all-gather)
 */
typedef struct gss_comm gss_comm;
/* NCCL-free bootstrap (any out-of-band all-gather, e.g. torch.distributed /
 * MPI): create -> export this rank's 128-byte CUDA-IPC handle -> all-gather
 * (rank order) -> connect.  Fixed terms: all-gather gss_engine_get_fixed_terms,
 * sum in rank order, gss_engine_set_fixed_terms on every rank. */
int gss_comm_create(int nranks, int rank, int device, gss_comm** out);
int gss_comm_ipc_handle(gss_comm* c, unsigned char* out128);
int gss_comm_connect(gss_comm* c, const unsigned char* all_handles);
int gss_engine_set_fixed_terms(gss_engine* e, const double* in, int64_t p);
/* max |x| per column of the engine's dataset (the fast overflow bound); shards
 * must share the global maximum: all-gather, max, set on every rank (the
 * setter writes the dataset's bound, shared by its engines) */
int gss_engine_get_colmax(gss_engine* e, double* out, int64_t p);
int gss_engine_set_colmax(gss_engine* e, const double* in, int64_t p);
int gss_comm_unique_id(unsigned char* out128);
int gss_comm_init(int nranks, int rank, const unsigned char* uid128, int device, gss_comm** out);
int gss_comm_local(gss_engine* const* shards, int count, gss_comm** comms_out);
int gss_comm_rank(const gss_comm* c, int* nranks, int* rank);
int gss_engine_attach_comm(gss_engine* e, gss_comm* c);
void gss_comm_destroy(gss_comm* c);
int gss_sharded_fit_local(gss_engine* const* shards, int count, const gss_penalty_spec* pen,
                          const gss_fit_config* cfg, double* beta_out, gss_fit_result* res,
                          double* device_seconds);

/* Device time (ms) of the last fit's coordinate cycles, for bench. */
int gss_engine_last_timing(gss_engine* e, double* scan_ms, int64_t* launches);
/* Per-cycle statistics of the last fit: CUDA-event device time of each
 * cycle's graph (ms) and the accepted-update count after each cycle.
 * Returns the number of cycles written (<= max). */
int64_t gss_engine_cycle_stats(gss_engine* e, double* ms, int64_t* accepted, int64_t max);

#ifdef __cplusplus
}
#endif
#endif /* GSS_H */
