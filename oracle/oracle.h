/*
 * oracle.h — CPU restatement of the reference (survscan) CCD hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library, and only as the checker.
 * The product (libgss.so / _survscan) never links or calls it.
 *
 * Every function restates one reference routine serially (a single chunk, i.e.
 * ChunkPlan::serial(), left-to-right accumulation) and cites the reference
 * file:line it follows (paths relative to /root/reference/proj/).
 *
 * Parity is pinned against the compiled reference (oracle/_ref, built by
 * oracle/build_ref.sh) via the golden fixtures in tests/golden/ (made by
 * tests/golden/make_golden.py) — see tests/test_oracle.py.
 *
 * Data contract (the reference's in-memory layout, include/survscan/dataset.hpp:14-111):
 *   rows sorted by (stratum asc,) time desc, original row id asc;
 *   CSC columns: col_ptr[p+1] (int64), row_idx[nnz] (int32, strictly ascending
 *   per column), vals[nnz] (fp64; 1.0 for indicator columns);
 *   col_indicator[j] = 1 when every stored value of column j is 1.0 and the
 *   column is below the 25% density cutoff (SparseColumn::make,
 *   src/dataset.cpp:126-157) — it selects the e *= exp(delta) cache rule.
 *   strata: optional stratum_start[n] (1 at the first row of each stratum);
 *   NULL means one stratum.  The reference has no strata; the
 *   stratified values here are the COMPOSITION sum over strata of the
 *   reference computation on each stratum's rows.
 */
#ifndef SURVSCAN_ORACLE_H
#define SURVSCAN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_DOMAIN = 3, ORC_INVALID_COLUMN = 6, ORC_NONPOS_DEN = 7,
       ORC_OVERFLOW = 8, ORC_DEGENERATE = 9 };

typedef struct {
  int64_t n, p;
  const double* times;         /* [n] sorted desc within stratum          */
  const int32_t* status;       /* [n] 0 censored, 1 event, 2 competing     */
  const int64_t* col_ptr;      /* [p+1]                                    */
  const int32_t* row_idx;      /* [nnz]                                    */
  const double* vals;          /* [nnz]                                    */
  const uint8_t* col_indicator;/* [p]                                      */
  const uint8_t* stratum_start;/* [n] or NULL                              */
} orc_data;

/* Mutable per-fit state (engine.hpp:81-87). Arrays sized by the caller. */
typedef struct {
  int fine_gray;        /* weighted path iff fine_gray && any status==2    */
  double* beta;         /* [p] */
  double* eta;          /* [n] */
  double* e;            /* [n] exp(eta) cache */
  double* fixed;        /* [p] delta' X_j */
  double* u;            /* [n] IPCW u (fine-gray) */
  double* g;            /* [n] IPCW g (fine-gray) */
  int64_t accepted, refreshes, recompute_interval;
} orc_state;

/* Tied blocks and per-row block-end event counts (src/dataset.cpp:190-204). */
int orc_block_counts(const orc_data* d, double* count_at_end /* [n] */);
/* IPCW weights, per stratum (src/censoring.cpp:39-90). */
int orc_ipcw(const orc_data* d, double* u, double* g);
/* delta' X_j (src/engine.cpp:76-101). */
void orc_fixed_terms(const orc_data* d, double* fixed);
/* Engine construction + load_beta (src/engine.cpp:103-154). */
int orc_init(const orc_data* d, orc_state* s);
int orc_load_beta(const orc_data* d, orc_state* s, const double* beta);
/* update_xbeta_sparse (src/engine.cpp:162-218). */
int orc_update(const orc_data* d, orc_state* s, int64_t j, double delta);
/* fused_grad_hess + finish (include/survscan/scan_kernels.hpp:74-214,
 * src/engine.cpp:220-242). Outputs gradient, hessian, fixed term, and the raw
 * sums (grad_sum, hess_sum). */
int orc_grad_hessian(const orc_data* d, const orc_state* s, int64_t j,
                     double* grad, double* hess, double* fixed_term,
                     double* grad_sum, double* hess_sum);
/* log_likelihood (src/engine.cpp:331-341, src/scan.cpp:233-250, 275-367). */
int orc_log_likelihood(const orc_data* d, const orc_state* s, double* out);

/* coordinate_step (src/ccd.cpp:71-129). penalty_kind: 0 none, 1 l1, 2 l2. */
void orc_coordinate_step(double beta_j, double grad, double hess, int penalty_kind,
                         double strength, int penalized, double halfwidth,
                         double* new_beta, double* applied, double* new_halfwidth,
                         int* skipped);

/* fit_with_engine (src/ccd.cpp:131-184). exempt: [p] 0/1 or NULL.
 * trace must hold max_cycles+1 entries. */
typedef struct {
  double objective;
  int64_t cycles, converged, nonzero, skipped, violations;
} orc_fit_result;
int orc_fit(const orc_data* d, orc_state* s, int penalty_kind, double strength,
            const uint8_t* exempt, double tol, int64_t max_cycles,
            double trust_init, double* trace, orc_fit_result* out);

#ifdef __cplusplus
}
#endif
#endif
