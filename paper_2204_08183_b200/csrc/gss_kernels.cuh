// gss_kernels.cuh — kernel parameter blocks shared by gss_kernels.cu and the
// host side (gss_capi.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace gss {

// Per-engine device control block (zero-initialised at engine creation).
struct Ctl {
  // contended words each own a 128-byte line (atomics vs. polling)
  alignas(128) unsigned int tile_counter;   // dynamic tile ids (phase C)
  alignas(128) unsigned int ticket;         // CTA completion count (last CTA runs the tail)
  alignas(128) unsigned int items_a;        // phase-A work items claimed
  alignas(128) unsigned int groups_done;    // 32-tile groups scanned (last one scans groups)
  alignas(128) unsigned long long ready;    // epoch whose tile prefixes are published
  alignas(128) int tprev_valid;             // tsum holds fresh per-tile sums of the current e
  int pad2;
  unsigned long long epoch;    // launch generation tag for tile status words
  // deferred state change applied by the NEXT sweep's tile phase
  long long pend_col;          // -1: none
  double pend_delta;
  double pend_factor;          // exp(pend_delta), indicator cache rule
  int refresh_pending;         // recompute eta/e from beta (refresh())
  int halted;                  // an error stopped the cycle: later sweeps no-op
  int err_code;                // gss_status of the first error in the cycle
  int pad0;
  long long err_col;
  unsigned long long eta_absmax_bits;  // max |eta| at the last refresh/load (double bits)
  unsigned long long absmax_next_bits; // max |eta| gathered by a refresh sweep in flight
  double bound_slack;                  // sum |delta| * max|x| of updates since then
  long long accepted;          // Engine::accepted_ (engine.hpp:88)
  long long refreshes;         // Engine::refreshes_
  long long skipped;           // FitResult.skipped_steps (ccd.cpp:161-164)
  // results of the last sweep
  double grad_sum, hess_sum;   // GradHessSums
  double gradient, hessian, fixed_term;
  double ll_fixed, ll_logden, loglik;
  int bad;                     // denominator <= 0 / NaN seen
  int pad1;
};

enum SweepMode : int { kModeGradApi = 0, kModeGradCcd = 1, kModeLoglik = 2 };

struct SweepParams {
  // dataset (shared, read-only)
  int64_t n, npad, p;
  int ntiles;
  int has_vals;
  const int64_t* col_ptr;
  const int32_t* row_idx;      // padded by 4 ints
  const double* vals;          // parallel to row_idx (NULL => all 1.0)
  const uint8_t* col_ind;      // [p] indicator-column flags
  const uint32_t* tile_ptr;    // [p][ntiles+1] nnz offset of each tile start
  const int64_t* row_ptr;      // CSR [n+1]
  const int32_t* csr_col;      // CSR [nnz] ascending per row
  const double* csr_val;       // CSR values (NULL => all 1.0)
  const double* colmax;        // [p] max |x| per column
  // engine state
  double* eta;                 // [npad]
  double* e;                   // [npad] exp(eta) cache (0 for masked/pad rows)
  const uint32_t* code;        // [npad]
  const double* u;             // [npad] Fine-Gray IPCW u (NULL for cox)
  const double* g;             // [npad] Fine-Gray IPCW g
  double* beta;                // [p]
  double* halfwidth;           // [p]
  const uint8_t* penalized;    // [p]
  const double* fixed;         // [p]
  int pen_kind;
  int weighted;
  double pen_strength;
  long long recompute_interval;
  // carry scratch
  double* agg;                 // [ntiles][4] phase-A tile aggregates (f, a, b, c)
  double* prefix;              // [ntiles][4] exclusive tile prefixes inside the 32-tile group
  double* gsum;                // [ngroups][4] group totals
  double* gpre;                // [ngroups][4] exclusive group prefixes
  unsigned int* grp_cnt;       // [ngroups] phase-A tiles completed per group (reset by the tail)
  double* tsum;                // [2][ntiles][2] fresh per-tile (f, sum e) by launch parity
  const int32_t* tile_lastseg; // [ntiles] last stratum-start row in the tile, -1 if none
  int has_mask;                // some rows are masked out (row_mask engine)
  int has_strata;              // a stratum starts after row 0 (segmented scan needed)
  double* tile_part;           // [ntiles][4]
  Ctl* ctl;
  int64_t column;              // scan column for grad modes
  unsigned long long* trace;   // optional event trace [cap][2] (GSS_TRACE=1), else null
  unsigned int* trace_n;
  unsigned int trace_cap;
};

// launchers (gss_kernels.cu)
cudaError_t launch_sweep(int mode, const CUtensorMap* tm_e, const CUtensorMap* tm_code,
                         const SweepParams& prm, int grid, cudaStream_t s);
int sweep_max_active_ctas_per_sm();
int sweep_threads();
size_t sweep_smem_bytes();

cudaError_t launch_validate_csc(const int64_t* col_ptr, const int32_t* row_idx, int64_t p,
                                int64_t n, int* bad, cudaStream_t s);
cudaError_t launch_exclusive_scan(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s);
cudaError_t launch_build_tile_ptr(const int64_t* col_ptr, const int32_t* row_idx, int64_t p,
                                  int ntiles, uint32_t* tile_ptr, cudaStream_t s);
cudaError_t launch_colmax(const int64_t* col_ptr, const double* vals, int64_t p,
                          double* colmax, cudaStream_t s);
cudaError_t launch_csr_count(const int32_t* row_idx, int64_t nnz, int64_t* row_cnt,
                             cudaStream_t s);
cudaError_t launch_csr_fill(const int64_t* col_ptr, const int32_t* row_idx, const double* vals,
                            int64_t p, int64_t* cursor, int32_t* csr_col, double* csr_val,
                            cudaStream_t s);
cudaError_t launch_csr_sort_rows(const int64_t* row_ptr, int64_t n, int32_t* csr_col,
                                 double* csr_val, cudaStream_t s);
cudaError_t launch_fixed_terms(const int64_t* col_ptr, const int32_t* row_idx,
                               const double* vals, const uint8_t* col_ind,
                               const uint32_t* code, int64_t p, double* fixed,
                               cudaStream_t s);
// load_beta: fresh eta = X beta into scratch, overflow flag; then commit
cudaError_t launch_spmv_rows(const SweepParams& prm, const double* beta, double* eta_out,
                             int* overflow, cudaStream_t s);
cudaError_t launch_commit_eta(const SweepParams& prm, const double* eta_in, cudaStream_t s);
// API update: check (validate-before-mutate) then commit
cudaError_t launch_update_check(const SweepParams& prm, int64_t col, double delta, int* overflow,
                                cudaStream_t s);
cudaError_t launch_update_commit(const SweepParams& prm, int64_t col, double delta,
                                 double factor, cudaStream_t s);

}  // namespace gss
