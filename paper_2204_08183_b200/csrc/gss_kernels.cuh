// gss_kernels.cuh — parameter blocks shared by the device code (gss_cycle.cu,
// gss_aux.cu) and the host side of the C ABI (gss_capi.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace gss {

// Per-engine device control block (zero-initialised at engine creation).
// Written by CTA 0 of the cycle kernel at the end of a launch; read by every
// CTA at launch start.
struct Ctl {
  unsigned long long bar_base;         // grid-barrier counter value at launch start
  unsigned long long eta_absmax_bits;  // max |eta| at the last refresh/load (double bits)
  double bound_slack;                  // sum |delta| * max|x| of updates since then
  long long accepted;                  // Engine::accepted_ (engine.hpp:88)
  long long refreshes;                 // Engine::refreshes_
  long long skipped;                   // FitResult.skipped_steps (ccd.cpp:161-164)
  int rec_valid;                       // per-tile records serve a launch starting at rec_col
  int pad0;
  long long rec_col;
  int err_code;                        // gss_status of the first error (0 = none)
  int pad1;
  long long err_col;
  unsigned long long xr_base;          // cross-shard counter value at launch start
  unsigned long long xr_count;         // cross-shard exchanges so far (buffer parity)
  // results of the last slot of each kind
  double grad_sum, hess_sum, gradient, hessian, fixed_term;
  double ll_fixed, ll_logden, loglik;
};

// per-tile record (doubles) produced by the consumers of slot k for slot k+1:
//   fwd lanes  : a = sum e, b = sum e*x, c = sum e*x^2            (x = next column)
//   fwd s-parts: sums of the same over the rows of the slot-k column (the
//                pending update of slot k+1), for the exp(delta) correction
//   rev lanes  : the u-weighted versions (Fine-Gray)
enum RecField : int {
  kRa = 0, kRb, kRc, kRsa, kRsb, kRsc,
  kRua, kRub, kRuc, kRusa, kRusb, kRusc,
  kRecFields
};
constexpr int kRecStride = 12;
// per-tile in-range carries (uncorrected + s-parts), written before the slot barrier
//   0..5  : fwd segmented exclusive prefix inside the CTA range (a,b,c,sa,sb,sc)
//   6     : 1 if a stratum starts at or before this tile inside the range (no CTA carry-in)
//   8..13 : rev segmented inclusive suffix inside the CTA range (ua,ub,uc,usa,usb,usc)
//   14    : 1 if a stratum starts after this tile inside the range (no CTA carry-in)
constexpr int kCarStride = 16;
// CTA payload exchanged at the slot barrier (one 128-byte row per CTA, gathered
// with one bulk copy)
//   0..2 : slot partials (p0, p1, bad)
//   3    : 1 if any tile of the range starts a stratum
//   4..9 : fwd tail  (tiles from the last stratum-first tile): a,b,c,sa,sb,sc
//   10..15: rev head (tiles before the first stratum-first tile): ua,ub,uc,usa,usb,usc
// followed by the auxiliary rows [2][grid][kPayAux]: 0 max |eta| (refresh),
// 1 overflow flag (exact validation)
constexpr int kPayStride = 16;
constexpr int kPayAux = 2;

enum SlotKind : int { kSlotGrad = 0, kSlotLoglik = 1 };
enum LaunchMode : int { kModeApi = 0, kModeCcd = 1 };

struct CycleParams {
  // ---- dataset (shared, read-only) ----
  int64_t n, npad, p;
  int ntiles;
  int has_vals;
  const int64_t* col_ptr;
  const int32_t* row_idx;      // padded device positions, +4 ints of slack
  const double* vals;          // parallel to row_idx (NULL => all 1.0)
  const uint8_t* col_ind;      // [p] indicator-column flags
  const uint32_t* tile_ptr;    // [p][ntiles+1] nnz offset of each tile start
  const int64_t* row_ptr;      // CSR [npad+1]
  const int32_t* csr_col;      // CSR [nnz] ascending per row
  const double* csr_val;       // CSR values (NULL => all 1.0)
  const double* colmax;        // [p] max |x| per column
  const uint8_t* tile_first;   // [ntiles] 1 if a stratum starts at the tile's first row
  const int32_t* dense_idx;    // [p] dense-pool slot of a column with density >= 25%, else -1
  const double* dense_pool;    // [ndense][npad] dense column values by device position
  // ---- engine state ----
  double* eta;                 // [npad]
  double* e;                   // [npad] exp(eta) cache (0 for masked/pad rows)
  const uint32_t* code;        // [npad] row code words
  const double* g;             // [npad] Fine-Gray G(Y-) (NULL unless weighted)
  double* beta;                // [p]
  double* halfwidth;           // [p]
  const uint8_t* penalized;    // [p]
  const double* fixed;         // [p]
  int weighted;
  int pen_kind;
  double pen_strength;
  long long recompute_interval;
  // ---- launch ----
  const int32_t* slot_col;     // [nslots] column of each slot, -1 = log-likelihood slot
  int nslots;
  int mode;                    // LaunchMode
  int grid;                    // CTAs (<= co-resident capacity)
  const int32_t* cta_tile0;    // [grid+1] first tile of each CTA (cost-balanced), or NULL
  double* slot_out;            // optional [nslots][4] API results (gradient, hessian, fixed, ll)
  // ---- scratch ----
  double* trec;                // [ntiles][kRecStride]
  double* tcar;                // [ntiles][kCarStride]
  double* cpay;                // [2][grid][kPayStride] + [2][grid][kPayAux]
  unsigned int* bar;           // grid barrier counter
  Ctl* ctl;
  // optional event trace (GSS_TRACE=1): [cap][2] = (globaltimer ns, cta<<40|ev<<32|arg)
  unsigned long long* trace;
  unsigned int* trace_n;
  unsigned int trace_cap;
  int dbg;                     // debug/ablation bits (GSS_DEBUG): 1 skip tile work, 2 skip records,
                               // 4 skip scans/transform
  // ---- patient sharding (C5): this engine holds one contiguous row shard ----
  const double* ext;           // [8] carry from the other shards: fwd (a,b,c) into the first
                               // tile, [4..6] rev (ua,ub,uc) after the last; NULL = none
  double* shard_out;           // [8] this shard's aggregate after the prologue exchange:
                               // [0] stratum-start flag, [1..3] fwd tail, [4..6] rev head
  int prologue_only;           // stop after the prologue (records + shard aggregate)
  int reuse_records;           // API mode: records from a prologue-only launch are valid
  // ---- in-kernel cross-shard exchange (gss_comm): every grid exchange of
  // this shard's launch is followed by one exchange of the shard aggregates
  // (kXrStride doubles per rank) over peer memory, so all shards run the
  // same fixed-order reduction and the same coordinate step ----
  int nranks, rank;            // nranks > 1 enables it
  int xr_sys;                  // shards on several devices: system-scope release/acquire
  double* const* xr_pay;       // [nranks] rank q's buffer [2][nranks][kXrStride] (peer-mapped)
  unsigned int* const* xr_bar; // [nranks] rank q's arrival counter (peer-mapped)
};
constexpr int kXrStride = 24;

// Kernel parameter block of one cycle-kernel launch over K engines (fits):
// CTAs [cta_base[f], cta_base[f+1]) run engine f with its own parameters,
// TMA descriptors, grid barrier and payload buffers.  K = 1 is the single-fit
// launch; K = kMaxBatch the batched multi-fit launch (CV folds x lambda grid,
// bootstrap resamples).  Lives in the parameter (constant) bank.
constexpr int kMaxBatch = 24;
template <int K>
struct LaunchParams {
  CUtensorMap tm_e[K], tm_code[K], tm_g[K];
  CycleParams P[K];
  int nfit;
  int cta_base[K + 1];
};
struct BatchEntry {
  const CUtensorMap* tm_e;
  const CUtensorMap* tm_code;
  const CUtensorMap* tm_g;
  const CycleParams* prm;
};

// launchers (gss_cycle.cu)
cudaError_t launch_cycle(const CUtensorMap* tm_e, const CUtensorMap* tm_code,
                         const CUtensorMap* tm_g, const CycleParams& prm, cudaStream_t s);
// one launch for k <= kMaxBatch engines of the same kind (all weighted or
// none); their grids must fit the device together
cudaError_t launch_cycle_batch(const BatchEntry* entries, int k, cudaStream_t s);
int cycle_max_grid(int device, bool weighted);
size_t cycle_smem_bytes(bool weighted);

// separated (unfused) derivative path (gss_separated.cu): out2 = (grad_sum, hess_sum)
size_t separated_scratch_doubles(int64_t npad, int ntiles);
cudaError_t launch_separated(const CycleParams& prm, int64_t column, double* scratch, int* bad,
                             double* out2, cudaStream_t s);

// aux (gss_aux.cu)
cudaError_t launch_validate_csc(const int64_t* col_ptr, const int32_t* row_idx, int64_t p,
                                int64_t n, int* bad, cudaStream_t s);
cudaError_t launch_exclusive_scan(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s);
cudaError_t launch_remap_rows(int32_t* row_idx, int64_t nnz, const int64_t* dev_row,
                              cudaStream_t s);
cudaError_t launch_build_tile_ptr(const int64_t* col_ptr, const int32_t* row_idx, int64_t p,
                                  int ntiles, uint32_t* tile_ptr, cudaStream_t s);
// dense pool: pool[slot[j]][row_idx[k]] = vals[k] (or 1.0) for dense columns
cudaError_t launch_fill_dense(const int64_t* col_ptr, const int32_t* row_idx, const double* vals,
                              const int32_t* slot, int64_t p, int64_t npad, double* pool,
                              cudaStream_t s);
cudaError_t launch_colmax(const int64_t* col_ptr, const double* vals, int64_t p,
                          double* colmax, cudaStream_t s);
// e[i] = 0 if code[i] & kCodeMasked else 1 (engine start, beta = 0)
cudaError_t launch_init_e(const uint32_t* code, int64_t npad, double* e, cudaStream_t s);
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
cudaError_t launch_spmv_rows(const CycleParams& prm, const double* beta, double* eta_out,
                             int* overflow, cudaStream_t s);
cudaError_t launch_commit_eta(const CycleParams& prm, const double* eta_in, cudaStream_t s);
// API update: check (validate-before-mutate) then commit
cudaError_t launch_update_check(const CycleParams& prm, int64_t col, double delta, int* overflow,
                                cudaStream_t s);
cudaError_t launch_update_commit(const CycleParams& prm, int64_t col, double delta,
                                 double factor, cudaStream_t s);

}  // namespace gss
