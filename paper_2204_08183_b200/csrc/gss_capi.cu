// gss_capi.cu — host implementation of the C ABI in include/gss.h.
//
// Owns device memory, streams and TMA descriptors; builds the per-engine row
// code words and (Fine-Gray) censoring weights on the host, exactly as the
// reference builds them per Engine (src/engine.cpp:103-118,
// src/censoring.cpp:39-94); drives the persistent cycle kernel
// (gss_cycle.cu) once per CCD cycle / API evaluation.
//
// Device row layout: the reference's sorted order with every stratum padded
// to a whole number of 2048-row tiles (padding rows are masked: exp(eta) = 0),
// so no tile spans two strata.  dev_row[i] maps sorted row i to its device
// position.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/gss.h"
#include "gss_device.cuh"
#include "gss_kernels.cuh"

namespace gss {
int set_last_error(int code, const std::string& msg);
int engine_fixed_terms(gss_engine* e, double** dev_fixed, int64_t* p, int* device,
                       cudaStream_t* stream);
int engine_attach_comm(gss_engine* e, int nranks, int rank, double* const* pay_ptrs,
                       unsigned int* const* bar_ptrs, int sys_scope);
}
using namespace gss;

namespace {

thread_local std::string g_last_error;

// NVTX ranges (header-only nvtx3; free when no tool is attached): one per C ABI
// entry point, per pack stage and per CCD cycle, so an nsys/ncu timeline
// lines the device launches up with the host calls that issued them.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  Nvtx(const char* fmt, long long k) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), fmt, k);
    nvtxRangePushA(buf);
  }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
}  // namespace

// shared with the other C-ABI translation units (gss_ingest.cu)
int gss::set_last_error(int code, const std::string& msg) { return fail(code, msg); }

namespace {

#define GSS_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess)                                                              \
      return fail(_e == cudaErrorMemoryAllocation ? GSS_ERR_OOM : GSS_ERR_CUDA,         \
                  std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " #call); \
  } while (0)

// Host vectors whose resize() leaves elements uninitialised, so the pages of
// a 10M-row copy are first touched by the parallel fill below, not serially.
template <class T>
struct DefaultInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = DefaultInitAlloc<U>;
  };
  DefaultInitAlloc() = default;
  template <class U>
  DefaultInitAlloc(const DefaultInitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* q) noexcept {
    ::new (static_cast<void*>(q)) U;
  }
  template <class U, class... A>
  void construct(U* q, A&&... a) {
    ::new (static_cast<void*>(q)) U(std::forward<A>(a)...);
  }
};

// f(lo, hi) over [0, n) in contiguous chunks on up to 16 host threads
// (chunk c covers [n*c/T, n*(c+1)/T)); serial below 1M rows.
template <class F>
void host_parallel(int64_t n, F&& f) {
  const unsigned hc = std::thread::hardware_concurrency();
  const int T = n < (int64_t(1) << 20) ? 1 : static_cast<int>(std::min(16u, std::max(1u, hc)));
  if (T == 1) {
    f(0, 0, n);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(T);
  for (int c = 0; c < T; ++c) th.emplace_back([&f, c, n, T]() { f(c, n * c / T, n * (c + 1) / T); });
  for (auto& t : th) t.join();
}

template <class T>
cudaError_t dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  return cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
}

// Engine buffers come from the device's stream-ordered memory pool (release
// threshold raised once per device): creating and destroying hundreds of
// fold / held-out engines (C4) neither pays cudaMalloc latency nor
// serialises on cudaFree's implicit device synchronisation.
template <class T>
cudaError_t ealloc(T** p, size_t count, cudaStream_t s) {
  *p = nullptr;
  if (count == 0) count = 1;
  static std::once_flag once[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::call_once(once[dev & 63], [dev]() {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
  return cudaMallocAsync(reinterpret_cast<void**>(p), count * sizeof(T), s);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, []() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2D view [npad*elem/128][128 bytes] of a row-major per-row array; box = one
// 2048-row tile as 128-byte rows, 128B swizzle.
int make_tile_map(CUtensorMap* map, void* base, int64_t npad, CUtensorMapDataType dt,
                  int elem_bytes) {
  auto fn = encode_fn();
  if (!fn) return fail(GSS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int per_row = 128 / elem_bytes;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(per_row), static_cast<cuuint64_t>(npad / per_row)};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(per_row),
                       static_cast<cuuint32_t>(kTileRows / per_row)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dt, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(GSS_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return GSS_OK;
}

}  // namespace

struct gss_dataset {
  std::atomic<int> refs{1};
  int device = 0;
  int64_t n = 0, p = 0, nnz = 0, npad = 0;
  int ntiles = 0;
  bool has_vals = false;
  // host copies needed per engine (row codes, IPCW) — sorted order
  template <class T>
  using hvec = std::vector<T, DefaultInitAlloc<T>>;
  hvec<double> times;
  hvec<int32_t> status;
  hvec<int64_t> stratum_of;   // stratum ordinal per sorted row
  hvec<int64_t> dev_row;      // sorted row -> device position
  bool identity_rows = false;  // dev_row[i] == i (no stratum padding)
  std::vector<uint8_t> h_tile_first;
  // device
  int64_t* col_ptr = nullptr;
  int32_t* row_idx = nullptr;        // device positions
  double* vals = nullptr;
  uint8_t* col_ind = nullptr;
  uint32_t* tile_ptr = nullptr;
  int64_t* row_ptr = nullptr;
  int32_t* csr_col = nullptr;
  double* csr_val = nullptr;
  double* colmax = nullptr;
  uint8_t* tile_first = nullptr;
  int32_t* dense_idx = nullptr;      // [p] dense-pool slot or -1 (density >= 25%)
  double* dense_pool = nullptr;      // [ndense][npad]
  int64_t ndense = 0;
  int64_t bytes = 0;  // footprint including the CSR built on the first load_beta
  std::vector<int64_t> h_col_ptr;
  std::mutex csr_mu;
  bool csr_built = false;

  ~gss_dataset() {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    for (void* q : {(void*)col_ptr, (void*)row_idx, (void*)vals, (void*)col_ind, (void*)tile_ptr,
                    (void*)row_ptr, (void*)csr_col, (void*)csr_val, (void*)colmax,
                    (void*)tile_first, (void*)dense_idx, (void*)dense_pool})
      if (q) cudaFree(q);
    if (prev >= 0) cudaSetDevice(prev);
  }
};

struct gss_engine {
  gss_dataset* ds = nullptr;
  int model = 0;
  int64_t interval = 100;
  bool weighted = false;
  cudaStream_t stream = nullptr;
  int grid = 1;
  int max_grid = 1;               // co-resident capacity (payload buffers are sized for it)
  std::vector<uint32_t> h_code;   // device positions
  std::vector<double> h_u, h_g;   // sorted order (accessor)
  std::vector<double> h_beta;
  std::vector<int32_t> h_slots;   // slots of the staged CCD cycle
  // device
  double *eta = nullptr, *e = nullptr, *scratch = nullptr, *g = nullptr;
  double* gs = nullptr;  // streamed G: u = 1/G on competing rows without events (Fine-Gray)
  uint32_t* code = nullptr;
  double *beta = nullptr, *halfwidth = nullptr, *fixed = nullptr;
  uint8_t* penalized = nullptr;
  double *trec = nullptr, *tcar = nullptr, *cpay = nullptr, *slot_out = nullptr;
  double *ext = nullptr, *shard = nullptr;  // patient-shard carry in / aggregate out
  double* sep = nullptr;                    // separated-path scratch (lazy)
  int32_t* slot_col = nullptr;
  int32_t* cta_tile0 = nullptr;
  unsigned int* bar = nullptr;
  Ctl* ctl = nullptr;
  int* dflag = nullptr;
  Ctl* h_ctl = nullptr;  // pinned mirror
  CUtensorMap tm_e{}, tm_code{}, tm_g{};
  CycleParams prm{};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double last_ms = 0.0;
  int64_t last_launches = 0;
  std::vector<double> cycle_ms;
  std::vector<int64_t> cycle_accepted;
  // state of the fit in progress (fit_begin / fit_after_cycle / fit_end)
  struct FitState {
    gss_penalty_spec pen{};
    std::vector<uint8_t> exempt;
    gss_fit_config cfg{};
    std::vector<double> trace;
    gss_fit_result res{};
    double prev = 0.0;
    bool converged = false, done = false;
    bool need_init_obj = false;  // sharded (nranks > 1): objective at beta = 0 still to come
    int64_t cycle = 0;
    int err = GSS_OK;
    std::chrono::steady_clock::time_point t0;
    double dev_ms = 0.0;
  } fs;

  ~gss_engine() {
    cudaSetDevice(ds->device);
    if (stream) cudaStreamSynchronize(stream);
    // pool allocations (ealloc): stream-ordered frees, no device-wide sync
    for (void* q : {(void*)eta, (void*)e, (void*)scratch, (void*)g, (void*)gs, (void*)code, (void*)beta,
                    (void*)halfwidth, (void*)fixed, (void*)penalized, (void*)trec, (void*)tcar,
                    (void*)cpay, (void*)slot_out, (void*)slot_col, (void*)bar, (void*)ctl,
                    (void*)dflag, (void*)ext, (void*)shard, (void*)cta_tile0})
      if (q) cudaFreeAsync(q, stream);
    if (stream) cudaStreamSynchronize(stream);
    if (sep) cudaFree(sep);
    if (h_ctl) cudaFreeHost(h_ctl);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
    gss_dataset_release(ds);
  }
};

namespace {

int sync_ctl(gss_engine* E) {
  GSS_CUDA(cudaMemcpyAsync(E->h_ctl, E->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, E->stream));
  GSS_CUDA(cudaStreamSynchronize(E->stream));
  return GSS_OK;
}

int push_ctl(gss_engine* E) {
  GSS_CUDA(cudaMemcpyAsync(E->ctl, E->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, E->stream));
  GSS_CUDA(cudaStreamSynchronize(E->stream));
  return GSS_OK;
}

// Map a device error word to the reference exception class + message.
int device_error(gss_engine* E, const char* where) {
  const int code = E->h_ctl->err_code;
  const long long col = E->h_ctl->err_col;
  std::string msg;
  switch (code) {
    case GSS_ERR_NONPOS_DEN:
      msg = std::string(where) +
            ": accumulated risk-set denominator <= 0 or derivatives not finite (exp overflow?)";
      break;
    case GSS_ERR_OVERFLOW:
      msg = std::string(where) + ": |x'beta| would exceed 700";
      break;
    default:
      msg = std::string(where) + ": device error " + std::to_string(code);
  }
  if (col >= 0) msg += " (column " + std::to_string(col) + ")";
  // clear for the next call
  E->h_ctl->err_code = 0;
  E->h_ctl->err_col = -1;
  E->h_ctl->rec_valid = 0;
  push_ctl(E);
  return fail(code, msg);
}

// Per-engine row code words (device positions) over the visible rows
// (row_mask), stratum by stratum: maximal runs of equal time among visible
// rows form the tied blocks (src/dataset.cpp:190-204 applied to the subset,
// src/dataset.cpp:268-322); the run's status==1 count goes to its last
// visible row.  Padding rows are masked.
int build_codes(const gss_dataset* ds, const uint8_t* mask, std::vector<uint32_t>& code) {
  const int64_t n = ds->n;
  code.assign(static_cast<size_t>(ds->npad), kCodeMasked);
  // Chunks start at a stratum start or a time change, so no tied block spans
  // two chunks and each chunk is processed exactly as the serial walk would.
  std::vector<int> err(16, 0);
  auto starts_block = [&](int64_t i) {
    return i == 0 || i >= n || ds->stratum_of[i] != ds->stratum_of[i - 1] ||
           ds->times[i] != ds->times[i - 1];
  };
  host_parallel(n, [&](int ch, int64_t lo, int64_t hi) {
    while (!starts_block(lo)) ++lo;
    while (!starts_block(hi)) ++hi;
    int64_t last_vis = -1;
    double last_t = 0.0;
    uint32_t cnt = 0;
    for (int64_t i = lo; i < hi; ++i) {
      const bool seg = i == 0 || ds->stratum_of[i] != ds->stratum_of[i - 1];
      if (seg) {  // a new stratum closes the previous one's last block
        if (last_vis >= 0) code[ds->dev_row[last_vis]] |= cnt;
        last_vis = -1;
        cnt = 0;
      }
      uint32_t& c = code[ds->dev_row[i]];
      c = seg ? kCodeSeg : 0u;
      if (mask && !mask[i]) {
        c |= kCodeMasked;
        continue;
      }
      if (last_vis >= 0 && ds->times[i] != last_t) {
        code[ds->dev_row[last_vis]] |= cnt;
        cnt = 0;
      }
      if (ds->status[i] == 1) {
        if (++cnt > kCodeCount) {
          err[ch] = 1;
          return;
        }
        c |= kCodeEvent;
      } else if (ds->status[i] == 2) {
        c |= kCodeCompeting;
      }
      last_vis = i;
      last_t = ds->times[i];
    }
    if (last_vis >= 0) code[ds->dev_row[last_vis]] |= cnt;
  });
  for (int e : err)
    if (e) return fail(GSS_ERR_DOMAIN, "tied block exceeds 2^28 events");
  return GSS_OK;
}

// Kaplan-Meier of the censoring distribution over the visible rows of each
// stratum, failures before censorings on ties, then u = 1/G(Y-) on competing
// rows and g = G(Y-) (src/censoring.cpp:39-90).  Sorted order.
int build_ipcw_host(const gss_dataset* ds, const uint8_t* mask, std::vector<double>& u,
                    std::vector<double>& g) {
  const int64_t n = ds->n;
  u.assign(static_cast<size_t>(n), 0.0);
  g.assign(static_cast<size_t>(n), 1.0);
  std::vector<int64_t> rows, ends;
  int64_t s = 0;
  while (s < n) {
    int64_t e = s + 1;
    while (e < n && ds->stratum_of[e] == ds->stratum_of[s]) ++e;
    rows.clear();
    for (int64_t i = s; i < e; ++i)
      if (!mask || mask[i]) rows.push_back(i);
    ends.clear();
    for (size_t k = 0; k < rows.size(); ++k)
      if (k + 1 == rows.size() || ds->times[rows[k + 1]] != ds->times[rows[k]]) ends.push_back(k);
    double surv = 1.0;
    for (size_t b = ends.size(); b-- > 0;) {
      const size_t end = ends[b];
      const size_t start = b == 0 ? 0 : ends[b - 1] + 1;
      const double before = surv;
      int64_t censored = 0, failed = 0;
      for (size_t k = start; k <= end; ++k) {
        const int64_t i = rows[k];
        if (ds->status[i] == 0)
          ++censored;
        else
          ++failed;
        g[i] = before;
        if (ds->status[i] == 2) {
          if (!(before > 0.0))
            return fail(GSS_ERR_DEGENERATE,
                        "censoring curve vanishes before a competing event at time " +
                            std::to_string(ds->times[i]));
          u[i] = 1.0 / before;
        }
      }
      if (censored) {
        const double at_risk = static_cast<double>(static_cast<int64_t>(end) + 1 - failed);
        surv *= 1.0 - static_cast<double>(censored) / at_risk;
      }
    }
    s = e;
  }
  return GSS_OK;
}

int check_engine(gss_engine* E) {
  if (!E) return fail(GSS_ERR_DOMAIN, "null engine handle");
  cudaError_t err = cudaSetDevice(E->ds->device);
  if (err != cudaSuccess) return fail(GSS_ERR_CUDA, cudaGetErrorString(err));
  return GSS_OK;
}

// One launch of the cycle kernel over `slots` (API or CCD mode).  Shard
// options: ext = apply the external carry, prologue = records + shard aggregate only.
int run_slots(gss_engine* E, const std::vector<int32_t>& slots, int mode, bool want_out,
              bool ext = false, bool prologue = false) {
  if (slots.empty()) return GSS_OK;
  if (static_cast<int64_t>(slots.size()) > E->ds->p + 1)
    return fail(GSS_ERR_DOMAIN, "too many slots");
  GSS_CUDA(cudaMemcpyAsync(E->slot_col, slots.data(), slots.size() * sizeof(int32_t),
                           cudaMemcpyHostToDevice, E->stream));
  CycleParams P = E->prm;
  P.slot_col = E->slot_col;
  P.nslots = static_cast<int>(slots.size());
  P.mode = mode;
  // API calls on a shard of an in-kernel sharded fit are shard-local (the
  // cross-shard exchange runs in CCD launches, which every shard makes)
  if (mode != kModeCcd) P.nranks = 0;
  P.slot_out = want_out ? E->slot_out : nullptr;
  P.ext = ext ? E->ext : nullptr;
  P.shard_out = prologue ? E->shard : nullptr;
  P.prologue_only = prologue ? 1 : 0;
  P.reuse_records = ext ? 1 : 0;
  if (prologue) P.nslots = 0;  // nothing is streamed
  GSS_CUDA(launch_cycle(&E->tm_e, &E->tm_code, &E->tm_g, P, E->stream));
  return GSS_OK;
}

double penalty_value(const gss_penalty_spec* pen, const std::vector<double>& beta) {
  if (pen->kind == GSS_PEN_NONE) return 0.0;
  double acc = 0.0;
  for (size_t j = 0; j < beta.size(); ++j) {
    if (pen->exempt && pen->exempt[j]) continue;
    if (pen->kind == GSS_PEN_L1)
      acc += pen->strength * std::abs(beta[j]);
    else
      acc += beta[j] * beta[j] / (2.0 * pen->strength);
  }
  return acc;
}

// Static contiguous CTA tile ranges, balanced by estimated tile cost: a tile
// costs its streaming (1) plus its transform passes (8-row x 32-lane passes
// holding a tied-block end with events).  Sets E->grid / prm.grid / prm.cta_tile0.
int partition_ctas(gss_engine* E, int grid) {
  const int nt = E->ds->ntiles;
  grid = std::max(1, std::min(grid, std::min(nt, E->max_grid)));
  std::vector<double> w(static_cast<size_t>(nt), 1.0);
  // Per-tile cost model (Cox): 1 + 0.12 if any pass holds a transform + 0.04
  // per such pass.  A consumer group's tile costs the longest of its warps, so
  // the first transform pass costs most (tools/tile_cost_probe.py: ~5.8k
  // cycles without, ~7.9k with); the p = 512 C2-design fit measured 42.3 us
  // per coordinate with this model vs 43.4 with 1 + 0.05 per pass and 46.0
  // unweighted (tools/gpu_partition_sweep.sh).  Fine-Gray (8-warp groups, one
  // pass per warp) is best at 1 + 0.05 per pass: 79.6 vs 82.2 us (p = 512),
  // 79.2 vs 81.7 (p = 5000).  A per-event-block-end term (GSS_BE_W) made the
  // C2 bench slower at 0.05 / 0.1, so it defaults to 0.
  const bool fg_w = E->weighted;
  const double kPassW =
      std::getenv("GSS_PASS_W") ? std::atof(std::getenv("GSS_PASS_W")) : (fg_w ? 0.05 : 0.028);
  const double kBeW = std::getenv("GSS_BE_W") ? std::atof(std::getenv("GSS_BE_W")) : (fg_w ? 0.0 : 0.0023);
  const double kAnyW =
      std::getenv("GSS_ANY_W") ? std::atof(std::getenv("GSS_ANY_W")) : (fg_w ? 0.0 : 0.15);
  for (int t = 0; t < nt; ++t) {
    int work = 0, ends = 0;
    for (int pass = 0; pass < kTileRows / 256; ++pass) {
      int any = 0;
      for (int r = 0; r < 256; ++r)
        any += (E->h_code[size_t(t) * kTileRows + pass * 256 + r] & kCodeCount) != 0;
      work += any ? 1 : 0;
      ends += any;
    }
    // (distinct event times saturate at one transform per row: cap at 4)
    w[t] = std::min(4.0, 1.0 + kPassW * work + kBeW * double(ends) + (work ? kAnyW : 0.0));
    if (std::getenv("GSS_TILE_DUMP")) {  // per-tile features for the cost-model fit
      int ev = 0, wmax = 0;
      for (int r = 0; r < kTileRows; ++r) ev += (E->h_code[size_t(t) * kTileRows + r] & kCodeEvent) != 0;
      for (int gw = 0; gw < 4; ++gw) {
        int c = 0;
        for (int pp = 2 * gw; pp < 2 * gw + 2; ++pp) {
          int a = 0;
          for (int r = 0; r < 256; ++r)
            a |= (E->h_code[size_t(t) * kTileRows + pp * 256 + r] & kCodeCount) != 0;
          c += a;
        }
        wmax = std::max(wmax, c);
      }
      std::fprintf(stderr, "tile %d work %d ends %d events %d wmax %d\n", t, work, ends, ev, wmax);
    }
  }
  double tot = 0.0;
  for (double x : w) tot += x;
  std::vector<int32_t> t0(static_cast<size_t>(grid) + 1, 0);
  static const bool greedy = std::getenv("GSS_PART_GREEDY") != nullptr;
  if (!greedy && nt > grid) {
    // Min-max contiguous partition: the smallest bound B (bisected in
    // [tot/grid, tot/grid + max w], where greedy filling needs <= grid ranges)
    // under which greedy filling fits the grid, then the heaviest multi-tile
    // ranges are halved until there are exactly `grid`.  A share-crossing cut
    // leaves a CTA up to one whole tile above the mean; this bounds the
    // heaviest CTA by the optimum instead.
    double wmax = 0.0;
    for (double x : w) wmax = std::max(wmax, x);
    auto fill = [&](double B, std::vector<int32_t>* cuts) {
      int cnt = 1;
      double a = 0.0;
      if (cuts) cuts->assign(1, 0);
      for (int t = 0; t < nt; ++t) {
        if (a > 0.0 && a + w[t] > B) {
          ++cnt;
          a = 0.0;
          if (cuts) cuts->push_back(t);
        }
        a += w[t];
      }
      if (cuts) cuts->push_back(nt);
      return cnt;
    };
    double lo = tot / grid, hi = tot / grid + wmax;
    for (int it = 0; it < 60; ++it) {
      const double mid = 0.5 * (lo + hi);
      (fill(mid, nullptr) <= grid ? hi : lo) = mid;
    }
    std::vector<int32_t> cuts;
    fill(hi, &cuts);
    while (static_cast<int>(cuts.size()) - 1 < grid) {
      int best = -1;
      double bw = -1.0;
      for (size_t k = 0; k + 1 < cuts.size(); ++k) {
        if (cuts[k + 1] - cuts[k] < 2) continue;
        double wk = 0.0;
        for (int t = cuts[k]; t < cuts[k + 1]; ++t) wk += w[t];
        if (wk > bw) bw = wk, best = static_cast<int>(k);
      }
      double a = 0.0;
      int m = cuts[best] + 1;
      for (int t = cuts[best]; t < cuts[best + 1] - 1; ++t) {
        a += w[t];
        m = t + 1;
        if (a >= 0.5 * bw) break;
      }
      cuts.insert(cuts.begin() + best + 1, m);
    }
    t0.assign(cuts.begin(), cuts.end());
  } else {
    double acc = 0.0;
    int c = 1;
    for (int t = 0; t < nt && c < grid; ++t) {
      acc += w[t];
      // cut after tile t once CTA c-1 holds its share (every CTA keeps >= 1 tile)
      while (c < grid && acc >= tot * c / grid && t + 1 <= nt - (grid - c)) {
        t0[c] = t + 1;
        ++c;
      }
    }
    for (; c < grid; ++c) t0[c] = std::max(t0[c - 1] + 1, nt - (grid - c));
    t0[grid] = nt;
    for (int k = 1; k <= grid; ++k)
      if (t0[k] <= t0[k - 1]) t0[k] = t0[k - 1] + 1;  // never empty
  }
  if (std::getenv("GSS_VERBOSE")) {
    for (int k = 0; k < grid; ++k) {
      double wk = 0.0;
      for (int t = t0[k]; t < t0[k + 1]; ++t) wk += w[t];
      std::fprintf(stderr, "cta %d tiles [%d,%d) n=%d cost %.2f\n", k, t0[k], t0[k + 1],
                   t0[k + 1] - t0[k], wk);
    }
  }
  GSS_CUDA(cudaMemcpy(E->cta_tile0, t0.data(), (grid + 1) * sizeof(int32_t),
                      cudaMemcpyHostToDevice));
  E->grid = grid;
  E->prm.grid = grid;
  E->prm.cta_tile0 = E->cta_tile0;
  // per-tile records / carries of the previous partition are stale
  E->h_ctl->rec_valid = 0;
  return GSS_OK;
}

}  // namespace

extern "C" {

const char* gss_last_error(void) { return g_last_error.c_str(); }

const char* gss_version(void) {
  return "gss 0.2.0 (sm_100a; persistent cycle kernel; tile=2048 rows; fp64)";
}

int gss_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int gss_dataset_pack(const gss_host_dataset* h, int device, gss_dataset** out) {
  Nvtx nvtx_("gss_dataset_pack");
  if (!h || !out) return fail(GSS_ERR_DOMAIN, "null argument");
  *out = nullptr;
  if (h->n < 0 || h->p < 0) return fail(GSS_ERR_DOMAIN, "negative dimensions");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(GSS_ERR_NO_DEVICE, "no CUDA device available");
  if (device < 0 || device >= ndev) return fail(GSS_ERR_NO_DEVICE, "bad device index");
  GSS_CUDA(cudaSetDevice(device));
  const int64_t n = h->n, p = h->p;
  const int64_t nnz = p > 0 ? h->col_ptr[p] : 0;
  // GSS_PACK_TIMING: per-phase wall times (stream synchronised at each mark)
  const bool ptime = std::getenv("GSS_PACK_TIMING") != nullptr;
  auto tp = std::chrono::steady_clock::now();
  cudaStream_t* ps = nullptr;
  auto mark = [&](const char* what) {
    if (!ptime) return;
    if (ps) cudaStreamSynchronize(*ps);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "pack %-22s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - tp).count());
    tp = now;
  };
  // validate the layout contract (sorted rows, ascending CSC indices); the
  // first failing row decides the message, as in a serial pass
  {
    std::vector<int64_t> bad_row(16, -1);
    std::vector<int> bad_code(16, 0);
    host_parallel(n, [&](int c, int64_t lo, int64_t hi) {
      for (int64_t i = lo; i < hi; ++i) {
        int code = 0;
        if (!std::isfinite(h->times[i]) || h->times[i] < 0.0) code = 1;
        else if (h->status[i] < 0 || h->status[i] > 2) code = 2;
        else if (i > 0 && !(h->stratum_start && h->stratum_start[i]) && h->times[i] > h->times[i - 1])
          code = 3;
        if (code) {
          bad_row[c] = i;
          bad_code[c] = code;
          return;
        }
      }
    });
    for (int c = 0; c < 16; ++c) {
      if (bad_row[c] < 0) continue;
      if (bad_code[c] == 1) return fail(GSS_ERR_DOMAIN, "observation time must be finite and >= 0");
      if (bad_code[c] == 2) return fail(GSS_ERR_DOMAIN, "status must be 0, 1 or 2");
      return fail(GSS_ERR_DOMAIN, "rows must be sorted by decreasing time within a stratum");
    }
  }
  if (p > 0 && h->col_ptr[0] != 0) return fail(GSS_ERR_DOMAIN, "col_ptr[0] must be 0");
  auto* ds = new gss_dataset();
  ds->device = device;
  ds->n = n;
  ds->p = p;
  ds->nnz = nnz;
  ds->times.resize(static_cast<size_t>(n));
  ds->status.resize(static_cast<size_t>(n));
  // stratum-aligned device layout
  ds->stratum_of.resize(static_cast<size_t>(n));
  ds->dev_row.resize(static_cast<size_t>(n));
  {
    int64_t pos = 0;
    if (!h->stratum_start) {  // one stratum: device position = sorted row
      host_parallel(n, [&](int, int64_t lo, int64_t hi) {
        std::memcpy(ds->times.data() + lo, h->times + lo, (hi - lo) * sizeof(double));
        std::memcpy(ds->status.data() + lo, h->status + lo, (hi - lo) * sizeof(int32_t));
        for (int64_t i = lo; i < hi; ++i) {
          ds->stratum_of[i] = 0;
          ds->dev_row[i] = i;
        }
      });
      pos = n;
    } else {
      host_parallel(n, [&](int, int64_t lo, int64_t hi) {
        std::memcpy(ds->times.data() + lo, h->times + lo, (hi - lo) * sizeof(double));
        std::memcpy(ds->status.data() + lo, h->status + lo, (hi - lo) * sizeof(int32_t));
      });
      int64_t stratum = -1;
      for (int64_t i = 0; i < n; ++i) {
        if (i == 0 || h->stratum_start[i]) {
          ++stratum;
          pos = (pos + kTileRows - 1) / kTileRows * kTileRows;  // next tile boundary
        }
        ds->stratum_of[i] = stratum;
        ds->dev_row[i] = pos++;
      }
    }
    // positions rise by >= 1 per row, so the map is the identity iff the last row is
    ds->identity_rows = n == 0 || ds->dev_row[n - 1] == n - 1;
    int64_t npad = (pos + kTileRows - 1) / kTileRows * kTileRows;
    if (npad == 0) npad = kTileRows;
    if (npad >= (int64_t(1) << 31) - kTileRows) {
      delete ds;
      return fail(GSS_ERR_DOMAIN, "dataset too large for 32-bit row positions");
    }
    if (npad > 4 * n + 64 * int64_t(kTileRows)) {
      delete ds;
      return fail(GSS_ERR_DOMAIN, "too many small strata for the tile-aligned device layout");
    }
    ds->npad = npad;
    ds->ntiles = static_cast<int>(npad / kTileRows);
    ds->h_tile_first.assign(static_cast<size_t>(ds->ntiles), 0);
    // row 0 starts a stratum unless the caller marks it as continuing one from
    // a previous patient shard (stratum_start[0] == 0)
    ds->h_tile_first[0] = (h->stratum_start && n > 0) ? (h->stratum_start[0] ? 1 : 0) : 1;
    if (h->stratum_start)
      for (int64_t i = 1; i < n; ++i)
        if (ds->stratum_of[i] != ds->stratum_of[i - 1])
          ds->h_tile_first[ds->dev_row[i] / kTileRows] = 1;
  }
  ds->h_col_ptr.assign(h->col_ptr, h->col_ptr + p + 1);
  if (p == 0) ds->h_col_ptr.assign(1, 0);
  // indicator flags: given, or all-ones & density < 25% (src/dataset.cpp:126-157)
  std::vector<uint8_t> ind(static_cast<size_t>(p), 1);
  bool any_valued = false;
  for (int64_t j = 0; j < p; ++j) {
    if (h->col_indicator) {
      ind[j] = h->col_indicator[j] ? 1 : 0;
    } else if (h->vals) {
      const int64_t cnt = h->col_ptr[j + 1] - h->col_ptr[j];
      bool ones = true;
      for (int64_t k = h->col_ptr[j]; k < h->col_ptr[j + 1] && ones; ++k) ones = h->vals[k] == 1.0;
      const double dens = n ? double(cnt) / double(n) : 0.0;
      ind[j] = (ones && dens < 0.25) ? 1 : 0;
    }
    if (!ind[j]) any_valued = true;
  }
  ds->has_vals = h->vals != nullptr && any_valued;
  mark("host layout");
  cudaStream_t s;
  GSS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  ps = &s;
  auto cleanup = [&](int rc) {
    cudaStreamDestroy(s);
    if (rc != GSS_OK) delete ds;
    return rc;
  };
#define PK(call)                                                                        \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess)                                                              \
      return cleanup(fail(_e == cudaErrorMemoryAllocation ? GSS_ERR_OOM : GSS_ERR_CUDA, \
                          std::string("CUDA error in pack: ") + cudaGetErrorString(_e))); \
  } while (0)
  const int64_t npad = ds->npad;
  PK(dalloc(&ds->col_ptr, p + 1));
  PK(dalloc(&ds->row_idx, nnz + 4));
  PK(dalloc(&ds->col_ind, p));
  PK(dalloc(&ds->tile_ptr, p * (ds->ntiles + 1)));
  PK(dalloc(&ds->colmax, p));
  PK(dalloc(&ds->tile_first, ds->ntiles));
  if (ds->has_vals) {
    PK(dalloc(&ds->vals, nnz + 4));
  }
  ds->bytes = (p + 1) * 8 + (nnz + 4) * 8 + p + int64_t(p) * (ds->ntiles + 1) * 4 +
              (npad + 1) * 8 + p * 8 + ds->ntiles + (ds->has_vals ? (nnz + 4) * 16 : 0);
  mark("alloc");
  PK(cudaMemcpyAsync(ds->col_ptr, ds->h_col_ptr.data(), (p + 1) * sizeof(int64_t),
                     cudaMemcpyHostToDevice, s));
  PK(cudaMemsetAsync(ds->row_idx, 0, (nnz + 4) * sizeof(int32_t), s));
  if (nnz)
    PK(cudaMemcpyAsync(ds->row_idx, h->row_idx, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  if (p) PK(cudaMemcpyAsync(ds->col_ind, ind.data(), p, cudaMemcpyHostToDevice, s));
  if (ds->has_vals && nnz)
    PK(cudaMemcpyAsync(ds->vals, h->vals, nnz * sizeof(double), cudaMemcpyHostToDevice, s));
  PK(cudaMemcpyAsync(ds->tile_first, ds->h_tile_first.data(), ds->ntiles, cudaMemcpyHostToDevice,
                     s));
  mark("h2d");
  {
    Nvtx nv("pack: validate csc");
    int* bad = nullptr;
    PK(dalloc(&bad, 1));
    PK(cudaMemsetAsync(bad, 0, sizeof(int), s));
    PK(launch_validate_csc(ds->col_ptr, ds->row_idx, p, n, bad, s));
    int hb = 0;
    PK(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    PK(cudaStreamSynchronize(s));
    cudaFree(bad);
    if (hb & 2) return cleanup(fail(GSS_ERR_INDEX, "row index outside [0, n)"));
    if (hb) return cleanup(fail(GSS_ERR_DOMAIN, "CSC columns must have monotone col_ptr and "
                                                "strictly ascending row indices"));
  }
  mark("validate csc");
  if (!ds->identity_rows) {  // remap to the stratum-aligned positions (order preserving)
    int64_t* drow = nullptr;
    PK(dalloc(&drow, std::max<int64_t>(n, 1)));
    if (n)
      PK(cudaMemcpyAsync(drow, ds->dev_row.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    PK(launch_remap_rows(ds->row_idx, nnz, drow, s));
    PK(cudaStreamSynchronize(s));
    cudaFree(drow);
  }
  mark("remap");
  if (p) {
    Nvtx nv("pack: tile pointers + colmax");
    PK(launch_build_tile_ptr(ds->col_ptr, ds->row_idx, p, ds->ntiles, ds->tile_ptr, s));
    PK(launch_colmax(ds->col_ptr, ds->has_vals ? ds->vals : nullptr, p, ds->colmax, s));
  }
  // Dense columns (density >= 25%: the reference stores them as dense arrays,
  // SparseColumn::make src/dataset.cpp:126-157): values by device position in
  // a pool the cycle kernel reads row-wise instead of their tile index lists.
  mark("tile ptr + colmax");
  if (p) {
    Nvtx nv("pack: dense columns");
    std::vector<int32_t> slot(static_cast<size_t>(p), -1);
    for (int64_t j = 0; j < p; ++j) {
      const int64_t cnt = ds->h_col_ptr[j + 1] - ds->h_col_ptr[j];
      if (n && double(cnt) / double(n) >= 0.25) slot[j] = static_cast<int32_t>(ds->ndense++);
    }
    PK(dalloc(&ds->dense_idx, p));
    PK(cudaMemcpyAsync(ds->dense_idx, slot.data(), p * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    if (ds->ndense) {
      PK(dalloc(&ds->dense_pool, ds->ndense * npad));
      PK(cudaMemsetAsync(ds->dense_pool, 0, ds->ndense * npad * sizeof(double), s));
      PK(launch_fill_dense(ds->col_ptr, ds->row_idx, ds->has_vals ? ds->vals : nullptr,
                           ds->dense_idx, p, npad, ds->dense_pool, s));
      ds->bytes += ds->ndense * npad * 8;
    }
    ds->bytes += p * 4;
  }
  mark("dense");
#undef PK
  *out = ds;
  return cleanup(GSS_OK);
}

namespace {
// CSR transpose over device positions (count -> exclusive scan -> fill ->
// per-row sort), built on the first load_beta: the row-wise η = Xβ is its only
// reader, so a fit from β = 0 never pays for it.
int ensure_csr(gss_dataset* ds) {
  std::lock_guard<std::mutex> lk(ds->csr_mu);
  if (ds->csr_built) return GSS_OK;
  Nvtx nv("csr transpose");
  GSS_CUDA(cudaSetDevice(ds->device));
  const int64_t npad = ds->npad, nnz = ds->nnz, p = ds->p;
  struct Res {
    cudaStream_t s = nullptr;
    int64_t* cnt = nullptr;
    ~Res() {
      if (cnt) cudaFree(cnt);
      if (s) cudaStreamDestroy(s);
    }
  } r;
  GSS_CUDA(cudaStreamCreateWithFlags(&r.s, cudaStreamNonBlocking));
  if (!ds->row_ptr) GSS_CUDA(dalloc(&ds->row_ptr, npad + 1));
  if (!ds->csr_col) GSS_CUDA(dalloc(&ds->csr_col, nnz + 4));
  if (ds->has_vals && !ds->csr_val) GSS_CUDA(dalloc(&ds->csr_val, nnz + 4));
  GSS_CUDA(dalloc(&r.cnt, npad + 1));
  GSS_CUDA(cudaMemsetAsync(r.cnt, 0, (npad + 1) * sizeof(int64_t), r.s));
  GSS_CUDA(launch_csr_count(ds->row_idx, nnz, r.cnt, r.s));
  GSS_CUDA(launch_exclusive_scan(r.cnt, ds->row_ptr, npad + 1, r.s));
  GSS_CUDA(cudaMemcpyAsync(r.cnt, ds->row_ptr, (npad + 1) * sizeof(int64_t),
                           cudaMemcpyDeviceToDevice, r.s));
  GSS_CUDA(launch_csr_fill(ds->col_ptr, ds->row_idx, ds->has_vals ? ds->vals : nullptr, p, r.cnt,
                           ds->csr_col, ds->has_vals ? ds->csr_val : nullptr, r.s));
  GSS_CUDA(launch_csr_sort_rows(ds->row_ptr, npad, ds->csr_col,
                                ds->has_vals ? ds->csr_val : nullptr, r.s));
  GSS_CUDA(cudaStreamSynchronize(r.s));
  ds->csr_built = true;
  return GSS_OK;
}
}  // namespace

void gss_dataset_release(gss_dataset* ds) {
  if (ds && --ds->refs == 0) delete ds;
}

int64_t gss_dataset_device_bytes(const gss_dataset* ds) { return ds ? ds->bytes : 0; }

int gss_engine_create(gss_dataset* ds, int model, int64_t recompute_interval,
                      const uint8_t* row_mask, gss_engine** out) {
  Nvtx nvtx_("gss_engine_create");
  if (!ds || !out) return fail(GSS_ERR_DOMAIN, "null argument");
  *out = nullptr;
  if (recompute_interval < 1) return fail(GSS_ERR_DOMAIN, "recompute_interval must be at least 1");
  if (model != GSS_COX && model != GSS_FINE_GRAY) return fail(GSS_ERR_DOMAIN, "unknown model");
  bool competing = false;
  for (int64_t i = 0; i < ds->n; ++i)
    if (ds->status[i] == 2 && (!row_mask || row_mask[i])) competing = true;
  if (model == GSS_COX && competing)
    return fail(GSS_ERR_DOMAIN,
                "cox model cannot ingest competing-event rows; fit fine_gray instead");
  GSS_CUDA(cudaSetDevice(ds->device));
  auto* E = new gss_engine();
  ++ds->refs;
  E->ds = ds;
  E->model = model;
  E->interval = recompute_interval;
  E->weighted = model == GSS_FINE_GRAY && competing;  // src/engine.cpp:237
  {
    int rc = build_codes(ds, row_mask, E->h_code);
    if (rc) {
      delete E;
      return rc;
    }
  }
  if (E->weighted) {
    int rc = build_ipcw_host(ds, row_mask, E->h_u, E->h_g);
    if (rc) {
      delete E;
      return rc;
    }
  }
  const int64_t n = ds->n, p = ds->p, npad = ds->npad;
  const int nt = ds->ntiles;
  auto bail = [&](int rc) {
    delete E;
    return rc;
  };
#define EK(call)                                                                        \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess)                                                              \
      return bail(fail(_e == cudaErrorMemoryAllocation ? GSS_ERR_OOM : GSS_ERR_CUDA,    \
                       std::string("CUDA error in engine_create: ") + cudaGetErrorString(_e))); \
  } while (0)
  int maxg = cycle_max_grid(ds->device, E->weighted);
  if (maxg < 1) return bail(fail(GSS_ERR_CUDA, "cycle kernel cannot be resident on this device"));
  E->grid = std::max(1, std::min(nt, maxg));  // payload buffers sized for the largest grid
  EK(cudaStreamCreateWithFlags(&E->stream, cudaStreamNonBlocking));
  EK(cudaEventCreate(&E->ev0));
  EK(cudaEventCreate(&E->ev1));
  EK(ealloc(&E->eta, npad, E->stream));
  EK(ealloc(&E->e, npad, E->stream));
  EK(ealloc(&E->scratch, npad, E->stream));
  EK(ealloc(&E->code, npad, E->stream));
  EK(ealloc(&E->beta, p, E->stream));
  EK(ealloc(&E->halfwidth, p, E->stream));
  EK(ealloc(&E->fixed, p, E->stream));
  EK(ealloc(&E->penalized, p, E->stream));
  EK(ealloc(&E->trec, size_t(nt) * kRecStride, E->stream));
  EK(ealloc(&E->tcar, size_t(nt) * kCarStride, E->stream));
  EK(ealloc(&E->cpay, size_t(2) * E->grid * (kPayStride + kPayAux), E->stream));
  EK(ealloc(&E->slot_out, size_t(p + 1) * 4, E->stream));
  EK(ealloc(&E->slot_col, size_t(p + 1), E->stream));
  EK(ealloc(&E->bar, 1, E->stream));
  EK(ealloc(&E->ctl, 1, E->stream));
  EK(ealloc(&E->dflag, 4, E->stream));
  EK(ealloc(&E->ext, 8, E->stream));
  EK(ealloc(&E->shard, 8, E->stream));
  EK(cudaMemsetAsync(E->ext, 0, 8 * sizeof(double), E->stream));
  if (E->weighted) {
    EK(ealloc(&E->g, npad, E->stream));
    EK(ealloc(&E->gs, npad, E->stream));
  }
  EK(cudaMallocHost(reinterpret_cast<void**>(&E->h_ctl), sizeof(Ctl)));
  std::memset(E->h_ctl, 0, sizeof(Ctl));
  E->h_ctl->err_col = -1;
  E->h_ctl->rec_col = -2;
  cudaStream_t s = E->stream;
  EK(cudaMemsetAsync(E->bar, 0, sizeof(unsigned), s));
  EK(cudaMemsetAsync(E->trec, 0, size_t(nt) * kRecStride * sizeof(double), s));
  EK(cudaMemsetAsync(E->tcar, 0, size_t(nt) * kCarStride * sizeof(double), s));
  EK(cudaMemcpyAsync(E->code, E->h_code.data(), npad * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
  EK(cudaMemsetAsync(E->eta, 0, npad * sizeof(double), s));
  {
    EK(launch_init_e(E->code, npad, E->e, s));
    if (E->weighted) {
      std::vector<double> gd(static_cast<size_t>(npad), 1.0);
      for (int64_t i = 0; i < n; ++i) gd[ds->dev_row[i]] = E->h_g[i];
      EK(cudaMemcpyAsync(E->g, gd.data(), npad * sizeof(double), cudaMemcpyHostToDevice, s));
      // The streamed copy carries u = 1/G on competing rows (the reference's
      // 1.0 / before, src/censoring.cpp) and G elsewhere, so the scan does not
      // divide per row; the Breslow transform needs G at tied-block ends and
      // divides back there when the block-end row is competing.
      std::vector<double> gsd(gd);
      for (int64_t r = 0; r < npad; ++r)
        if (E->h_code[r] & kCodeCompeting) gsd[r] = 1.0 / gd[r];
      EK(cudaMemcpyAsync(E->gs, gsd.data(), npad * sizeof(double), cudaMemcpyHostToDevice, s));
      EK(cudaStreamSynchronize(s));
    } else {
      EK(cudaStreamSynchronize(s));
    }
  }
  EK(cudaMemsetAsync(E->beta, 0, std::max<int64_t>(p, 1) * sizeof(double), s));
  EK(cudaMemcpyAsync(E->ctl, E->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, s));
  EK(launch_fixed_terms(ds->col_ptr, ds->row_idx, ds->has_vals ? ds->vals : nullptr, ds->col_ind,
                        E->code, p, E->fixed, s));
  EK(cudaStreamSynchronize(s));
  E->h_beta.assign(static_cast<size_t>(p), 0.0);
  int rc = make_tile_map(&E->tm_e, E->e, npad, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8);
  if (rc) return bail(rc);
  rc = make_tile_map(&E->tm_code, E->code, npad, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4);
  if (rc) return bail(rc);
  if (E->weighted) {
    rc = make_tile_map(&E->tm_g, E->gs, npad, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8);
    if (rc) return bail(rc);
  } else {
    E->tm_g = E->tm_e;
  }
  CycleParams& P = E->prm;
  P.n = n;
  P.npad = npad;
  P.p = p;
  P.ntiles = nt;
  P.has_vals = ds->has_vals ? 1 : 0;
  P.col_ptr = ds->col_ptr;
  P.row_idx = ds->row_idx;
  P.vals = ds->vals;
  P.col_ind = ds->col_ind;
  P.tile_ptr = ds->tile_ptr;
  P.dense_idx = ds->ndense ? ds->dense_idx : nullptr;  // no dense column: no per-tile lookup
  P.dense_pool = ds->dense_pool;
  P.row_ptr = ds->row_ptr;
  P.csr_col = ds->csr_col;
  P.csr_val = ds->csr_val;
  P.colmax = ds->colmax;
  P.tile_first = ds->tile_first;
  P.eta = E->eta;
  P.e = E->e;
  P.code = E->code;
  P.g = E->g;
  P.beta = E->beta;
  P.halfwidth = E->halfwidth;
  P.penalized = E->penalized;
  P.fixed = E->fixed;
  P.weighted = E->weighted ? 1 : 0;
  P.pen_kind = 0;
  P.pen_strength = 0.0;
  P.recompute_interval = recompute_interval;
  P.grid = E->grid;
  {
    int mg = maxg;
    if (const char* cap = std::getenv("GSS_MAX_GRID")) {
      const int c = std::atoi(cap);
      if (c > 0) mg = std::min(mg, c);
    }
    EK(ealloc(&E->cta_tile0, maxg + 1, E->stream));
    E->max_grid = maxg;
    int rc2 = partition_ctas(E, std::max(1, std::min(nt, mg)));
    if (rc2) return bail(rc2);
  }
  P.trec = E->trec;
  P.tcar = E->tcar;
  P.cpay = E->cpay;
  P.bar = E->bar;
  P.ctl = E->ctl;
  if (const char* dbg = std::getenv("GSS_DEBUG")) P.dbg = std::atoi(dbg);
  if (const char* tr = std::getenv("GSS_TRACE")) {
    if (tr[0] == '1') {
      P.trace_cap = 32u << 16;  // 32 warps x 65536 events (CTA 0)
      EK(dalloc(&P.trace, size_t(P.trace_cap) * 2));
      EK(cudaMemset(P.trace, 0, size_t(P.trace_cap) * 16));
    }
  }
#undef EK
  *out = E;
  return GSS_OK;
}

void gss_engine_destroy(gss_engine* e) { delete e; }

int gss_engine_set_grid(gss_engine* E, int grid) {
  int rc = check_engine(E);
  if (rc) return rc;
  if (grid < 0) return fail(GSS_ERR_DOMAIN, "grid must be >= 0");
  rc = sync_ctl(E);
  if (rc) return rc;
  rc = partition_ctas(E, grid == 0 ? E->max_grid : grid);
  if (rc) return rc;
  return push_ctl(E);
}

int gss_engine_grid(gss_engine* E) { return E ? E->grid : 0; }

int gss_engine_load_beta(gss_engine* E, const double* beta, int64_t p) {
  Nvtx nvtx_("gss_engine_load_beta");
  int rc = check_engine(E);
  if (rc) return rc;
  if (p != E->ds->p)
    return fail(GSS_ERR_INVALID_COLUMN, "load_beta: expected " + std::to_string(E->ds->p) +
                                            " coefficients, got " + std::to_string(p));
  for (int64_t j = 0; j < p; ++j)
    if (!std::isfinite(beta[j])) return fail(GSS_ERR_DOMAIN, "load_beta: non-finite coefficient");
  double* dbeta = nullptr;
  GSS_CUDA(dalloc(&dbeta, p));
  cudaStream_t s = E->stream;
  if (p) GSS_CUDA(cudaMemcpyAsync(dbeta, beta, p * sizeof(double), cudaMemcpyHostToDevice, s));
  {
    int rc2 = sync_ctl(E);
    if (rc2) {
      cudaFree(dbeta);
      return rc2;
    }
  }
  // beta = 0 on indicator data (every fit's start, ccd.cpp:137): the row sums
  // are +0.0 + 0 * 1.0 + ... = +0.0 exactly, so eta is a memset and the CSR is
  // not needed.  Valued data keeps the product path (a non-finite value would
  // make 0 * x NaN there, as in the reference).
  bool zero = !E->ds->has_vals;
  for (int64_t j = 0; j < p && zero; ++j) zero = beta[j] == 0.0;
  GSS_CUDA(cudaMemsetAsync(E->dflag, 0, sizeof(int), s));
  if (zero) {
    GSS_CUDA(cudaMemsetAsync(E->scratch, 0, E->ds->npad * sizeof(double), s));
  } else {
    const int rc2 = ensure_csr(E->ds);
    if (rc2) {
      cudaFree(dbeta);
      return rc2;
    }
    GSS_CUDA(cudaSetDevice(E->ds->device));
    E->prm.row_ptr = E->ds->row_ptr;
    E->prm.csr_col = E->ds->csr_col;
    E->prm.csr_val = E->ds->csr_val;
    GSS_CUDA(launch_spmv_rows(E->prm, dbeta, E->scratch, E->dflag, s));
  }
  int over = 0;
  GSS_CUDA(cudaMemcpyAsync(&over, E->dflag, sizeof(int), cudaMemcpyDeviceToHost, s));
  GSS_CUDA(cudaStreamSynchronize(s));
  if (over) {
    cudaFree(dbeta);
    return fail(GSS_ERR_OVERFLOW, "load_beta: |x'beta| exceeds 700");
  }
  if (p) GSS_CUDA(cudaMemcpyAsync(E->beta, dbeta, p * sizeof(double), cudaMemcpyDeviceToDevice, s));
  E->h_ctl->rec_valid = 0;        // e rewritten outside the cycle kernel
  E->h_ctl->eta_absmax_bits = 0;  // fresh eta: the bound is rebuilt exactly by the commit
  E->h_ctl->bound_slack = 0.0;
  GSS_CUDA(cudaMemcpyAsync(E->ctl, E->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, s));
  GSS_CUDA(launch_commit_eta(E->prm, E->scratch, s));
  GSS_CUDA(cudaStreamSynchronize(s));
  cudaFree(dbeta);
  E->h_beta.assign(beta, beta + p);
  return sync_ctl(E);
}

int gss_engine_refresh(gss_engine* E) {
  int rc = check_engine(E);
  if (rc) return rc;
  std::vector<double> b = E->h_beta;
  rc = gss_engine_load_beta(E, b.data(), static_cast<int64_t>(b.size()));
  if (rc) return rc;
  rc = sync_ctl(E);
  if (rc) return rc;
  E->h_ctl->refreshes += 1;
  return push_ctl(E);
}

int gss_engine_update(gss_engine* E, int64_t column, double delta) {
  Nvtx nvtx_("gss_engine_update");
  int rc = check_engine(E);
  if (rc) return rc;
  if (column < 0 || column >= E->ds->p)
    return fail(GSS_ERR_INVALID_COLUMN, "update: column " + std::to_string(column) +
                                            " outside [0, " + std::to_string(E->ds->p) + ")");
  if (!std::isfinite(delta)) return fail(GSS_ERR_DOMAIN, "update: non-finite delta");
  if (delta == 0.0) return GSS_OK;
  cudaStream_t s = E->stream;
  GSS_CUDA(cudaMemsetAsync(E->dflag, 0, sizeof(int), s));
  GSS_CUDA(launch_update_check(E->prm, column, delta, E->dflag, s));
  int over = 0;
  GSS_CUDA(cudaMemcpyAsync(&over, E->dflag, sizeof(int), cudaMemcpyDeviceToHost, s));
  GSS_CUDA(cudaStreamSynchronize(s));
  if (over) return fail(GSS_ERR_OVERFLOW, "update: |x'beta| would exceed 700");
  GSS_CUDA(launch_update_commit(E->prm, column, delta, std::exp(delta), s));
  E->h_beta[column] += delta;
  GSS_CUDA(cudaMemcpyAsync(E->beta + column, &E->h_beta[column], sizeof(double),
                           cudaMemcpyHostToDevice, s));
  rc = sync_ctl(E);
  if (rc) return rc;
  E->h_ctl->accepted += 1;
  E->h_ctl->rec_valid = 0;  // e changed outside the cycle kernel
  const bool refresh = E->h_ctl->accepted % E->interval == 0;
  rc = push_ctl(E);
  if (rc) return rc;
  if (refresh) return gss_engine_refresh(E);
  return GSS_OK;
}

int gss_engine_grad_hessian(gss_engine* E, int64_t column, double* gradient, double* hessian,
                            double* fixed_term) {
  Nvtx nvtx_("gss_engine_grad_hessian");
  int rc = check_engine(E);
  if (rc) return rc;
  if (column < 0 || column >= E->ds->p)
    return fail(GSS_ERR_INVALID_COLUMN, "grad_hessian: column " + std::to_string(column) +
                                            " outside [0, " + std::to_string(E->ds->p) + ")");
  rc = run_slots(E, {static_cast<int32_t>(column)}, kModeApi, false);
  if (rc) return rc;
  rc = sync_ctl(E);
  if (rc) return rc;
  if (E->h_ctl->err_code) return device_error(E, "grad_hessian");
  if (gradient) *gradient = E->h_ctl->gradient;
  if (hessian) *hessian = E->h_ctl->hessian;
  if (fixed_term) *fixed_term = E->h_ctl->fixed_term;
  return GSS_OK;
}

int gss_engine_grad_hessian_separated(gss_engine* E, int64_t column, double* gradient,
                                      double* hessian, double* fixed_term) {
  int rc = check_engine(E);
  if (rc) return rc;
  if (column < 0 || column >= E->ds->p)
    return fail(GSS_ERR_INVALID_COLUMN, "grad_hessian: column " + std::to_string(column) +
                                            " outside [0, " + std::to_string(E->ds->p) + ")");
  cudaStream_t s = E->stream;
  const size_t nsep = separated_scratch_doubles(E->ds->npad, E->ds->ntiles);
  if (!E->sep) {
    cudaError_t err = dalloc(&E->sep, nsep);
    if (err != cudaSuccess) {
      E->sep = nullptr;
      return fail(err == cudaErrorMemoryAllocation ? GSS_ERR_OOM : GSS_ERR_CUDA,
                  std::string("separated path scratch: ") + cudaGetErrorString(err));
    }
  }
  GSS_CUDA(cudaMemsetAsync(E->dflag + 1, 0, sizeof(int), s));
  double* out2 = E->sep + nsep - 2;
  GSS_CUDA(launch_separated(E->prm, column, E->sep, E->dflag + 1, out2, s));
  double sums[2] = {0.0, 0.0}, fixed = 0.0;
  int bad = 0;
  GSS_CUDA(cudaMemcpyAsync(sums, out2, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  GSS_CUDA(cudaMemcpyAsync(&bad, E->dflag + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  GSS_CUDA(cudaMemcpyAsync(&fixed, E->fixed + column, sizeof(double), cudaMemcpyDeviceToHost, s));
  GSS_CUDA(cudaStreamSynchronize(s));
  if (bad)
    return fail(GSS_ERR_NONPOS_DEN, "separated path: accumulated risk-set denominator <= 0");
  // Engine::finish (src/engine.cpp:220-230)
  const double g = fixed - sums[0];
  double h = -sums[1];
  if (h > 0.0) h = 0.0;
  if (!std::isfinite(g) || !std::isfinite(h))
    return fail(GSS_ERR_NONPOS_DEN, "derivatives overflowed; risk-set sums are not finite");
  if (gradient) *gradient = g;
  if (hessian) *hessian = h;
  if (fixed_term) *fixed_term = fixed;
  return GSS_OK;
}

int gss_engine_log_likelihood(gss_engine* E, double* out) {
  Nvtx nvtx_("gss_engine_log_likelihood");
  int rc = check_engine(E);
  if (rc) return rc;
  rc = run_slots(E, {-1}, kModeApi, false);
  if (rc) return rc;
  rc = sync_ctl(E);
  if (rc) return rc;
  if (E->h_ctl->err_code) return device_error(E, "log-likelihood");
  *out = E->h_ctl->loglik;
  return GSS_OK;
}

int gss_engine_get_beta(gss_engine* E, double* out, int64_t p) {
  int rc = check_engine(E);
  if (rc) return rc;
  if (p != E->ds->p) return fail(GSS_ERR_INVALID_COLUMN, "get_beta: size mismatch");
  std::copy(E->h_beta.begin(), E->h_beta.end(), out);
  return GSS_OK;
}

static int get_rows(gss_engine* E, const double* src, double* out, int64_t n) {
  int rc = check_engine(E);
  if (rc) return rc;
  if (n != E->ds->n) return fail(GSS_ERR_DOMAIN, "row array size mismatch");
  std::vector<double> tmp(static_cast<size_t>(E->ds->npad));
  GSS_CUDA(cudaMemcpyAsync(tmp.data(), src, E->ds->npad * sizeof(double), cudaMemcpyDeviceToHost,
                           E->stream));
  GSS_CUDA(cudaStreamSynchronize(E->stream));
  for (int64_t i = 0; i < n; ++i) out[i] = tmp[E->ds->dev_row[i]];
  return GSS_OK;
}

int gss_engine_get_xbeta(gss_engine* E, double* out, int64_t n) { return get_rows(E, E->eta, out, n); }
int gss_engine_get_exp_xbeta(gss_engine* E, double* out, int64_t n) {
  return get_rows(E, E->e, out, n);
}

int gss_engine_get_fixed_terms(gss_engine* E, double* out, int64_t p) {
  int rc = check_engine(E);
  if (rc) return rc;
  if (p != E->ds->p) return fail(GSS_ERR_INVALID_COLUMN, "fixed terms: size mismatch");
  if (p) GSS_CUDA(cudaMemcpyAsync(out, E->fixed, p * sizeof(double), cudaMemcpyDeviceToHost, E->stream));
  GSS_CUDA(cudaStreamSynchronize(E->stream));
  return GSS_OK;
}

int gss_engine_set_fixed_terms(gss_engine* E, const double* in, int64_t p) {
  int rc = check_engine(E);
  if (rc) return rc;
  if (!in && p) return fail(GSS_ERR_DOMAIN, "null argument");
  if (p != E->ds->p) return fail(GSS_ERR_INVALID_COLUMN, "fixed terms: size mismatch");
  if (p) GSS_CUDA(cudaMemcpyAsync(E->fixed, in, p * sizeof(double), cudaMemcpyHostToDevice, E->stream));
  GSS_CUDA(cudaStreamSynchronize(E->stream));
  return GSS_OK;
}

// max |x| per column (the fast overflow bound): patient shards must share
// the global bound so every shard takes the same validate-before-mutate path
int gss_engine_get_colmax(gss_engine* E, double* out, int64_t p) {
  int rc = check_engine(E);
  if (rc) return rc;
  if (p != E->ds->p) return fail(GSS_ERR_INVALID_COLUMN, "colmax: size mismatch");
  if (p) GSS_CUDA(cudaMemcpy(out, E->ds->colmax, p * sizeof(double), cudaMemcpyDeviceToHost));
  return GSS_OK;
}

int gss_engine_set_colmax(gss_engine* E, const double* in, int64_t p) {
  int rc = check_engine(E);
  if (rc) return rc;
  if (!in && p) return fail(GSS_ERR_DOMAIN, "null argument");
  if (p != E->ds->p) return fail(GSS_ERR_INVALID_COLUMN, "colmax: size mismatch");
  if (p) GSS_CUDA(cudaMemcpy(E->ds->colmax, in, p * sizeof(double), cudaMemcpyHostToDevice));
  return GSS_OK;
}

int gss_engine_get_ipcw(gss_engine* E, double* u, double* g, int64_t n) {
  int rc = check_engine(E);
  if (rc) return rc;
  if (n != E->ds->n) return fail(GSS_ERR_DOMAIN, "ipcw: size mismatch");
  for (int64_t i = 0; i < n; ++i) {
    u[i] = E->h_u.empty() ? 0.0 : E->h_u[i];
    g[i] = E->h_g.empty() ? 1.0 : E->h_g[i];
  }
  return GSS_OK;
}

int gss_sharded_fit_local(gss_engine* const* shards, int count, const gss_penalty_spec* pen,
                          const gss_fit_config* cfg, double* beta_out, gss_fit_result* res,
                          double* device_seconds) {
  Nvtx nvtx_("gss_sharded_fit_local");
  if (!shards || count < 1 || !pen || !cfg || !res) return fail(GSS_ERR_DOMAIN, "null argument");
  for (int r = 0; r < count; ++r) {
    if (!shards[r] || shards[r]->prm.nranks != count || shards[r]->prm.rank != r)
      return fail(GSS_ERR_DOMAIN, "gss_sharded_fit_local: shard r must carry rank r of a local comm");
    if (shards[r]->ds->device != shards[0]->ds->device)
      return fail(GSS_ERR_DOMAIN, "gss_sharded_fit_local: shards must share one device "
                                  "(one process per GPU uses gss_engine_fit)");
  }
  if (count > kMaxBatch || count > shards[0]->max_grid)
    return fail(GSS_ERR_DOMAIN, "gss_sharded_fit_local: too many shards for one launch");
  // all shards in ONE batched launch per cycle (their kernels wait on each
  // other's exchange rows, so they must be co-resident)
  std::vector<gss_penalty_spec> pens(static_cast<size_t>(count), *pen);
  std::vector<gss_fit_result> rs(static_cast<size_t>(count));
  std::vector<int32_t> st(static_cast<size_t>(count));
  const int64_t p = shards[0]->ds->p;
  std::vector<double> betas(static_cast<size_t>(count * p));
  const int rc = gss_fit_batch(shards, count, pens.data(), cfg, count, betas.data(), rs.data(),
                               st.data(), device_seconds);
  if (rc) return rc;
  *res = rs[0];
  if (beta_out) std::copy(betas.begin(), betas.begin() + p, beta_out);
  return GSS_OK;
}

int gss_engine_counters(gss_engine* E, int64_t* accepted, int64_t* refreshes) {
  int rc = check_engine(E);
  if (rc) return rc;
  rc = sync_ctl(E);
  if (rc) return rc;
  if (accepted) *accepted = E->h_ctl->accepted;
  if (refreshes) *refreshes = E->h_ctl->refreshes;
  return GSS_OK;
}

}  // extern "C"

namespace {

// fit_with_engine (src/ccd.cpp:131-184) in three phases, so that one engine
// (gss_engine_fit) or many (gss_fit_batch: one launch per cycle for all of
// them) share the same per-fit host logic.
int fit_begin(gss_engine* E, const gss_penalty_spec* pen, const gss_fit_config* cfg) {
  int rc = check_engine(E);
  if (rc) return rc;
  if (!pen || !cfg) return fail(GSS_ERR_DOMAIN, "null argument");
  auto& F = E->fs;
  F = gss_engine::FitState{};
  F.t0 = std::chrono::steady_clock::now();
  const int64_t p = E->ds->p;
  // PenaltySpec::validate / FitConfig::validate (src/ccd.cpp:37-69)
  if (pen->kind < 0 || pen->kind > 2) return fail(GSS_ERR_DOMAIN, "unknown penalty");
  if (pen->kind == GSS_PEN_L1 && (!std::isfinite(pen->strength) || pen->strength < 0.0))
    return fail(GSS_ERR_DOMAIN, "l1 strength must be finite and >= 0");
  if (pen->kind == GSS_PEN_L2 && (!std::isfinite(pen->strength) || pen->strength <= 0.0))
    return fail(GSS_ERR_DOMAIN, "l2 strength must be finite and > 0");
  if (!std::isfinite(cfg->tolerance) || cfg->tolerance <= 0.0)
    return fail(GSS_ERR_DOMAIN, "tolerance must be > 0");
  if (cfg->max_cycles < 1) return fail(GSS_ERR_DOMAIN, "max_cycles must be >= 1");
  if (!std::isfinite(cfg->trust_init) || cfg->trust_init <= 0.0)
    return fail(GSS_ERR_DOMAIN, "trust_init must be > 0");
  F.pen = *pen;
  if (pen->exempt) {
    F.exempt.assign(pen->exempt, pen->exempt + p);
    F.pen.exempt = F.exempt.data();
  }
  F.cfg = *cfg;
  F.trace.assign(static_cast<size_t>(cfg->max_cycles) + 1, 0.0);
  std::vector<double> zero(static_cast<size_t>(p), 0.0);
  rc = gss_engine_load_beta(E, zero.data(), p);  // ccd.cpp:137
  if (rc) return rc;
  cudaStream_t s = E->stream;
  {
    std::vector<double> hw(static_cast<size_t>(p), cfg->trust_init);
    std::vector<uint8_t> pz(static_cast<size_t>(p), 0);
    for (int64_t j = 0; j < p; ++j)
      pz[j] = (pen->kind != GSS_PEN_NONE && !(pen->exempt && pen->exempt[j])) ? 1 : 0;
    if (p) {
      GSS_CUDA(cudaMemcpyAsync(E->halfwidth, hw.data(), p * sizeof(double), cudaMemcpyHostToDevice, s));
      GSS_CUDA(cudaMemcpyAsync(E->penalized, pz.data(), p, cudaMemcpyHostToDevice, s));
    }
    GSS_CUDA(cudaStreamSynchronize(s));
  }
  E->prm.pen_kind = pen->kind;
  E->prm.pen_strength = pen->strength;
  rc = sync_ctl(E);
  if (rc) return rc;
  E->h_ctl->skipped = 0;
  E->h_ctl->err_code = 0;
  E->h_ctl->err_col = -1;
  rc = push_ctl(E);
  if (rc) return rc;
  if (E->prm.nranks > 1) {
    // patient shard: the objective at beta = 0 needs every shard's carries;
    // it is a CCD launch of the objective slot alone, made by all shards
    // together (init_objective) before the first cycle
    F.need_init_obj = true;
  } else {
    double ll = 0.0;
    rc = gss_engine_log_likelihood(E, &ll);
    if (rc) return rc;
    F.prev = ll - penalty_value(&F.pen, E->h_beta);
    F.trace[0] = F.prev;
  }
  F.converged = p == 0;
  F.done = F.converged;
  E->cycle_ms.clear();
  E->cycle_accepted.clear();
  // one cycle = p coordinate slots + the objective slot
  std::vector<int32_t> slots(static_cast<size_t>(p + 1));
  for (int64_t j = 0; j < p; ++j) slots[j] = static_cast<int32_t>(j);
  slots[p] = -1;
  E->h_slots = slots;
  GSS_CUDA(cudaMemcpyAsync(E->slot_col, slots.data(), slots.size() * sizeof(int32_t),
                           cudaMemcpyHostToDevice, s));
  GSS_CUDA(cudaStreamSynchronize(s));
  return GSS_OK;
}

// parameters of one CCD-cycle launch of E (slots staged by fit_begin)
CycleParams cycle_params(const gss_engine* E) {
  CycleParams P = E->prm;
  P.slot_col = E->slot_col;
  P.nslots = static_cast<int>(E->h_slots.size());
  P.mode = kModeCcd;
  P.slot_out = nullptr;
  P.ext = nullptr;
  P.shard_out = nullptr;
  P.prologue_only = 0;
  P.reuse_records = 0;
  return P;
}

// after a cycle launch of E completed (stream synchronised by the caller)
// The objective at beta = 0 of sharded engines (need_init_obj): one launch of
// the objective slot in CCD mode (the cross-shard exchange runs), for all the
// given shards together (a batched launch: they must be co-resident).
int init_objective(gss_engine* const* es, int count) {
  std::vector<CycleParams> prm(static_cast<size_t>(count));
  std::vector<BatchEntry> ent(static_cast<size_t>(count));
  for (int a = 0; a < count; ++a) {
    gss_engine* E = es[a];
    prm[a] = cycle_params(E);
    prm[a].slot_col = E->slot_col + E->ds->p;  // the cycle's last slot: -1 (objective)
    prm[a].nslots = 1;
    ent[a] = BatchEntry{&E->tm_e, &E->tm_code, &E->tm_g, &prm[a]};
  }
  GSS_CUDA(count == 1 ? launch_cycle(ent[0].tm_e, ent[0].tm_code, ent[0].tm_g, prm[0], es[0]->stream)
                      : launch_cycle_batch(ent.data(), count, es[0]->stream));
  GSS_CUDA(cudaStreamSynchronize(es[0]->stream));
  for (int a = 0; a < count; ++a) {
    gss_engine* E = es[a];
    if (int rc = sync_ctl(E)) return rc;
    if (E->h_ctl->err_code) return device_error(E, "fit");
    E->fs.prev = E->h_ctl->loglik - penalty_value(&E->fs.pen, E->h_beta);
    E->fs.trace[0] = E->fs.prev;
    E->fs.need_init_obj = false;
  }
  return GSS_OK;
}

int fit_after_cycle(gss_engine* E, double ms) {
  auto& F = E->fs;
  const int64_t p = E->ds->p;
  int rc = sync_ctl(E);
  if (rc) return F.err = rc;
  ++F.cycle;
  F.dev_ms += ms;
  E->cycle_ms.push_back(ms);
  E->cycle_accepted.push_back(E->h_ctl->accepted);
  if (p) GSS_CUDA(cudaMemcpy(E->h_beta.data(), E->beta, p * sizeof(double), cudaMemcpyDeviceToHost));
  if (E->h_ctl->err_code) {
    F.err = device_error(E, "fit");
    F.done = true;
    return F.err;
  }
  F.res.cycles = F.cycle;
  const double obj = E->h_ctl->loglik - penalty_value(&F.pen, E->h_beta);
  F.trace[F.cycle] = obj;
  if (obj < F.prev - 1e-10) ++F.res.monotonicity_violations;
  if (std::abs(obj - F.prev) / std::max(1.0, std::abs(obj)) < F.cfg.tolerance) F.converged = true;
  F.prev = obj;
  if (F.converged || F.cycle >= F.cfg.max_cycles) F.done = true;
  return GSS_OK;
}

int fit_end(gss_engine* E, double* beta_out, double* trace_out, gss_fit_result* res) {
  auto& F = E->fs;
  E->last_ms = F.dev_ms;
  E->last_launches = F.res.cycles;
  if (F.err) return F.err;
  F.res.converged = F.converged ? 1 : 0;
  F.res.objective = F.prev;
  F.res.skipped_steps = E->h_ctl->skipped;
  F.res.nonzero_count = 0;
  const int64_t p = E->ds->p;
  for (int64_t j = 0; j < p; ++j) F.res.nonzero_count += E->h_beta[j] != 0.0;
  if (beta_out) std::copy(E->h_beta.begin(), E->h_beta.end(), beta_out);
  if (trace_out) std::copy(F.trace.begin(), F.trace.begin() + F.cycle + 1, trace_out);
  F.res.device_seconds = F.dev_ms * 1e-3;
  F.res.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - F.t0).count();
  *res = F.res;
  return GSS_OK;
}

}  // namespace

extern "C" {

int gss_engine_fit(gss_engine* E, const gss_penalty_spec* pen, const gss_fit_config* cfg,
                   double* beta_out, double* trace_out, gss_fit_result* res) {
  Nvtx nvtx_("gss_engine_fit");
  if (!res) return fail(GSS_ERR_DOMAIN, "null argument");
  *res = gss_fit_result{};
  int rc = fit_begin(E, pen, cfg);
  if (rc) return rc;
  if (E->fs.need_init_obj) {  // one process per GPU: every rank makes this launch
    rc = init_objective(&E, 1);
    if (rc) return rc;
  }
  cudaStream_t s = E->stream;
  while (!E->fs.done) {
    Nvtx nvtx_cycle("ccd cycle %lld", static_cast<long long>(E->fs.cycle + 1));
    const CycleParams P = cycle_params(E);
    cudaEventRecord(E->ev0, s);
    GSS_CUDA(launch_cycle(&E->tm_e, &E->tm_code, &E->tm_g, P, s));
    cudaEventRecord(E->ev1, s);
    GSS_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, E->ev0, E->ev1);
    if (fit_after_cycle(E, ms)) break;
  }
  return fit_end(E, beta_out, trace_out, res);
}

int gss_fit_batch(gss_engine* const* engines, int64_t count, const gss_penalty_spec* pens,
                  const gss_fit_config* cfg, int max_active, double* beta_out,
                  gss_fit_result* results, int32_t* status, double* device_seconds) {
  Nvtx nvtx_("gss_fit_batch");
  if (count < 0 || (count > 0 && (!engines || !pens || !cfg || !results)))
    return fail(GSS_ERR_DOMAIN, "null argument");
  if (count == 0) return GSS_OK;
  const int dev = engines[0]->ds->device;
  for (int64_t i = 0; i < count; ++i) {
    if (!engines[i]) return fail(GSS_ERR_DOMAIN, "null engine handle");
    if (engines[i]->ds->device != dev)
      return fail(GSS_ERR_DOMAIN, "gss_fit_batch: all engines must live on one device");
    for (int64_t j = 0; j < i; ++j)
      if (engines[j] == engines[i]) return fail(GSS_ERR_DOMAIN, "gss_fit_batch: repeated engine");
  }
  GSS_CUDA(cudaSetDevice(dev));
  const int64_t p0 = engines[0]->ds->p;
  std::vector<int> grid0(static_cast<size_t>(count));
  for (int64_t i = 0; i < count; ++i) {
    results[i] = gss_fit_result{};
    if (status) status[i] = GSS_OK;
    grid0[i] = engines[i]->grid;
  }
  double total_ms = 0.0;
  // engines of one launch share the kernel instantiation: weighted
  // (Fine-Gray with competing rows) and unweighted fits go in separate queues
  int first_err = GSS_OK;
  std::string first_msg;
  for (int pass = 0; pass < 2; ++pass) {
    const bool weighted = pass == 1;
    std::vector<int64_t> queue;
    for (int64_t i = 0; i < count; ++i)
      if (engines[i]->weighted == weighted) queue.push_back(i);
    if (queue.empty()) continue;
    const int maxg = engines[queue[0]]->max_grid;
    // fits per launch at the default concurrency (a process-wide constant, so
    // every fit's CTA share is the same in every call)
    static const int kBatchW = [] {
      const char* b = std::getenv("GSS_BATCH_MAX");
      return b ? std::max(1, std::min(kMaxBatch, std::atoi(b))) : kMaxBatch;
    }();
    int slots = max_active > 0 ? max_active : kBatchW;
    if (max_active <= 0)
      if (const char* a = std::getenv("GSS_BATCH_ACTIVE")) slots = std::max(1, std::atoi(a));
    slots = std::max(1, std::min({slots, kBatchW, maxg, static_cast<int>(queue.size())}));
    // CTAs per fit: with the default concurrency every fit gets maxg / kMaxBatch
    // CTAs whatever the batch holds, so a fit's CTA partition (hence its
    // summation order) never depends on how many fits share its launch: CV and
    // bootstrap results are bit-identical across worker and device counts (the
    // reference's guarantee, tests/acceptance.cpp:346-383)
    const int share = std::max(1, maxg / (max_active > 0 ? slots : kBatchW));
    size_t next = 0;
    std::vector<int64_t> active;
    auto finish = [&](int64_t i, int rc) {
      gss_engine* E = engines[i];
      if (rc == GSS_OK)
        rc = fit_end(E, beta_out ? beta_out + i * p0 : nullptr, nullptr, &results[i]);
      if (E->grid != grid0[i]) {  // give the engine its own grid back
        const int rc2 = partition_ctas(E, grid0[i]);
        if (rc2 == GSS_OK) push_ctl(E);
      }
      if (status) status[i] = rc;
      if (rc && first_err == GSS_OK) {
        first_err = rc;
        first_msg = g_last_error;
      }
    };
    auto join = [&]() {
      while (active.size() < static_cast<size_t>(slots) && next < queue.size()) {
        const int64_t i = queue[next++];
        gss_engine* E = engines[i];
        if (E->ds->p != p0) {
          finish(i, fail(GSS_ERR_DOMAIN, "gss_fit_batch: engines differ in p"));
          continue;
        }
        int rc = partition_ctas(E, share);
        if (!rc) rc = push_ctl(E);
        if (!rc) rc = fit_begin(E, &pens[i], cfg);
        if (rc || E->fs.done) {
          finish(i, rc);
          continue;
        }
        active.push_back(i);
      }
    };
    join();
    cudaStream_t s = engines[queue[0]]->stream;
    cudaEvent_t e0 = engines[queue[0]]->ev0, e1 = engines[queue[0]]->ev1;
    std::vector<CycleParams> prm;
    std::vector<BatchEntry> ent;
    {  // sharded engines (gss_sharded_fit_local): objective at beta = 0, together
      std::vector<gss_engine*> need;
      for (int64_t i : active)
        if (engines[i]->fs.need_init_obj) need.push_back(engines[i]);
      if (!need.empty()) {
        const int rc = init_objective(need.data(), static_cast<int>(need.size()));
        if (rc) return rc;
      }
    }
    while (!active.empty()) {
      Nvtx nvtx_cycle("batched ccd cycle (%lld fits)", static_cast<long long>(active.size()));
      prm.resize(active.size());
      ent.resize(active.size());
      for (size_t a = 0; a < active.size(); ++a) {
        gss_engine* E = engines[active[a]];
        prm[a] = cycle_params(E);
        ent[a] = BatchEntry{&E->tm_e, &E->tm_code, &E->tm_g, &prm[a]};
      }
      cudaEventRecord(e0, s);
      GSS_CUDA(launch_cycle_batch(ent.data(), static_cast<int>(ent.size()), s));
      cudaEventRecord(e1, s);
      GSS_CUDA(cudaStreamSynchronize(s));
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      total_ms += ms;
      std::vector<int64_t> still;
      for (int64_t i : active) {
        gss_engine* E = engines[i];
        const int rc = fit_after_cycle(E, ms);
        if (rc || E->fs.done)
          finish(i, rc);
        else
          still.push_back(i);
      }
      active.swap(still);
      join();
    }
  }
  if (device_seconds) *device_seconds = total_ms * 1e-3;
  if (first_err) {
    g_last_error = first_msg;
    return first_err;
  }
  return GSS_OK;
}

int gss_engine_grad_hessian_all(gss_engine* E, double* gradient, double* hessian,
                                double* fixed_term) {
  Nvtx nvtx_("gss_engine_grad_hessian_all");
  int rc = check_engine(E);
  if (rc) return rc;
  const int64_t p = E->ds->p;
  if (p == 0) return GSS_OK;
  std::vector<int32_t> slots(static_cast<size_t>(p));
  for (int64_t j = 0; j < p; ++j) slots[j] = static_cast<int32_t>(j);
  rc = run_slots(E, slots, kModeApi, true);
  if (rc) return rc;
  rc = sync_ctl(E);
  if (rc) return rc;
  if (E->h_ctl->err_code) return device_error(E, "grad_hessian");
  std::vector<double> outv(static_cast<size_t>(p) * 4);
  GSS_CUDA(cudaMemcpy(outv.data(), E->slot_out, outv.size() * sizeof(double),
                      cudaMemcpyDeviceToHost));
  for (int64_t j = 0; j < p; ++j) {
    if (gradient) gradient[j] = outv[j * 4];
    if (hessian) hessian[j] = outv[j * 4 + 1];
    if (fixed_term) fixed_term[j] = outv[j * 4 + 2];
  }
  return GSS_OK;
}

int gss_engine_max_abs_gradient(gss_engine* E, double* out) {
  const int64_t p = E ? E->ds->p : 0;
  std::vector<double> g(static_cast<size_t>(p));
  int rc = gss_engine_grad_hessian_all(E, g.data(), nullptr, nullptr);
  if (rc) return rc;
  double top = 0.0;
  for (double v : g) top = std::max(top, std::abs(v));
  *out = top;
  return GSS_OK;
}

// ---- patient sharding (config C5): see include/gss.h ----------------------
int gss_shard_aggregate(gss_engine* E, int64_t column, double* out8) {
  int rc = check_engine(E);
  if (rc) return rc;
  if (column < -1 || column >= E->ds->p) return fail(GSS_ERR_INVALID_COLUMN, "shard: bad column");
  rc = run_slots(E, {static_cast<int32_t>(column)}, kModeApi, false, false, true);
  if (rc) return rc;
  GSS_CUDA(cudaMemcpyAsync(out8, E->shard, 8 * sizeof(double), cudaMemcpyDeviceToHost, E->stream));
  rc = sync_ctl(E);
  if (rc) return rc;
  if (E->h_ctl->err_code) return device_error(E, "shard aggregate");
  return GSS_OK;
}

int gss_shard_sums(gss_engine* E, int64_t column, const double* carry8, double* s0, double* s1) {
  int rc = check_engine(E);
  if (rc) return rc;
  if (column < -1 || column >= E->ds->p) return fail(GSS_ERR_INVALID_COLUMN, "shard: bad column");
  GSS_CUDA(cudaMemcpyAsync(E->ext, carry8, 8 * sizeof(double), cudaMemcpyHostToDevice, E->stream));
  rc = run_slots(E, {static_cast<int32_t>(column)}, kModeApi, false, true, false);
  if (rc) return rc;
  rc = sync_ctl(E);
  if (rc) return rc;
  if (E->h_ctl->err_code) return device_error(E, "shard sums");
  if (column >= 0) {
    *s0 = E->h_ctl->grad_sum;
    *s1 = E->h_ctl->hess_sum;
  } else {
    *s0 = E->h_ctl->ll_fixed;
    *s1 = E->h_ctl->ll_logden;
  }
  return GSS_OK;
}

int gss_engine_update_validate(gss_engine* E, int64_t column, double delta, int32_t* overflow) {
  int rc = check_engine(E);
  if (rc) return rc;
  if (column < 0 || column >= E->ds->p) return fail(GSS_ERR_INVALID_COLUMN, "validate: bad column");
  cudaStream_t s = E->stream;
  GSS_CUDA(cudaMemsetAsync(E->dflag, 0, sizeof(int), s));
  GSS_CUDA(launch_update_check(E->prm, column, delta, E->dflag, s));
  int over = 0;
  GSS_CUDA(cudaMemcpyAsync(&over, E->dflag, sizeof(int), cudaMemcpyDeviceToHost, s));
  GSS_CUDA(cudaStreamSynchronize(s));
  *overflow = over;
  return GSS_OK;
}

int gss_engine_last_timing(gss_engine* E, double* scan_ms, int64_t* launches) {
  if (!E) return fail(GSS_ERR_DOMAIN, "null engine");
  if (scan_ms) *scan_ms = E->last_ms;
  if (launches) *launches = E->last_launches;
  return GSS_OK;
}

// Debug: copy the event trace (GSS_TRACE=1) to host and reset it; returns events copied.
// Debug: copy the CTA-0 event trace (trace build + GSS_TRACE=1) and clear it.
// Layout [32 warps][65536][2] (timestamp 0 = unused); returns the entries copied.
int64_t gss_engine_trace(gss_engine* E, unsigned long long* out, int64_t max_events) {
  if (!E || !E->prm.trace) return 0;
  const int64_t k = std::min<int64_t>(E->prm.trace_cap, max_events);
  if (out && k) cudaMemcpy(out, E->prm.trace, size_t(k) * 16, cudaMemcpyDeviceToHost);
  cudaMemset(E->prm.trace, 0, size_t(E->prm.trace_cap) * 16);
  return k;
}

int64_t gss_engine_cycle_stats(gss_engine* E, double* ms, int64_t* accepted, int64_t max) {
  if (!E) return 0;
  const int64_t k = std::min<int64_t>(max, static_cast<int64_t>(E->cycle_ms.size()));
  for (int64_t i = 0; i < k; ++i) {
    if (ms) ms[i] = E->cycle_ms[i];
    if (accepted) accepted[i] = E->cycle_accepted[i];
  }
  return k;
}

}  // extern "C"

// ---- gss_comm.cu support -------------------------------------------------
int gss::engine_fixed_terms(gss_engine* e, double** dev_fixed, int64_t* p, int* device,
                            cudaStream_t* stream) {
  if (!e) return fail(GSS_ERR_DOMAIN, "null engine handle");
  *dev_fixed = e->fixed;
  *p = e->ds->p;
  *device = e->ds->device;
  *stream = e->stream;
  return GSS_OK;
}

int gss::engine_attach_comm(gss_engine* e, int nranks, int rank, double* const* pay_ptrs,
                            unsigned int* const* bar_ptrs, int sys_scope) {
  if (!e) return fail(GSS_ERR_DOMAIN, "null engine handle");
  if (e->weighted)
    return fail(GSS_ERR_DOMAIN, "patient sharding supports the Cox model (Fine-Gray needs the "
                                "global censoring distribution)");
  if (nranks > 16) return fail(GSS_ERR_DOMAIN, "patient sharding supports at most 16 shards");
  cudaSetDevice(e->ds->device);
  if (int rc = sync_ctl(e)) return rc;
  e->prm.nranks = nranks;
  e->prm.rank = rank;
  e->prm.xr_sys = sys_scope;
  e->prm.xr_pay = pay_ptrs;
  e->prm.xr_bar = bar_ptrs;
  e->h_ctl->xr_base = 0;
  e->h_ctl->xr_count = 0;
  e->h_ctl->rec_valid = 0;
  return push_ctl(e);
}
