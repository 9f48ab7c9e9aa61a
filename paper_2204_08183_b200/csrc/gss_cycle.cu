// gss_cycle.cu — the sm_100a CCD hot path: ONE persistent kernel per call
// that walks a list of "slots" (coordinates of a CCD cycle, or a
// log-likelihood evaluation) over the time-ordered rows.
//
// Per slot it computes what the reference computes per coordinate
//   * the fused reverse-time risk-set scan -> Breslow transform -> reduce of
//     detail::fused_grad_hess (/root/reference/proj/include/survscan/scan_kernels.hpp:74-214),
//     Cox (3 lanes) or Fine-Gray (3 forward + 3 u-weighted backward lanes),
//     plus Engine::finish (src/engine.cpp:220-230);
//   * or the log-likelihood of Engine::log_likelihood (src/engine.cpp:331-341,
//     src/scan.cpp:233-250, 275-367);
//   * in CCD mode, coordinate_step (src/ccd.cpp:71-129) and the sparse
//     eta/exp(eta) update of Engine::update_xbeta_sparse (src/engine.cpp:162-218),
//     with the periodic refresh (src/engine.cpp:120-160).
//
// Layout.  Rows live in 2048-row tiles (strata padded so a tile never spans
// two strata).  CTA c owns a fixed contiguous tile range.  Per CTA:
//   producer warp : streams (slot, tile) positions through an S-stage smem ring
//                   — exp(eta) and row codes (and Fine-Gray G(Y-)) as 2D TMA
//                   boxes, plus the tile's slice of three CSC index lists
//                   (pending-update column, scan column, next column) as 1D
//                   bulk copies.  It runs ahead across slot boundaries.
//   consumer warps: 16, in tile groups (4 warps for Cox, 8 for Fine-Gray),
//                   a group per tile: patch the pending update into the staged
//                   tile and commit it, thread-serial 8-row aggregates -> warp
//                   scans -> group exchange, transform at tied-block ends, and
//                   the next slot's per-tile record (in shared memory).
//   control warp  : owns every cross-slot value (in shared memory); folds the
//                   records into the in-range carry scan as tiles retire, then
//                   publishes the CTA payload, joins the grid barrier, gathers
//                   all payload rows with one bulk copy, runs the replicated
//                   Engine::finish + coordinate_step and hands the consumers
//                   the next slot (or a rare all-warp task) at a named barrier.
// Carry.  A tile's risk-set carry is the sum of all earlier rows.  It is
// assembled from per-tile records written by the previous slot's consumers;
// the exp(delta) change of the pending indicator update enters linearly
// ((phi-1) * s-part), so ONE grid-wide exchange per slot suffices: each CTA
// publishes its partial sums + range aggregates, every CTA reduces them in a
// fixed order and computes the identical coordinate step, then the carries.
// Valued pending columns and refreshes take an extra exchange.
// Determinism: every sum has a fixed order independent of scheduling, so
// results are bitwise reproducible run to run (scan_kernels.hpp:8-10).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <mutex>

#include "gss_device.cuh"
#include "gss_kernels.cuh"

namespace gss {

namespace {

constexpr double kXbetaBound = 700.0;  // src/engine.cpp:12
constexpr double kHwFloor = 1e-300;    // src/ccd.cpp:13
constexpr double kFastBound = 700.0 * (1.0 - 1e-12);
constexpr int kErrNonPos = 7;     // GSS_ERR_NONPOS_DEN (include/gss.h)
constexpr int kErrOverflow = 8;   // GSS_ERR_OVERFLOW

template <bool FG>
struct Geo {
  static constexpr int kW = 16;           // consumer warps
  static constexpr int kGW = FG ? 8 : 4;  // warps per tile group (kPasses / kGW passes each)
  static_assert(kPasses % kGW == 0 && kW % kGW == 0, "group geometry");
  static constexpr int kNG = kW / kGW;    // tile groups (tiles in process at once)
  static constexpr int kS = FG ? 4 : 6;   // ring stages
  static constexpr int kCap = kNnzCap;    // per-list smem capacity (ints)
  static constexpr uint32_t kEBytes = kTileRows * 8;
  static constexpr uint32_t kCBytes = kTileRows * 4;
  static constexpr uint32_t kGBytes = FG ? kTileRows * 8 : 0;
  static constexpr uint32_t kLBytes = kCap * 4;
  static constexpr uint32_t kOffC = kEBytes;
  static constexpr uint32_t kOffG = kEBytes + kCBytes;
  static constexpr uint32_t kOffL = kEBytes + kCBytes + kGBytes;
  static constexpr uint32_t kStage = (kOffL + 3 * kLBytes + 1023) / 1024 * 1024;
  static constexpr int kP = 1;            // producer warps (independent issue chains)
  static constexpr int kThreads = 32 * (kW + 1 + kP);  // consumers, control warp, producer(s)
  static_assert(kStage % 1024 == 0, "stage alignment");
};

struct ListRef {
  long long lo;   // global index of the first entry of the tile's slice
  int cnt;        // entries
  int off;        // smem index of entry 0 (lo - aligned base), -1 => read global
};

struct StageInfo {
  int tile, slot, li;  // li = tile index inside the CTA range
  ListRef l[3];  // 0 pending column, 1 scan column, 2 next column
};

struct SlotState {
  long long col;   // scan column of the slot (-1: log-likelihood slot)
  long long pcol;  // pending-update column (-1: none)
  long long ncol;  // next slot's column (-1: none / objective)
  double delta, phi;
  int pind;        // pending column is an indicator column
  int cind;        // scan column is an indicator column
  int nind;        // next column is an indicator column
  int refresh;     // staged exp(eta) is stale (a refresh ran): reload from global
  int fused;       // Cox CCD slot with indicator scan + next columns: fused records
  int dry;         // halted: stream without work
  int kind;
  double cin_f[6];   // corrected fwd carry into the CTA range (a,b,c) + spare
  double cin_r[6];   // corrected rev carry into the CTA range (ua,ub,uc)
};

struct SlotFields {
  long long col, ncol;
  int kind, cind, nind, fused, valid;
};

// replicated CCD state, owned by thread 0 (kept in shared memory: registers
// holding it across the consume phase would spill to local memory, which
// misses L1 under this shared-memory carve-out)
struct CcdState {
  double absmax, slack;
  long long accepted, refreshes, skipped, err_col;
  int err;
  unsigned bar_target;
  unsigned long long xr_base, xr_count;  // cross-shard counter base / exchanges done
  unsigned long long tgo, tcons;         // GSS_DEBUG & 65536: per-CTA consume time
  // step inputs of the current slot, prefetched at slot start
  double in_fixed, in_beta, in_hw, in_cmax;
  int in_pen, in_ind;
  SlotFields nf;
  // phase profile (GSS_DEBUG & 256, one CTA): clock64 sums per phase
  long long ph[16];
  long long ph_t, ph_ref;
  long long gfirst[4], glast[4];
  int prev_rf, n_rf;
  // control-warp loop state (shared memory is its home: no local-memory spills)
  int xi, cstar, cend;
  unsigned qbase;
  long long to_refresh;
  long long col, ncol;
};

// tiles per CTA with shared-memory records / carries (Fine-Gray: fewer, its
// stages are larger)
template <bool FG>
struct MaxTc {
  static constexpr int v = FG ? 40 : 64;
};
constexpr int kMaxGrid = 148;  // CTAs (one per SM; B200)

// lightweight phase profile (GSS_DEBUG bit 256) on thread 0 of CTA kProfCta
constexpr int kProfCta = 5;
#define PROF_ON (((P.dbg & 256) != 0) && cta == kProfCta)
#define PROF_MARK(i)                                   \
  do {                                                 \
    if (PROF_ON && tid == 0) {                         \
      const long long _n = clock64();                  \
      cst.ph[i] += _n - cst.ph_t;                      \
      cst.ph_t = _n;                                   \
    }                                                  \
  } while (0)

template <bool FG>
struct Tail {
  static constexpr int W = Geo<FG>::kW, S = Geo<FG>::kS;
  uint64_t full[S];
  uint64_t empty[S];
  StageInfo info[S];
  static constexpr int NG = Geo<FG>::kNG, GW = Geo<FG>::kGW;
  uint32_t xm[NG][2][256];  // per-group scan-column bitmask per thread-row (+ first-entry
                            // offset), double-buffered by the group's tile parity
  uint32_t xn[NG][2][256];  // per-group next-column bitmask (fused records)
  double gx[NG][GW][8];  // per-warp pass-group totals (group exchange)
  double gr[NG][GW][10]; // per-warp record partials (group exchange)
  double gc[NG][16];     // the tile's carries (group exchange)
  double wpart[W][4];
  unsigned int progress[NG];
  SlotState ss;
  double bcast[8];
  double gs[16];
  uint8_t cflag[256];   // CTA range holds a stratum-first tile (grid <= 256)
  int flag;
  int need_exact, refresh, valued;
  int task;                  // consumer task handed out at the GO barrier
  unsigned issued;           // stream positions issued by the producer (in order)
  long long tcol, tncol;     // task parameters
  double tdelta;
  uint8_t tfirst[MaxTc<FG>::v];  // tile_first of the CTA's first MaxTc tiles
  int cstar, cend;
  int ext_f, ext_r;
  double xext[12];      // cross-shard carry: fwd (a,b,c,sa,sb,sc) of earlier shards,
                        // rev (ua..usc) of later shards (in-kernel exchange)
  double xaux[2];       // cross-shard aux: max |eta| (refresh), overflow flag (validation)
  volatile unsigned mark[32];  // last phase reached by each warp (watchdog report)
  CcdState cs;
  // per-tile records and in-range carries of the CTA's first kMaxTc tiles live
  // in shared memory (tiles beyond use the global arrays); records are loaded
  // from / flushed to global at launch start / end
  alignas(128) double gbuf[kMaxGrid][kPayStride];  // staged CTA payloads (gather)
  uint64_t gbar;                                    // gather bulk-copy barrier
  uint32_t gphase;
  double gred[32][FG ? 15 : 9];                      // gather cross-lane partials
  double srec[MaxTc<FG>::v][FG ? 12 : 6];
  double scar[MaxTc<FG>::v][FG ? 16 : 8];
};

template <bool FG>
__device__ __forceinline__ double* rec_at(const CycleParams& P, Tail<FG>* tl, int t, int li) {
  return li < MaxTc<FG>::v ? tl->srec[li] : P.trec + size_t(t) * kRecStride;
}
template <bool FG>
__device__ __forceinline__ double* car_at(const CycleParams& P, Tail<FG>* tl, int t, int li) {
  return li < MaxTc<FG>::v ? tl->scar[li] : P.tcar + size_t(t) * kCarStride;
}
// load through the right path (global fallback entries bypass L1)
template <bool FG>
__device__ __forceinline__ double ld_rc(const double* p, int li) {
  return li < MaxTc<FG>::v ? *p : __ldcg(p);
}

template <bool FG>
__host__ __device__ constexpr size_t smem_total() {
  return 1024 + size_t(Geo<FG>::kS) * Geo<FG>::kStage + sizeof(Tail<FG>);
}

// consumer <-> control warp handshake (named barriers; 1 = consumers only,
// 2.. = tile groups): consumers ARRIVE at kBarDone when their slot (or task) is
// finished and SYNC at kBarGo; the control warp does the opposite
constexpr int kBarDone = 8, kBarGo = 9;
enum ConsumerTask : int { kTaskNext = 0, kTaskExit, kTaskExact, kTaskRefresh, kTaskValued };
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_sync_n(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void consumer_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void red_add_f64(double* p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

__device__ __forceinline__ double sgn(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// CTA-scope message flags in shared memory (stream progress, issue count):
// release store by the publisher, acquire loads by the pollers, so the data
// written before the flag (records, committed updates) is visible after it.
__device__ __forceinline__ void flag_release(unsigned* p, unsigned v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned flag_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

// swizzled element addresses inside a staged tile: TMA boxes of 128-byte rows
// (16 doubles / 32 codes) with 128B swizzle; a lane's 8-row thread-row is half
// (exp(eta), G) or a quarter (codes) of a box row, and the lane pattern of the
// consumers stays bank-conflict free.
__device__ __forceinline__ double* e_at(unsigned char* base, int lr) {
  return reinterpret_cast<double*>(base + swz<128>(lr * 8));
}
__device__ __forceinline__ uint32_t code_at(const unsigned char* base, int lr) {
  return *reinterpret_cast<const uint32_t*>(base + swz<128>(lr * 4));
}

// coordinate_step (src/ccd.cpp:71-129), scalar, no FMA contraction.
struct Step {
  double new_beta, applied, new_hw;
  bool skipped;
};
__device__ __forceinline__ Step coordinate_step_dev(double beta_j, double grad, double hess, int kind,
                                    double strength, bool penalized, double hw) {
  double geff = grad, heff = hess;
  bool at_zero_l1 = false;
  if (penalized) {
    if (kind == 2) {
      geff = __dsub_rn(geff, __ddiv_rn(beta_j, strength));
      heff = __dsub_rn(heff, __ddiv_rn(1.0, strength));
    } else if (kind == 1) {
      if (beta_j != 0.0)
        geff = __dsub_rn(geff, __dmul_rn(strength, sgn(beta_j)));
      else
        at_zero_l1 = true;
    }
  }
  Step s{beta_j, 0.0, hw, false};
  if (at_zero_l1) {
    if (fabs(geff) <= strength) {
      s.new_hw = fmax(hw / 2.0, kHwFloor);
      return s;
    }
    geff = __dsub_rn(geff, __dmul_rn(strength, sgn(geff)));
  }
  if (!(heff < 0.0)) {
    if (geff != 0.0) {
      s.skipped = true;
      return s;
    }
    s.new_hw = fmax(hw / 2.0, kHwFloor);
    return s;
  }
  double raw = __ddiv_rn(-geff, heff);
  if (penalized && kind == 1 && beta_j != 0.0 && sgn(__dadd_rn(beta_j, raw)) != sgn(beta_j))
    raw = -beta_j;
  const double a = __dmul_rn(sgn(raw), fmin(fabs(raw), hw));
  s.applied = a;
  s.new_beta = __dadd_rn(beta_j, a);
  s.new_hw = fmax(fmax(__dmul_rn(2.0, fabs(a)), hw / 2.0), kHwFloor);
  return s;
}

// optional event trace: compiled in only with -DGSS_ENABLE_TRACE=1 (tools/trace_cycle.py;
// build with GSS_TRACE_BUILD=1), and then active only when the engine was created with
// GSS_TRACE=1
#ifndef GSS_ENABLE_TRACE
#define GSS_ENABLE_TRACE 0
#endif
constexpr unsigned kTrPerWarp = 1u << 16;  // events per traced warp (CTA 0 only)
__device__ __forceinline__ unsigned& trace_slot(int warp) {
  __shared__ unsigned tr_n[32];
  return tr_n[warp];
}
// lane-0 only; no atomics: warp w of CTA 0 owns trace[w * kTrPerWarp ...]
__device__ __forceinline__ void trace_ev(const CycleParams& P, int ev, int arg) {
  if (!GSS_ENABLE_TRACE || !P.trace || blockIdx.x != 0 || (P.dbg & 32)) return;
  const int warp = threadIdx.x >> 5;
  unsigned& n = trace_slot(warp);
  const unsigned i = atomicAdd(&n, 1u);  // smem atomic: several lanes may trace
  if (i < kTrPerWarp) {
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    unsigned long long* o = P.trace + 2 * (size_t(warp) * kTrPerWarp + i);
    o[0] = ns;
    o[1] = (static_cast<unsigned long long>(ev) << 32) | static_cast<unsigned>(arg);
  }
}
// per-CTA slot timestamps of ALL CTAs (trace build): region of warp 31, [slot][cta]
__device__ __forceinline__ void trace_cta(const CycleParams& P, int ev, int slot, int region = 31) {
  if (!GSS_ENABLE_TRACE || !P.trace) return;
  const unsigned i = static_cast<unsigned>(slot) * gridDim.x + blockIdx.x;
  if (i < kTrPerWarp) {
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    unsigned long long* o = P.trace + 2 * (size_t(region) * kTrPerWarp + i);
    o[0] = ns;
    o[1] = (static_cast<unsigned long long>(ev) << 32) | static_cast<unsigned>(blockIdx.x);
  }
}
__device__ __forceinline__ void trace_c0(const CycleParams& P, int ev, int arg) {
  trace_ev(P, ev, arg);
}
__device__ __forceinline__ void trace_w0(const CycleParams& P, int ev, int arg) {
  if ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) == 0) trace_ev(P, ev, arg);
}

__device__ __forceinline__ bool gt0(int warp, int lane, int gw) {
  return lane == 0 && (warp % gw) == 0;
}

// list entry i of a staged list (smem copy or global fallback)
__device__ __forceinline__ int32_t list_at(const int32_t* ls, const ListRef& L, const int32_t* glob,
                                           int i) {
  return L.off >= 0 ? ls[L.off + i] : glob[L.lo + i];
}

// ---------------------------------------------------------------------------
// watchdog: every spin-wait gives up after kWatchdogNs and traps with a
// message, so a protocol bug surfaces as a launch error, never a hung device
// ---------------------------------------------------------------------------
constexpr unsigned long long kWatchdogNs = 10ull * 1000 * 1000 * 1000;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long ns;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
  return ns;
}
__device__ __noinline__ void watchdog_trap(const char* what, unsigned a, unsigned b,
                                           const volatile unsigned* marks = nullptr) {
  if (marks)
    printf("gss watchdog: %s stuck (cta %d thread %d: %u %u) marks %x %x %x %x | %x %x %x %x | "
           "%x %x %x %x | %x %x %x %x | producer %x %x %x %x %x %x %x\n",
           what, blockIdx.x, threadIdx.x, a, b, marks[0], marks[1], marks[2], marks[3], marks[4],
           marks[5], marks[6], marks[7], marks[8], marks[9], marks[10], marks[11], marks[12],
           marks[13], marks[14], marks[15], marks[16], marks[17], marks[18], marks[19], marks[20],
           marks[21], marks[22]);
  else
    printf("gss watchdog: %s stuck (cta %d thread %d: %u %u)\n", what, blockIdx.x, threadIdx.x,
           a, b);
  __trap();
}

// ---------------------------------------------------------------------------
// grid barrier over the co-resident CTAs (monotonic counter, no reset)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void grid_arrive_wait(unsigned int* bar, unsigned target) {
  // release-reduction: orders this thread's prior writes (the payload) before
  // the arrival without a separate fence round trip
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
  const unsigned long long t0 = gtimer();
  unsigned it = 0;
  while (static_cast<int>(ld_acquire_u32(bar) - target) < 0) {
    if ((++it & 1023u) == 0 && gtimer() - t0 > 2 * kWatchdogNs)
      watchdog_trap("grid barrier", ld_acquire_u32(bar), target);
  }
}

// bounded wait on an mbarrier phase (consumers: data landed)
__device__ __forceinline__ void mbar_wait_wd(uint64_t* bar, uint32_t parity, const char* what,
                                             unsigned info,
                                             const volatile unsigned* marks = nullptr) {
  if (mbar_try_wait(bar, parity)) return;
  const unsigned long long t0 = gtimer();
  unsigned it = 0;
  // try_wait suspends the warp in hardware until the phase completes or a
  // time limit passes, so the retry needs no software back-off (measured:
  // a 64 ns sleep here cost 0.4% per coordinate)
  while (!mbar_try_wait(bar, parity)) {
    if ((++it & 63u) == 0 && gtimer() - t0 > kWatchdogNs) watchdog_trap(what, info, parity, marks);
  }
}

// ---------------------------------------------------------------------------
// per-slot kernel context
// ---------------------------------------------------------------------------
template <bool FG>
struct Ctx {
  const CycleParams* P;
  unsigned char* smem;
  Tail<FG>* tl;
  int cta, t0, tc;         // tile range [t0, t0 + tc)
  unsigned bar_target;     // next grid-barrier target
  int par;                 // payload buffer parity
};

// ---------------------------------------------------------------------------
// producer: streams every (slot, tile) position of this CTA through the ring
// ---------------------------------------------------------------------------
template <bool FG>
__device__ __forceinline__ void producer(const CycleParams& P, unsigned char* smem, Tail<FG>* tl,
                                      int t0, int tc, const CUtensorMap* tm_e,
                                      const CUtensorMap* tm_code, const CUtensorMap* tm_g,
                                      int pw) {
  using G = Geo<FG>;
  constexpr int S = G::kS, NP = G::kP;
  const int lane = threadIdx.x & 31;
  // positions are 32-bit (slots x tiles-per-CTA < 2^31): no 64-bit divisions
  const unsigned total = static_cast<unsigned>(P.nslots) * static_cast<unsigned>(tc);
  const size_t nt1 = static_cast<size_t>(P.ntiles) + 1;
  const unsigned utc = static_cast<unsigned>(tc);
  // producer warp pw owns positions q == pw (mod NP), in increasing order (the
  // warps run independent latency chains); waves of 32 of its positions: lane
  // l resolves position q0 + l*NP (list slices), then lane 0 waits the stages
  // in order and lane l issues its position as soon as its stage is free
  for (unsigned q0 = static_cast<unsigned>(pw); q0 < total; q0 += 32u * NP) {
    const unsigned qq = q0 + static_cast<unsigned>(lane) * NP;
    long long lo[3] = {0, 0, 0};
    int cnt[3] = {0, 0, 0};
    int slot = 0, tloc = 0;
    if (qq < total) {
      slot = static_cast<int>(qq / utc);
      tloc = static_cast<int>(qq - static_cast<unsigned>(slot) * utc);
      const int tile = t0 + tloc;
      long long cols[3];
      cols[0] = (P.mode == kModeCcd && slot > 0) ? P.slot_col[slot - 1] : -1;
      cols[1] = P.slot_col[slot];
      cols[2] = (slot + 1 < P.nslots) ? P.slot_col[slot + 1]
                                      : (P.mode == kModeCcd ? P.slot_col[0] : -1);
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        if (cols[l] >= 0) {
          const long long cb = P.col_ptr[cols[l]];
          const uint32_t a = P.tile_ptr[size_t(cols[l]) * nt1 + tile];
          const uint32_t b = P.tile_ptr[size_t(cols[l]) * nt1 + tile + 1];
          lo[l] = cb + a;
          cnt[l] = static_cast<int>(b - a);
        }
      }
    }
    for (int i = 0; i < 32; ++i) {
      const unsigned qw = q0 + static_cast<unsigned>(i) * NP;
      if (qw >= total) break;
      const int s = static_cast<int>(qw % S);
      const int tl_i = __shfl_sync(0xffffffffu, tloc, i);
      if (lane == 0) {
        tl->mark[16 + s] = 0xA0u | (qw << 8);
        trace_c0(P, 24, static_cast<int>(qw));
        mbar_wait_wd(&tl->empty[s], ((qw / S) & 1u) ^ 1u, "producer empty-stage wait", qw, tl->mark);
        trace_c0(P, 25, static_cast<int>(qw));
        // the same tile of the previous slot must have committed its pending
        // update (the committing group fenced generic -> async proxy before
        // publishing its progress)
        if (qw >= utc) {
          const unsigned prevq = qw - utc;
          const unsigned* pr = &tl->progress[tl_i % G::kNG];
          if (flag_acquire(pr) < prevq + 1) {
            const unsigned long long tw = gtimer();
            while (flag_acquire(pr) < prevq + 1) {
              __nanosleep(32);
              if (gtimer() - tw > kWatchdogNs)
                watchdog_trap("producer progress wait", qw, flag_acquire(pr), tl->mark);
            }
          }
        }
      }
      __syncwarp();
      if (lane != i) continue;
      const int tile = t0 + tloc;
      trace_c0(P, 23, static_cast<int>(qq));
      unsigned char* sb = smem + size_t(s) * G::kStage;
      StageInfo& inf = tl->info[s];
      inf.tile = tile;
      inf.slot = slot;
      inf.li = tloc;
      uint32_t bytes = G::kEBytes + G::kCBytes + G::kGBytes;
      int32_t* lbase = reinterpret_cast<int32_t*>(sb + G::kOffL);
      uint32_t lbytes[3];
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        inf.l[l].lo = lo[l];
        inf.l[l].cnt = cnt[l];
        lbytes[l] = 0;
        if (cnt[l] > 0) {
          const long long base = lo[l] & ~3LL;
          const long long end = (lo[l] + cnt[l] + 3) & ~3LL;
          if (end - base <= G::kCap) {
            inf.l[l].off = static_cast<int>(lo[l] - base);
            lbytes[l] = static_cast<uint32_t>((end - base) * 4);
            bytes += lbytes[l];
          } else {
            inf.l[l].off = -1;
          }
        } else {
          inf.l[l].off = 0;
        }
      }
      trace_c0(P, 20, static_cast<int>(qq));
      mbar_arrive_expect_tx(&tl->full[s], bytes);
      // 128-byte box rows: 16 doubles / 32 codes per row, 128B swizzle
      tma_load_2d(sb, tm_e, 0, tile * (kTileRows / 16), &tl->full[s]);
      tma_load_2d(sb + G::kOffC, tm_code, 0, tile * (kTileRows / 32), &tl->full[s]);
      if constexpr (FG) tma_load_2d(sb + G::kOffG, tm_g, 0, tile * (kTileRows / 16), &tl->full[s]);
#pragma unroll
      for (int l = 0; l < 3; ++l)
        if (lbytes[l])
          bulk_load_1d(lbase + l * G::kCap, P.row_idx + (lo[l] & ~3LL), lbytes[l], &tl->full[s]);
      trace_c0(P, 26, static_cast<int>(qq));
      // positions are issued in order: publish the count (consumers check it
      // before their parity wait, see the consumer loop)
      flag_release(&tl->issued, qq + 1);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// consumer: one tile of one slot, processed by a group of kGW warps
// (warp gw of the group owns passes [gw*PPW, (gw+1)*PPW) of the tile)
// ---------------------------------------------------------------------------
// staged Fine-Gray weight of a row (gss_engine::gs): u = 1/G(Y-) on
// competing rows, G elsewhere
__device__ __forceinline__ double u_of(uint32_t code, double staged) {
  return (code & kCodeCompeting) ? staged : 0.0;
}
__device__ __forceinline__ double g_of(uint32_t code, double staged) {
  return (code & kCodeCompeting) ? __drcp_rn(staged) : staged;
}

template <int L>
struct Lanes {
  double v[L];
};

template <bool FG>
__device__ __forceinline__ void mark(Tail<FG>* tl, unsigned code) {
  if ((threadIdx.x & 31) == 0) tl->mark[threadIdx.x >> 5] = code;
}

template <bool FG>
__device__ __forceinline__ void group_sync(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(2 + g), "r"(32 * Geo<FG>::kGW) : "memory");
}

// FUSED (Cox, CCD, indicator scan + next columns): the next slot's record
// sums ride along the scan as two extra lanes (next-column e, and e on rows of
// both columns), so the tile totals ARE the record.
template <bool FG, bool IND, int KIND, bool FUSED = false>
__device__ __forceinline__ void process_tile(const CycleParams& P, Tail<FG>* tl, unsigned char* sb,
                                             const StageInfo& inf, const SlotState& ss, int g,
                                             int gw, int lane, int par, double& acc0,
                                             double& acc1, int& bad, uint64_t* empty_bar) {
  using G = Geo<FG>;
  constexpr int GW = G::kGW, PPW = kPasses / GW, GT = 32 * GW;
  constexpr int NF = (KIND == kSlotLoglik) ? 1 : (IND ? 2 : 3);
  constexpr int NU = FG ? NF : 0;
  constexpr int NX = FUSED ? 2 : 0;
  constexpr int L = NF + NU + NX;
  static_assert(!FUSED || (!FG && IND && KIND == kSlotGrad), "fused records: Cox indicator only");
  const int gt = gw * 32 + lane;  // thread index inside the group
  const int t = inf.tile;
  const long long row0 = static_cast<long long>(t) * kTileRows;
  const unsigned char* sc = sb + G::kOffC;
  const unsigned char* sg = sb + G::kOffG;
  const int32_t* lbase = reinterpret_cast<const int32_t*>(sb + G::kOffL);
  const int32_t* lp = lbase;
  const int32_t* lcur = lbase + G::kCap;
  const int32_t* lnext = lbase + 2 * G::kCap;
  const ListRef& Lp = inf.l[0];
  const ListRef& Lc = inf.l[1];
  const ListRef& Ln = inf.l[2];
  uint32_t* xm = tl->xm[g][par];
  uint32_t* xn = tl->xn[g][par];
  {  // the other buffers served the group's previous tile (released): clear them
    uint32_t* om = tl->xm[g][par ^ 1];
    uint32_t* on = tl->xn[g][par ^ 1];
    for (int i = gt; i < 256; i += GT) {
      om[i] = 0u;
      on[i] = 0u;
    }
  }
  const bool has_cur = KIND == kSlotGrad && ss.col >= 0;
  // dense columns (density >= 25%, SparseColumn::make src/dataset.cpp:126-157):
  // values by row from the dense pool instead of the tile's index list
  auto dense_of = [&](long long c) -> const double* {
    if (c < 0 || !P.dense_idx) return nullptr;
    const int k = P.dense_idx[c];
    return k < 0 ? nullptr : P.dense_pool + size_t(k) * size_t(P.npad);
  };
  const double* dcur = (!IND && has_cur) ? dense_of(ss.col) : nullptr;
  const double* dpen = (ss.pcol >= 0 && !ss.pind) ? dense_of(ss.pcol) : nullptr;
  const double* dnxt = ss.nind ? nullptr : dense_of(ss.ncol);

  // The pre-barrier list work is spread over the group's warps (each loop
  // is one dependent chain per entry): the patch on warp 0, the scan-column
  // bitmask from warp 1, the next-column bitmask from warp 2, the carries on
  // the last warp.
  const int gt1 = ((gw + GW - 1) % GW) * 32 + lane;  // warp 1 first
  const int gt2 = ((gw + GW - 2) % GW) * 32 + lane;  // warp 2 first
  // ---- tile carries -> group smem (visible after the first group barrier) ----
  if (gw == GW - 1 && lane < (FG ? 15 : 7)) tl->gc[g][lane] = ld_rc<FG>(car_at<FG>(P, tl, t, inf.li) + lane, inf.li);
  const double* tcv = tl->gc[g];

  // ---- stale tile after a refresh: reload exp(eta) from global ----
  if (ss.refresh) {
    for (int i = gt; i < kTileRows; i += GT) *e_at(sb, i) = __ldcg(P.e + row0 + i);
  } else if (dpen) {
    // ---- dense pending column: own rows, e = exp(eta + x*delta) ----
    for (int lr = gt; lr < kTileRows; lr += GT) {
      const double x = __ldg(dpen + row0 + lr);
      if (x == 0.0 || (code_at(sc, lr) & kCodeMasked)) continue;
      const long long r = row0 + lr;
      const double ne = __dadd_rn(__ldcg(P.eta + r), __dmul_rn(x, ss.delta));
      const double en = exp(ne);
      P.eta[r] = ne;
      *e_at(sb, lr) = en;
      if constexpr (FG)
        atomicExch(reinterpret_cast<unsigned long long*>(P.e + r),
                   static_cast<unsigned long long>(__double_as_longlong(en)));
      else
        P.e[r] = en;
    }
  } else if (ss.pcol >= 0) {
    // ---- patch + commit the pending update (src/engine.cpp:192-215) ----
    for (int i = gt; i < Lp.cnt; i += GT) {
      const int32_t r = list_at(lp, Lp, P.row_idx, i);
      const int lr = static_cast<int>(r - row0);
      if (code_at(sc, lr) & kCodeMasked) continue;
      double* pe = e_at(sb, lr);
      double en;
      if (ss.pind) {
        en = __dmul_rn(*pe, ss.phi);
        red_add_f64(P.eta + r, ss.delta);  // xbeta_[i] += 1.0 * delta, fire-and-forget
      } else {
        const double ne = __dadd_rn(__ldcg(P.eta + r), __dmul_rn(P.vals[Lp.lo + i], ss.delta));
        en = exp(ne);
        P.eta[r] = ne;
      }
      *pe = en;
      if constexpr (FG)  // L2 atomic store: measured 2% faster for Fine-Gray, not for Cox
        atomicExch(reinterpret_cast<unsigned long long*>(P.e + r),
                   static_cast<unsigned long long>(__double_as_longlong(en)));
      else
        P.e[r] = en;
    }
  }
  // ---- scan-column bitmask per thread-row (xm is all-zero on entry) ----
  if (has_cur && !dcur) {
    for (int i = gt1; i < Lc.cnt; i += GT) {
      const int32_t r = list_at(lcur, Lc, P.row_idx, i);
      const int lr = static_cast<int>(r - row0);
      uint32_t w = 1u << (lr & 7);
      if (!IND) {
        const bool first =
            i == 0 || ((list_at(lcur, Lc, P.row_idx, i - 1) - row0) >> 3) != (lr >> 3);
        if (first) w |= static_cast<uint32_t>(i) << 8;
      }
      atomicOr(&xm[lr >> 3], w);
    }
  }
  if constexpr (FUSED) {
    for (int i = gt2; i < Ln.cnt; i += GT) {
      const int lr = static_cast<int>(list_at(lnext, Ln, P.row_idx, i) - row0);
      atomicOr(&xn[lr >> 3], 1u << (lr & 7));
    }
  }
  mark<FG>(tl, 0x11u | (static_cast<unsigned>(t & 0xffff) << 8));
  group_sync<FG>(g);
  trace_w0(P, 10, t);

  // per-row lane values of thread-row tr
  struct Rows {
    double ev[kIpt];
    uint32_t cw[kIpt];
    double gv[FG ? kIpt : 1], uv[FG ? kIpt : 1];
    double xv[(KIND == kSlotGrad && !IND) ? kIpt : 1];
    uint32_t xb, nb;
  };
  auto load_rows = [&](int tr, Rows& R) {
#pragma unroll
    for (int c = 0; c < kIpt / 2; ++c) {
      const double2 v =
          *reinterpret_cast<const double2*>(sb + swz<128>(tr * (kIpt * 8) + c * 16));
      R.ev[2 * c] = v.x;
      R.ev[2 * c + 1] = v.y;
    }
#pragma unroll
    for (int c = 0; c < kIpt / 4; ++c) {
      const uint4 v = *reinterpret_cast<const uint4*>(sc + swz<128>(tr * (kIpt * 4) + c * 16));
      R.cw[4 * c] = v.x;
      R.cw[4 * c + 1] = v.y;
      R.cw[4 * c + 2] = v.z;
      R.cw[4 * c + 3] = v.w;
    }
    if constexpr (FG) {
#pragma unroll
      for (int c = 0; c < kIpt / 2; ++c) {
        const double2 v =
            *reinterpret_cast<const double2*>(sg + swz<128>(tr * (kIpt * 8) + c * 16));
        R.gv[2 * c] = v.x;
        R.gv[2 * c + 1] = v.y;
      }
#pragma unroll
      for (int m = 0; m < kIpt; ++m) R.uv[m] = u_of(R.cw[m], R.gv[m]);
    }
    R.xb = 0;
    R.nb = 0;
    if constexpr (FUSED) R.nb = xn[tr];
    if constexpr (KIND == kSlotGrad) {
      if (has_cur) R.xb = xm[tr];
      if constexpr (!IND) {
        if (dcur) {  // dense scan column: the thread-row's values, coalesced
#pragma unroll
          for (int c = 0; c < kIpt / 2; ++c) {
            const double2 v = __ldg(reinterpret_cast<const double2*>(dcur + row0 + tr * kIpt) + c);
            R.xv[2 * c] = v.x;
            R.xv[2 * c + 1] = v.y;
          }
          uint32_t bits = 0;
#pragma unroll
          for (int m = 0; m < kIpt; ++m) bits |= (R.xv[m] != 0.0 ? 1u : 0u) << m;
          R.xb = bits;
          return;
        }
        const uint32_t bits = R.xb & 0xffu;
        const long long k0 = Lc.lo + (R.xb >> 8);
        int k = 0;
#pragma unroll
        for (int m = 0; m < kIpt; ++m) {
          R.xv[m] = 0.0;
          if ((bits >> m) & 1u) {
            R.xv[m] = P.vals[k0 + k];
            ++k;
          }
        }
      }
    }
  };
  auto row_val = [&](const Rows& R, int m) {
    Lanes<L> rv;
    rv.v[0] = R.ev[m];
    if constexpr (NF >= 2) {
      if constexpr (IND) {
        rv.v[1] = ((R.xb >> m) & 1u) ? R.ev[m] : 0.0;
      } else {
        const double ex = __dmul_rn(R.ev[m], R.xv[m]);
        rv.v[1] = ex;
        rv.v[2] = __dmul_rn(ex, R.xv[m]);
      }
    }
    if constexpr (FG) {
#pragma unroll
      for (int i = 0; i < NU; ++i) rv.v[NF + i] = __dmul_rn(R.uv[m], rv.v[i]);
    }
    if constexpr (FUSED) {
      const bool nx = (R.nb >> m) & 1u;
      rv.v[NF] = nx ? R.ev[m] : 0.0;                          // next column: e * x_next
      rv.v[NF + 1] = (nx && ((R.xb >> m) & 1u)) ? R.ev[m] : 0.0;  // rows of both columns
    }
    return rv;
  };
  constexpr uint32_t kWork = (KIND == kSlotLoglik) ? (kCodeCount | kCodeEvent) : kCodeCount;

  // ---- phase 1: thread aggregates of this warp's PPW passes ----
  Lanes<L> st[PPW];
  uint32_t work = 0;  // bit pp: this lane's rows of pass pp hold a block end (or event)
#pragma unroll
  for (int pp = 0; pp < PPW; ++pp) {
    Rows R;
    load_rows((gw * PPW + pp) * 32 + lane, R);
#pragma unroll
    for (int i = 0; i < L; ++i) st[pp].v[i] = 0.0;
    uint32_t w = 0;
#pragma unroll
    for (int m = 0; m < kIpt; ++m) {
      const Lanes<L> rv = row_val(R, m);
#pragma unroll
      for (int i = 0; i < L; ++i) st[pp].v[i] = __dadd_rn(st[pp].v[i], rv.v[i]);
      w |= R.cw[m] & kWork;
    }
    if (w) work |= 1u << pp;
  }
  // ---- phase 2: warp inclusive scans (PPW interleaved) ----
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
    for (int pp = 0; pp < PPW; ++pp) {
#pragma unroll
      for (int i = 0; i < L; ++i) {
        const double o = __shfl_up_sync(0xffffffffu, st[pp].v[i], d);
        if (lane >= d) st[pp].v[i] = __dadd_rn(o, st[pp].v[i]);
      }
    }
  }
  // exclusive prefix inside this warp's passes; warp total -> group exchange
  Lanes<L> wt;
#pragma unroll
  for (int i = 0; i < L; ++i) wt.v[i] = 0.0;
#pragma unroll
  for (int pp = 0; pp < PPW; ++pp) {
#pragma unroll
    for (int i = 0; i < L; ++i) {
      double ex = __shfl_up_sync(0xffffffffu, st[pp].v[i], 1);
      if (lane == 0) ex = 0.0;
      const double tot = __shfl_sync(0xffffffffu, st[pp].v[i], 31);
      st[pp].v[i] = __dadd_rn(wt.v[i], ex);
      wt.v[i] = __dadd_rn(wt.v[i], tot);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < L; ++i) tl->gx[g][gw][i] = wt.v[i];
  }
  const unsigned wany = __reduce_or_sync(0xffffffffu, work);
  mark<FG>(tl, 0x12u | (static_cast<unsigned>(t & 0xffff) << 8));
  group_sync<FG>(g);
  // offset of this warp's passes inside the tile (fixed order) and the tile total
  Lanes<L> off, ttot;
#pragma unroll
  for (int i = 0; i < L; ++i) off.v[i] = ttot.v[i] = 0.0;
#pragma unroll
  for (int w2 = 0; w2 < GW; ++w2) {
#pragma unroll
    for (int i = 0; i < L; ++i) {
      const double x = tl->gx[g][w2][i];
      if (w2 < gw) off.v[i] = __dadd_rn(off.v[i], x);
      ttot.v[i] = __dadd_rn(ttot.v[i], x);
    }
  }
  trace_w0(P, 11, t);

  // ---- phase 3: transform at tied-block ends (Breslow), passes with work only ----
  if (wany) {
    double cf[NF], cr[NU > 0 ? NU : 1];
    {
      const double k1 = __dsub_rn(ss.phi, 1.0);
      const bool reset_f = tcv[6] != 0.0;
#pragma unroll
      for (int i = 0; i < NF; ++i) {
        const int f = (NF == 2 && i == 1) ? 1 : i;  // IND: lanes (a, b)
        double v = __dadd_rn(tcv[f], __dmul_rn(k1, tcv[3 + f]));
        if (!reset_f) v = __dadd_rn(ss.cin_f[f], v);
        cf[i] = v;
      }
      if constexpr (FG) {
        const bool reset_r = tcv[14] != 0.0;
#pragma unroll
        for (int i = 0; i < NU; ++i) {
          const int f = (NU == 2 && i == 1) ? 1 : i;
          double v = __dadd_rn(tcv[8 + f], __dmul_rn(k1, tcv[11 + f]));
          if (!reset_r) v = __dadd_rn(v, ss.cin_r[f]);
          cr[i] = v;  // u-weighted rows of this tile and the rest of the stratum
        }
      }
    }
#pragma unroll
    for (int pp = 0; pp < PPW; ++pp) {
      if (!((wany >> pp) & 1u)) continue;
      const int tr = (gw * PPW + pp) * 32 + lane;
      Rows R;
      load_rows(tr, R);
      Lanes<L> run;
#pragma unroll
      for (int i = 0; i < L; ++i) run.v[i] = __dadd_rn(off.v[i], st[pp].v[i]);
#pragma unroll
      for (int m = 0; m < kIpt; ++m) {
        const Lanes<L> rv = row_val(R, m);
#pragma unroll
        for (int i = 0; i < L; ++i) run.v[i] = __dadd_rn(run.v[i], rv.v[i]);
        if (!(R.cw[m] & kWork)) continue;
        if (KIND == kSlotLoglik && (R.cw[m] & kCodeEvent))
          acc0 = __dadd_rn(acc0, __ldcg(P.eta + row0 + tr * kIpt + m));
        const uint32_t d = R.cw[m] & kCodeCount;
        if (!d) continue;
        double den = __dadd_rn(cf[0], run.v[0]);
        double n1 = 0.0, n2 = 0.0;
        if constexpr (NF >= 2) {
          n1 = __dadd_rn(cf[1], run.v[1]);
          n2 = IND ? n1 : __dadd_rn(cf[NF - 1], run.v[NF - 1]);
        }
        if constexpr (FG) {
          // u-weighted suffix strictly after this row, inside the stratum:
          // S(k+1) = RcarryTot - inclusive in-tile prefix
          const double gk = g_of(R.cw[m], R.gv[m]);  // G at the block end
          den = __dadd_rn(den, __dmul_rn(gk, __dsub_rn(cr[0], run.v[NF])));
          if constexpr (NF >= 2) {
            n1 = __dadd_rn(n1, __dmul_rn(gk, __dsub_rn(cr[1], run.v[NF + 1])));
            if constexpr (!IND)
              n2 = __dadd_rn(n2, __dmul_rn(gk, __dsub_rn(cr[NU - 1], run.v[NF + NU - 1])));
            else
              n2 = n1;
          }
        }
        const double cnt = static_cast<double>(d);
        if (!(den > 0.0)) {
          bad = 1;
        } else if constexpr (KIND == kSlotGrad) {
          const double rinv = __drcp_rn(den);
          const double Gm = __dmul_rn(n1, rinv);
          const double Hm = IND ? Gm : __dmul_rn(n2, rinv);
          acc0 = __dadd_rn(acc0, __dmul_rn(cnt, Gm));
          acc1 = __dadd_rn(acc1, __dmul_rn(cnt, __dsub_rn(Hm, __dmul_rn(Gm, Gm))));
        } else {
          acc1 = __dadd_rn(acc1, __dmul_rn(cnt, log(den)));
        }
      }
    }
  }
  trace_w0(P, 12, t);

  // ---- the next slot's per-tile record (from the patched staged tile) ----
  if constexpr (FUSED) {
    if (gw == 0 && lane == 0) {
      double* rec = rec_at<FG>(P, tl, t, inf.li);
      rec[kRa] = ttot.v[0];
      rec[kRb] = ttot.v[NF];
      rec[kRc] = ttot.v[NF];
      rec[kRsa] = ttot.v[1];  // indicator scan column: its b lane is sum e over its rows
      rec[kRsb] = ttot.v[NF + 1];
      rec[kRsc] = ttot.v[NF + 1];
    }
  } else if (!(P.dbg & 2)) {
    double rb = 0.0, rc = 0.0, rsa = 0.0, rsb = 0.0, rsc = 0.0;
    double rub = 0.0, ruc = 0.0, rusa = 0.0, rusb = 0.0, rusc = 0.0;
    const bool n_ind = ss.nind != 0;
    const bool ccd_cur = P.mode == kModeCcd && has_cur;
    auto in_cur = [&](int lr) {
      return dcur ? (__ldg(dcur + row0 + lr) != 0.0) : (((xm[lr >> 3] >> (lr & 7)) & 1u) != 0u);
    };
    // dense next column: own rows; else the tile's slice of its index list
    const int nlim = dnxt ? kTileRows : Ln.cnt;
    for (int i = gt; i < nlim; i += GT) {
      int lr;
      double x;
      if (dnxt) {
        lr = i;
        x = __ldg(dnxt + row0 + lr);
        if (x == 0.0) continue;
      } else {
        lr = static_cast<int>(list_at(lnext, Ln, P.row_idx, i) - row0);
        x = n_ind ? 1.0 : P.vals[Ln.lo + i];
      }
      const double ev = *e_at(sb, lr);
      const double eb = __dmul_rn(ev, x);
      const double ec = __dmul_rn(eb, x);
      rb = __dadd_rn(rb, eb);
      rc = __dadd_rn(rc, ec);
      double u = 0.0;
      if constexpr (FG) {
        if (code_at(sc, lr) & kCodeCompeting)
          u = u_of(code_at(sc, lr), *reinterpret_cast<const double*>(sg + swz<128>(lr * 8)));
        rub = __dadd_rn(rub, __dmul_rn(u, eb));
        ruc = __dadd_rn(ruc, __dmul_rn(u, ec));
      }
      if (ccd_cur && in_cur(lr)) {
        rsb = __dadd_rn(rsb, eb);
        rsc = __dadd_rn(rsc, ec);
        if constexpr (FG) {
          rusb = __dadd_rn(rusb, __dmul_rn(u, eb));
          rusc = __dadd_rn(rusc, __dmul_rn(u, ec));
        }
      }
    }
    if (ccd_cur) {
      const int clim = dcur ? kTileRows : Lc.cnt;
      for (int i = gt; i < clim; i += GT) {
        int lr;
        if (dcur) {
          lr = i;
          if (__ldg(dcur + row0 + lr) == 0.0) continue;
        } else {
          lr = static_cast<int>(list_at(lcur, Lc, P.row_idx, i) - row0);
        }
        const double ev = *e_at(sb, lr);
        rsa = __dadd_rn(rsa, ev);
        if constexpr (FG) {
          if (code_at(sc, lr) & kCodeCompeting)
            rusa = __dadd_rn(
                rusa, __dmul_rn(u_of(code_at(sc, lr), *reinterpret_cast<const double*>(sg + swz<128>(lr * 8))),
                                ev));
        }
      }
    }
    constexpr int NR = FG ? 10 : 5;
    double rv[NR] = {rb, rc, rsa, rsb, rsc};
    if constexpr (FG) {
      rv[5] = rub;
      rv[6] = ruc;
      rv[7] = rusa;
      rv[8] = rusb;
      rv[9] = rusc;
    }
    // Fine-Gray (8-warp groups, 10 partials): warps past both slices summed
    // nothing (their partials are +0.0 exactly), so they skip the shuffles
    // (warp-uniform).  Cox keeps the unconditional form: the branch changed
    // the whole kernel's register allocation and cost 7% on the fused path.
    const bool warp_had =
        !FG || gw * 32 < nlim || (ccd_cur && gw * 32 < (dcur ? kTileRows : Lc.cnt));
    if (warp_had) {
#pragma unroll
      for (int i = 0; i < NR; ++i) rv[i] = warp_sum(rv[i]);
    }
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < NR; ++i) tl->gr[g][gw][i] = rv[i];
    }
  }
  mark<FG>(tl, 0x13u | (static_cast<unsigned>(t & 0xffff) << 8));
  if constexpr (!FUSED) group_sync<FG>(g);
  if (!FUSED && gw == 0 && lane == 0 && !(P.dbg & 2)) {
    constexpr int NR = FG ? 10 : 5;
    double s[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) s[i] = 0.0;
    for (int w2 = 0; w2 < GW; ++w2) {
#pragma unroll
      for (int i = 0; i < NR; ++i) s[i] = __dadd_rn(s[i], tl->gr[g][w2][i]);
    }
    double* rec = rec_at<FG>(P, tl, t, inf.li);
    rec[kRa] = ttot.v[0];
    rec[kRb] = s[0];
    rec[kRc] = s[1];
    rec[kRsa] = s[2];
    rec[kRsb] = s[3];
    rec[kRsc] = s[4];
    if constexpr (FG) {
      rec[kRua] = ttot.v[NF];
      rec[kRub] = s[5];
      rec[kRuc] = s[6];
      rec[kRusa] = s[7];
      rec[kRusb] = s[8];
      rec[kRusc] = s[9];
    }
  }
  trace_w0(P, 13, t);
}

// returns true if the stage was already released (fused path)
template <bool FG>
__device__ __forceinline__ bool consume_tile(const CycleParams& P, Tail<FG>* tl, unsigned char* sb,
                                             const StageInfo& inf, const SlotState& ss, int g,
                                             int gw, int lane, int par, double& acc0,
                                             double& acc1, int& bad, uint64_t* empty_bar) {
  if constexpr (!FG) {
    if (ss.fused) {
      process_tile<false, true, kSlotGrad, true>(P, tl, sb, inf, ss, g, gw, lane, par, acc0, acc1,
                                                 bad, empty_bar);
      return false;
    }
  }
  if (ss.kind == kSlotLoglik)
    process_tile<FG, true, kSlotLoglik>(P, tl, sb, inf, ss, g, gw, lane, par, acc0, acc1, bad, empty_bar);
  else if (ss.cind)
    process_tile<FG, true, kSlotGrad>(P, tl, sb, inf, ss, g, gw, lane, par, acc0, acc1, bad, empty_bar);
  else
    process_tile<FG, false, kSlotGrad>(P, tl, sb, inf, ss, g, gw, lane, par, acc0, acc1, bad, empty_bar);
  return false;
}

// ---------------------------------------------------------------------------
// records computed from global memory (launch prologue, refresh): for every
// tile of the range, warp per tile.  Optional virtual pending update is not
// needed here: callers commit first.
// ---------------------------------------------------------------------------
template <bool FG>
__device__ __forceinline__ void records_from_global(const CycleParams& P, Tail<FG>* tl, int t0, int tc,
                                                 long long ncol, int warp, int lane) {
  constexpr int W = Geo<FG>::kW;
  const size_t nt1 = size_t(P.ntiles) + 1;
  const bool n_ind = ncol >= 0 && (!P.has_vals || P.col_ind[ncol]);
  for (int i = warp; i < tc; i += W) {
    const int t = t0 + i;
    const long long row0 = static_cast<long long>(t) * kTileRows;
    double a = 0.0, ua = 0.0;
    for (int k = lane; k < kTileRows; k += 32) {
      const double ev = __ldcg(P.e + row0 + k);
      a = __dadd_rn(a, ev);
      if constexpr (FG) {
        if (P.code[row0 + k] & kCodeCompeting) ua = __dadd_rn(ua, __dmul_rn(__drcp_rn(P.g[row0 + k]), ev));
      }
    }
    double rb = 0.0, rc = 0.0, rub = 0.0, ruc = 0.0;
    if (ncol >= 0) {
      const long long cb = P.col_ptr[ncol];
      const long long lo = cb + P.tile_ptr[size_t(ncol) * nt1 + t];
      const long long hi = cb + P.tile_ptr[size_t(ncol) * nt1 + t + 1];
      for (long long k = lo + lane; k < hi; k += 32) {
        const int32_t r = P.row_idx[k];
        const double ev = __ldcg(P.e + r);
        const double x = n_ind ? 1.0 : P.vals[k];
        const double eb = __dmul_rn(ev, x), ec = __dmul_rn(eb, x);
        rb = __dadd_rn(rb, eb);
        rc = __dadd_rn(rc, ec);
        if constexpr (FG) {
          if (P.code[r] & kCodeCompeting) {
            const double u = __drcp_rn(P.g[r]);
            rub = __dadd_rn(rub, __dmul_rn(u, eb));
            ruc = __dadd_rn(ruc, __dmul_rn(u, ec));
          }
        }
      }
    }
    a = warp_sum(a);
    rb = warp_sum(rb);
    rc = warp_sum(rc);
    if constexpr (FG) {
      ua = warp_sum(ua);
      rub = warp_sum(rub);
      ruc = warp_sum(ruc);
    }
    if (lane == 0) {
      double* rec = rec_at<FG>(P, tl, t, i);
      rec[kRa] = a;
      rec[kRb] = rb;
      rec[kRc] = rc;
      rec[kRsa] = rec[kRsb] = rec[kRsc] = 0.0;
      if constexpr (FG) {
        rec[kRua] = ua;
        rec[kRub] = rub;
        rec[kRuc] = ruc;
        rec[kRusa] = rec[kRusb] = rec[kRusc] = 0.0;
      }
    }
  }
}

// In-kernel refresh (src/engine.cpp:120-160 via :217): the accepted update of
// column `col` is applied to eta over this CTA's rows, then exp(eta) is
// rebuilt for every row from the incrementally maintained eta (the eta drift
// is a few ulps; load_beta()/refresh() API calls rebuild eta = X beta), and the
// tile records are recomputed from the fresh values.  Returns max |eta|.
template <bool FG>
__device__ __forceinline__ double refresh_tiles(const CycleParams& P, Tail<FG>* tl, int t0, int tc,
                                             long long col, double delta, long long ncol, int warp,
                                             int lane) {
  constexpr int W = Geo<FG>::kW;
  const size_t nt1 = size_t(P.ntiles) + 1;
  const bool c_ind = !P.has_vals || P.col_ind[col];
  const bool n_ind = ncol >= 0 && (!P.has_vals || P.col_ind[ncol]);
  double mx = 0.0;
  for (int i = warp; i < tc; i += W) {
    const int t = t0 + i;
    const long long row0 = static_cast<long long>(t) * kTileRows;
    {  // eta += x * delta over the tile's rows of the updated column
      const long long cb = P.col_ptr[col];
      const long long lo = cb + P.tile_ptr[size_t(col) * nt1 + t];
      const long long hi = cb + P.tile_ptr[size_t(col) * nt1 + t + 1];
      for (long long k = lo + lane; k < hi; k += 32) {
        const int32_t r = P.row_idx[k];
        if (P.code[r] & kCodeMasked) continue;
        P.eta[r] = __dadd_rn(__ldcg(P.eta + r), __dmul_rn(c_ind ? 1.0 : P.vals[k], delta));
      }
      __syncwarp();
      __threadfence_block();
    }
    double a = 0.0, ua = 0.0;
    // lane owns row pairs (2*lane + 64*j): 16-byte loads, 8 pairs in flight
    // (masked / padding rows keep exp(eta) = 0)
#pragma unroll 8
    for (int j = 0; j < kTileRows / 64; ++j) {
      const long long r = row0 + 2 * lane + 64 * j;
      const uint2 cw = __ldcg(reinterpret_cast<const uint2*>(P.code + r));
      const double2 et = __ldcg(reinterpret_cast<const double2*>(P.eta + r));
      const bool m0 = (cw.x & kCodeMasked) != 0, m1 = (cw.y & kCodeMasked) != 0;
      double2 ev;
      ev.x = m0 ? 0.0 : exp(et.x);
      ev.y = m1 ? 0.0 : exp(et.y);
      *reinterpret_cast<double2*>(P.e + r) = ev;
      if (!m0) {
        mx = fmax(mx, fabs(et.x));
        a = __dadd_rn(a, ev.x);
      }
      if (!m1) {
        mx = fmax(mx, fabs(et.y));
        a = __dadd_rn(a, ev.y);
      }
      if constexpr (FG) {
        if (cw.x & kCodeCompeting) ua = __dadd_rn(ua, __dmul_rn(__drcp_rn(P.g[r]), ev.x));
        if (cw.y & kCodeCompeting) ua = __dadd_rn(ua, __dmul_rn(__drcp_rn(P.g[r + 1]), ev.y));
      }
    }
    __syncwarp();
    __threadfence_block();
    double rb = 0.0, rc = 0.0, rub = 0.0, ruc = 0.0;
    if (ncol >= 0) {
      const long long cb = P.col_ptr[ncol];
      const long long lo = cb + P.tile_ptr[size_t(ncol) * nt1 + t];
      const long long hi = cb + P.tile_ptr[size_t(ncol) * nt1 + t + 1];
      for (long long k = lo + lane; k < hi; k += 32) {
        const int32_t r = P.row_idx[k];
        const double ev = __ldcg(P.e + r);
        const double x = n_ind ? 1.0 : P.vals[k];
        const double eb = __dmul_rn(ev, x), ec = __dmul_rn(eb, x);
        rb = __dadd_rn(rb, eb);
        rc = __dadd_rn(rc, ec);
        if constexpr (FG) {
          if (P.code[r] & kCodeCompeting) {
            const double u = __drcp_rn(P.g[r]);
            rub = __dadd_rn(rub, __dmul_rn(u, eb));
            ruc = __dadd_rn(ruc, __dmul_rn(u, ec));
          }
        }
      }
    }
    a = warp_sum(a);
    rb = warp_sum(rb);
    rc = warp_sum(rc);
    if constexpr (FG) {
      ua = warp_sum(ua);
      rub = warp_sum(rub);
      ruc = warp_sum(ruc);
    }
    if (lane == 0) {
      double* rec = rec_at<FG>(P, tl, t, i);
      rec[kRa] = a;
      rec[kRb] = rb;
      rec[kRc] = rc;
      rec[kRsa] = rec[kRsb] = rec[kRsc] = 0.0;
      if constexpr (FG) {
        rec[kRua] = ua;
        rec[kRub] = rub;
        rec[kRuc] = ruc;
        rec[kRusa] = rec[kRusb] = rec[kRusc] = 0.0;
      }
    }
  }
  return mx;
}

// Sparse correction of the records for a VALUED pending update (exp is not
// linear in delta): rec += sum over the pending rows of (e_new - e_old) terms.
template <bool FG>
__device__ __forceinline__ void correct_records_valued(const CycleParams& P, Tail<FG>* tl, int t0, int tc,
                                                    long long pcol, double delta, long long ncol,
                                                    int warp, int lane) {
  constexpr int W = Geo<FG>::kW;
  const size_t nt1 = size_t(P.ntiles) + 1;
  const bool n_ind = ncol >= 0 && (!P.has_vals || P.col_ind[ncol]);
  for (int i = warp; i < tc; i += W) {
    const int t = t0 + i;
    const long long cb = P.col_ptr[pcol];
    const long long lo = cb + P.tile_ptr[size_t(pcol) * nt1 + t];
    const long long hi = cb + P.tile_ptr[size_t(pcol) * nt1 + t + 1];
    long long nlo = 0, nhi = 0;
    if (ncol >= 0) {
      const long long nb = P.col_ptr[ncol];
      nlo = nb + P.tile_ptr[size_t(ncol) * nt1 + t];
      nhi = nb + P.tile_ptr[size_t(ncol) * nt1 + t + 1];
    }
    double da = 0.0, db = 0.0, dc = 0.0, dua = 0.0, dub = 0.0, duc = 0.0;
    for (long long k = lo + lane; k < hi; k += 32) {
      const int32_t r = P.row_idx[k];
      if (P.code[r] & kCodeMasked) continue;
      const double eo = __ldcg(P.e + r);
      const double en = exp(__dadd_rn(__ldcg(P.eta + r), __dmul_rn(P.vals[k], delta)));
      const double de = __dsub_rn(en, eo);
      double u = 0.0;
      if constexpr (FG) {
        if (P.code[r] & kCodeCompeting) u = __drcp_rn(P.g[r]);
      }
      da = __dadd_rn(da, de);
      if constexpr (FG) dua = __dadd_rn(dua, __dmul_rn(u, de));
      // is r also a row of the next column?
      long long a = nlo, b = nhi;
      while (a < b) {
        const long long mid = (a + b) >> 1;
        if (P.row_idx[mid] < r)
          a = mid + 1;
        else
          b = mid;
      }
      if (a < nhi && P.row_idx[a] == r) {
        const double x = n_ind ? 1.0 : P.vals[a];
        const double eb = __dmul_rn(de, x), ec = __dmul_rn(eb, x);
        db = __dadd_rn(db, eb);
        dc = __dadd_rn(dc, ec);
        if constexpr (FG) {
          dub = __dadd_rn(dub, __dmul_rn(u, eb));
          duc = __dadd_rn(duc, __dmul_rn(u, ec));
        }
      }
    }
    da = warp_sum(da);
    db = warp_sum(db);
    dc = warp_sum(dc);
    if constexpr (FG) {
      dua = warp_sum(dua);
      dub = warp_sum(dub);
      duc = warp_sum(duc);
    }
    if (lane == 0) {
      double* rec = rec_at<FG>(P, tl, t, i);
      rec[kRa] = __dadd_rn(rec[kRa], da);
      rec[kRb] = __dadd_rn(rec[kRb], db);
      rec[kRc] = __dadd_rn(rec[kRc], dc);
      rec[kRsa] = rec[kRsb] = rec[kRsc] = 0.0;
      if constexpr (FG) {
        rec[kRua] = __dadd_rn(rec[kRua], dua);
        rec[kRub] = __dadd_rn(rec[kRub], dub);
        rec[kRuc] = __dadd_rn(rec[kRuc], duc);
        rec[kRusa] = rec[kRusb] = rec[kRusc] = 0.0;
      }
    }
  }
}

// Exact validate-before-mutate over this CTA's rows (src/engine.cpp:171-190).
__device__ __forceinline__ int validate_rows(const CycleParams& P, int t0, int tc, long long col, double delta,
                             int tid, int nthr) {
  const size_t nt1 = size_t(P.ntiles) + 1;
  const long long cb = P.col_ptr[col];
  const long long lo = cb + P.tile_ptr[size_t(col) * nt1 + t0];
  const long long hi = cb + P.tile_ptr[size_t(col) * nt1 + t0 + tc];
  const bool ind = !P.has_vals || P.col_ind[col];
  int over = 0;
  for (long long k = lo + tid; k < hi; k += nthr) {
    const int32_t r = P.row_idx[k];
    if (P.code[r] & kCodeMasked) continue;
    const double x = ind ? 1.0 : P.vals[k];
    if (fabs(__dadd_rn(__ldcg(P.eta + r), __dmul_rn(x, delta))) > kXbetaBound) over = 1;
  }
  return over;
}

// ---------------------------------------------------------------------------
// In-range segmented scans of the per-tile records (warp 0): per-tile carries
// (uncorrected value + s-part) and the CTA payload aggregates.
// ---------------------------------------------------------------------------
template <bool FG>
__device__ __forceinline__ void range_scan(const CycleParams& P, Tail<FG>* tl, int t0, int tc, double* pay,
                                        int lane, bool fwd = true) {
  // forward: exclusive segmented prefix, flags at stratum-first tiles
  double carry[6] = {0, 0, 0, 0, 0, 0};
  int seen = 0;  // a stratum-first tile was passed inside the range
  for (int ch = 0; fwd && ch < tc; ch += 32) {
    const int i = ch + lane;
    const bool valid = i < tc;
    const int t = t0 + i;
    double v[6];
    int f = 0;
    if (valid) {
      const double* rec = rec_at<FG>(P, tl, t, i);
#pragma unroll
      for (int k = 0; k < 6; ++k) v[k] = ld_rc<FG>(rec + k, i);
      f = P.tile_first[t] ? 1 : 0;
    } else {
#pragma unroll
      for (int k = 0; k < 6; ++k) v[k] = 0.0;
    }
    // segmented inclusive scan (x earlier, y later): y.f ? y.v : x.v + y.v
    int sf = f;
    double s[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) s[k] = v[k];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int of = __shfl_up_sync(0xffffffffu, sf, d);
      double o[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) o[k] = __shfl_up_sync(0xffffffffu, s[k], d);
      if (lane >= d) {
        if (!sf) {
#pragma unroll
          for (int k = 0; k < 6; ++k) s[k] = __dadd_rn(o[k], s[k]);
        }
        sf |= of;
      }
    }
    // exclusive: previous lane's inclusive, combined after the chunk carry
    int ef = __shfl_up_sync(0xffffffffu, sf, 1);
    double ex[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) ex[k] = __shfl_up_sync(0xffffffffu, s[k], 1);
    if (lane == 0) {
      ef = 0;
#pragma unroll
      for (int k = 0; k < 6; ++k) ex[k] = 0.0;
    }
    double outv[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) outv[k] = ef ? ex[k] : __dadd_rn(carry[k], ex[k]);
    const int reset = seen | ef | f;
    if (f) {
#pragma unroll
      for (int k = 0; k < 6; ++k) outv[k] = 0.0;
    }
    if (valid) {
      double* tcp = car_at<FG>(P, tl, t, i);
#pragma unroll
      for (int k = 0; k < 6; ++k) tcp[k] = outv[k];
      tcp[6] = reset ? 1.0 : 0.0;
    }
    // chunk total -> carry
    const int last = min(31, tc - ch - 1);
    const int tf = __shfl_sync(0xffffffffu, sf, last);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const double tv = __shfl_sync(0xffffffffu, s[k], last);
      carry[k] = tf ? tv : __dadd_rn(carry[k], tv);
    }
    seen |= tf;
  }
  if (lane == 0 && fwd) {
    pay[3] = seen ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) pay[4 + k] = carry[k];
  }
  if constexpr (FG) {
    // reverse: inclusive segmented suffix; element i is cut from i+1 when
    // tile i+1 starts a stratum
    double rc[6] = {0, 0, 0, 0, 0, 0};
    int rseen = 0;  // a stratum-first tile lies after the current position
    const int nch = (tc + 31) / 32;
    for (int cc = nch - 1; cc >= 0; --cc) {
      const int ch = cc * 32;
      const int i = ch + 31 - lane;  // lane 0 = highest tile of the chunk
      const bool valid = i < tc;
      const int t = t0 + i;
      double v[6];
      int fnext = 0;  // tile i+1 (inside the range) starts a stratum
      if (valid) {
        const double* rec = rec_at<FG>(P, tl, t, i);
#pragma unroll
        for (int k = 0; k < 6; ++k) v[k] = ld_rc<FG>(rec + 6 + k, i);
        fnext = (i + 1 < tc && P.tile_first[t + 1]) ? 1 : 0;
      } else {
#pragma unroll
        for (int k = 0; k < 6; ++k) v[k] = 0.0;
      }
      int sf = fnext;
      double s[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) s[k] = v[k];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int of = __shfl_up_sync(0xffffffffu, sf, d);
        double o[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) o[k] = __shfl_up_sync(0xffffffffu, s[k], d);
        if (lane >= d) {
          if (!sf) {
#pragma unroll
            for (int k = 0; k < 6; ++k) s[k] = __dadd_rn(o[k], s[k]);
          }
          sf |= of;
        }
      }
      // inclusive value at tile i, plus the carry from higher chunks unless cut
      double outv[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) outv[k] = sf ? s[k] : __dadd_rn(rc[k], s[k]);
      const int reset = sf | rseen;
      if (valid) {
        double* tcp = car_at<FG>(P, tl, t, i);
#pragma unroll
        for (int k = 0; k < 6; ++k) tcp[8 + k] = outv[k];
        tcp[14] = reset ? 1.0 : 0.0;
      }
      // carry for the next (lower) chunk: the value at the chunk's lowest valid tile
      const int lowest = 31 - 0;  // lane holding i = ch (always valid)
      const int lf = __shfl_sync(0xffffffffu, sf, lowest);
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const double tv = __shfl_sync(0xffffffffu, s[k], lowest);
        rc[k] = lf ? tv : __dadd_rn(rc[k], tv);
      }
      rseen |= lf;
      // a stratum start at the chunk's lowest tile cuts everything below it
      const int low_first = P.tile_first[t0 + ch] ? 1 : 0;
      if (low_first) {
#pragma unroll
        for (int k = 0; k < 6; ++k) rc[k] = 0.0;
        rseen = 1;
      }
    }
    // head = rows before the first stratum-first tile of the range
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 6; ++k) pay[10 + k] = rc[k];
    }
  }
}

// The control warp reads the published payloads (lane l <- CTAs l, l+32, ...)
// and reduces them in a fixed order: the slot partials over all CTAs (the same
// order in every CTA => identical results everywhere), the fwd tails of CTAs
// [cstar, cta) and the rev heads of CTAs (cta, cend] (segmented by strata).
// Result: tl->gs[0..2] partials, [3..8] fwd (a,b,c,sa,sb,sc), [9..14] rev.
template <bool FG>
__device__ __forceinline__ void gather_warp(const CycleParams& P, const double* pay_all, int cta,
                                            int cstar, int cend, Tail<FG>* tl, int lane) {
  constexpr int NV = FG ? 15 : 9;
  double v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = 0.0;
  // every CTA's payload row in shared memory with ONE bulk copy (large
  // transactions: the rows are read by all CTAs at once), then reduce there
  const int G = P.grid;
  const long long gt0 = clock64();
  if (lane == 0) {
    const uint32_t bytes = static_cast<uint32_t>(G) * kPayStride * 8u;
    fence_proxy_async_global();  // generic-proxy payload writes -> async-proxy read
    mbar_arrive_expect_tx(&tl->gbar, bytes);
    bulk_load_1d(&tl->gbuf[0][0], pay_all, bytes, &tl->gbar);
  }
  mbar_wait(&tl->gbar, tl->gphase);
  __syncwarp();
  if (lane == 0) tl->gphase ^= 1u;
  const long long gt1 = clock64();
  for (int c = lane; c < G; c += 32) {
    const double* x = tl->gbuf[c];
    v[0] = __dadd_rn(v[0], x[0]);
    v[1] = __dadd_rn(v[1], x[1]);
    v[2] = __dadd_rn(v[2], x[2]);
    if (c >= cstar && c < cta) {
#pragma unroll
      for (int i = 0; i < 6; ++i) v[3 + i] = __dadd_rn(v[3 + i], x[4 + i]);
    }
    if constexpr (FG) {
      if (c > cta && c <= cend) {
#pragma unroll
        for (int i = 0; i < 6; ++i) v[9 + i] = __dadd_rn(v[9 + i], x[10 + i]);
      }
    }
  }
  const long long gt2 = clock64();
  // cross-lane reduction through shared memory (fixed lane order; lane i sums value i)
#pragma unroll
  for (int i = 0; i < NV; ++i) tl->gred[lane][i] = v[i];
  __syncwarp();
  if (lane < NV) {
    double r = 0.0;
#pragma unroll 8
    for (int l = 0; l < 32; ++l) r = __dadd_rn(r, tl->gred[l][lane]);
    tl->gs[lane] = r;
  }
  __syncwarp();
  const long long gt3 = clock64();
  if (lane == 0 && (P.dbg & 256)) {
    tl->cs.ph[6] += gt1 - gt0;
    tl->cs.ph[7] += gt2 - gt1;
    tl->cs.ph[8] += gt3 - gt2;
  }
}

// corrected CTA carries from the gathered sums (thread 0)
template <bool FG>
__device__ __forceinline__ void set_carry_in(const CycleParams& P, Tail<FG>* tl, double k1) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double v = __dadd_rn(tl->gs[3 + i], __dmul_rn(k1, tl->gs[6 + i]));
    if (tl->ext_f) {  // shards before this one
      const double x = P.nranks > 1 ? __dadd_rn(tl->xext[i], __dmul_rn(k1, tl->xext[3 + i]))
                                    : __ldcg(P.ext + i);
      v = __dadd_rn(x, v);
    }
    tl->ss.cin_f[i] = v;
  }
  if constexpr (FG) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double v = __dadd_rn(tl->gs[9 + i], __dmul_rn(k1, tl->gs[12 + i]));
      if (tl->ext_r) {  // shards after this one
        const double x = P.nranks > 1 ? __dadd_rn(tl->xext[6 + i], __dmul_rn(k1, tl->xext[9 + i]))
                                      : __ldcg(P.ext + 4 + i);
        v = __dadd_rn(v, x);
      }
      tl->ss.cin_r[i] = v;
    }
  }
}

// This shard's aggregate from the CTA payloads (warp 0 of CTA 0; fixed order):
// fwd tail = tails of CTAs from the last stratum-start CTA on, rev head =
// heads of CTAs up to the first stratum-start CTA (carry sums of other shards
// are composed by the host, segmented over shards).
template <bool FG>
__device__ void shard_aggregate(const CycleParams& P, const double* pall, const Tail<FG>* tl,
                                int lane) {
  const int G = P.grid;
  int last = -1, first = G;
  for (int c = 0; c < G; ++c)
    if (tl->cflag[c]) {
      if (last < c) last = c;
      if (first > c) first = c;
    }
  double f[3] = {0, 0, 0}, r[3] = {0, 0, 0};
  for (int c = lane; c < G; c += 32) {
    const double* py = pall + size_t(c) * kPayStride;
    if (c >= (last < 0 ? 0 : last)) {
#pragma unroll
      for (int k = 0; k < 3; ++k) f[k] = __dadd_rn(f[k], __ldcg(py + 4 + k));
    }
    if (FG && c <= (first == G ? G - 1 : first)) {
#pragma unroll
      for (int k = 0; k < 3; ++k) r[k] = __dadd_rn(r[k], __ldcg(py + 10 + k));
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    f[k] = warp_sum(f[k]);
    r[k] = warp_sum(r[k]);
  }
  if (lane == 0) {
    P.shard_out[0] = last >= 0 ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      P.shard_out[1 + k] = f[k];
      P.shard_out[4 + k] = r[k];
    }
    P.shard_out[7] = first == 0 ? 1.0 : 0.0;  // the shard's first tile starts a stratum
  }
}

// ---------------------------------------------------------------------------
// consumer side of the rare all-warp tasks (exact validation, refresh,
// valued-update record correction): wait at GO, run the task, arrive at DONE,
// until the control warp hands out NEXT (the next slot) or EXIT
// ---------------------------------------------------------------------------
template <bool FG>
__device__ __forceinline__ void consumer_tasks(const CycleParams& P, Tail<FG>* tl, int t0, int tc,
                                               int warp, int lane, int tid) {
  constexpr int NC = 32 * Geo<FG>::kW, NB = NC + 32;
  for (;;) {
    bar_sync_n(kBarGo, NB);
    const int task = *reinterpret_cast<volatile int*>(&tl->task);
    if (task == kTaskNext || task == kTaskExit) return;
    const long long col = tl->tcol, ncol = tl->tncol;
    const double delta = tl->tdelta;
    if (task == kTaskExact) {
      if (validate_rows(P, t0, tc, col, delta, tid, NC)) tl->flag = 1;
    } else if (task == kTaskRefresh) {
      double m = refresh_tiles<FG>(P, tl, t0, tc, col, delta, ncol, warp, lane);
      fence_proxy_async_global();
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, d));
      if (lane == 0) tl->wpart[warp][3] = m;
      __threadfence();
    } else if (task == kTaskValued) {
      correct_records_valued<FG>(P, tl, t0, tc, col, delta, ncol, warp, lane);
      __threadfence();
    }
    __threadfence_block();
    bar_arrive_n(kBarDone, NB);
  }
}

// ---------------------------------------------------------------------------
// Cross-shard exchange (patient-sharded fit, config C5): after a grid exchange
// and gather, CTA 0 of every shard publishes the shard's aggregate — slot
// partials, the segmented fwd tail from its last stratum-starting CTA (with
// s-parts), the rev head up to its first one, aux values — to every shard's
// buffer with peer stores, then a system-scope release arrival on every
// shard's counter; every CTA of every shard waits for all arrivals and
// combines the rows in RANK order: identical partial sums (hence identical
// coordinate steps) everywhere, and the carries from the other shards
// (src/scan_kernels.hpp:114-134 combines chunks the same way).  Lane 0.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <bool FG>
__device__ void cross_shard(const CycleParams& P, Tail<FG>* tl, int cta, double aux0, double aux1) {
  const int R = P.nranks, me = P.rank, G = P.grid;
  CcdState& cs = tl->cs;
  const unsigned long long xc = cs.xr_count;
  const size_t slot = (xc & 1ull) * size_t(R);
  if (cta == 0) {
    double row[kXrStride];
#pragma unroll
    for (int i = 0; i < kXrStride; ++i) row[i] = 0.0;
    row[0] = tl->gs[0];
    row[1] = tl->gs[1];
    row[2] = tl->gs[2];
    int last = -1, first = G;
    for (int c = 0; c < G; ++c)
      if (tl->cflag[c]) {
        last = c;
        if (first == G) first = c;
      }
    row[3] = last >= 0 ? 1.0 : 0.0;
    for (int c = (last < 0 ? 0 : last); c < G; ++c)
#pragma unroll
      for (int i = 0; i < 6; ++i) row[4 + i] = __dadd_rn(row[4 + i], tl->gbuf[c][4 + i]);
    if constexpr (FG) {
      const int end = first == G ? G - 1 : first;
      for (int c = 0; c <= end; ++c)
#pragma unroll
        for (int i = 0; i < 6; ++i) row[10 + i] = __dadd_rn(row[10 + i], tl->gbuf[c][10 + i]);
    }
    row[16] = aux0;
    row[17] = aux1;
    for (int q = 0; q < R; ++q) {
      double* dst = P.xr_pay[q] + (slot + me) * kXrStride;
      for (int i = 0; i < 18; ++i) dst[i] = row[i];
    }
    // release-reduction at system scope: orders this thread's row stores
    // before the arrival (no separate fence round trip)
    if (P.xr_sys)  // peers on other GPUs (NVLink): system scope
      for (int q = 0; q < R; ++q)
        asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(P.xr_bar[q]) : "memory");
    else  // every shard on this device: gpu scope suffices
      for (int q = 0; q < R; ++q)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(P.xr_bar[q]) : "memory");
  }
  const unsigned target = static_cast<unsigned>(cs.xr_base + (xc + 1) * static_cast<unsigned long long>(R));
  const unsigned* mybar = P.xr_bar[me];
  const unsigned long long t0 = gtimer();
  unsigned it = 0;
  auto arrived = [&]() { return P.xr_sys ? ld_acquire_sys_u32(mybar) : ld_acquire_u32(mybar); };
  while (static_cast<int>(arrived() - target) < 0) {
    if ((++it & 1023u) == 0 && gtimer() - t0 > 2 * kWatchdogNs)
      watchdog_trap("cross-shard exchange", arrived(), target);
  }
  const double* rows = P.xr_pay[me] + slot * kXrStride;
  double g0 = 0.0, g1 = 0.0, g2 = 0.0, a0 = 0.0, a1 = 0.0;
  for (int q = 0; q < R; ++q) {
    const double* r = rows + size_t(q) * kXrStride;
    g0 = __dadd_rn(g0, __ldcv(r + 0));
    g1 = __dadd_rn(g1, __ldcv(r + 1));
    g2 = __dadd_rn(g2, __ldcv(r + 2));
    a0 = fmax(a0, __ldcv(r + 16));
    a1 = fmax(a1, __ldcv(r + 17));
  }
  tl->gs[0] = g0;
  tl->gs[1] = g1;
  tl->gs[2] = g2;
  tl->xaux[0] = a0;
  tl->xaux[1] = a1;
  // fwd: tails of shards start .. me-1 (start = the last earlier shard with a
  // stratum start); rev: heads of shards me+1 .. end (end = the first later
  // shard with a stratum start)
  int start = 0;
  for (int q = me - 1; q >= 0; --q)
    if (__ldcv(rows + size_t(q) * kXrStride + 3) != 0.0) {
      start = q;
      break;
    }
  double f[6] = {0, 0, 0, 0, 0, 0};
  for (int q = start; q < me; ++q)
#pragma unroll
    for (int i = 0; i < 6; ++i) f[i] = __dadd_rn(f[i], __ldcv(rows + size_t(q) * kXrStride + 4 + i));
#pragma unroll
  for (int i = 0; i < 6; ++i) tl->xext[i] = f[i];
  if constexpr (FG) {
    int end = R - 1;
    for (int q = me + 1; q < R; ++q)
      if (__ldcv(rows + size_t(q) * kXrStride + 3) != 0.0) {
        end = q;
        break;
      }
    double r6[6] = {0, 0, 0, 0, 0, 0};
    for (int q = me + 1; q <= end; ++q)
#pragma unroll
      for (int i = 0; i < 6; ++i)
        r6[i] = __dadd_rn(r6[i], __ldcv(rows + size_t(q) * kXrStride + 10 + i));
#pragma unroll
    for (int i = 0; i < 6; ++i) tl->xext[6 + i] = r6[i];
  }
  cs.xr_count = xc + 1;
}

// ---------------------------------------------------------------------------
// the control warp: per slot, the in-range carry scan of the records as the
// consumers release tiles, then (once the slot is consumed) the partial sums,
// the grid exchange, the fixed-order gather, Engine::finish + coordinate_step
// (replicated in every CTA) and the next slot's state.  Lane 0 runs the
// serial parts; the warp runs the gathers and full range scans.
// ---------------------------------------------------------------------------
template <bool FG>
__device__ __forceinline__ void control_warp(const CycleParams& P, Tail<FG>* tl, int cta, int t0,
                                          int tc, int lane) {
  using Gm = Geo<FG>;
  constexpr int W = Gm::kW, NB = 32 * W + 32;
  const int G = P.grid;
  Ctl* ctl = P.ctl;
  SlotState& ss = tl->ss;
  const bool prof = (P.dbg & 256) && cta == kProfCta && lane == 0;
  // phase profile in shared memory (no local-memory array)
  long long* ph = tl->cs.ph;
  if (lane == 0)
    for (int i = 0; i < 16; ++i) ph[i] = 0;
  tl->cs.ph_t = clock64();
  auto pmark = [&](int i) {
    if (prof) {
      const long long n = clock64();
      ph[i] += n - tl->cs.ph_t;
      tl->cs.ph_t = n;
    }
  };
  // replicated CCD state (identical in every CTA: same inputs, same order),
  // kept in shared memory (written by lane 0)
  CcdState& cs = tl->cs;
  if (lane == 0) {
    cs.bar_target = static_cast<unsigned>(ctl->bar_base);
    cs.xr_base = ctl->xr_base;
    cs.xr_count = ctl->xr_count;
    cs.absmax = __longlong_as_double(static_cast<long long>(ctl->eta_absmax_bits));
    cs.slack = ctl->bound_slack;
    cs.accepted = ctl->accepted;
    cs.refreshes = ctl->refreshes;
    cs.skipped = ctl->skipped;
    cs.err = ctl->err_code;
    cs.err_col = ctl->err_col;
    cs.xi = 0;
    cs.qbase = 0;
    cs.tgo = 0;
    cs.tcons = 0;
    // accepted updates until the next refresh (accepted % interval == 0)
    cs.to_refresh = P.recompute_interval - (cs.accepted % P.recompute_interval);
  }
  __syncwarp();
  unsigned& bar_target = cs.bar_target;
  double& absmax = cs.absmax;
  double& slack = cs.slack;
  long long& accepted = cs.accepted;
  long long& refreshes = cs.refreshes;
  long long& skipped = cs.skipped;
  int& err = cs.err;
  long long& err_col = cs.err_col;
  int& xi = cs.xi;  // payload double buffer, indexed by the exchange count
  auto wbuf = [&]() { return P.cpay + (size_t(xi & 1) * G + cta) * kPayStride; };
  auto rbuf = [&](int x) { return P.cpay + size_t(x & 1) * G * kPayStride; };
  // auxiliary payload fields (rare paths)
  auto waux = [&]() {
    return P.cpay + size_t(2) * G * kPayStride + (size_t(xi & 1) * G + cta) * kPayAux;
  };
  auto raux = [&](int x) { return P.cpay + size_t(2) * G * kPayStride + size_t(x & 1) * G * kPayAux; };
  // one gpu-scope fence + release by lane 0 (the cooperative-groups grid.sync pattern)
  auto exchange = [&]() {
    __syncwarp();
    if (lane == 0) {
      bar_target += static_cast<unsigned>(G);
      grid_arrive_wait(P.bar, bar_target);
      ++xi;
    }
    __syncwarp();
  };
  int& cstar = cs.cstar;
  int& cend = cs.cend;
  // full range scan of the records + publish + exchange + gather
  // cross-shard step after a gather (patient-sharded launches only): aux0 /
  // aux1 are this shard's max |eta| / overflow flag, combined into tl->xaux
  auto xshard = [&](double aux0, double aux1) {
    if (P.nranks <= 1) return;
    __syncwarp();
    if (lane == 0) cross_shard<FG>(P, tl, cta, aux0, aux1);
    __syncwarp();
  };
  auto publish_full = [&](double p0, double p1, double pb, int auxmode = 0) {
    double* pm = wbuf();
    range_scan<FG>(P, tl, t0, tc, pm, lane);
    if (lane == 0) {
      pm[0] = p0;
      pm[1] = p1;
      pm[2] = pb;
    }
    exchange();
    gather_warp<FG>(P, rbuf(xi - 1), cta, cstar, cend, tl, lane);
    double mm = 0.0;
    if (auxmode == 1 && lane == 0 && P.nranks > 1) {  // refresh: this shard's max |eta|
      const double* pa = raux(xi - 1);
      for (int c = 0; c < G; ++c) mm = fmax(mm, __ldcg(pa + size_t(c) * kPayAux + 0));
    }
    xshard(mm, 0.0);
  };
  auto slot_fields = [&](int kk) {
    SlotFields f{};
    f.valid = kk < P.nslots;
    if (!f.valid) return f;
    const long long c = P.slot_col[kk];
    const long long nc =
        (kk + 1 < P.nslots) ? P.slot_col[kk + 1] : (P.mode == kModeCcd ? P.slot_col[0] : -1);
    f.col = c;
    f.ncol = nc;
    f.kind = c >= 0 ? kSlotGrad : kSlotLoglik;
    f.cind = c >= 0 ? ((!P.has_vals || P.col_ind[c]) ? 1 : 0) : 1;
    f.nind = nc >= 0 ? ((!P.has_vals || P.col_ind[nc]) ? 1 : 0) : 1;
    f.fused = (!FG && P.mode == kModeCcd && c >= 0 && nc >= 0 && f.cind && f.nind &&
               !(P.dbg & 8)) ? 1 : 0;
    return f;
  };
  auto set_slot_fields = [&](const SlotFields& f) {
    if (!f.valid) return;
    ss.col = f.col;
    ss.ncol = f.ncol;
    ss.kind = f.kind;
    ss.cind = f.cind;
    ss.nind = f.nind;
    ss.fused = f.fused;
  };
  auto go = [&](int task) {
    if (lane == 0) tl->task = task;
    __syncwarp();
    bar_arrive_n(kBarGo, NB);
  };
  auto wait_done = [&]() { bar_sync_n(kBarDone, NB); };

  // ---- prologue: records for slot 0 (consumers), then the slot-0 carries ----
  wait_done();
  if (lane == 0) {
    cstar = tl->cstar;
    cend = tl->cend;
  }
  __syncwarp();
  publish_full(0.0, 0.0, 0.0);
  if (P.shard_out && cta == 0) shard_aggregate<FG>(P, rbuf(xi - 1), tl, lane);
  if (P.prologue_only) {
    if (lane == 0 && cta == 0) {
      ctl->bar_base = bar_target;
      ctl->xr_count = cs.xr_count;
      ctl->rec_valid = err ? 0 : 1;  // the records serve the launch that follows
      ctl->rec_col = P.slot_col[0];
    }
    go(kTaskExit);
    return;
  }
  if (lane == 0) {
    set_carry_in<FG>(P, tl, 0.0);
    ss.pcol = -1;
    ss.delta = 0.0;
    ss.phi = 1.0;
    ss.pind = 1;
    ss.refresh = 0;
    ss.dry = err ? 1 : 0;
    set_slot_fields(slot_fields(0));
  }
  go(kTaskNext);
  pmark(5);

  unsigned& qbase = cs.qbase;
  for (int k = 0; k < P.nslots; ++k) {
    // step inputs and the next slot's fields: loaded while the slot streams
    long long& col = cs.col;
    long long& ncol = cs.ncol;
    double& in_fixed = cs.in_fixed;
    double& in_beta = cs.in_beta;
    double& in_hw = cs.in_hw;
    double& in_cmax = cs.in_cmax;
    int& in_pen = cs.in_pen;
    int& in_ind = cs.in_ind;
    SlotFields& nf = cs.nf;
    if (lane == 0) {
      in_ind = 1;
      col = P.slot_col[k];
      ncol = (k + 1 < P.nslots) ? P.slot_col[k + 1] : (P.mode == kModeCcd ? P.slot_col[0] : -1);
      if (col >= 0) {
        in_fixed = __ldcg(P.fixed + col);
        in_beta = __ldcg(P.beta + col);
        in_hw = __ldcg(P.halfwidth + col);
        in_cmax = __ldcg(P.colmax + col);
        in_pen = P.penalized[col];
        in_ind = (!P.has_vals || P.col_ind[col]) ? 1 : 0;
      }
      nf = slot_fields(k + 1);
    }
    // ---- in-range forward carry scan as the records appear (Cox; for
    // Fine-Gray the full scan after the slot measured faster) ----
    {
      if (!FG && lane == 0 && !(P.dbg & (16 | 512))) {
        double car[6] = {0, 0, 0, 0, 0, 0};
        int seen = 0;
        const unsigned* prog = tl->progress;
        for (int i = 0; i < tc; ++i) {
          const unsigned need = qbase + static_cast<unsigned>(i) + 1u;
          const int g = i % Gm::kNG;
          if (flag_acquire(prog + g) < need) {
            const unsigned long long tw = gtimer();
            unsigned it = 0;
            while (flag_acquire(prog + g) < need) {
              __nanosleep(64);
              if ((++it & 63u) == 0 && gtimer() - tw > kWatchdogNs)
                watchdog_trap("control record wait", need, flag_acquire(prog + g));
            }
          }
          const int t = t0 + i;
          const double* rec = rec_at<FG>(P, tl, t, i);
          const int f = (i < MaxTc<FG>::v) ? tl->tfirst[i] : (P.tile_first[t] ? 1 : 0);
          double* tcp = car_at<FG>(P, tl, t, i);
#pragma unroll
          for (int m = 0; m < 6; ++m) tcp[m] = f ? 0.0 : car[m];
          tcp[6] = (seen | f) ? 1.0 : 0.0;
#pragma unroll
          for (int m = 0; m < 6; ++m) {
            const double r = ld_rc<FG>(rec + m, i);
            car[m] = f ? r : __dadd_rn(car[m], r);
          }
          seen |= f;
        }
        double* pm = wbuf();
        pm[3] = seen ? 1.0 : 0.0;
#pragma unroll
        for (int m = 0; m < 6; ++m) pm[4 + m] = car[m];
      }
    }
    wait_done();  // slot consumed: partials in wpart
    if ((P.dbg & 65536) && lane == 0 && k > 0) cs.tcons += gtimer() - cs.tgo;
    pmark(0);
    if (lane == 0) qbase += static_cast<unsigned>(tc);
    __syncwarp();
    if (P.dbg & 16) {  // ablation: stream only
      if ((P.dbg & 65536) && lane == 0) cs.tgo = gtimer();
      go(kTaskNext);
      continue;
    }
    double r0 = 0.0, r1 = 0.0, rb = 0.0;
    if (lane == 0) {
      for (int w = 0; w < W; ++w) {
        r0 = __dadd_rn(r0, tl->wpart[w][0]);
        r1 = __dadd_rn(r1, tl->wpart[w][1]);
        rb = __dadd_rn(rb, tl->wpart[w][2]);
      }
    }
    if (FG || (P.dbg & 512)) {
      publish_full(r0, r1, rb);
    } else {
      if (lane == 0) {
        double* pm = wbuf();
        pm[0] = r0;
        pm[1] = r1;
        pm[2] = rb;
      }
      exchange();
      pmark(1);
      gather_warp<FG>(P, rbuf(xi - 1), cta, cstar, cend, tl, lane);
      xshard(0.0, 0.0);
    }
    pmark(2);
    // ---- finish + coordinate step (lane 0, replicated in every CTA) ----
    double delta = 0.0, phi = 1.0, step_slack = 0.0;
    int need_exact = 0, do_refresh = 0, valued = 0;
    const bool dry = ss.dry != 0;
    if (lane == 0) {
      const double g0 = tl->gs[0], g1 = tl->gs[1];
      const bool badden = tl->gs[2] != 0.0;
      if (!dry) {
        if (col < 0) {
          const double ll = __dsub_rn(g0, g1);
          if (badden && !err) {
            err = kErrNonPos;
            err_col = -1;
          }
          if (cta == 0) {
            ctl->ll_fixed = g0;
            ctl->ll_logden = g1;
            ctl->loglik = ll;
            if (P.slot_out) P.slot_out[size_t(k) * 4 + 3] = ll;
          }
        } else {
          // Engine::finish (src/engine.cpp:220-230)
          const double grad = __dsub_rn(in_fixed, g0);
          double hess = -g1;
          if (hess > 0.0) hess = 0.0;
          const bool nonfinite = !isfinite(grad) || !isfinite(hess);
          if (cta == 0) {
            ctl->grad_sum = g0;
            ctl->hess_sum = g1;
            ctl->gradient = grad;
            ctl->hessian = hess;
            ctl->fixed_term = in_fixed;
            if (P.slot_out) {
              P.slot_out[size_t(k) * 4 + 0] = grad;
              P.slot_out[size_t(k) * 4 + 1] = hess;
              P.slot_out[size_t(k) * 4 + 2] = in_fixed;
            }
          }
          if (badden || nonfinite) {
            if (!err) {
              err = kErrNonPos;
              err_col = col;
            }
          } else if (P.mode == kModeCcd && !err) {
            // coordinate_step + update decision (src/ccd.cpp:152-167)
            const Step stp = coordinate_step_dev(in_beta, grad, hess, P.pen_kind, P.pen_strength,
                                                 in_pen != 0, in_hw);
            if (stp.skipped) {
              ++skipped;
            } else {
              if (cta == 0) P.halfwidth[col] = stp.new_hw;
              if (stp.applied != 0.0) {
                step_slack = __dmul_rn(in_cmax, fabs(stp.applied));
                delta = stp.applied;
                // fast validate: max|eta| at the last refresh/load plus the
                // accumulated |delta|*max|x| bounds every row
                need_exact = (absmax + slack + step_slack <= kFastBound) ? 0 : 1;
              }
            }
          }
        }
      }
      phi = (delta != 0.0) ? exp(delta) : 1.0;
      // carries for slot k+1 (linear path; refresh / valued paths redo them)
      pmark(9);
      set_carry_in<FG>(P, tl, __dsub_rn(phi, 1.0));
      pmark(10);
    }
    need_exact = __shfl_sync(0xffffffffu, need_exact, 0);
    pmark(11);
    // ---- exact validate-before-mutate (rare): consumers check, one more exchange ----
    if (need_exact) {
      if (lane == 0) {
        tl->flag = 0;
        tl->tcol = col;
        tl->tdelta = delta;
      }
      go(kTaskExact);
      wait_done();
      if (lane == 0) waux()[1] = tl->flag ? 1.0 : 0.0;
      exchange();
      double anyd = 0.0;
      if (lane == 0) {
        const double* pa = raux(xi - 1);
        for (int c = 0; c < G; ++c) anyd = fmax(anyd, __ldcg(pa + size_t(c) * kPayAux + 1));
      }
      if (P.nranks > 1) {  // OR over shards (validate-before-mutate on every shard)
        __syncwarp();
        if (lane == 0) {
          tl->gs[0] = tl->gs[1] = tl->gs[2] = 0.0;
          cross_shard<FG>(P, tl, cta, 0.0, anyd);
          anyd = tl->xaux[1];
        }
        __syncwarp();
      }
      if (lane == 0) {
        const bool any = anyd != 0.0;
        if (any) {
          if (!err) {
            err = kErrOverflow;
            err_col = col;
          }
          if (cta == 0) P.halfwidth[col] = in_hw;  // unchanged on the exception path
          delta = 0.0;
          phi = 1.0;
          set_carry_in<FG>(P, tl, 0.0);
        }
      }
    }
    // ---- accept: beta_[column] += delta, refresh cadence (src/engine.cpp:216-217) ----
    if (lane == 0) {
      if (delta != 0.0) {
        if (cta == 0) P.beta[col] = __dadd_rn(in_beta, delta);
        slack = __dadd_rn(slack, step_slack);
        ++accepted;
        if (--cs.to_refresh == 0) {
          cs.to_refresh = P.recompute_interval;
          do_refresh = 1;  // refresh subsumes the incremental update
          ++refreshes;
        }
      }
      valued = (delta != 0.0 && !do_refresh && !in_ind) ? 1 : 0;
      tl->refresh = do_refresh;
    }
    do_refresh = __shfl_sync(0xffffffffu, do_refresh, 0);
    pmark(4);
    valued = __shfl_sync(0xffffffffu, valued, 0);
    if (do_refresh) {
      if (lane == 0) {
        tl->tcol = col;
        tl->tdelta = delta;
        tl->tncol = ncol;
      }
      pmark(4);
      go(kTaskRefresh);
      wait_done();
      pmark(12);
      if (prof) ph[13] += 1;
      if (lane == 0) {
        double mm = 0.0;
        for (int w = 0; w < W; ++w) mm = fmax(mm, tl->wpart[w][3]);
        waux()[0] = mm;
      }
      publish_full(0.0, 0.0, 0.0, 1);
      if (lane == 0) {
        set_carry_in<FG>(P, tl, 0.0);
        const double* pa = raux(xi - 1);
        double mm = 0.0;
        for (int c = 0; c < G; ++c) mm = fmax(mm, __ldcg(pa + size_t(c) * kPayAux + 0));
        if (P.nranks > 1) mm = tl->xaux[0];  // max over shards
        absmax = mm;  // the bound is exact again
        slack = 0.0;
      }
    } else if (valued) {
      if (lane == 0) {
        tl->tcol = col;
        tl->tdelta = delta;
        tl->tncol = ncol;
      }
      go(kTaskValued);
      wait_done();
      publish_full(0.0, 0.0, 0.0);
      if (lane == 0) set_carry_in<FG>(P, tl, 0.0);
    }
    // ---- the next slot's pending update and fields ----
    if (lane == 0) {
      ss.pcol = (delta != 0.0 && !do_refresh) ? col : -1;
      ss.delta = delta;
      ss.phi = phi;
      ss.pind = in_ind;
      ss.refresh = do_refresh;
      ss.dry = err ? 1 : 0;
      set_slot_fields(nf);
    }
    pmark(3);
    if ((P.dbg & 65536) && lane == 0) cs.tgo = gtimer();
    go(kTaskNext);
  }
  if ((P.dbg & 65536) && lane == 0)
    printf("gss cta %d tiles %d [%d, %d) consume_us %.2f\n", cta, tc, t0, t0 + tc,
           P.nslots > 1 ? double(cs.tcons) / (P.nslots - 1) / 1000.0 : 0.0);

  // ---- epilogue: CTA 0 persists the replicated state ----
  if (lane == 0 && cta == 0) {
    ctl->bar_base = bar_target;
    ctl->xr_count = cs.xr_count;
    ctl->eta_absmax_bits = static_cast<unsigned long long>(__double_as_longlong(absmax));
    ctl->bound_slack = slack;
    ctl->accepted = accepted;
    ctl->refreshes = refreshes;
    ctl->skipped = skipped;
    ctl->err_code = err;
    ctl->err_col = err_col;
    ctl->rec_valid = (P.mode == kModeCcd && !err) ? 1 : 0;
    ctl->rec_col = P.slot_col[0];
  }
  if (prof) {
    const double ns = P.nslots > 0 ? static_cast<double>(P.nslots) : 1.0;
    printf("gss prof cta %d slots %d (cycles/slot, control warp): consume %.0f publish+barrier %.0f "
           "gather %.0f step+tasks %.0f (prologue %lld) | gather: wait %.0f sum %.0f reduce %.0f | "
           "step %.0f carry %.0f shfl %.0f accept %.0f | refreshes %lld task %.0f\n",
           cta, P.nslots, ph[0] / ns, ph[1] / ns, ph[2] / ns, ph[3] / ns, ph[5], ph[6] / ns,
           ph[7] / ns, ph[8] / ns, ph[9] / ns, ph[10] / ns, ph[11] / ns, ph[4] / ns, ph[13],
           ph[13] ? static_cast<double>(ph[12]) / ph[13] : 0.0);
  }
}

// ---------------------------------------------------------------------------
// the persistent cycle kernel
// ---------------------------------------------------------------------------
template <bool FG, int K>
__global__ void __launch_bounds__(Geo<FG>::kThreads, 1)
    cycle_kernel(const __grid_constant__ LaunchParams<K> L) {
  using Gm = Geo<FG>;
  constexpr int W = Gm::kW, S = Gm::kS;
  constexpr int NC = 32 * W;  // consumer threads
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  Tail<FG>* tl = reinterpret_cast<Tail<FG>*>(smem + size_t(S) * Gm::kStage);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // this CTA's engine (fit) and its CTA index inside that engine's grid
  int f = 0;
  if constexpr (K > 1) {
    while (f + 1 < L.nfit && static_cast<int>(blockIdx.x) >= L.cta_base[f + 1]) ++f;
  }
  const CycleParams& P = L.P[f];
  const int bid = static_cast<int>(blockIdx.x) - (K > 1 ? L.cta_base[f] : 0);
  const int cta = (P.dbg & 64) ? P.grid - 1 - bid : bid;
  const int G = P.grid;
  // static contiguous tile ranges, balanced by estimated tile cost (host,
  // per engine); P.cta_tile0[c] = first tile of CTA c, [G] = ntiles
  auto range_lo = [&](int c) {
    return P.cta_tile0 ? P.cta_tile0[c]
                       : static_cast<int>((static_cast<long long>(c) * P.ntiles) / G);
  };
  const int t0 = range_lo(cta);
  const int tc = range_lo(cta + 1) - t0;
  Ctl* ctl = P.ctl;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&tl->full[s], 1);
      mbar_init(&tl->empty[s], 1);
    }
    mbar_init(&tl->gbar, 1);
    tl->gphase = 0u;
    tl->issued = 0u;
    fence_mbar_init();
  }
  if (tid < Gm::kNG) tl->progress[tid] = 0u;
  if (tid < 32) trace_slot(tid) = 0u;
  for (int i = tid; i < Gm::kNG * 512; i += blockDim.x) {
    (&tl->xm[0][0][0])[i] = 0u;
    (&tl->xn[0][0][0])[i] = 0u;
  }
  for (int i = tid; i < min(tc, MaxTc<FG>::v); i += blockDim.x) tl->tfirst[i] = P.tile_first[t0 + i];
  if (tid == 0) tl->task = kTaskNext;
  // static stratum flags of every CTA range (carry segmentation bounds)
  for (int c = tid; c < G; c += blockDim.x) {
    uint8_t f = 0;
    for (int t = range_lo(c); t < range_lo(c + 1); ++t) f |= P.tile_first[t];
    tl->cflag[c] = f;
  }
  __syncthreads();
  if (tid == 0) {
    int cs = 0, fs = 0;
    for (int c = cta - 1; c >= 0; --c)
      if (tl->cflag[c]) {
        cs = c;
        fs = 1;
        break;
      }
    int ce = G - 1, fe = 0;
    for (int c = cta + 1; c < G; ++c)
      if (tl->cflag[c]) {
        ce = c;
        fe = 1;
        break;
      }
    tl->cstar = cs;
    tl->cend = ce;
    // carry from other shards reaches this CTA when no stratum starts between
    tl->ext_f = ((P.ext || P.nranks > 1) && !fs) ? 1 : 0;
    tl->ext_r = ((P.ext || P.nranks > 1) && !fe) ? 1 : 0;
    for (int i = 0; i < 12; ++i) tl->xext[i] = 0.0;
  }

  if (warp > W) {
    producer<FG>(P, smem, tl, t0, tc, &L.tm_e[f], &L.tm_code[f], &L.tm_g[f], warp - W - 1);
    return;
  }
  const bool rec_ok = (P.mode == kModeCcd || P.reuse_records) && ctl->rec_valid &&
                      ctl->rec_col == P.slot_col[0];
  SlotState& ss = tl->ss;
  if (warp == W) {
    control_warp<FG>(P, tl, cta, t0, tc, lane);
    return;
  }

  // ------------------------------ consumer warps ------------------------------
  // Consumers only stream tiles and run the all-warp tasks the control warp
  // hands them; every value that lives across slots is in shared memory
  // (the control warp owns it), so nothing is spilled across the tile loop.
  if (!rec_ok) {
    records_from_global<FG>(P, tl, t0, tc, P.slot_col[0], warp, lane);
  } else {  // records of the previous launch (global) -> shared memory
    constexpr int R = FG ? 12 : 6;
    const int nl = min(tc, MaxTc<FG>::v);
    for (int i = tid; i < nl * R; i += NC)
      tl->srec[i / R][i % R] = __ldcg(P.trec + size_t(t0 + i / R) * kRecStride + i % R);
  }
  __threadfence_block();
  bar_arrive_n(kBarDone, NC + 32);
  consumer_tasks<FG>(P, tl, t0, tc, warp, lane, tid);
  unsigned qbase = 0;  // stream position of the slot's first tile
  int gpar = 0;        // this warp's group: mask buffer of its next tile
  const int nsl = (tl->task == kTaskExit) ? 0 : P.nslots;
  for (int k = 0; k < nsl; ++k) {
    double acc0 = 0.0, acc1 = 0.0;
    int bad = 0;
    const bool dry = ss.dry != 0;
    {
      constexpr int NGr = Gm::kNG, GWr = Gm::kGW;
      const int g = warp / GWr, gw = warp % GWr;
      // Progress (the producer's licence to reload a tile for the next slot,
      // and the control warp's licence to read the tile's record) is
      // published with the stage release; the threads that committed the
      // pending update fence generic -> async proxy first.
      for (int i = g; i < tc; i += NGr) {
        const unsigned q = qbase + static_cast<unsigned>(i);
        const int s = static_cast<int>(q % S);
        const uint32_t ph = (q / S) & 1u;
        // A parity wait only tells apart consecutive phases of a stage: a group
        // that runs two ring cycles ahead of a slow group would see the phase
        // of position q - 2S as "complete". Wait until the producer has issued
        // q (it issues q only after q - S was released), then the parity test
        // is exact.
        {
          const unsigned* iss = &tl->issued;
          if (flag_acquire(iss) <= q) {
            const unsigned long long tw = gtimer();
            unsigned it = 0;
            while (flag_acquire(iss) <= q) {
              __nanosleep(32);
              if ((++it & 63u) == 0 && gtimer() - tw > kWatchdogNs)
                watchdog_trap("consumer issue wait", q, flag_acquire(iss),
                              lane == 0 ? tl->mark : nullptr);
            }
          }
        }
        mbar_wait_wd(&tl->full[s], ph, "consumer full-stage wait", q, lane == 0 ? tl->mark : nullptr);
        // per-tile cost probe (GSS_DEBUG bit 524288 + GSS_TRACE=1): cycles from
        // stage-ready to the end of the tile, for the slot in the middle
        const bool tprobe = GSS_ENABLE_TRACE && (P.dbg & 524288) && P.trace && k == P.nslots / 2 &&
                            gw == 0 && lane == 0;
        const long long tp0 = tprobe ? clock64() : 0;
        unsigned char* sb = smem + size_t(s) * Gm::kStage;
        if (!dry && !(P.dbg & 1))
          consume_tile<FG>(P, tl, sb, tl->info[s], ss, g, gw, lane, gpar, acc0, acc1, bad,
                           &tl->empty[s]);
        gpar ^= 1;
        if (ss.pcol >= 0 && !ss.refresh && (gw * 32 + lane) < tl->info[s].l[0].cnt)
          fence_proxy_async_global();
        mark<FG>(tl, 0x15u | (q << 8));
        group_sync<FG>(g);
        if (gw == 0 && lane == 0) {
          flag_release(&tl->progress[g], q + 1);  // the tile's record before its progress
          mbar_arrive(&tl->empty[s]);
        }
        if (tprobe && t0 + i < static_cast<int>(P.trace_cap))
          P.trace[t0 + i] = static_cast<unsigned long long>(clock64() - tp0);
      }
    }
    qbase += static_cast<unsigned>(tc);
    acc0 = warp_sum(acc0);
    acc1 = warp_sum(acc1);
    const double badw = warp_sum(static_cast<double>(bad));
    if (lane == 0) {
      tl->wpart[warp][0] = acc0;
      tl->wpart[warp][1] = acc1;
      tl->wpart[warp][2] = badw;
    }
    __threadfence_block();
    bar_arrive_n(kBarDone, NC + 32);
    consumer_tasks<FG>(P, tl, t0, tc, warp, lane, tid);
  }
  // shared-memory records -> global (they outlive the launch)
  {
    constexpr int R = FG ? 12 : 6;
    consumer_sync(NC);
    const int nl = min(tc, MaxTc<FG>::v);
    for (int i = tid; i < nl * R; i += NC)
      P.trec[size_t(t0 + i / R) * kRecStride + i % R] = tl->srec[i / R][i % R];
  }
}

}  // namespace

size_t cycle_smem_bytes(bool weighted) {
  return weighted ? smem_total<true>() : smem_total<false>();
}

namespace {
template <bool FG, int K>
void set_smem_attr() {
  cudaFuncSetAttribute(cycle_kernel<FG, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem_total<FG>()));
}

template <bool FG, int K>
cudaError_t launch_k(const LaunchParams<K>& L, int grid, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (grid barriers)
  attr[0].val.cooperative = 1;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(Geo<FG>::kThreads);
  cfg.dynamicSmemBytes = smem_total<FG>();
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, cycle_kernel<FG, K>, L);
}
}  // namespace

int cycle_max_grid(int device, bool weighted) {
  int sms = 0, n = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (weighted) {
    set_smem_attr<true, 1>();
    set_smem_attr<true, kMaxBatch>();
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, cycle_kernel<true, 1>, Geo<true>::kThreads,
                                                  smem_total<true>());
  } else {
    set_smem_attr<false, 1>();
    set_smem_attr<false, kMaxBatch>();
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, cycle_kernel<false, 1>, Geo<false>::kThreads,
                                                  smem_total<false>());
  }
  return n > 0 ? (sms < kMaxGrid ? sms : kMaxGrid) : 0;
}

cudaError_t launch_cycle(const CUtensorMap* tm_e, const CUtensorMap* tm_code,
                         const CUtensorMap* tm_g, const CycleParams& prm, cudaStream_t s) {
  LaunchParams<1> L;
  L.tm_e[0] = *tm_e;
  L.tm_code[0] = *tm_code;
  L.tm_g[0] = *tm_g;
  L.P[0] = prm;
  L.nfit = 1;
  L.cta_base[0] = 0;
  L.cta_base[1] = prm.grid;
  return prm.weighted ? launch_k<true, 1>(L, prm.grid, s) : launch_k<false, 1>(L, prm.grid, s);
}

cudaError_t launch_cycle_batch(const BatchEntry* en, int k, cudaStream_t s) {
  if (k < 1 || k > kMaxBatch) return cudaErrorInvalidValue;
  if (k == 1) return launch_cycle(en[0].tm_e, en[0].tm_code, en[0].tm_g, *en[0].prm, s);
  static LaunchParams<kMaxBatch> L;  // 17 KB: not on the host stack (callers serialise per device)
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  const bool w = en[0].prm->weighted != 0;
  int base = 0;
  for (int i = 0; i < k; ++i) {
    if ((en[i].prm->weighted != 0) != w) return cudaErrorInvalidValue;
    L.tm_e[i] = *en[i].tm_e;
    L.tm_code[i] = *en[i].tm_code;
    L.tm_g[i] = *en[i].tm_g;
    L.P[i] = *en[i].prm;
    L.cta_base[i] = base;
    base += en[i].prm->grid;
  }
  L.cta_base[k] = base;
  L.nfit = k;
  return w ? launch_k<true, kMaxBatch>(L, base, s) : launch_k<false, kMaxBatch>(L, base, s);
}

}  // namespace gss
