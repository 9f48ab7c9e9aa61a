// gss_kernels.cu — sm_100a per-coordinate kernel of the Cox CCD hot path.
//
// `sweep_kernel` is ONE persistent, single-pass scan -> transform -> reduce
// over the time-ordered rows: the reference's two-phase chunked
// fused_grad_hess (/root/reference/proj/include/survscan/scan_kernels.hpp:74-214)
// plus Engine::finish (src/engine.cpp:220-230).  Around the scan it fuses
//   * the previous coordinate's deferred sparse eta/exp(eta) update
//     (Engine::update_xbeta_sparse, src/engine.cpp:162-218) or the periodic
//     refresh (src/engine.cpp:120-160);
//   * in CCD mode, coordinate_step (src/ccd.cpp:71-129), run by the last CTA,
//     which validates and defers the next update.
//
// Single pass without a serial look-back.  The per-tile carry of the
// reverse-time risk-set scan is known BEFORE the dense data is read:
//   Phase A (all warps, dynamic work items, O(nnz) traffic): tile aggregate
//     A[t] = (f, a, b, c) where a = this tile's fresh sum of exp(eta) from the
//     previous sweep (written by its consumers) + the sparse correction of the
//     pending update, and b, c = sums of e*x, e*x^2 over the scan column's
//     in-tile nonzeros (gathers).  The CTA that completes the last item scans
//     the tile aggregates in a fixed order and publishes prefix[t] + a ready
//     flag (epoch tagged).
//   Phase C (warp specialised): a producer warp claims tiles dynamically and
//     streams the 2048-row tiles of exp(eta) (fp64) and row codes (u32) with 2D
//     TMA (64B/32B swizzle) plus a 1D bulk copy of the in-tile row indices;
//     8 consumer warps patch the pending update into the staged tile, block-
//     scan it (writing the tile's fresh sum for the next sweep), take prefix[t]
//     and evaluate the Breslow transform at tied-block ends.  Tiles never wait
//     on each other; loading overlaps phase A.
// Determinism: every prefix is a fixed-order function of fixed-order tile
// aggregates; tile partials are reduced in tile order by the last CTA; results
// are bitwise reproducible run to run (the reference's guarantee,
// scan_kernels.hpp:8-10) for any schedule.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gss_device.cuh"
#include "gss_kernels.cuh"

namespace gss {

namespace {

constexpr uint32_t kEBytes = kTileRows * 8;      // 16 KB
constexpr uint32_t kCodeBytes = kTileRows * 4;   // 8 KB
constexpr uint32_t kNnzBytes = kNnzCap * 4;      // 1 KB
constexpr uint32_t kStageBytes = kEBytes + kCodeBytes + 2 * kNnzBytes;  // 26 KB
static_assert(kStageBytes % 1024 == 0, "stage alignment");
constexpr int kConsumerWarps = kThreads / 32;  // 8
constexpr int kProducerWarp = kConsumerWarps;   // 8
constexpr int kWarps = kConsumerWarps + 1;
constexpr int kSweepThreads = 32 * kWarps;      // 288
constexpr int kScratchInts = 128;               // per-warp phase-A scratch (smem)
constexpr double kXbetaBound = 700.0;           // src/engine.cpp:12
constexpr double kHwFloor = 1e-300;             // src/ccd.cpp:13
constexpr double kFastBound = 700.0 * (1.0 - 1e-12);

struct StageInfo {
  int tile;
  int smem_s, smem_u;
  int pad;
  long long lo_s, hi_s, base_s;  // scan column nnz range [lo, hi); smem copy starts at base
  long long lo_u, hi_u, base_u;  // pending-update column nnz range
};

struct SmemTail {
  uint64_t full[kStages];   // producer -> consumers (TMA tx)
  uint64_t empty[kStages];  // consumers -> producer
  StageInfo info[kStages];
  double red[kWarps][8];
  double scan[2][kConsumerWarps][4];  // block-scan warp totals, double-buffered by tile parity
  double part[2][kConsumerWarps][4];  // per-warp tile partials, double-buffered by tile parity
  double bcast[8];
  int32_t scratch[kConsumerWarps][kScratchInts];  // phase-A pending-column lists
  int flag;
};

__host__ __device__ constexpr size_t smem_total() {
  return 1024 /*align slack*/ + size_t(kStages) * kStageBytes + sizeof(SmemTail);
}

__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
}

__device__ __forceinline__ double sgn(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }

__device__ __forceinline__ void red_add_f64(double* p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// optional event trace: word0 = globaltimer ns, word1 = (cta << 40) | (event << 32) | tile
__device__ __forceinline__ void trace_ev(const SweepParams& P, int ev, int tile) {
  if (!P.trace) return;
  unsigned long long ns;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
  const unsigned i = atomicAdd(P.trace_n, 1u);
  if (i < P.trace_cap) {
    P.trace[2 * i] = ns;
    P.trace[2 * i + 1] = (static_cast<unsigned long long>(blockIdx.x) << 40) |
                         (static_cast<unsigned long long>(ev) << 32) | static_cast<unsigned>(tile);
  }
}

__device__ __forceinline__ double* e_at(unsigned char* se, int lr) {
  return reinterpret_cast<double*>(se + swz<kIpt * 8>(lr * 8));
}

// Exclusive scan across the 256 consumer threads (thread order), plus total.
// One barrier: the warp-total buffer alternates with the tile parity, and
// consecutive uses of one buffer are separated by the next tile's barrier.
template <int L>
__device__ __forceinline__ Seg<L> block_exclusive_scan(Seg<L> v, Seg<L>& total, SmemTail* st,
                                                       int tid, int par) {
  const int lane = tid & 31, warp = tid >> 5;
  const Seg<L> inc = warp_inclusive_scan(v, lane);
  if (lane == 31) {
    st->scan[par][warp][0] = inc.f ? 1.0 : 0.0;
#pragma unroll
    for (int i = 0; i < L; ++i) st->scan[par][warp][1 + i] = inc.v[i];
  }
  consumer_sync();
  Seg<L> wpre = Seg<L>::zero(), tot = Seg<L>::zero();
#pragma unroll
  for (int w = 0; w < kConsumerWarps; ++w) {
    Seg<L> x;
    x.f = st->scan[par][w][0] != 0.0 ? 1u : 0u;
#pragma unroll
    for (int i = 0; i < L; ++i) x.v[i] = st->scan[par][w][1 + i];
    if (w < warp) wpre = seg_combine(wpre, x);
    tot = seg_combine(tot, x);
  }
  Seg<L> exc = shfl_up_seg(inc, 1);
  if (lane == 0) exc = Seg<L>::zero();
  total = tot;
  return seg_combine(wpre, exc);
}

// Three sums at once (fixed order); results broadcast to all consumers.
__device__ __forceinline__ void block_sum3(double v[3], SmemTail* st, int tid) {
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int i = 0; i < 3; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) st->red[warp][5 + i] = v[i];
  }
  consumer_sync();
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double r = 0.0;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) r = __dadd_rn(r, st->red[w][5 + i]);
    v[i] = r;
  }
  consumer_sync();
}

// Tile partial = fixed warp-order sum of the per-warp partials of tile t.
__device__ __forceinline__ void flush_partial(const SweepParams& P, const SmemTail* st, int t,
                                              int par) {
  double r0 = 0.0, r1 = 0.0, r2 = 0.0;
#pragma unroll
  for (int w = 0; w < kConsumerWarps; ++w) {
    r0 = __dadd_rn(r0, st->part[par][w][0]);
    r1 = __dadd_rn(r1, st->part[par][w][1]);
    r2 = __dadd_rn(r2, st->part[par][w][2]);
  }
  double* tp = P.tile_part + size_t(t) * 4;
  tp[0] = r0;
  tp[1] = r1;
  tp[2] = r2;
}

// Lower bound of `row` in the nonzero list [lo, hi) (smem copy or global).
__device__ __forceinline__ long long lower_bound_rows(const int32_t* list_smem, long long base,
                                                      const int32_t* list_glob, long long lo,
                                                      long long hi, int32_t row, bool use_smem) {
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    const int32_t v = use_smem ? list_smem[mid - base] : list_glob[mid];
    if (v < row)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// coordinate_step (src/ccd.cpp:71-129), scalar, no FMA contraction.
struct Step {
  double new_beta, applied, new_hw;
  bool skipped;
};
__device__ Step coordinate_step_dev(double beta_j, double grad, double hess, int kind,
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

// Per-launch view of the control block, read once at kernel entry.
struct Pending {
  long long col;   // pending-update column (valid iff active)
  double delta, factor;
  bool active;     // deferred sparse update to apply in this launch
  bool refresh;    // deferred full refresh to apply in this launch
  bool ind;        // pending column is an indicator column
};

// exp(eta) of row r after the pending update of list entry k (src/engine.cpp:192-215)
__device__ __forceinline__ double updated_e(const SweepParams& P, const Pending& pd, long long k,
                                            int32_t r, double e_old) {
  if (pd.ind) return __dmul_rn(e_old, pd.factor);
  return exp(__dadd_rn(__ldcg(P.eta + r), __dmul_rn(P.vals[k], pd.delta)));
}

// ---------------------------------------------------------------------------
// Phase A: aggregate of tile t by one warp.  Returns (f, a, b, c) in lane 0.
// ---------------------------------------------------------------------------
template <int L>
__device__ Seg<3> phase_a_tile(const SweepParams& P, const Pending& pd, int t, long long col,
                               bool tprev_valid, const double* t_in, int32_t* scratch, int lane,
                               double* absmax) {
  const long long row0 = static_cast<long long>(t) * kTileRows;
  const int lastseg = P.tile_lastseg[t];
  const int from = lastseg < 0 ? 0 : lastseg;
  const size_t nt1 = size_t(P.ntiles) + 1;
  double a = 0.0, da = 0.0, b = 0.0, c = 0.0;
  if (pd.refresh) {
    // Engine::refresh -> load_beta (src/engine.cpp:120-160): each lane
    // recomputes eta_r = sum_j beta_j x_rj over its rows' CSR entries
    double mx = 0.0;
    for (int lr = lane; lr < kTileRows; lr += 32) {
      const long long r = row0 + lr;
      if (r >= P.n) break;
      if (P.has_mask && (P.code[r] & kCodeMasked)) continue;
      const long long k0 = P.row_ptr[r], k1 = P.row_ptr[r + 1];
      double acc = 0.0;
      long long k = k0;
      for (; k + 4 <= k1; k += 4) {
        int32_t cc[4];
        double xx[4], bb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) cc[q] = P.csr_col[k + q];
#pragma unroll
        for (int q = 0; q < 4; ++q) xx[q] = P.csr_val ? P.csr_val[k + q] : 1.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) bb[q] = P.beta[cc[q]];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc = __dadd_rn(acc, __dmul_rn(bb[q], xx[q]));
      }
      for (; k < k1; ++k)
        acc = __dadd_rn(acc, __dmul_rn(P.beta[P.csr_col[k]], P.csr_val ? P.csr_val[k] : 1.0));
      const double ev = exp(acc);
      P.eta[r] = acc;
      P.e[r] = ev;
      if (lr >= from) a = __dadd_rn(a, ev);
      mx = fmax(mx, fabs(acc));
    }
    *absmax = fmax(*absmax, mx);
    __syncwarp();
  } else {
    if (tprev_valid) {
      if (lane == 0) a = t_in[2 * t + 1];
    } else {
      for (int lr = from + lane; lr < kTileRows; lr += 32) a = __dadd_rn(a, __ldcg(P.e + row0 + lr));
    }
    if (pd.active) {
      const long long cb = P.col_ptr[pd.col];
      const long long lo = cb + P.tile_ptr[size_t(pd.col) * nt1 + t];
      const long long hi = cb + P.tile_ptr[size_t(pd.col) * nt1 + t + 1];
      for (long long k = lo + lane; k < hi; k += 32) {
        const int32_t r = P.row_idx[k];
        if (hi - lo <= kScratchInts) scratch[k - lo] = r;
        if (static_cast<int>(r - row0) < from) continue;
        if (P.has_mask && (P.code[r] & kCodeMasked)) continue;
        const double eo = __ldcg(P.e + r);
        da = __dadd_rn(da, __dsub_rn(updated_e(P, pd, k, r, eo), eo));
      }
      __syncwarp();
    }
  }
  if (L == 3) {
    const long long cb = P.col_ptr[col];
    const long long lo = cb + P.tile_ptr[size_t(col) * nt1 + t];
    const long long hi = cb + P.tile_ptr[size_t(col) * nt1 + t + 1];
    const bool ind_s = !P.has_vals || P.col_ind[col];
    long long ulo = 0, uhi = 0, ucb = 0;
    if (pd.active) {
      ucb = P.col_ptr[pd.col];
      ulo = ucb + P.tile_ptr[size_t(pd.col) * nt1 + t];
      uhi = ucb + P.tile_ptr[size_t(pd.col) * nt1 + t + 1];
    }
    for (long long k = lo + lane; k < hi; k += 32) {
      const int32_t r = P.row_idx[k];
      if (static_cast<int>(r - row0) < from) continue;
      if (P.has_mask && (P.code[r] & kCodeMasked)) continue;
      double ev = __ldcg(P.e + r);
      if (pd.active && uhi > ulo) {
        // is r also a row of the pending column? (its e changes this launch)
        long long q0 = ulo, q1 = uhi;
        const bool sm = uhi - ulo <= kScratchInts;
        while (q0 < q1) {
          const long long mid = (q0 + q1) >> 1;
          const int32_t v = sm ? scratch[mid - ulo] : P.row_idx[mid];
          if (v < r)
            q0 = mid + 1;
          else
            q1 = mid;
        }
        if (q0 < uhi && (sm ? scratch[q0 - ulo] : P.row_idx[q0]) == r)
          ev = updated_e(P, pd, q0, r, ev);
      }
      const double x = ind_s ? 1.0 : P.vals[k];
      const double ex = __dmul_rn(ev, x);
      b = __dadd_rn(b, ex);
      c = __dadd_rn(c, __dmul_rn(ex, x));
    }
  }
  Seg<3> A;
  A.f = lastseg >= 0 ? 1u : 0u;
  A.v[0] = __dadd_rn(warp_sum(a), warp_sum(da));
  A.v[1] = warp_sum(b);
  A.v[2] = warp_sum(c);
  return A;
}

__device__ __forceinline__ Seg<3> load_seg(const double* a) {
  Seg<3> x;
  x.f = __ldcg(a) != 0.0 ? 1u : 0u;
  x.v[0] = __ldcg(a + 1);
  x.v[1] = __ldcg(a + 2);
  x.v[2] = __ldcg(a + 3);
  return x;
}
__device__ __forceinline__ void store_seg(double* a, const Seg<3>& x) {
  a[0] = x.f ? 1.0 : 0.0;
  a[1] = x.v[0];
  a[2] = x.v[1];
  a[3] = x.v[2];
}

// In-group scan by the warp that completed the group's last tile aggregate:
// ipre[t] = exclusive prefix inside the 32-tile group, gsum[g] = group total
// (fixed warp tree => canonical).
__device__ void group_scan(const SweepParams& P, int g, int gsize, int lane) {
  const int t = g * 32 + lane;
  const Seg<3> x = lane < gsize ? load_seg(P.agg + size_t(t) * 4) : Seg<3>::zero();
  const Seg<3> inc = warp_inclusive_scan(x, lane);
  Seg<3> exc = shfl_up_seg(inc, 1);
  if (lane == 0) exc = Seg<3>::zero();
  if (lane < gsize) store_seg(P.prefix + size_t(t) * 4, exc);
  if (lane == 31) store_seg(P.gsum + size_t(g) * 4, inc);
}

// Exclusive scan of the group totals by the warp that completed the last
// group: gpre[g] (lane-contiguous chunks, fixed tree).
__device__ void final_scan(const SweepParams& P, int ng, int lane) {
  const int per = (ng + 31) / 32;
  const int g0 = min(ng, lane * per), g1 = min(ng, g0 + per);
  // loads batched 8 at a time (independent), folded in order
  constexpr int kB = 8;
  Seg<3> own = Seg<3>::zero();
  for (int b = g0; b < g1; b += kB) {
    Seg<3> x[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q)
      x[q] = b + q < g1 ? load_seg(P.gsum + size_t(b + q) * 4) : Seg<3>::zero();
#pragma unroll
    for (int q = 0; q < kB; ++q) own = seg_combine(own, x[q]);
  }
  const Seg<3> inc = warp_inclusive_scan(own, lane);
  Seg<3> run = shfl_up_seg(inc, 1);
  if (lane == 0) run = Seg<3>::zero();
  for (int b = g0; b < g1; b += kB) {
    Seg<3> x[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q)
      x[q] = b + q < g1 ? load_seg(P.gsum + size_t(b + q) * 4) : Seg<3>::zero();
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      if (b + q < g1) store_seg(P.gpre + size_t(b + q) * 4, run);
      run = seg_combine(run, x[q]);
    }
  }
}

// ---------------------------------------------------------------------------
// Phase-C consumer loop, specialised on the column kind and on strata:
//   IND    : indicator column, x in {0,1} held as a bitmask; lane c == lane b
//   STRATA : some stratum starts inside the data (segmented operator); without
//            strata the only segment start is row 0, whose prefix is zero, so
//            plain sums are exact and the selects disappear
// ---------------------------------------------------------------------------
template <int L, bool STRATA>
__device__ __forceinline__ Seg<L> comb(const Seg<L>& x, const Seg<L>& y) {
  if constexpr (STRATA) {
    return seg_combine(x, y);
  } else {
    Seg<L> r;
    r.f = 0u;
#pragma unroll
    for (int i = 0; i < L; ++i) r.v[i] = __dadd_rn(x.v[i], y.v[i]);
    return r;
  }
}

template <int L, bool STRATA>
__device__ __forceinline__ Seg<L> warp_scan_incl(Seg<L> s, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    Seg<L> o;
    o.f = STRATA ? __shfl_up_sync(0xffffffffu, s.f, d) : 0u;
#pragma unroll
    for (int i = 0; i < L; ++i) o.v[i] = __shfl_up_sync(0xffffffffu, s.v[i], d);
    if (lane >= d) s = comb<L, STRATA>(o, s);
  }
  return s;
}

template <int MODE, bool IND, bool STRATA>
__device__ __forceinline__ void consume(const SweepParams& P, const Pending& pd, SmemTail* st,
                                        unsigned char* smem, double* t_out,
                                        unsigned long long epoch, Ctl* ctl, long long col,
                                        int tid) {
  // lanes: a = sum e, b = sum e*x, c = sum e*x^2 (c == b for indicators)
  constexpr int L = (MODE == kModeLoglik) ? 1 : (IND ? 2 : 3);
  const int warp = tid >> 5, lane = tid & 31;
  bool ready_seen = false;
  int prev_t = -1;  // tile whose per-warp partials await the fixed-order sum
  int last_par = 0;
  for (int it = 0;; ++it) {
    const int s = it % kStages;
    const uint32_t ph = (it / kStages) & 1;
    const int par = it & 1;
    mbar_wait(&st->full[s], ph);
    const StageInfo& inf = st->info[s];
    const int t = inf.tile;
    if (t < 0) break;
    if (tid == 0) trace_ev(P, 7, t);
    const long long row0 = static_cast<long long>(t) * kTileRows;
    unsigned char* sb = smem + size_t(s) * kStageBytes;
    const unsigned char* sc = sb + kEBytes;
    const int32_t* nnz_s = reinterpret_cast<const int32_t*>(sb + kEBytes + kCodeBytes);
    const int32_t* nnz_u = nnz_s + kNnzCap;
    const int lr0 = tid * kIpt;
    // prefix loads issued early; consumed only after the block scan, so their
    // latency overlaps the local pass (raw values, no arithmetic here)
    double pg[1 + L], pq[1 + L];
    auto load_prefix = [&]() {
      const double* g = P.gpre + size_t(t / 32) * 4;
      const double* q = P.prefix + size_t(t) * 4;
#pragma unroll
      for (int i = 0; i < L; ++i) {
        pg[1 + i] = __ldcg(g + 1 + i);
        pq[1 + i] = __ldcg(q + 1 + i);
      }
      pg[0] = STRATA ? __ldcg(g) : 0.0;
      pq[0] = STRATA ? __ldcg(q) : 0.0;
    };
    if (ready_seen) load_prefix();

    // ---- patch the deferred update into this warp's rows (smem only) ----
    if (pd.active) {
      const int w0 = warp * 32 * kIpt;
      for (long long k = inf.lo_u + lane; k < inf.hi_u; k += 32) {
        const int32_t r = inf.smem_u ? nnz_u[k - inf.base_u] : P.row_idx[k];
        const int lr = static_cast<int>(r - row0);
        if (lr < w0 || lr >= w0 + 32 * kIpt) continue;
        const uint32_t cwr = *reinterpret_cast<const uint32_t*>(sc + swz<kIpt * 4>(lr * 4));
        if (cwr & kCodeMasked) continue;
        double* pe = e_at(sb, lr);
        *pe = updated_e(P, pd, k, r, *pe);
      }
      __syncwarp();
    }

    // ---- thread-contiguous rows: exp(eta), code, x_j ----
    double ev[kIpt];
    uint32_t cw[kIpt];
#pragma unroll
    for (int c = 0; c < kIpt / 2; ++c) {
      const double2 v =
          *reinterpret_cast<const double2*>(sb + swz<kIpt * 8>(tid * (kIpt * 8) + c * 16));
      ev[2 * c] = v.x;
      ev[2 * c + 1] = v.y;
    }
#pragma unroll
    for (int c = 0; c < kIpt / 4; ++c) {
      const uint4 v =
          *reinterpret_cast<const uint4*>(sc + swz<kIpt * 4>(tid * (kIpt * 4) + c * 16));
      cw[4 * c] = v.x;
      cw[4 * c + 1] = v.y;
      cw[4 * c + 2] = v.z;
      cw[4 * c + 3] = v.w;
    }
    uint32_t xb = 0;                    // IND: bit m = row m holds a nonzero
    double xv[IND ? 1 : kIpt];          // valued: x per row
    if constexpr (!IND) {
#pragma unroll
      for (int m = 0; m < kIpt; ++m) xv[m] = 0.0;
    }
    if (MODE != kModeLoglik && inf.hi_s > inf.lo_s) {
      const int32_t rfirst = static_cast<int32_t>(row0 + lr0);
      long long k = lower_bound_rows(nnz_s, inf.base_s, P.row_idx, inf.lo_s, inf.hi_s, rfirst,
                                     inf.smem_s != 0);
      while (k < inf.hi_s) {
        const int32_t r = inf.smem_s ? nnz_s[k - inf.base_s] : P.row_idx[k];
        const int m = r - rfirst;
        if (m >= kIpt) break;
        if constexpr (IND) {
          xb |= 1u << m;
        } else {
#pragma unroll
          for (int q = 0; q < kIpt; ++q)
            if (q == m) xv[q] = P.vals[k];
        }
        ++k;
      }
    }
    auto row_val = [&](int m) {
      Seg<L> rv;
      rv.f = STRATA ? ((cw[m] & kCodeSeg) ? 1u : 0u) : 0u;
      rv.v[0] = ev[m];
      if constexpr (L >= 2) {
        if constexpr (IND) {
          rv.v[1] = ((xb >> m) & 1u) ? ev[m] : 0.0;
        } else {
          const double ex = __dmul_rn(ev[m], xv[m]);
          rv.v[1] = ex;
          rv.v[2] = __dmul_rn(ex, xv[m]);
        }
      }
      return rv;
    };
    // ---- thread aggregate -> exclusive prefix within the tile ----
    Seg<L> own = Seg<L>::zero();
#pragma unroll
    for (int m = 0; m < kIpt; ++m) own = comb<L, STRATA>(own, row_val(m));
    const Seg<L> inc = warp_scan_incl<L, STRATA>(own, lane);
    if (lane == 31) {
      st->scan[par][warp][0] = inc.f ? 1.0 : 0.0;
#pragma unroll
      for (int i = 0; i < L; ++i) st->scan[par][warp][1 + i] = inc.v[i];
    }
    consumer_sync();
    Seg<L> excl = Seg<L>::zero(), tot = Seg<L>::zero();
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) {
      Seg<L> x;
      x.f = STRATA ? (st->scan[par][w][0] != 0.0 ? 1u : 0u) : 0u;
#pragma unroll
      for (int i = 0; i < L; ++i) x.v[i] = st->scan[par][w][1 + i];
      if (w < warp) excl = comb<L, STRATA>(excl, x);
      tot = comb<L, STRATA>(tot, x);
    }
    {
      Seg<L> e1;
      e1.f = STRATA ? __shfl_up_sync(0xffffffffu, inc.f, 1) : 0u;
#pragma unroll
      for (int i = 0; i < L; ++i) e1.v[i] = __shfl_up_sync(0xffffffffu, inc.v[i], 1);
      if (lane > 0) excl = comb<L, STRATA>(excl, e1);
    }
    if (tid == 0) {
      // the tile's fresh exp(eta) sum for the next launch's phase A
      t_out[2 * t] = tot.f ? 1.0 : 0.0;
      t_out[2 * t + 1] = tot.v[0];
      // previous tile's partials are visible after the scan barrier
      if (prev_t >= 0) flush_partial(P, st, prev_t, par ^ 1);
    }
    prev_t = t;
    // ---- the tile prefix (published once by the last phase-A warp) ----
    if (!ready_seen) {
      if (tid == 0)
        while (ld_acquire_u64(&ctl->ready) != epoch) __nanosleep(64);
      consumer_sync();
      ready_seen = true;
      load_prefix();
    }
    if (tid == 0) trace_ev(P, 9, t);
    // ---- commit the deferred update to global memory (phase A has read it) ----
    if (pd.active) {
      const int w0 = warp * 32 * kIpt;
      for (long long k = inf.lo_u + lane; k < inf.hi_u; k += 32) {
        const int32_t r = inf.smem_u ? nnz_u[k - inf.base_u] : P.row_idx[k];
        const int lr = static_cast<int>(r - row0);
        if (lr < w0 || lr >= w0 + 32 * kIpt) continue;
        const uint32_t cwr = *reinterpret_cast<const uint32_t*>(sc + swz<kIpt * 4>(lr * 4));
        if (cwr & kCodeMasked) continue;
        P.e[r] = *e_at(sb, lr);
        if (pd.ind)
          red_add_f64(&P.eta[r], pd.delta);  // eta += delta
        else
          P.eta[r] = __dadd_rn(__ldcg(P.eta + r), __dmul_rn(P.vals[k], pd.delta));
      }
      if (MODE == kModeLoglik) consumer_sync();  // eta read below
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&st->empty[s]);  // stage may be refilled now
    Seg<L> run, rq;
    run.f = STRATA ? (pg[0] != 0.0 ? 1u : 0u) : 0u;
    rq.f = STRATA ? (pq[0] != 0.0 ? 1u : 0u) : 0u;
#pragma unroll
    for (int i = 0; i < L; ++i) {
      run.v[i] = pg[1 + i];
      rq.v[i] = pq[1 + i];
    }
    run = comb<L, STRATA>(comb<L, STRATA>(run, rq), excl);

    // ---- transform at tied-block ends and reduce ----
    double acc0 = 0.0, acc1 = 0.0;
    int bad = 0;
#pragma unroll
    for (int m = 0; m < kIpt; ++m) {
      run = comb<L, STRATA>(run, row_val(m));
      const uint32_t d = cw[m] & kCodeCount;
      if (d) {
        const double den = run.v[0];
        const double cnt = static_cast<double>(d);
        if (!(den > 0.0)) {
          bad = 1;
        } else if constexpr (L >= 2) {
          const double rinv = __drcp_rn(den);
          const double G = __dmul_rn(run.v[1], rinv);
          const double H = IND ? G : __dmul_rn(run.v[L - 1], rinv);
          acc0 = __dadd_rn(acc0, __dmul_rn(cnt, G));
          acc1 = __dadd_rn(acc1, __dmul_rn(cnt, __dsub_rn(H, __dmul_rn(G, G))));
        } else {
          acc1 = __dadd_rn(acc1, __dmul_rn(cnt, log(den)));
        }
      }
      if constexpr (MODE == kModeLoglik) {
        if (cw[m] & kCodeEvent) acc0 = __dadd_rn(acc0, __ldcg(P.eta + row0 + lr0 + m));
      }
    }
    // per-warp partials; summed in warp order after the next barrier
    acc0 = warp_sum(acc0);
    acc1 = warp_sum(acc1);
    const double badw = warp_sum(static_cast<double>(bad));
    if (lane == 0) {
      st->part[par][warp][0] = acc0;
      st->part[par][warp][1] = acc1;
      st->part[par][warp][2] = badw;
    }
    if (tid == 0) trace_ev(P, 10, t);
    last_par = par;
  }
  consumer_sync();
  if (tid == 0 && prev_t >= 0) flush_partial(P, st, prev_t, last_par);
}

// ---------------------------------------------------------------------------
// the fused sweep kernel
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kSweepThreads, 2)
    sweep_kernel(const __grid_constant__ CUtensorMap tm_e,
                 const __grid_constant__ CUtensorMap tm_code, const SweepParams P) {
  constexpr int L = (MODE == kModeLoglik) ? 1 : 3;
  extern __shared__ unsigned char smem_raw[];
  // 1024B-align by pointer arithmetic on the shared array itself, so the
  // compiler keeps the shared address space (LDS, not generic LD)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  SmemTail* st = reinterpret_cast<SmemTail*>(smem + size_t(kStages) * kStageBytes);
  Ctl* ctl = P.ctl;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  if (ctl->halted) return;  // an earlier coordinate of this cycle failed
  const unsigned long long epoch = ctl->epoch;
  Pending pd;
  pd.refresh = ctl->refresh_pending != 0;
  pd.col = ctl->pend_col;
  pd.delta = ctl->pend_delta;
  pd.factor = ctl->pend_factor;
  pd.active = !pd.refresh && pd.col >= 0 && pd.delta != 0.0;
  pd.ind = pd.active ? (P.col_ind[pd.col] != 0 || !P.has_vals) : true;
  const bool tprev_valid = ctl->tprev_valid != 0;
  const long long col = P.column;
  const int ntiles = P.ntiles;
  const double* t_in = P.tsum + size_t(epoch & 1) * 2 * ntiles;
  double* t_out = P.tsum + size_t((epoch & 1) ^ 1) * 2 * ntiles;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&st->full[s], 1);
      mbar_init(&st->empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) trace_ev(P, 0, 0);

  // ------------------------------ phase A ------------------------------------
  // consumer warps only: the producer starts streaming tiles immediately
  if (warp != kProducerWarp) {
    int32_t* scratch = st->scratch[warp];
    double absmax = 0.0;
    for (;;) {
      unsigned t = 0;
      if (lane == 0) t = atomicAdd(&ctl->items_a, 1u);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= static_cast<unsigned>(ntiles)) break;
      if (lane == 0) trace_ev(P, 2, static_cast<int>(t));
      const Seg<3> A = phase_a_tile<L>(P, pd, static_cast<int>(t), col, tprev_valid, t_in,
                                       scratch, lane, &absmax);
      // publish A[t]; the warp completing a 32-tile group scans it, the warp
      // completing the last group scans the group totals and raises `ready`
      const int g = static_cast<int>(t) / 32;
      const int gsize = min(32, ntiles - g * 32);
      unsigned done = 0;
      if (lane == 0) {
        store_seg(P.agg + size_t(t) * 4, A);
        __threadfence();
        trace_ev(P, 3, static_cast<int>(t));
        done = atomicAdd(&P.grp_cnt[g], 1u);
      }
      done = __shfl_sync(0xffffffffu, done, 0);
      if (done == static_cast<unsigned>(gsize) - 1) {
        __threadfence();
        group_scan(P, g, gsize, lane);
        __syncwarp();
        unsigned gd = 0;
        if (lane == 0) {
          __threadfence();
          gd = atomicAdd(&ctl->groups_done, 1u);
        }
        gd = __shfl_sync(0xffffffffu, gd, 0);
        const int ngroups = (ntiles + 31) / 32;
        if (gd == static_cast<unsigned>(ngroups) - 1) {
          __threadfence();
          if (lane == 0) trace_ev(P, 4, 0);
          final_scan(P, ngroups, lane);
          __syncwarp();
          if (lane == 0) {
            __threadfence();
            st_release_u64(&ctl->ready, epoch);
            trace_ev(P, 5, 0);
          }
        }
      }
    }
    if (pd.refresh) {
      // exact max |eta| of the refreshed rows -> the next fast-path bound
#pragma unroll
      for (int d = 16; d > 0; d >>= 1)
        absmax = fmax(absmax, __shfl_xor_sync(0xffffffffu, absmax, d));
      if (lane == 0 && absmax > 0.0)
        atomicMax(&ctl->absmax_next_bits,
                  static_cast<unsigned long long>(__double_as_longlong(absmax)));
    }
  }
  if (tid == 0) trace_ev(P, 1, 0);

  // ------------------------------ phase C ------------------------------------
  if (warp == kProducerWarp) {
    if (lane == 0) {
      if (pd.refresh) {  // tiles must be read after phase A rewrote them
        while (ld_acquire_u64(&ctl->ready) != epoch) __nanosleep(64);
      }
      const uint32_t* tp_s =
          (MODE != kModeLoglik) ? P.tile_ptr + size_t(col) * (ntiles + 1) : nullptr;
      const uint32_t* tp_u = pd.active ? P.tile_ptr + size_t(pd.col) * (ntiles + 1) : nullptr;
      const long long cb_s = (MODE != kModeLoglik) ? P.col_ptr[col] : 0;
      const long long cb_u = pd.active ? P.col_ptr[pd.col] : 0;
      unsigned t = atomicAdd(&ctl->tile_counter, 1u);
      for (int it = 0;; ++it) {
        const int s = it % kStages;
        const uint32_t ph = (it / kStages) & 1;
        mbar_wait(&st->empty[s], ph ^ 1);
        StageInfo& inf = st->info[s];
        if (t >= static_cast<unsigned>(ntiles)) {
          inf.tile = -1;
          mbar_arrive(&st->full[s]);
          break;
        }
        unsigned char* sb = smem + size_t(s) * kStageBytes;
        // the dense tiles first: their latency overlaps the index lookups below
        mbar_expect_tx(&st->full[s], kEBytes + kCodeBytes);
        tma_load_2d(sb, &tm_e, 0, static_cast<int>(t) * kThreads, &st->full[s]);
        tma_load_2d(sb + kEBytes, &tm_code, 0, static_cast<int>(t) * kThreads, &st->full[s]);
        const unsigned tnext = atomicAdd(&ctl->tile_counter, 1u);
        int32_t* nnz_s = reinterpret_cast<int32_t*>(sb + kEBytes + kCodeBytes);
        int32_t* nnz_u = nnz_s + kNnzCap;
        const uint32_t s0 = tp_s ? tp_s[t] : 0, s1 = tp_s ? tp_s[t + 1] : 0;
        const uint32_t u0 = tp_u ? tp_u[t] : 0, u1 = tp_u ? tp_u[t + 1] : 0;
        inf.tile = static_cast<int>(t);
        inf.lo_s = cb_s + s0;
        inf.hi_s = cb_s + s1;
        inf.lo_u = cb_u + u0;
        inf.hi_u = cb_u + u1;
        inf.base_s = inf.lo_s & ~3LL;
        inf.base_u = inf.lo_u & ~3LL;
        const long long as1 = (inf.hi_s + 3) & ~3LL, au1 = (inf.hi_u + 3) & ~3LL;
        const bool cs = inf.hi_s > inf.lo_s && as1 - inf.base_s <= kNnzCap;
        const bool cu = inf.hi_u > inf.lo_u && au1 - inf.base_u <= kNnzCap;
        uint32_t extra = 0;
        if (cs) extra += static_cast<uint32_t>((as1 - inf.base_s) * 4);
        if (cu) extra += static_cast<uint32_t>((au1 - inf.base_u) * 4);
        inf.smem_s = cs ? 1 : 0;
        inf.smem_u = cu ? 1 : 0;
        if (extra) mbar_expect_tx(&st->full[s], extra);
        if (cs)
          bulk_load_1d(nnz_s, P.row_idx + inf.base_s,
                       static_cast<uint32_t>((as1 - inf.base_s) * 4), &st->full[s]);
        if (cu)
          bulk_load_1d(nnz_u, P.row_idx + inf.base_u,
                       static_cast<uint32_t>((au1 - inf.base_u) * 4), &st->full[s]);
        mbar_arrive(&st->full[s]);
        t = tnext;
      }
    }
  } else {
    // ------------------------------ consumers -----------------------------
    const bool ind_s = (MODE != kModeLoglik) ? (P.col_ind[col] != 0 || !P.has_vals) : true;
    if (MODE == kModeLoglik || ind_s) {
      if (P.has_strata)
        consume<MODE, true, true>(P, pd, st, smem, t_out, epoch, ctl, col, tid);
      else
        consume<MODE, true, false>(P, pd, st, smem, t_out, epoch, ctl, col, tid);
    } else if (MODE != kModeLoglik) {
      if (P.has_strata)
        consume<MODE, false, true>(P, pd, st, smem, t_out, epoch, ctl, col, tid);
      else
        consume<MODE, false, false>(P, pd, st, smem, t_out, epoch, ctl, col, tid);
    }
  }

  // ------------------------------ completion + tail ------------------------
  __syncthreads();
  __shared__ unsigned int s_last;
  if (tid == 0) {
    __threadfence();
    s_last = (atomicAdd(&ctl->ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid >= kThreads) return;  // tail uses the consumer threads only

  // deterministic reduction of the per-tile partials (tile order)
  double r0 = 0.0, r1 = 0.0, rb = 0.0;
#pragma unroll 4
  for (int t = tid; t < ntiles; t += kThreads) {
    const double* tp = P.tile_part + size_t(t) * 4;
    r0 = __dadd_rn(r0, __ldcg(tp));
    r1 = __dadd_rn(r1, __ldcg(tp + 1));
    rb = __dadd_rn(rb, __ldcg(tp + 2));
  }
  {
    double t3[3] = {r0, r1, rb};
    block_sum3(t3, st, tid);
    r0 = t3[0];
    r1 = t3[1];
    rb = t3[2];
  }
  const bool badden = rb != 0.0;

  if (tid == 0 && pd.refresh) {
    // refresh finished: the bound is exact again
    ctl->eta_absmax_bits = ctl->absmax_next_bits;
    ctl->absmax_next_bits = 0ULL;
    ctl->bound_slack = 0.0;
  }

  if constexpr (MODE == kModeLoglik) {
    if (tid == 0) {
      ctl->ll_fixed = r0;
      ctl->ll_logden = r1;
      ctl->loglik = __dsub_rn(r0, r1);
      ctl->bad = badden;
      if (badden && ctl->err_code == 0) {
        ctl->err_code = 7;
        ctl->err_col = -1;
      }
      if (ctl->err_code) ctl->halted = 1;
      ctl->pend_col = -1;
      ctl->pend_delta = 0.0;
      ctl->refresh_pending = 0;
    }
  } else {
    // Engine::finish (src/engine.cpp:220-230)
    const double fixed = P.fixed[col];
    const double grad = __dsub_rn(fixed, r0);
    double hess = -r1;
    if (hess > 0.0) hess = 0.0;
    const bool nonfinite = !isfinite(grad) || !isfinite(hess);
    if constexpr (MODE == kModeGradApi) {
      if (tid == 0) {
        ctl->grad_sum = r0;
        ctl->hess_sum = r1;
        ctl->gradient = grad;
        ctl->hessian = hess;
        ctl->fixed_term = fixed;
        ctl->bad = badden;
        if ((badden || nonfinite) && ctl->err_code == 0) {
          ctl->err_code = 7;
          ctl->err_col = col;
        }
        ctl->pend_col = -1;
        ctl->pend_delta = 0.0;
        ctl->refresh_pending = 0;
      }
    } else {
      // CCD: coordinate_step + deferred update decision (src/ccd.cpp:152-167)
      __shared__ double s_delta;
      __shared__ int s_need_exact;
      if (tid == 0) {
        ctl->grad_sum = r0;
        ctl->hess_sum = r1;
        ctl->gradient = grad;
        ctl->hessian = hess;
        ctl->fixed_term = fixed;
        ctl->pend_col = -1;
        ctl->pend_delta = 0.0;
        ctl->refresh_pending = 0;
        s_delta = 0.0;
        s_need_exact = 0;
        if (badden || nonfinite) {
          ctl->err_code = 7;
          ctl->err_col = col;
          ctl->halted = 1;
        } else {
          const double bj = P.beta[col];
          const Step stp = coordinate_step_dev(bj, grad, hess, P.pen_kind, P.pen_strength,
                                               P.penalized[col] != 0, P.halfwidth[col]);
          if (stp.skipped) {
            ctl->skipped += 1;
          } else {
            st->bcast[1] = P.halfwidth[col];  // kept if the update overflows
            P.halfwidth[col] = stp.new_hw;
            if (stp.applied != 0.0) {
              // fast validate: exact max|eta| at the last refresh/load + the
              // accumulated |delta|*max|x| of later updates bounds every row
              const double bound =
                  __longlong_as_double(static_cast<long long>(ctl->eta_absmax_bits)) +
                  ctl->bound_slack;
              const double step_slack = P.colmax[col] * fabs(stp.applied);
              s_delta = stp.applied;
              s_need_exact = (bound + step_slack <= kFastBound) ? 0 : 1;
              st->bcast[2] = step_slack;
            }
          }
        }
      }
      consumer_sync();
      const double delta = s_delta;
      if (delta != 0.0) {
        int over = 0;
        if (s_need_exact) {
          // exact validate-before-mutate (src/engine.cpp:171-190)
          const long long k0 = P.col_ptr[col], k1 = P.col_ptr[col + 1];
          const bool ind = P.col_ind[col] != 0 || !P.has_vals;
          for (long long k = k0 + tid; k < k1; k += kThreads) {
            const int32_t r = P.row_idx[k];
            if (P.code[r] & kCodeMasked) continue;
            const double x = ind ? 1.0 : P.vals[k];
            if (fabs(__dadd_rn(__ldcg(P.eta + r), __dmul_rn(x, delta))) > kXbetaBound) over = 1;
          }
        }
        if (tid == 0) st->flag = 0;
        consumer_sync();
        if (over) st->flag = 1;
        consumer_sync();
        over = st->flag;
        if (tid == 0) {
          if (over) {
            ctl->err_code = 8;
            ctl->err_col = col;
            ctl->halted = 1;
            P.halfwidth[col] = st->bcast[1];  // unchanged on failure (exception path)
          } else {
            P.beta[col] = __dadd_rn(P.beta[col], delta);  // beta_[column] += delta
            ctl->pend_col = col;
            ctl->pend_delta = delta;
            ctl->pend_factor = exp(delta);
            ctl->bound_slack = ctl->bound_slack + st->bcast[2];
            ctl->accepted += 1;
            if (ctl->accepted % P.recompute_interval == 0) {
              ctl->refresh_pending = 1;  // refresh subsumes the incremental update
              ctl->refreshes += 1;
            }
          }
        }
      }
    }
  }
  for (int g = tid; g < (ntiles + 31) / 32; g += kThreads) P.grp_cnt[g] = 0u;
  if (tid == 0) {
    ctl->tile_counter = 0;
    ctl->items_a = 0;
    ctl->groups_done = 0;
    ctl->ticket = 0;
    ctl->tprev_valid = 1;
    ctl->epoch = epoch + 1;
    trace_ev(P, 12, 0);
  }
}

}  // namespace

size_t sweep_smem_bytes() { return smem_total(); }
int sweep_threads() { return kSweepThreads; }

int sweep_max_active_ctas_per_sm() {
  int n = 0;
  cudaFuncSetAttribute(sweep_kernel<kModeGradCcd>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem_total()));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sweep_kernel<kModeGradCcd>, kSweepThreads,
                                                smem_total());
  return n;
}

cudaError_t launch_sweep(int mode, const CUtensorMap* tm_e, const CUtensorMap* tm_code,
                         const SweepParams& prm, int grid, cudaStream_t s) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(sweep_kernel<kModeGradApi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem_total()));
    cudaFuncSetAttribute(sweep_kernel<kModeGradCcd>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem_total()));
    cudaFuncSetAttribute(sweep_kernel<kModeLoglik>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem_total()));
    attr_done = true;
  }
  switch (mode) {
    case kModeGradApi:
      sweep_kernel<kModeGradApi><<<grid, kSweepThreads, smem_total(), s>>>(*tm_e, *tm_code, prm);
      break;
    case kModeGradCcd:
      sweep_kernel<kModeGradCcd><<<grid, kSweepThreads, smem_total(), s>>>(*tm_e, *tm_code, prm);
      break;
    default:
      sweep_kernel<kModeLoglik><<<grid, kSweepThreads, smem_total(), s>>>(*tm_e, *tm_code, prm);
      break;
  }
  return cudaGetLastError();
}

}  // namespace gss
