// gss_kernels.cu — sm_100a kernels of the Cox CCD hot path.
//
// The per-coordinate kernel (`sweep_kernel`) is ONE persistent, single-pass,
// decoupled-look-back scan -> transform -> reduce over the time-ordered rows
// (the reference's two-phase chunked fused_grad_hess,
// /root/reference/proj/include/survscan/scan_kernels.hpp:74-214, plus
// Engine::finish, src/engine.cpp:220-230).  Around the scan it fuses:
//   * the previous coordinate's deferred sparse eta/exp(eta) update
//     (Engine::update_xbeta_sparse, src/engine.cpp:162-218) or the periodic
//     full refresh (src/engine.cpp:120-160), applied tile by tile while the
//     tile is resident in shared memory;
//   * in CCD mode, the coordinate step (src/ccd.cpp:71-129) run by the last
//     CTA, which also decides the next deferred update.
// Data movement: one producer warp per CTA claims tiles dynamically (atomic
// counter => look-back forward progress without co-residency), loads the
// 2048-row tile of exp(eta) (fp64) and the per-row code word (int32) with 2D
// TMA (swizzled, bank-conflict-free for the thread-contiguous read), and
// bulk-copies the tile's slice of the column's row indices.  Consumer warps
// (256 threads x 8 rows) do the segmented fp64 scan.
//
// Determinism: every tile's exclusive prefix is P[checkpoint] ⊕ ordered
// tree-sum of the A's of its group, and the final reduction runs over
// per-tile partials in tile order, so results are bitwise reproducible run
// to run (the reference's guarantee, scan_kernels.hpp:8-10).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gss_device.cuh"
#include "gss_kernels.cuh"

namespace gss {

namespace {

constexpr int kSlot = 8;                         // doubles per look-back slot
constexpr uint32_t kEBytes = kTileRows * 8;      // 16 KB
constexpr uint32_t kCodeBytes = kTileRows * 4;   // 8 KB
constexpr uint32_t kNnzBytes = kNnzCap * 4;      // 2 KB
constexpr uint32_t kStageBytes = kEBytes + kCodeBytes + 2 * kNnzBytes;  // 28 KB
static_assert(kStageBytes % 1024 == 0, "stage alignment");
constexpr double kXbetaBound = 700.0;          // src/engine.cpp:12
constexpr double kHwFloor = 1e-300;            // src/ccd.cpp:13
constexpr double kFastBound = 700.0 * (1.0 - 1e-12);

struct StageInfo {
  int tile;
  int smem_s, smem_u;
  int pad;
  long long lo_s, hi_s, base_s;  // scan column nnz range [lo, hi); smem copy starts at base
  long long lo_u, hi_u, base_u;  // pending-update column nnz range
};

struct SmemTail {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  StageInfo info[kStages];
  double red[kThreads / 32][kSlot];  // per-warp partials
  double bcast[kSlot];
  int flag;
};

__host__ __device__ constexpr size_t smem_total() {
  return 1024 /*align slack*/ + size_t(kStages) * kStageBytes + sizeof(SmemTail);
}

__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
}

__device__ __forceinline__ double sgn(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }

// Reduce a Seg<L> held by every consumer thread in thread order; result is
// broadcast to all consumers. Fixed tree => deterministic.
template <int L>
__device__ __forceinline__ Seg<L> block_ordered_reduce(Seg<L> v, SmemTail* st, int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  v = warp_ordered_reduce(v);
  if (lane == 0) {
    st->red[warp][0] = v.f ? 1.0 : 0.0;
#pragma unroll
    for (int i = 0; i < L; ++i) st->red[warp][1 + i] = v.v[i];
  }
  consumer_sync();
  Seg<L> r = Seg<L>::zero();
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    Seg<L> x;
    x.f = st->red[w][0] != 0.0 ? 1u : 0u;
#pragma unroll
    for (int i = 0; i < L; ++i) x.v[i] = st->red[w][1 + i];
    r = seg_combine(r, x);
  }
  consumer_sync();
  return r;
}

// Exclusive scan across consumer threads (thread order); also returns the total.
template <int L>
__device__ __forceinline__ Seg<L> block_exclusive_scan(Seg<L> v, Seg<L>& total, SmemTail* st,
                                                       int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  const Seg<L> inc = warp_inclusive_scan(v, lane);
  if (lane == 31) {
    st->red[warp][0] = inc.f ? 1.0 : 0.0;
#pragma unroll
    for (int i = 0; i < L; ++i) st->red[warp][1 + i] = inc.v[i];
  }
  consumer_sync();
  Seg<L> wpre = Seg<L>::zero();
  Seg<L> tot = Seg<L>::zero();
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    Seg<L> x;
    x.f = st->red[w][0] != 0.0 ? 1u : 0u;
#pragma unroll
    for (int i = 0; i < L; ++i) x.v[i] = st->red[w][1 + i];
    if (w < warp) wpre = seg_combine(wpre, x);
    tot = seg_combine(tot, x);
  }
  consumer_sync();
  Seg<L> exc = shfl_up_seg(inc, 1);
  if (lane == 0) exc = Seg<L>::zero();
  total = tot;
  return seg_combine(wpre, exc);
}

__device__ __forceinline__ double block_sum(double v, SmemTail* st, int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  v = warp_sum(v);
  if (lane == 0) st->red[warp][7] = v;
  consumer_sync();
  double r = 0.0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) r = __dadd_rn(r, st->red[w][7]);
  consumer_sync();
  return r;
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
    for (int w = 0; w < kThreads / 32; ++w) r = __dadd_rn(r, st->red[w][5 + i]);
    v[i] = r;
  }
  consumer_sync();
}

__device__ __forceinline__ void atomic_max_abs(Ctl* ctl, double v) {
  v = fabs(v);
  atomicMax(&ctl->eta_absmax_bits, static_cast<unsigned long long>(__double_as_longlong(v)));
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

// coordinate_step (src/ccd.cpp:71-129), scalar.
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

// ---------------------------------------------------------------------------
// the fused sweep kernel
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kCtaThreads, 2)
    sweep_kernel(const __grid_constant__ CUtensorMap tm_e,
                 const __grid_constant__ CUtensorMap tm_code, const SweepParams P) {
  constexpr int L = (MODE == kModeLoglik) ? 1 : 3;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  SmemTail* st = reinterpret_cast<SmemTail*>(smem + size_t(kStages) * kStageBytes);
  Ctl* ctl = P.ctl;
  const int tid = threadIdx.x;

  if (ctl->halted) return;  // an earlier coordinate of this cycle failed
  const unsigned long long epoch = ctl->epoch;
  const bool refresh = ctl->refresh_pending != 0;
  const long long pcol = ctl->pend_col;
  const double pdelta = ctl->pend_delta;
  const double pfactor = ctl->pend_factor;
  const bool pend = !refresh && pcol >= 0 && pdelta != 0.0;
  const long long col = P.column;
  const int ntiles = P.ntiles;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&st->full[s], 1);
      mbar_init(&st->empty[s], kThreads / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (tid >= kThreads) {
    // ------------------------------ producer warp ------------------------
    if (tid == kThreads) {
      const uint32_t* tp_s =
          (MODE != kModeLoglik) ? P.tile_ptr + size_t(col) * (ntiles + 1) : nullptr;
      const uint32_t* tp_u = pend ? P.tile_ptr + size_t(pcol) * (ntiles + 1) : nullptr;
      const long long cb_s = (MODE != kModeLoglik) ? P.col_ptr[col] : 0;
      const long long cb_u = pend ? P.col_ptr[pcol] : 0;
      for (int it = 0;; ++it) {
        const int s = it % kStages;
        const uint32_t ph = (it / kStages) & 1;
        mbar_wait(&st->empty[s], ph ^ 1);
        const unsigned t = atomicAdd(&ctl->tile_counter, 1u);
        StageInfo& inf = st->info[s];
        if (t >= static_cast<unsigned>(ntiles)) {
          inf.tile = -1;
          mbar_arrive(&st->full[s]);
          break;
        }
        unsigned char* sb = smem + size_t(s) * kStageBytes;
        int32_t* nnz_s = reinterpret_cast<int32_t*>(sb + kEBytes + kCodeBytes);
        int32_t* nnz_u = nnz_s + kNnzCap;
        uint32_t bytes = kEBytes + kCodeBytes;
        inf.tile = static_cast<int>(t);
        inf.smem_s = inf.smem_u = 0;
        inf.lo_s = inf.hi_s = inf.lo_u = inf.hi_u = 0;
        long long cs_a0 = 0, cu_a0 = 0;
        uint32_t cs_bytes = 0, cu_bytes = 0;
        if (tp_s) {
          inf.lo_s = cb_s + tp_s[t];
          inf.hi_s = cb_s + tp_s[t + 1];
          cs_a0 = inf.lo_s & ~3LL;
          const long long a1 = (inf.hi_s + 3) & ~3LL;
          if (inf.hi_s > inf.lo_s && a1 - cs_a0 <= kNnzCap) {
            inf.smem_s = 1;
            cs_bytes = static_cast<uint32_t>((a1 - cs_a0) * 4);
            bytes += cs_bytes;
          }
          inf.base_s = cs_a0;
        }
        if (tp_u) {
          inf.lo_u = cb_u + tp_u[t];
          inf.hi_u = cb_u + tp_u[t + 1];
          cu_a0 = inf.lo_u & ~3LL;
          const long long a1 = (inf.hi_u + 3) & ~3LL;
          if (inf.hi_u > inf.lo_u && a1 - cu_a0 <= kNnzCap) {
            inf.smem_u = 1;
            cu_bytes = static_cast<uint32_t>((a1 - cu_a0) * 4);
            bytes += cu_bytes;
          }
          inf.base_u = cu_a0;
        }
        mbar_arrive_expect_tx(&st->full[s], bytes);
        tma_load_2d(sb, &tm_e, 0, static_cast<int>(t) * kThreads, &st->full[s]);
        tma_load_2d(sb + kEBytes, &tm_code, 0, static_cast<int>(t) * kThreads, &st->full[s]);
        if (cs_bytes) bulk_load_1d(nnz_s, P.row_idx + cs_a0, cs_bytes, &st->full[s]);
        if (cu_bytes) bulk_load_1d(nnz_u, P.row_idx + cu_a0, cu_bytes, &st->full[s]);
      }
    }
  } else {
    // ------------------------------ consumer warps -----------------------
    const int lane = tid & 31;
    const bool ind_s = (MODE != kModeLoglik) ? (P.col_ind[col] != 0 || !P.has_vals) : true;
    const bool ind_u = pend ? (P.col_ind[pcol] != 0 || !P.has_vals) : true;
    for (int it = 0;; ++it) {
      const int s = it % kStages;
      const uint32_t ph = (it / kStages) & 1;
      mbar_wait(&st->full[s], ph);
      const StageInfo inf = st->info[s];
      if (inf.tile < 0) break;
      const int t = inf.tile;
      const long long row0 = static_cast<long long>(t) * kTileRows;
      unsigned char* sb = smem + size_t(s) * kStageBytes;
      double* se = reinterpret_cast<double*>(sb);
      const uint32_t* scode = reinterpret_cast<const uint32_t*>(sb + kEBytes);
      const int32_t* nnz_s = reinterpret_cast<const int32_t*>(sb + kEBytes + kCodeBytes);
      const int32_t* nnz_u = nnz_s + kNnzCap;

      // ---- (1) deferred state change for rows of this tile ----------------
      bool wrote = false;
      if (refresh) {
        // Engine::refresh -> load_beta (src/engine.cpp:120-160): eta_i =
        // sum_j beta_j x_ij over the row's CSR entries (ascending j), warp per row.
        const int warp = tid >> 5;
        for (int lr = warp; lr < kTileRows; lr += kThreads / 32) {
          const long long r = row0 + lr;
          if (r >= P.n) break;
          const uint32_t cw =
              *reinterpret_cast<const uint32_t*>(reinterpret_cast<const unsigned char*>(scode) +
                                                 swz<kIpt * 4>(lr * 4));
          if (cw & kCodeMasked) continue;
          const long long k0 = P.row_ptr[r], k1 = P.row_ptr[r + 1];
          double acc = 0.0;
          for (long long k = k0 + lane; k < k1; k += 32) {
            const int32_t c = P.csr_col[k];
            const double x = P.csr_val ? P.csr_val[k] : 1.0;
            acc = __dadd_rn(acc, __dmul_rn(P.beta[c], x));
          }
          acc = warp_sum(acc);
          if (lane == 0) {
            if (fabs(acc) > kXbetaBound && ctl->err_code == 0) {
              ctl->err_code = 8;  // OverflowError from refresh
              ctl->err_col = -1;
            }
            const double ev = exp(acc);
            P.eta[r] = acc;
            P.e[r] = ev;
            *reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(se) +
                                       swz<kIpt * 8>(lr * 8)) = ev;
            atomic_max_abs(ctl, acc);
          }
        }
        wrote = true;
      } else if (pend) {
        // Engine::update_xbeta_sparse commit half (src/engine.cpp:192-215);
        // validation already happened in the tail that deferred it.
        double mx = 0.0;
        for (long long k = inf.lo_u + tid; k < inf.hi_u; k += kThreads) {
          const int32_t r = inf.smem_u ? nnz_u[k - inf.base_u] : P.row_idx[k];
          const int lr = static_cast<int>(r - row0);
          const uint32_t cw = *reinterpret_cast<const uint32_t*>(
              reinterpret_cast<const unsigned char*>(scode) +
              swz<kIpt * 4>(lr * 4));
          if (cw & kCodeMasked) continue;
          double* pe = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(se) +
                                                 swz<kIpt * 8>(lr * 8));
          const double x = ind_u ? 1.0 : P.vals[k];
          const double ne = __dadd_rn(P.eta[r], __dmul_rn(x, pdelta));
          const double ev = ind_u ? __dmul_rn(*pe, pfactor) : exp(ne);
          P.eta[r] = ne;
          P.e[r] = ev;
          *pe = ev;
          mx = fmax(mx, fabs(ne));
        }
        if (mx > 0.0) atomic_max_abs(ctl, mx);
        wrote = true;
      }
      if (wrote) consumer_sync();

      // ---- (2) thread-contiguous rows: exp(eta), code, x_j ----------------
      const int lr0 = tid * kIpt;
      double ev[kIpt];
      uint32_t cw[kIpt];
      {
        const unsigned char* eb = reinterpret_cast<const unsigned char*>(se);
#pragma unroll
        for (int c = 0; c < kIpt / 2; ++c) {
          const double2 v =
              *reinterpret_cast<const double2*>(eb + swz<kIpt * 8>(tid * (kIpt * 8) + c * 16));
          ev[2 * c] = v.x;
          ev[2 * c + 1] = v.y;
        }
        const unsigned char* cb = reinterpret_cast<const unsigned char*>(scode);
#pragma unroll
        for (int c = 0; c < kIpt / 4; ++c) {
          const uint4 v =
              *reinterpret_cast<const uint4*>(cb + swz<kIpt * 4>(tid * (kIpt * 4) + c * 16));
          cw[4 * c] = v.x;
          cw[4 * c + 1] = v.y;
          cw[4 * c + 2] = v.z;
          cw[4 * c + 3] = v.w;
        }
      }
      double xv[kIpt];
#pragma unroll
      for (int m = 0; m < kIpt; ++m) xv[m] = 0.0;
      if (MODE != kModeLoglik && inf.hi_s > inf.lo_s) {
        const int32_t rfirst = static_cast<int32_t>(row0 + lr0);
        long long k = lower_bound_rows(nnz_s, inf.base_s, P.row_idx, inf.lo_s, inf.hi_s, rfirst,
                                       inf.smem_s != 0);
        while (k < inf.hi_s) {
          const int32_t r = inf.smem_s ? nnz_s[k - inf.base_s] : P.row_idx[k];
          const int m = r - rfirst;
          if (m >= kIpt) break;
          xv[m] = ind_s ? 1.0 : P.vals[k];
          ++k;
        }
      }
      if (wrote) fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&st->empty[s]);  // stage may be refilled now

      // ---- (3) thread aggregate, block scan, tile aggregate ---------------
      Seg<L> own = Seg<L>::zero();
#pragma unroll
      for (int m = 0; m < kIpt; ++m) {
        Seg<L> rv;
        rv.f = (cw[m] & kCodeSeg) ? 1u : 0u;
        rv.v[0] = ev[m];
        if constexpr (L == 3) {
          const double ex = __dmul_rn(ev[m], xv[m]);
          rv.v[1] = ex;
          rv.v[2] = __dmul_rn(ex, xv[m]);
        }
        own = seg_combine(own, rv);
      }
      Seg<L> tile_tot;
      const Seg<L> excl = block_exclusive_scan(own, tile_tot, st, tid);

      // publish the tile aggregate A[t]
      if (tid == 0) {
        double* slot = P.aggA + size_t(t) * kSlot;
        slot[0] = static_cast<double>(tile_tot.f);
#pragma unroll
        for (int i = 0; i < L; ++i) slot[1 + i] = tile_tot.v[i];
        st_release_u64(&P.statA[t], epoch);
      }

      // ---- (4) look-back: prefix = P[group-1] ⊕ (A[B] ⊕ ... ⊕ A[t-1]) ------
      const int grp = t / kGroup;
      const int B = grp * kGroup;
      Seg<L> mine = Seg<L>::zero();
      if (B + tid < t) {
        const int idx = B + tid;
        while (ld_acquire_u64(&P.statA[idx]) != epoch) __nanosleep(32);
        const double* slot = P.aggA + size_t(idx) * kSlot;
        mine.f = ld_relaxed_f64(slot) != 0.0 ? 1u : 0u;
#pragma unroll
        for (int i = 0; i < L; ++i) mine.v[i] = ld_relaxed_f64(slot + 1 + i);
      }
      const Seg<L> ingroup = block_ordered_reduce(mine, st, tid);
      Seg<L> ck = Seg<L>::zero();
      if (grp > 0) {
        // every consumer reads the same checkpoint (L2-resident broadcast)
        while (ld_acquire_u64(&P.statP[grp - 1]) != epoch) __nanosleep(32);
        const double* slot = P.aggP + size_t(grp - 1) * kSlot;
        ck.f = ld_relaxed_f64(slot) != 0.0 ? 1u : 0u;
#pragma unroll
        for (int i = 0; i < L; ++i) ck.v[i] = ld_relaxed_f64(slot + 1 + i);
      }
      const Seg<L> tile_prefix = seg_combine(ck, ingroup);
      if (tid == 0 && (t % kGroup) == kGroup - 1) {
        const Seg<L> incl = seg_combine(tile_prefix, tile_tot);
        double* slot = P.aggP + size_t(grp) * kSlot;
        slot[0] = static_cast<double>(incl.f);
#pragma unroll
        for (int i = 0; i < L; ++i) slot[1 + i] = incl.v[i];
        st_release_u64(&P.statP[grp], epoch);
      }

      // ---- (5) transform at tied-block ends and reduce --------------------
      Seg<L> run = seg_combine(tile_prefix, excl);
      double acc0 = 0.0, acc1 = 0.0;
      int bad = 0;
#pragma unroll
      for (int m = 0; m < kIpt; ++m) {
        Seg<L> rv;
        rv.f = (cw[m] & kCodeSeg) ? 1u : 0u;
        rv.v[0] = ev[m];
        if constexpr (L == 3) {
          const double ex = __dmul_rn(ev[m], xv[m]);
          rv.v[1] = ex;
          rv.v[2] = __dmul_rn(ex, xv[m]);
        }
        run = seg_combine(run, rv);
        const uint32_t d = cw[m] & kCodeCount;
        if (d) {
          const double den = run.v[0];
          const double cnt = static_cast<double>(d);
          if (!(den > 0.0)) {
            bad = 1;
          } else if constexpr (L == 3) {
            const double rinv = __drcp_rn(den);
            const double G = __dmul_rn(run.v[1], rinv);
            const double H = __dmul_rn(run.v[2], rinv);
            acc0 = __dadd_rn(acc0, __dmul_rn(cnt, G));
            acc1 = __dadd_rn(acc1, __dmul_rn(cnt, __dsub_rn(H, __dmul_rn(G, G))));
          } else {
            acc1 = __dadd_rn(acc1, __dmul_rn(cnt, log(den)));
          }
        }
        if constexpr (MODE == kModeLoglik) {
          if (cw[m] & kCodeEvent) acc0 = __dadd_rn(acc0, P.eta[row0 + lr0 + m]);
        }
      }
      double t3[3] = {acc0, acc1, static_cast<double>(bad)};
      block_sum3(t3, st, tid);
      if (tid == 0) {
        double* tp = P.tile_part + size_t(t) * 4;
        tp[0] = t3[0];
        tp[1] = t3[1];
        tp[2] = t3[2];
      }
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
  for (int t = tid; t < ntiles; t += kThreads) {
    const double* tp = P.tile_part + size_t(t) * 4;
    r0 = __dadd_rn(r0, ld_relaxed_f64(tp));
    r1 = __dadd_rn(r1, ld_relaxed_f64(tp + 1));
    rb = __dadd_rn(rb, ld_relaxed_f64(tp + 2));
  }
  {
    double t3[3] = {r0, r1, rb};
    block_sum3(t3, st, tid);
    r0 = t3[0];
    r1 = t3[1];
    rb = t3[2];
  }
  const bool badden = rb != 0.0;

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
    double grad = __dsub_rn(fixed, r0);
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
            if (stp.applied != 0.0) {
              const double bound = __longlong_as_double(
                  static_cast<long long>(ctl->eta_absmax_bits));
              const double worst = bound + P.colmax[col] * fabs(stp.applied);
              s_delta = stp.applied;
              s_need_exact = (worst <= kFastBound) ? 0 : 1;
            }
            st->bcast[1] = P.halfwidth[col];  // kept if the update overflows
            P.halfwidth[col] = stp.new_hw;
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
            if (fabs(__dadd_rn(P.eta[r], __dmul_rn(x, delta))) > kXbetaBound) over = 1;
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
  if (tid == 0) {
    ctl->tile_counter = 0;
    ctl->ticket = 0;
    ctl->epoch = epoch + 1;
  }
}

}  // namespace

size_t sweep_smem_bytes() { return smem_total(); }

int sweep_max_active_ctas_per_sm() {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sweep_kernel<kModeGradCcd>, kCtaThreads,
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
      sweep_kernel<kModeGradApi><<<grid, kCtaThreads, smem_total(), s>>>(*tm_e, *tm_code, prm);
      break;
    case kModeGradCcd:
      sweep_kernel<kModeGradCcd><<<grid, kCtaThreads, smem_total(), s>>>(*tm_e, *tm_code, prm);
      break;
    default:
      sweep_kernel<kModeLoglik><<<grid, kCtaThreads, smem_total(), s>>>(*tm_e, *tm_code, prm);
      break;
  }
  return cudaGetLastError();
}

}  // namespace gss
