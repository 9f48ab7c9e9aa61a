// gss_separated.cu — the unfused "separated" derivative path
// (Engine::grad_hessian_separated, src/engine.cpp:244-329 + tuple3_scan,
// src/scan.cpp:141-214).  It exists as the fusion ablation of the reference
// (acceptance check 5, tests/acceptance.cpp:196-235; test_engine.cpp:165-176):
// the same (g', g'') as the fused cycle kernel, computed in separate passes
// over materialised lanes:
//
//   1. lanes       a = e, b = e*x, c = e*x^2            (3 x npad fp64 written)
//   2. suffix scan of u*(a,b,c) per tile (Fine-Gray with competing rows only)
//   3. prefix scan of (a,b,c) per tile, in place
//   4. tile carries: segmented (by stratum) exclusive prefix / suffix of the
//      tile totals, one CTA
//   5. Breslow transform at tied-block ends + per-tile partial sums
//   6. fixed-order reduction of the tile partials
//
// Tiles are the dataset's 2048-row, stratum-aligned tiles (no tile spans two
// strata), so the scans are plain inside a tile and segmented over tiles.
// HBM-bound like the fused path but with ~4x its traffic; it is not on the
// CCD hot path.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "gss_device.cuh"
#include "gss_kernels.cuh"

namespace gss {

namespace {

constexpr int kSepThreads = 256;
constexpr int kSepRows = kTileRows / kSepThreads;  // 8 rows per thread
static_assert(kSepRows * kSepThreads == kTileRows, "tile split");

struct L3 {
  double a, b, c;
};

__device__ __forceinline__ L3 l3_add(L3 x, L3 y) { return {x.a + y.a, x.b + y.b, x.c + y.c}; }

// Block-wide inclusive scan of one L3 per thread (fixed order: warp shuffle
// scan, then a scan of the 8 warp totals).  Returns the inclusive value;
// *total receives the block total.
__device__ L3 block_scan_l3(L3 v, L3* total) {
  __shared__ L3 wsum[kSepThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double a = __shfl_up_sync(0xffffffffu, v.a, d);
    const double b = __shfl_up_sync(0xffffffffu, v.b, d);
    const double c = __shfl_up_sync(0xffffffffu, v.c, d);
    if (lane >= d) v = l3_add(L3{a, b, c}, v);
  }
  if (lane == 31) wsum[w] = v;
  __syncthreads();
  if (w == 0 && lane < kSepThreads / 32) {
    L3 s = wsum[lane];
#pragma unroll
    for (int d = 1; d < kSepThreads / 32; d <<= 1) {
      const double a = __shfl_up_sync(0xffu, s.a, d);
      const double b = __shfl_up_sync(0xffu, s.b, d);
      const double c = __shfl_up_sync(0xffu, s.c, d);
      if (lane >= d) s = l3_add(L3{a, b, c}, s);
    }
    wsum[lane] = s;
  }
  __syncthreads();
  if (w > 0) v = l3_add(wsum[w - 1], v);
  *total = wsum[kSepThreads / 32 - 1];
  __syncthreads();
  return v;
}

// 1. a = e over all rows, b = c = 0 (grid-stride)
__global__ void sep_lanes_init(const double* __restrict__ e, int64_t npad, double* __restrict__ la,
                               double* __restrict__ lb, double* __restrict__ lc) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npad;
       i += int64_t(gridDim.x) * blockDim.x) {
    la[i] = e[i];
    lb[i] = 0.0;
    lc[i] = 0.0;
  }
}

// 1b. scatter the column: b = e*x, c = (e*x)*x (engine.cpp:255-259)
__global__ void sep_lanes_scatter(const int32_t* __restrict__ rows, const double* __restrict__ vals,
                                  int64_t nnz, const double* __restrict__ e, double* __restrict__ lb,
                                  double* __restrict__ lc) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nnz;
       k += int64_t(gridDim.x) * blockDim.x) {
    const int32_t i = rows[k];
    const double x = vals ? vals[k] : 1.0;
    const double ex = e[i] * x;
    lb[i] = ex;
    lc[i] = ex * x;
  }
}

// 2./3. one CTA per tile: in-tile inclusive scan (forward = ascending device
// position; backward = descending, of the u-weighted lanes).  Thread t owns 8
// consecutive rows (in scan order).  Writes the in-tile scan to out and the
// tile total to tot[t*3..].
template <bool kBackward>
__global__ void __launch_bounds__(kSepThreads)
sep_scan_tile(const double* la, const double* lb, const double* lc,  // may alias oa/ob/oc
              const uint32_t* __restrict__ code, const double* __restrict__ g, double* oa,
              double* ob, double* oc, double* __restrict__ tot) {
  const int64_t base = int64_t(blockIdx.x) * kTileRows;
  L3 v[kSepRows];
  L3 run{0.0, 0.0, 0.0};
#pragma unroll
  for (int k = 0; k < kSepRows; ++k) {
    const int r = kBackward ? kTileRows - 1 - (threadIdx.x * kSepRows + k) : threadIdx.x * kSepRows + k;
    const int64_t i = base + r;
    L3 x{la[i], lb[i], lc[i]};
    if (kBackward) {
      // u = 1/G(Y-) on visible competing rows, else 0 (src/censoring.cpp:65-90)
      const double u = (code[i] & kCodeCompeting) ? 1.0 / g[i] : 0.0;
      x = {u * x.a, u * x.b, u * x.c};
    }
    run = l3_add(run, x);
    v[k] = run;
  }
  L3 total;
  const L3 incl = block_scan_l3(run, &total);
  // exclusive offset of this thread = the previous thread's inclusive value
  __shared__ L3 sh[kSepThreads];
  sh[threadIdx.x] = incl;
  __syncthreads();
  const L3 ex = threadIdx.x ? sh[threadIdx.x - 1] : L3{0.0, 0.0, 0.0};
#pragma unroll
  for (int k = 0; k < kSepRows; ++k) {
    const int r = kBackward ? kTileRows - 1 - (threadIdx.x * kSepRows + k) : threadIdx.x * kSepRows + k;
    const int64_t i = base + r;
    const L3 s = l3_add(ex, v[k]);
    oa[i] = s.a;
    ob[i] = s.b;
    oc[i] = s.c;
  }
  if (threadIdx.x == 0) {
    tot[3 * blockIdx.x + 0] = total.a;
    tot[3 * blockIdx.x + 1] = total.b;
    tot[3 * blockIdx.x + 2] = total.c;
  }
}

// 4. segmented carries over tiles (one CTA of 1024 threads, chunked).
//    fwd: car_f[t] = sum tot_f over tiles [start of t's stratum, t)
//    bwd: car_b[t] = sum tot_b over tiles (t, end of t's stratum]
__global__ void __launch_bounds__(1024)
sep_carries(const double* __restrict__ tot_f, const double* __restrict__ tot_b,
            const uint8_t* __restrict__ tile_first, int nt, double* __restrict__ car_f,
            double* __restrict__ car_b) {
  __shared__ double agg[1024][3];
  __shared__ int flag[1024];
  const int per = (nt + 1023) / 1024;
  const int t0 = min(nt, int(threadIdx.x) * per), t1 = min(nt, t0 + per);
  // forward: chunk aggregate since the last stratum start inside the chunk
  {
    L3 s{0.0, 0.0, 0.0};
    int f = 0;
    for (int t = t0; t < t1; ++t) {
      if (tile_first[t]) {
        s = {0.0, 0.0, 0.0};
        f = 1;
      }
      s = l3_add(s, L3{tot_f[3 * t], tot_f[3 * t + 1], tot_f[3 * t + 2]});
    }
    agg[threadIdx.x][0] = s.a;
    agg[threadIdx.x][1] = s.b;
    agg[threadIdx.x][2] = s.c;
    flag[threadIdx.x] = f;
    __syncthreads();
    if (threadIdx.x == 0) {  // serial exclusive segmented scan of the chunk aggregates
      L3 acc{0.0, 0.0, 0.0};
      for (int k = 0; k < 1024; ++k) {
        const L3 a{agg[k][0], agg[k][1], agg[k][2]};
        const int fk = flag[k];
        agg[k][0] = acc.a;
        agg[k][1] = acc.b;
        agg[k][2] = acc.c;
        acc = fk ? a : l3_add(acc, a);
      }
    }
    __syncthreads();
    L3 c{agg[threadIdx.x][0], agg[threadIdx.x][1], agg[threadIdx.x][2]};
    for (int t = t0; t < t1; ++t) {
      if (tile_first[t]) c = {0.0, 0.0, 0.0};
      car_f[3 * t] = c.a;
      car_f[3 * t + 1] = c.b;
      car_f[3 * t + 2] = c.c;
      c = l3_add(c, L3{tot_f[3 * t], tot_f[3 * t + 1], tot_f[3 * t + 2]});
    }
    __syncthreads();
  }
  if (!tot_b) return;
  // backward: a stratum ends after tile t iff t is last or tile_first[t+1]
  {
    L3 s{0.0, 0.0, 0.0};
    int f = 0;  // chunk contains a stratum end (other than possibly its last tile)
    for (int t = t1 - 1; t >= t0; --t) {
      if (t + 1 == nt || tile_first[t + 1]) {
        s = {0.0, 0.0, 0.0};
        f = 1;
      }
      s = l3_add(s, L3{tot_b[3 * t], tot_b[3 * t + 1], tot_b[3 * t + 2]});
    }
    agg[threadIdx.x][0] = s.a;
    agg[threadIdx.x][1] = s.b;
    agg[threadIdx.x][2] = s.c;
    flag[threadIdx.x] = f;
    __syncthreads();
    if (threadIdx.x == 0) {
      L3 acc{0.0, 0.0, 0.0};
      for (int k = 1023; k >= 0; --k) {
        const L3 a{agg[k][0], agg[k][1], agg[k][2]};
        const int fk = flag[k];
        agg[k][0] = acc.a;
        agg[k][1] = acc.b;
        agg[k][2] = acc.c;
        acc = fk ? a : l3_add(acc, a);
      }
    }
    __syncthreads();
    L3 c{agg[threadIdx.x][0], agg[threadIdx.x][1], agg[threadIdx.x][2]};
    for (int t = t1 - 1; t >= t0; --t) {
      if (t + 1 == nt || tile_first[t + 1]) c = {0.0, 0.0, 0.0};
      car_b[3 * t] = c.a;
      car_b[3 * t + 1] = c.b;
      car_b[3 * t + 2] = c.c;
      c = l3_add(c, L3{tot_b[3 * t], tot_b[3 * t + 1], tot_b[3 * t + 2]});
    }
  }
}

// 5. Breslow transform at block ends (engine.cpp:295-318) + per-tile partials
__global__ void __launch_bounds__(kSepThreads)
sep_transform(const double* __restrict__ pa, const double* __restrict__ pb,
              const double* __restrict__ pc, const double* __restrict__ car_f,
              const double* __restrict__ sa, const double* __restrict__ sb,
              const double* __restrict__ sc, const double* __restrict__ car_b,
              const uint32_t* __restrict__ code, const double* __restrict__ g,
              const uint8_t* __restrict__ tile_first, int nt, double* __restrict__ part,
              int* __restrict__ bad) {
  const int t = blockIdx.x;
  const int64_t base = int64_t(t) * kTileRows;
  const L3 cf{car_f[3 * t], car_f[3 * t + 1], car_f[3 * t + 2]};
  double lg = 0.0, lh = 0.0;
  bool nonpos = false;
#pragma unroll
  for (int k = 0; k < kSepRows; ++k) {
    const int r = threadIdx.x * kSepRows + k;
    const int64_t i = base + r;
    const uint32_t cnt = code[i] & kCodeCount;
    if (!cnt) continue;
    double den = pa[i] + cf.a, n1 = pb[i] + cf.b, n2 = pc[i] + cf.c;
    if (sa) {
      // suffix from the next row, inside the stratum
      L3 s{0.0, 0.0, 0.0};
      if (r + 1 < kTileRows)
        s = {sa[i + 1] + car_b[3 * t], sb[i + 1] + car_b[3 * t + 1], sc[i + 1] + car_b[3 * t + 2]};
      else if (t + 1 < nt && !tile_first[t + 1])
        s = {sa[i + 1] + car_b[3 * (t + 1)], sb[i + 1] + car_b[3 * (t + 1) + 1],
             sc[i + 1] + car_b[3 * (t + 1) + 2]};
      const double gi = g[i];
      den += gi * s.a;
      n1 += gi * s.b;
      n2 += gi * s.c;
    }
    if (!(den > 0.0)) {
      nonpos = true;
      continue;
    }
    const double G = n1 / den;
    const double H = n2 / den;
    const double d = static_cast<double>(cnt);
    lg += d * G;
    lh += d * (H - G * G);
  }
  if (nonpos) atomicOr(bad, 1);
  // fixed-order tree over the block
  __shared__ double rg[kSepThreads], rh[kSepThreads];
  rg[threadIdx.x] = lg;
  rh[threadIdx.x] = lh;
  __syncthreads();
  for (int s = kSepThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      rg[threadIdx.x] += rg[threadIdx.x + s];
      rh[threadIdx.x] += rh[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * t] = rg[0];
    part[2 * t + 1] = rh[0];
  }
}

// 6. fixed-order reduction of the tile partials: out = (grad_sum, hess_sum)
__global__ void __launch_bounds__(1024)
sep_reduce(const double* __restrict__ part, int nt, double* __restrict__ out) {
  __shared__ double rg[1024], rh[1024];
  double lg = 0.0, lh = 0.0;
  for (int t = threadIdx.x; t < nt; t += 1024) {
    lg += part[2 * t];
    lh += part[2 * t + 1];
  }
  rg[threadIdx.x] = lg;
  rh[threadIdx.x] = lh;
  __syncthreads();
  for (int s = 512; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      rg[threadIdx.x] += rg[threadIdx.x + s];
      rh[threadIdx.x] += rh[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = rg[0];
    out[1] = rh[0];
  }
}

}  // namespace

size_t separated_scratch_doubles(int64_t npad, int ntiles) {
  return size_t(6) * npad + size_t(ntiles) * 14 + 2;
}

cudaError_t launch_separated(const CycleParams& P, int64_t column, double* scratch, int* bad,
                             double* out2, cudaStream_t s) {
  const int64_t npad = P.npad;
  const int nt = P.ntiles;
  double* la = scratch;
  double* lb = la + npad;
  double* lc = lb + npad;
  double* sa = lc + npad;
  double* sb = sa + npad;
  double* sc = sb + npad;
  double* tot_f = sc + npad;
  double* tot_b = tot_f + 3 * size_t(nt);
  double* car_f = tot_b + 3 * size_t(nt);
  double* car_b = car_f + 3 * size_t(nt);
  double* part = car_b + 3 * size_t(nt);
  int64_t c0 = 0, c1 = 0;
  cudaError_t err = cudaMemcpyAsync(&c0, P.col_ptr + column, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (err != cudaSuccess) return err;
  err = cudaMemcpyAsync(&c1, P.col_ptr + column + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (err != cudaSuccess) return err;
  err = cudaStreamSynchronize(s);
  if (err != cudaSuccess) return err;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  sep_lanes_init<<<sms * 8, 256, 0, s>>>(P.e, npad, la, lb, lc);
  if (c1 > c0) {
    const int64_t nnz = c1 - c0;
    const int blocks = static_cast<int>(std::min<int64_t>((nnz + 255) / 256, int64_t(sms) * 16));
    sep_lanes_scatter<<<blocks, 256, 0, s>>>(P.row_idx + c0, P.has_vals ? P.vals + c0 : nullptr,
                                             nnz, P.e, lb, lc);
  }
  const bool w = P.weighted != 0;
  if (w)
    sep_scan_tile<true><<<nt, kSepThreads, 0, s>>>(la, lb, lc, P.code, P.g, sa, sb, sc, tot_b);
  sep_scan_tile<false><<<nt, kSepThreads, 0, s>>>(la, lb, lc, P.code, P.g, la, lb, lc, tot_f);
  sep_carries<<<1, 1024, 0, s>>>(tot_f, w ? tot_b : nullptr, P.tile_first, nt, car_f, car_b);
  sep_transform<<<nt, kSepThreads, 0, s>>>(la, lb, lc, car_f, w ? sa : nullptr, sb, sc, car_b,
                                           P.code, P.g, P.tile_first, nt, part, bad);
  sep_reduce<<<1, 1024, 0, s>>>(part, nt, out2);
  return cudaGetLastError();
}

}  // namespace gss
