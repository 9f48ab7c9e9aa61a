// gss_simgen.cu — device generator of synthetic sparse survival designs at
// benchmark scale (N = 1e7 .. 1e8), producing the reference's sorted layout
// directly (rows by decreasing time, ties by original row id; CSC over the
// sorted positions).
//
// Same design family as the reference generator (src/simgen.cpp:31-151):
// binary covariates at `density`, true beta_j ~ N(0,1) zeroed with
// probability beta_sparsity, event times Exponential(rate = exp(x'beta)),
// optional administrative censoring at the `censoring_quantile` of the times
// (type-7 quantile, util.hpp:33-42), plus optional time quantisation
// t <- ceil(t * q) / q that creates Breslow ties.
// The random streams are counter-based (splitmix64), not libstdc++'s, so
// values differ from simulate_cox for the same seed; parity tests never rely
// on this generator — they use reference-made fixtures.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gss_sim.h"

namespace {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

struct Rng {
  uint64_t s;
  __device__ explicit Rng(uint64_t seed) : s(seed) {}
  __device__ __forceinline__ double uniform() {  // (0, 1)
    s = mix64(s);
    return (static_cast<double>(s >> 11) + 0.5) * (1.0 / 9007199254740992.0);
  }
};

__global__ void beta_kernel(int64_t p, double sparsity, uint64_t seed, double* beta) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < p;
       j += int64_t(gridDim.x) * blockDim.x) {
    Rng r(mix64(seed ^ 0x5bd1e995ULL) ^ mix64(uint64_t(j) + 1));
    const double keep = r.uniform();
    const double u1 = r.uniform(), u2 = r.uniform();
    const double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    beta[j] = keep < sparsity ? 0.0 : z;
  }
}

// Columns of row i by geometric skipping over [0, p) (Bernoulli(density) each).
template <bool FILL>
__global__ void rows_kernel(int64_t n, int64_t p, double density, uint64_t seed,
                            const double* __restrict__ beta, const int64_t* __restrict__ rptr,
                            int32_t* __restrict__ cnt, uint64_t* __restrict__ keys,
                            double* __restrict__ eta) {
  const double lq = log1p(-density);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    Rng r(mix64(seed ^ 0x2545f4914f6cdd1dULL) ^ mix64(uint64_t(i) * 2 + 1));
    int64_t pos = -1;
    int32_t c = 0;
    double acc = 0.0;
    int64_t out = FILL ? rptr[i] : 0;
    if (density > 0.0) {
      for (;;) {
        const double u = r.uniform();
        const double skip = density >= 1.0 ? 0.0 : floor(log(u) / lq);
        if (skip >= double(p)) break;
        pos += 1 + static_cast<int64_t>(skip);
        if (pos >= p) break;
        ++c;
        if (FILL) {
          acc += beta[pos];
          keys[out++] = (uint64_t(pos) << 32);  // row part filled after sorting rows
        }
      }
    }
    if (!FILL) cnt[i] = c;
    if (FILL) eta[i] = acc;
  }
}

// Cox: Exponential(rate exp(x'beta)).  Fine-Gray (p_mix > 0): the primary
// event with probability 1 - (1 - p_mix)^exp(x'beta), its time by inverting the
// subdistribution 1 - [1 - p_mix (1 - e^-t)]^exp(x'beta); otherwise a competing
// event at Exponential(rate exp(-x'beta)) (simgen.hpp:33-37 design).
__global__ void times_kernel(int64_t n, uint64_t seed, const double* __restrict__ eta,
                             double p_mix, double* __restrict__ t, int32_t* __restrict__ cause,
                             int64_t* __restrict__ ids) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    Rng r(mix64(seed ^ 0x71d67fffeda60000ULL) ^ mix64(uint64_t(i) + 7));
    const double rate = exp(eta[i]);
    int32_t c = 1;
    double ti;
    if (p_mix <= 0.0) {
      ti = -log(r.uniform()) / rate;
    } else {
      const double p1 = -expm1(rate * log1p(-p_mix));
      if (r.uniform() < p1) {
        ti = INFINITY;
        for (int k = 0; k < 64 && !isfinite(ti); ++k) {
          const double v = r.uniform() * p1;
          const double w = -expm1(log1p(-v) / rate) / p_mix;
          ti = -log1p(-w);
        }
        if (!isfinite(ti)) ti = 1e300;
      } else {
        ti = -log(r.uniform()) * rate;
        c = 2;
      }
    }
    t[i] = ti;
    cause[i] = c;
    ids[i] = i;
  }
}

__global__ void censor_kernel(int64_t n, double cutoff, double quantum, double* __restrict__ t,
                              int32_t* __restrict__ status) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    double ti = t[i];
    int32_t s = status[i];  // cause from times_kernel
    if (cutoff > 0.0 && ti > cutoff) {
      ti = cutoff;
      s = 0;
    }
    if (quantum > 0.0) ti = ceil(ti * quantum) / quantum;
    t[i] = ti;
    status[i] = s;
  }
}

__global__ void inv_perm_kernel(int64_t n, const int64_t* __restrict__ perm,
                                int32_t* __restrict__ inv) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n;
       k += int64_t(gridDim.x) * blockDim.x)
    inv[perm[k]] = static_cast<int32_t>(k);
}

// attach the sorted position of each entry's row (entries are grouped by row)
__global__ void attach_rows_kernel(int64_t n, const int64_t* __restrict__ rptr,
                                   const int32_t* __restrict__ inv, uint64_t* __restrict__ keys) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t pos = static_cast<uint32_t>(inv[i]);
    for (int64_t k = rptr[i]; k < rptr[i + 1]; ++k) keys[k] |= pos;
  }
}

__global__ void split_keys_kernel(int64_t nnz, const uint64_t* __restrict__ keys,
                                  int32_t* __restrict__ row_idx, unsigned long long* colcnt) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nnz;
       k += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t key = keys[k];
    row_idx[k] = static_cast<int32_t>(key & 0xffffffffULL);
    atomicAdd(&colcnt[key >> 32], 1ULL);
  }
}

__global__ void gather_kernel(int64_t n, const int64_t* __restrict__ perm,
                              const double* __restrict__ t_sorted_src,
                              const int32_t* __restrict__ status, int32_t* __restrict__ st_out) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n;
       k += int64_t(gridDim.x) * blockDim.x)
    st_out[k] = status[perm[k]];
}

thread_local std::string g_sim_error;

int grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  return static_cast<int>(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

}  // namespace

#define SIM_CUDA(call)                                                     \
  do {                                                                     \
    cudaError_t _e = (call);                                               \
    if (_e != cudaSuccess) {                                               \
      g_sim_error = std::string(#call) + ": " + cudaGetErrorString(_e);    \
      return 100;                                                          \
    }                                                                      \
  } while (0)

extern "C" {

const char* gss_sim_last_error(void) { return g_sim_error.c_str(); }

void gss_sim_free(gss_sim_out* o) {
  if (!o) return;
  for (void* q : {(void*)o->times, (void*)o->status, (void*)o->col_ptr, (void*)o->row_idx,
                  (void*)o->beta_true})
    if (q) cudaFreeHost(q);
  std::memset(o, 0, sizeof(*o));
}

int gss_simulate_cox(const gss_sim_config* c, int device, gss_sim_out* o) {
  gss_sim_config cc = *c;
  cc.p_mix = 0.0;
  return gss_simulate(&cc, device, o);
}

int gss_simulate(const gss_sim_config* c, int device, gss_sim_out* o) {
  std::memset(o, 0, sizeof(*o));
  if (c->n <= 0 || c->p < 0 || c->n >= (int64_t(1) << 31) || c->p >= (int64_t(1) << 31)) {
    g_sim_error = "bad dimensions";
    return 3;
  }
  SIM_CUDA(cudaSetDevice(device));
  cudaStream_t s;
  SIM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const int64_t n = c->n, p = c->p;
  double* beta = nullptr;
  int32_t* cnt = nullptr;
  int64_t* rptr = nullptr;
  SIM_CUDA(cudaMalloc(&beta, sizeof(double) * (p + 1)));
  SIM_CUDA(cudaMalloc(&cnt, sizeof(int32_t) * (n + 1)));
  SIM_CUDA(cudaMalloc(&rptr, sizeof(int64_t) * (n + 1)));
  beta_kernel<<<grid(p), 256, 0, s>>>(p, c->beta_sparsity, c->seed, beta);
  rows_kernel<false><<<grid(n), 256, 0, s>>>(n, p, c->density, c->seed, beta, nullptr, cnt,
                                              nullptr, nullptr);
  // row pointers (exclusive scan of counts)
  SIM_CUDA(cudaMemsetAsync(rptr, 0, sizeof(int64_t), s));
  {
    void* tmp = nullptr;
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, cnt, rptr + 1, n, s);
    SIM_CUDA(cudaMalloc(&tmp, tb));
    cub::DeviceScan::InclusiveSum(tmp, tb, cnt, rptr + 1, n, s);
    SIM_CUDA(cudaStreamSynchronize(s));
    cudaFree(tmp);
  }
  int64_t nnz = 0;
  SIM_CUDA(cudaMemcpy(&nnz, rptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost));
  uint64_t *keys = nullptr, *keys2 = nullptr;
  double *eta = nullptr, *t = nullptr, *t2 = nullptr;
  int64_t *ids = nullptr, *perm = nullptr;
  int32_t *status = nullptr, *status_sorted = nullptr, *inv = nullptr, *row_idx = nullptr;
  unsigned long long* colcnt = nullptr;
  SIM_CUDA(cudaMalloc(&keys, sizeof(uint64_t) * (nnz + 1)));
  SIM_CUDA(cudaMalloc(&eta, sizeof(double) * n));
  rows_kernel<true><<<grid(n), 256, 0, s>>>(n, p, c->density, c->seed, beta, rptr, nullptr, keys,
                                             eta);
  SIM_CUDA(cudaMalloc(&t, sizeof(double) * n));
  SIM_CUDA(cudaMalloc(&t2, sizeof(double) * n));
  SIM_CUDA(cudaMalloc(&ids, sizeof(int64_t) * n));
  SIM_CUDA(cudaMalloc(&perm, sizeof(int64_t) * n));
  SIM_CUDA(cudaMalloc(&status, sizeof(int32_t) * n));
  SIM_CUDA(cudaMalloc(&status_sorted, sizeof(int32_t) * n));
  SIM_CUDA(cudaMalloc(&inv, sizeof(int32_t) * n));
  times_kernel<<<grid(n), 256, 0, s>>>(n, c->seed, eta, c->p_mix, t, status, ids);
  double cutoff = -1.0;
  if (c->censoring_quantile > 0.0 && c->censoring_quantile < 1.0) {
    // type-7 quantile of the event times (util.hpp:33-42)
    void* tmp = nullptr;
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, t, t2, n, 0, 64, s);
    SIM_CUDA(cudaMalloc(&tmp, tb));
    cub::DeviceRadixSort::SortKeys(tmp, tb, t, t2, n, 0, 64, s);
    SIM_CUDA(cudaStreamSynchronize(s));
    cudaFree(tmp);
    const double h = c->censoring_quantile * double(n - 1);
    const int64_t lo = static_cast<int64_t>(h);
    double a = 0, b = 0;
    SIM_CUDA(cudaMemcpy(&a, t2 + lo, sizeof(double), cudaMemcpyDeviceToHost));
    b = a;
    if (lo + 1 < n) SIM_CUDA(cudaMemcpy(&b, t2 + lo + 1, sizeof(double), cudaMemcpyDeviceToHost));
    const double frac = h - double(lo);
    cutoff = frac == 0.0 ? a : a + frac * (b - a);
  }
  censor_kernel<<<grid(n), 256, 0, s>>>(n, cutoff, c->time_quantum, t, status);
  // sort rows by time descending; stable => ties keep ascending original id
  {
    void* tmp = nullptr;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, t, t2, ids, perm, n, 0, 64, s);
    SIM_CUDA(cudaMalloc(&tmp, tb));
    cub::DeviceRadixSort::SortPairsDescending(tmp, tb, t, t2, ids, perm, n, 0, 64, s);
    SIM_CUDA(cudaStreamSynchronize(s));
    cudaFree(tmp);
  }
  inv_perm_kernel<<<grid(n), 256, 0, s>>>(n, perm, inv);
  attach_rows_kernel<<<grid(n), 256, 0, s>>>(n, rptr, inv, keys);
  gather_kernel<<<grid(n), 256, 0, s>>>(n, perm, t2, status, status_sorted);
  int end_bit = 32;
  while ((int64_t(1) << (end_bit - 32)) < p + 1) ++end_bit;
  SIM_CUDA(cudaMalloc(&keys2, sizeof(uint64_t) * (nnz + 1)));
  {
    void* tmp = nullptr;
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, keys2, nnz, 0, end_bit, s);
    SIM_CUDA(cudaMalloc(&tmp, tb));
    cub::DeviceRadixSort::SortKeys(tmp, tb, keys, keys2, nnz, 0, end_bit, s);
    SIM_CUDA(cudaStreamSynchronize(s));
    cudaFree(tmp);
  }
  cudaFree(keys);
  keys = nullptr;
  SIM_CUDA(cudaMalloc(&row_idx, sizeof(int32_t) * (nnz + 1)));
  SIM_CUDA(cudaMalloc(&colcnt, sizeof(unsigned long long) * (p + 1)));
  SIM_CUDA(cudaMemsetAsync(colcnt, 0, sizeof(unsigned long long) * (p + 1), s));
  split_keys_kernel<<<grid(nnz), 256, 0, s>>>(nnz, keys2, row_idx, colcnt);
  SIM_CUDA(cudaStreamSynchronize(s));
  SIM_CUDA(cudaGetLastError());
  // host (pinned) outputs
  o->n = n;
  o->p = p;
  o->nnz = nnz;
  SIM_CUDA(cudaMallocHost(&o->times, sizeof(double) * n));
  SIM_CUDA(cudaMallocHost(&o->status, sizeof(int32_t) * n));
  SIM_CUDA(cudaMallocHost(&o->col_ptr, sizeof(int64_t) * (p + 1)));
  SIM_CUDA(cudaMallocHost(&o->row_idx, sizeof(int32_t) * (nnz + 1)));
  SIM_CUDA(cudaMallocHost(&o->beta_true, sizeof(double) * (p + 1)));
  SIM_CUDA(cudaMemcpy(o->times, t2, sizeof(double) * n, cudaMemcpyDeviceToHost));
  SIM_CUDA(cudaMemcpy(o->status, status_sorted, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  SIM_CUDA(cudaMemcpy(o->row_idx, row_idx, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost));
  SIM_CUDA(cudaMemcpy(o->beta_true, beta, sizeof(double) * p, cudaMemcpyDeviceToHost));
  {
    std::vector<unsigned long long> cc(static_cast<size_t>(p + 1));
    SIM_CUDA(cudaMemcpy(cc.data(), colcnt, sizeof(unsigned long long) * p, cudaMemcpyDeviceToHost));
    o->col_ptr[0] = 0;
    for (int64_t j = 0; j < p; ++j) o->col_ptr[j + 1] = o->col_ptr[j] + int64_t(cc[j]);
  }
  for (void* q : {(void*)beta, (void*)cnt, (void*)rptr, (void*)keys2, (void*)eta, (void*)t,
                  (void*)t2, (void*)ids, (void*)perm, (void*)status, (void*)status_sorted,
                  (void*)inv, (void*)row_idx, (void*)colcnt})
    if (q) cudaFree(q);
  cudaStreamDestroy(s);
  return 0;
}

}  // extern "C"
