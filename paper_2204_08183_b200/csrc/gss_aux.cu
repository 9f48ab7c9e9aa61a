// gss_aux.cu — the non-scan kernels of the engine: dataset packing
// (tile-blocked column pointers, CSR transpose, per-column max |x|), fixed
// terms, load_beta's full X*beta, and the API-mode validate/commit update.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdint>

#include "gss_device.cuh"
#include "gss_kernels.cuh"

namespace gss {

namespace {

constexpr double kXbetaBound = 700.0;  // src/engine.cpp:12

// tile_ptr[j][b] = (first nonzero of column j with row >= b*kTileRows) - col_ptr[j]
__global__ void tile_ptr_kernel(const int64_t* __restrict__ col_ptr,
                                const int32_t* __restrict__ row_idx, int64_t p, int ntiles,
                                uint32_t* __restrict__ tile_ptr) {
  const int64_t total = p * (ntiles + 1);
  for (int64_t id = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; id < total;
       id += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = id / (ntiles + 1);
    const int b = static_cast<int>(id % (ntiles + 1));
    const int64_t base = col_ptr[j];
    int64_t lo = base, hi = col_ptr[j + 1];
    const int64_t target = int64_t(b) * kTileRows;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (row_idx[mid] < target)
        lo = mid + 1;
      else
        hi = mid;
    }
    tile_ptr[id] = static_cast<uint32_t>(lo - base);
  }
}

// device row positions of the padded (stratum-aligned) layout
__global__ void remap_rows_kernel(int32_t* __restrict__ row_idx, int64_t nnz,
                                  const int64_t* __restrict__ dev_row) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nnz;
       k += int64_t(gridDim.x) * blockDim.x)
    row_idx[k] = static_cast<int32_t>(dev_row[row_idx[k]]);
}

// warp per column
// e = exp(0) on visible rows, 0 on masked rows and padding (engine start)
__global__ void init_e_kernel(const uint32_t* __restrict__ code, int64_t npad,
                              double* __restrict__ e) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npad;
       i += int64_t(gridDim.x) * blockDim.x)
    e[i] = (code[i] & kCodeMasked) ? 0.0 : 1.0;
}

__global__ void colmax_kernel(const int64_t* __restrict__ col_ptr, const double* __restrict__ vals,
                              int64_t p, double* __restrict__ colmax) {
  const int lane = threadIdx.x & 31;
  for (int64_t j = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; j < p;
       j += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    double m = 0.0;
    if (vals) {
      for (int64_t k = col_ptr[j] + lane; k < col_ptr[j + 1]; k += 32) m = fmax(m, fabs(vals[k]));
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, d));
    } else {
      m = col_ptr[j + 1] > col_ptr[j] ? 1.0 : 0.0;
    }
    if (lane == 0) colmax[j] = m;
  }
}

__global__ void fill_dense_kernel(const int64_t* __restrict__ col_ptr, const int32_t* __restrict__ row_idx,
                                  const double* __restrict__ vals, const int32_t* __restrict__ slot,
                                  int64_t p, int64_t npad, double* __restrict__ pool) {
  const int lane = threadIdx.x & 31;
  for (int64_t j = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; j < p;
       j += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    if (slot[j] < 0) continue;
    double* col = pool + size_t(slot[j]) * size_t(npad);
    for (int64_t k = col_ptr[j] + lane; k < col_ptr[j + 1]; k += 32)
      col[row_idx[k]] = vals ? vals[k] : 1.0;
  }
}

__global__ void csr_count_kernel(const int32_t* __restrict__ row_idx, int64_t nnz,
                                 int64_t* __restrict__ cnt) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nnz;
       k += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[row_idx[k]]), 1ULL);
}

// warp per column; order of arrival inside a row is fixed up by the sort pass
__global__ void csr_fill_kernel(const int64_t* __restrict__ col_ptr,
                                const int32_t* __restrict__ row_idx,
                                const double* __restrict__ vals, int64_t p,
                                int64_t* __restrict__ cursor, int32_t* __restrict__ csr_col,
                                double* __restrict__ csr_val) {
  const int lane = threadIdx.x & 31;
  for (int64_t j = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; j < p;
       j += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    for (int64_t k = col_ptr[j] + lane; k < col_ptr[j + 1]; k += 32) {
      const int32_t r = row_idx[k];
      const int64_t pos = static_cast<int64_t>(
          atomicAdd(reinterpret_cast<unsigned long long*>(&cursor[r]), 1ULL));
      csr_col[pos] = static_cast<int32_t>(j);
      if (csr_val) csr_val[pos] = vals ? vals[k] : 1.0;
    }
  }
}

// thread per row: insertion sort of the row's (col, val) pairs by column
__global__ void csr_sort_kernel(const int64_t* __restrict__ row_ptr, int64_t n,
                                int32_t* __restrict__ csr_col, double* __restrict__ csr_val) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t a = row_ptr[r], b = row_ptr[r + 1];
    for (int64_t i = a + 1; i < b; ++i) {
      const int32_t c = csr_col[i];
      const double v = csr_val ? csr_val[i] : 0.0;
      int64_t k = i - 1;
      while (k >= a && csr_col[k] > c) {
        csr_col[k + 1] = csr_col[k];
        if (csr_val) csr_val[k + 1] = csr_val[k];
        --k;
      }
      csr_col[k + 1] = c;
      if (csr_val) csr_val[k + 1] = v;
    }
  }
}

// delta' X_j over visible rows (src/engine.cpp:76-101); warp per column,
// lane-strided then fixed xor tree => deterministic.
__global__ void fixed_terms_kernel(const int64_t* __restrict__ col_ptr,
                                   const int32_t* __restrict__ row_idx,
                                   const double* __restrict__ vals,
                                   const uint8_t* __restrict__ col_ind,
                                   const uint32_t* __restrict__ code, int64_t p,
                                   double* __restrict__ fixed) {
  const int lane = threadIdx.x & 31;
  for (int64_t j = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; j < p;
       j += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const bool ind = !vals || col_ind[j];
    double acc = 0.0;
    for (int64_t k = col_ptr[j] + lane; k < col_ptr[j + 1]; k += 32) {
      if (code[row_idx[k]] & kCodeEvent) acc = __dadd_rn(acc, ind ? 1.0 : vals[k]);
    }
    acc = warp_sum(acc);
    if (lane == 0) fixed[j] = acc;
  }
}

// eta_out[r] = sum_j beta_j x_rj, accumulated in ascending column order
// exactly as Engine::load_beta does (src/engine.cpp:120-154); thread per row.
__global__ void spmv_rows_kernel(const int64_t* __restrict__ row_ptr,
                                 const int32_t* __restrict__ csr_col,
                                 const double* __restrict__ csr_val,
                                 const uint32_t* __restrict__ code, int64_t n,
                                 const double* __restrict__ beta, double* __restrict__ eta_out,
                                 int* __restrict__ overflow) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k)
      acc = __dadd_rn(acc, __dmul_rn(beta[csr_col[k]], csr_val ? csr_val[k] : 1.0));
    eta_out[r] = acc;
    if (!(code[r] & kCodeMasked) && fabs(acc) > kXbetaBound) *overflow = 1;
  }
}

__global__ void commit_eta_kernel(const double* __restrict__ eta_in,
                                  const uint32_t* __restrict__ code, int64_t n,
                                  double* __restrict__ eta, double* __restrict__ e, Ctl* ctl) {
  double mx = 0.0;
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const double v = eta_in[r];
    const bool vis = !(code[r] & kCodeMasked);
    eta[r] = v;
    e[r] = vis ? exp(v) : 0.0;
    if (vis) mx = fmax(mx, fabs(v));
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
  if ((threadIdx.x & 31) == 0 && mx > 0.0)
    atomicMax(&ctl->eta_absmax_bits, static_cast<unsigned long long>(__double_as_longlong(mx)));
}

__global__ void update_check_kernel(CycleParams P, int64_t col, double delta, int* overflow) {
  const int64_t k0 = P.col_ptr[col], k1 = P.col_ptr[col + 1];
  const bool ind = !P.has_vals || P.col_ind[col];
  for (int64_t k = k0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < k1;
       k += int64_t(gridDim.x) * blockDim.x) {
    const int32_t r = P.row_idx[k];
    if (P.code[r] & kCodeMasked) continue;
    const double x = ind ? 1.0 : P.vals[k];
    if (fabs(__dadd_rn(P.eta[r], __dmul_rn(x, delta))) > kXbetaBound) *overflow = 1;
  }
}

__global__ void update_commit_kernel(CycleParams P, int64_t col, double delta, double factor) {
  const int64_t k0 = P.col_ptr[col], k1 = P.col_ptr[col + 1];
  const bool ind = !P.has_vals || P.col_ind[col];
  double mx = 0.0;
  for (int64_t k = k0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < k1;
       k += int64_t(gridDim.x) * blockDim.x) {
    const int32_t r = P.row_idx[k];
    if (P.code[r] & kCodeMasked) continue;
    const double x = ind ? 1.0 : P.vals[k];
    const double ne = __dadd_rn(P.eta[r], __dmul_rn(x, delta));
    P.eta[r] = ne;
    P.e[r] = ind ? __dmul_rn(P.e[r], factor) : exp(ne);
    mx = fmax(mx, fabs(ne));
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
  if ((threadIdx.x & 31) == 0 && mx > 0.0)
    atomicMax(&P.ctl->eta_absmax_bits, static_cast<unsigned long long>(__double_as_longlong(mx)));
}

// layout contract of the CSC input: indices in [0, n), strictly ascending per column
__global__ void validate_csc_kernel(const int64_t* __restrict__ col_ptr,
                                    const int32_t* __restrict__ row_idx, int64_t p, int64_t n,
                                    int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  for (int64_t j = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; j < p;
       j += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const int64_t a = col_ptr[j], b = col_ptr[j + 1];
    if (b < a) {
      if (lane == 0) atomicOr(bad, 1);
      continue;
    }
    for (int64_t k = a + lane; k < b; k += 32) {
      const int32_t r = row_idx[k];
      if (r < 0 || r >= n) atomicOr(bad, 2);
      if (k > a && row_idx[k - 1] >= r) atomicOr(bad, 4);
    }
  }
}

int grid_for(int64_t work, int block) {
  int64_t g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return static_cast<int>(g);
}

}  // namespace

cudaError_t launch_validate_csc(const int64_t* col_ptr, const int32_t* row_idx, int64_t p,
                                int64_t n, int* bad, cudaStream_t s) {
  if (p == 0) return cudaSuccess;
  validate_csc_kernel<<<grid_for(p * 32, 256), 256, 0, s>>>(col_ptr, row_idx, p, n, bad);
  return cudaGetLastError();
}

cudaError_t launch_exclusive_scan(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s);
  if (e != cudaSuccess) return e;
  void* tmp = nullptr;
  e = cudaMallocAsync(&tmp, tb, s);
  if (e != cudaSuccess) return e;
  e = cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, n, s);
  cudaFreeAsync(tmp, s);
  return e;
}

cudaError_t launch_remap_rows(int32_t* row_idx, int64_t nnz, const int64_t* dev_row,
                              cudaStream_t s) {
  if (nnz == 0) return cudaSuccess;
  remap_rows_kernel<<<grid_for(nnz, 256), 256, 0, s>>>(row_idx, nnz, dev_row);
  return cudaGetLastError();
}

cudaError_t launch_build_tile_ptr(const int64_t* col_ptr, const int32_t* row_idx, int64_t p,
                                  int ntiles, uint32_t* tile_ptr, cudaStream_t s) {
  tile_ptr_kernel<<<grid_for(p * (ntiles + 1), 256), 256, 0, s>>>(col_ptr, row_idx, p, ntiles,
                                                                   tile_ptr);
  return cudaGetLastError();
}

cudaError_t launch_fill_dense(const int64_t* col_ptr, const int32_t* row_idx, const double* vals,
                              const int32_t* slot, int64_t p, int64_t npad, double* pool,
                              cudaStream_t s) {
  if (p == 0) return cudaSuccess;
  fill_dense_kernel<<<grid_for(p * 32, 256), 256, 0, s>>>(col_ptr, row_idx, vals, slot, p, npad,
                                                          pool);
  return cudaGetLastError();
}

cudaError_t launch_init_e(const uint32_t* code, int64_t npad, double* e, cudaStream_t s) {
  init_e_kernel<<<grid_for(npad, 256), 256, 0, s>>>(code, npad, e);
  return cudaGetLastError();
}

cudaError_t launch_colmax(const int64_t* col_ptr, const double* vals, int64_t p, double* colmax,
                          cudaStream_t s) {
  colmax_kernel<<<grid_for(p * 32, 256), 256, 0, s>>>(col_ptr, vals, p, colmax);
  return cudaGetLastError();
}

cudaError_t launch_csr_count(const int32_t* row_idx, int64_t nnz, int64_t* row_cnt,
                             cudaStream_t s) {
  if (nnz == 0) return cudaSuccess;
  csr_count_kernel<<<grid_for(nnz, 256), 256, 0, s>>>(row_idx, nnz, row_cnt);
  return cudaGetLastError();
}

cudaError_t launch_csr_fill(const int64_t* col_ptr, const int32_t* row_idx, const double* vals,
                            int64_t p, int64_t* cursor, int32_t* csr_col, double* csr_val,
                            cudaStream_t s) {
  if (p == 0) return cudaSuccess;
  csr_fill_kernel<<<grid_for(p * 32, 256), 256, 0, s>>>(col_ptr, row_idx, vals, p, cursor,
                                                        csr_col, csr_val);
  return cudaGetLastError();
}

cudaError_t launch_csr_sort_rows(const int64_t* row_ptr, int64_t n, int32_t* csr_col,
                                 double* csr_val, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  csr_sort_kernel<<<grid_for(n, 128), 128, 0, s>>>(row_ptr, n, csr_col, csr_val);
  return cudaGetLastError();
}

cudaError_t launch_fixed_terms(const int64_t* col_ptr, const int32_t* row_idx, const double* vals,
                               const uint8_t* col_ind, const uint32_t* code, int64_t p,
                               double* fixed, cudaStream_t s) {
  if (p == 0) return cudaSuccess;
  fixed_terms_kernel<<<grid_for(p * 32, 256), 256, 0, s>>>(col_ptr, row_idx, vals, col_ind, code,
                                                           p, fixed);
  return cudaGetLastError();
}

cudaError_t launch_spmv_rows(const CycleParams& prm, const double* beta, double* eta_out,
                             int* overflow, cudaStream_t s) {
  if (prm.npad == 0) return cudaSuccess;
  spmv_rows_kernel<<<grid_for(prm.npad, 256), 256, 0, s>>>(
      prm.row_ptr, prm.csr_col, prm.csr_val, prm.code, prm.npad, beta, eta_out, overflow);
  return cudaGetLastError();
}

cudaError_t launch_commit_eta(const CycleParams& prm, const double* eta_in, cudaStream_t s) {
  if (prm.npad == 0) return cudaSuccess;
  commit_eta_kernel<<<grid_for(prm.npad, 256), 256, 0, s>>>(eta_in, prm.code, prm.npad, prm.eta, prm.e,
                                                         prm.ctl);
  return cudaGetLastError();
}

cudaError_t launch_update_check(const CycleParams& prm, int64_t col, double delta, int* overflow,
                                cudaStream_t s) {
  update_check_kernel<<<grid_for(1 << 16, 256), 256, 0, s>>>(prm, col, delta, overflow);
  return cudaGetLastError();
}

cudaError_t launch_update_commit(const CycleParams& prm, int64_t col, double delta, double factor,
                                 cudaStream_t s) {
  update_commit_kernel<<<grid_for(1 << 16, 256), 256, 0, s>>>(prm, col, delta, factor);
  return cudaGetLastError();
}

}  // namespace gss
