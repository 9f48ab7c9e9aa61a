// gss_ingest.cu — device ingestion: the reference's dataset_from_coo /
// sort_and_block (/root/reference/proj/src/dataset.cpp:190-262) on the GPU.
//
//   1. row order: (stratum asc,) time desc, row id asc — two stable CUB radix
//      sorts of the row ids (time key first, then the stratum key), so equal
//      keys keep ascending ids exactly like the reference's comparison sort;
//   2. entry checks in input order (row / column range, finite value; zero
//      values are absent cells) — the FIRST failing entry is reported, with
//      the class of its first failing check, as the host loop would;
//   3. CSC: one radix sort of (column * n + sorted position) keys with the
//      values as payload; the first adjacent equal key is the reference's
//      DuplicateEntryError; column pointers by binary search.
// The host keeps its SurvivalDataset (the drop-in API is host-resident); this
// replaces its O(N log N + nnz log nnz) comparison sorts, the ingestion
// bottleneck at C5 scale.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/gss.h"

namespace gss {
int set_last_error(int code, const std::string& msg);  // gss_capi.cu
}

namespace {

constexpr unsigned long long kNone = ~0ull;

// order-preserving map of a double to uint64, then complemented: ascending
// radix order == descending time
__device__ __forceinline__ unsigned long long time_key_desc(double t) {
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(t));
  b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  return ~b;
}

__global__ void row_keys_kernel(const double* __restrict__ times, int64_t n,
                                unsigned long long* __restrict__ key, int64_t* __restrict__ id) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    key[i] = time_key_desc(times[i] + 0.0);  // -0.0 ties with +0.0, as in the comparison sort
    id[i] = i;
  }
}

__global__ void stratum_keys_kernel(const int64_t* __restrict__ strata, const int64_t* __restrict__ order,
                                    int64_t n, unsigned long long* __restrict__ key) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    key[i] = static_cast<unsigned long long>(strata[order[i]]) ^ 0x8000000000000000ull;
}

__global__ void pos_of_kernel(const int64_t* __restrict__ order, int64_t n, int64_t* __restrict__ pos) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    pos[order[i]] = i;
}

// per entry: validity checks (first failure = min over k*4 + class, classes
// 1 row, 2 column, 3 value), CSC key (or kNone for absent / invalid cells)
__global__ void entry_keys_kernel(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                                  const double* __restrict__ vals, int64_t nnz, int64_t n, int64_t p,
                                  const int64_t* __restrict__ pos_of,
                                  unsigned long long* __restrict__ key, double* __restrict__ val,
                                  unsigned long long* __restrict__ first_bad,
                                  unsigned long long* __restrict__ kept) {
  unsigned long long local = 0;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nnz;
       k += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = rows[k], c = cols[k];
    const double v = vals[k];
    int cls = 0;
    if (r < 0 || r >= n)
      cls = 1;
    else if (c < 0 || c >= p)
      cls = 2;
    else if (!isfinite(v))
      cls = 3;
    if (cls) {
      atomicMin(first_bad, static_cast<unsigned long long>(k) * 4ull + cls);
      key[k] = kNone;
    } else if (v == 0.0) {  // absent cell
      key[k] = kNone;
    } else {
      key[k] = static_cast<unsigned long long>(c) * static_cast<unsigned long long>(n) +
               static_cast<unsigned long long>(pos_of[r]);
      ++local;
    }
    val[k] = v;
  }
  if (local) atomicAdd(kept, local);
}

__global__ void first_dup_kernel(const unsigned long long* __restrict__ key, int64_t m,
                                 unsigned long long* __restrict__ first) {
  for (int64_t i = 1 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
       i += int64_t(gridDim.x) * blockDim.x)
    if (key[i] == key[i - 1]) atomicMin(first, static_cast<unsigned long long>(i));
}

__global__ void csc_kernel(const unsigned long long* __restrict__ key, int64_t m, int64_t n, int64_t p,
                           int64_t* __restrict__ col_ptr, int32_t* __restrict__ row_pos) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
       i += int64_t(gridDim.x) * blockDim.x)
    row_pos[i] = static_cast<int32_t>(key[i] % static_cast<unsigned long long>(n));
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j <= p;
       j += int64_t(gridDim.x) * blockDim.x) {
    const unsigned long long target = static_cast<unsigned long long>(j) * n;
    int64_t lo = 0, hi = m;  // first key >= j*n
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (key[mid] < target)
        lo = mid + 1;
      else
        hi = mid;
    }
    col_ptr[j] = lo;
  }
}

int grid_for(int64_t work) {
  int64_t g = (work + 255) / 256;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<int>(g);
}

struct Buf {
  std::vector<void*> ptrs;
  ~Buf() {
    for (void* q : ptrs) cudaFree(q);
  }
  template <class T>
  cudaError_t get(T** p, size_t count) {
    *p = nullptr;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), (count ? count : 1) * sizeof(T));
    if (e == cudaSuccess) ptrs.push_back(*p);
    return e;
  }
};

}  // namespace

extern "C" int gss_coo_sort(int device, int64_t n, const double* times, const int64_t* strata,
                            int64_t nnz, const int64_t* rows, const int64_t* cols,
                            const double* vals, int64_t p, int64_t* order_out, int64_t* col_ptr_out,
                            int32_t* row_pos_out, double* vals_out, int64_t* nnz_out,
                            int64_t* err_info) {
  using gss::set_last_error;
  if (!order_out || !col_ptr_out || !nnz_out || !err_info || (n && !times) ||
      (nnz && (!rows || !cols || !vals)))
    return set_last_error(GSS_ERR_DOMAIN, "gss_coo_sort: null argument");
  err_info[0] = err_info[1] = -1;
  if (n >= (int64_t(1) << 31) || nnz >= (int64_t(1) << 31))
    return set_last_error(GSS_ERR_DOMAIN, "gss_coo_sort: n and nnz must be below 2^31 per call");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return set_last_error(GSS_ERR_NO_DEVICE, "gss_coo_sort: no such CUDA device");
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  struct Restore {
    int d;
    ~Restore() {
      if (d >= 0) cudaSetDevice(d);
    }
  } restore{prev};
  cudaStream_t s;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess)
    return set_last_error(GSS_ERR_CUDA, "gss_coo_sort: stream creation failed");
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{s};
  Buf B;
#define IK(call)                                                                              \
  do {                                                                                        \
    cudaError_t _e = (call);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      return set_last_error(_e == cudaErrorMemoryAllocation ? GSS_ERR_OOM : GSS_ERR_CUDA,     \
                            std::string("gss_coo_sort: ") + cudaGetErrorString(_e));          \
  } while (0)
  // ---- 1. row order --------------------------------------------------------
  double* d_t = nullptr;
  unsigned long long *k0 = nullptr, *k1 = nullptr;
  int64_t *i0 = nullptr, *i1 = nullptr, *pos = nullptr;
  IK(B.get(&d_t, n));
  IK(B.get(&k0, n));
  IK(B.get(&k1, n));
  IK(B.get(&i0, n));
  IK(B.get(&i1, n));
  IK(B.get(&pos, n));
  if (n) IK(cudaMemcpyAsync(d_t, times, n * sizeof(double), cudaMemcpyHostToDevice, s));
  row_keys_kernel<<<grid_for(n), 256, 0, s>>>(d_t, n, k0, i0);
  IK(cudaGetLastError());
  size_t tmp_bytes = 0, need = 0;
  void* tmp = nullptr;
  const int64_t big = n > nnz ? n : nnz;
  cub::DeviceRadixSort::SortPairs(nullptr, need, k0, k1, i0, i1, static_cast<int>(big > 0 ? big : 1),
                                  0, 64, s);
  tmp_bytes = need;
  {
    size_t need2 = 0;
    unsigned long long* kk = nullptr;
    double* vv = nullptr;
    cub::DeviceRadixSort::SortPairs(nullptr, need2, kk, kk, vv, vv, static_cast<int>(big > 0 ? big : 1),
                                    0, 64, s);
    if (need2 > tmp_bytes) tmp_bytes = need2;
  }
  IK(B.get(reinterpret_cast<unsigned char**>(&tmp), tmp_bytes));
  if (n) IK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, i0, i1, static_cast<int>(n), 0, 64, s));
  int64_t* order = i1;
  if (strata && n) {
    int64_t* d_s = nullptr;
    IK(B.get(&d_s, n));
    IK(cudaMemcpyAsync(d_s, strata, n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    stratum_keys_kernel<<<grid_for(n), 256, 0, s>>>(d_s, i1, n, k0);
    IK(cudaGetLastError());
    IK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, i1, i0, static_cast<int>(n), 0, 64, s));
    order = i0;
  }
  pos_of_kernel<<<grid_for(n), 256, 0, s>>>(order, n, pos);
  IK(cudaGetLastError());
  if (n) IK(cudaMemcpyAsync(order_out, order, n * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  // ---- 2. entry checks and CSC keys -----------------------------------------
  int64_t *d_r = nullptr, *d_c = nullptr;
  double *d_v = nullptr, *v1 = nullptr;
  unsigned long long *ek0 = nullptr, *ek1 = nullptr, *flags = nullptr;
  IK(B.get(&d_r, nnz));
  IK(B.get(&d_c, nnz));
  IK(B.get(&d_v, nnz));
  IK(B.get(&v1, nnz));
  IK(B.get(&ek0, nnz));
  IK(B.get(&ek1, nnz));
  IK(B.get(&flags, 3));
  const unsigned long long init[3] = {kNone, 0ull, kNone};  // first bad, kept, first dup
  IK(cudaMemcpyAsync(flags, init, sizeof(init), cudaMemcpyHostToDevice, s));
  if (nnz) {
    IK(cudaMemcpyAsync(d_r, rows, nnz * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    IK(cudaMemcpyAsync(d_c, cols, nnz * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    IK(cudaMemcpyAsync(d_v, vals, nnz * sizeof(double), cudaMemcpyHostToDevice, s));
    entry_keys_kernel<<<grid_for(nnz), 256, 0, s>>>(d_r, d_c, d_v, nnz, n, p, pos, ek0, v1,
                                                    flags, flags + 1);
    IK(cudaGetLastError());
  }
  unsigned long long hf[3];
  IK(cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, s));
  IK(cudaStreamSynchronize(s));
  if (hf[0] != kNone) {
    err_info[0] = static_cast<int64_t>(hf[0] / 4);
    const int cls = static_cast<int>(hf[0] % 4);
    return set_last_error(cls == 3 ? GSS_ERR_DOMAIN : GSS_ERR_INDEX,
                          cls == 1 ? "matrix row outside [0, n)"
                                   : (cls == 2 ? "matrix column outside [0, p)"
                                               : "matrix value must be finite"));
  }
  const int64_t m = static_cast<int64_t>(hf[1]);
  // ---- 3. CSC ----------------------------------------------------------------
  if (nnz) IK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, ek0, ek1, v1, d_v, static_cast<int>(nnz), 0, 64, s));
  if (m > 1) {
    first_dup_kernel<<<grid_for(m), 256, 0, s>>>(ek1, m, flags + 2);
    IK(cudaGetLastError());
  }
  int64_t* d_cp = nullptr;
  int32_t* d_rp = nullptr;
  IK(B.get(&d_cp, p + 1));
  IK(B.get(&d_rp, m));
  csc_kernel<<<grid_for(m > p + 1 ? m : p + 1), 256, 0, s>>>(ek1, m, n > 0 ? n : 1, p, d_cp, d_rp);
  IK(cudaGetLastError());
  IK(cudaMemcpyAsync(hf + 2, flags + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  IK(cudaStreamSynchronize(s));
  if (hf[2] != kNone) {
    unsigned long long dk = 0;
    IK(cudaMemcpy(&dk, ek1 + hf[2], sizeof(dk), cudaMemcpyDeviceToHost));
    err_info[0] = static_cast<int64_t>(dk % static_cast<unsigned long long>(n));  // sorted position
    err_info[1] = static_cast<int64_t>(dk / static_cast<unsigned long long>(n));  // column
    return set_last_error(GSS_ERR_DUPLICATE, "matrix cell appears more than once");
  }
  IK(cudaMemcpyAsync(col_ptr_out, d_cp, (p + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  if (m) {
    IK(cudaMemcpyAsync(row_pos_out, d_rp, m * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    IK(cudaMemcpyAsync(vals_out, d_v, m * sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  IK(cudaStreamSynchronize(s));
#undef IK
  *nnz_out = m;
  return GSS_OK;
}
