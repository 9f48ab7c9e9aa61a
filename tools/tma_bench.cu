// Microbenchmark: throughput of the sweep kernel's data path alone.
//   mode 0: producer warp + dynamic tile claims + 2D TMA (e, code); consumers
//           wait full, touch one value, release.
//   mode 1: same but static tile assignment (no atomics).
//   mode 2: plain vectorized LDG streaming of the same bytes (no TMA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_bench.cu -o /tmp/tma_bench
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <vector>

#include "../paper_2204_08183_b200/csrc/gss_device.cuh"

using namespace gss;
constexpr int kS = 4;
constexpr uint32_t kEB = kTileRows * 8, kCB = kTileRows * 4, kSB = kEB + kCB + 2048;

__global__ void __launch_bounds__(288, 2) tma_kernel(const __grid_constant__ CUtensorMap tm_e,
                                                     const __grid_constant__ CUtensorMap tm_c,
                                                     int ntiles, unsigned* counter, int mode,
                                                     double* sink) {
  extern __shared__ unsigned char raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kS], empty[kS];
  __shared__ int tiles[kS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    fence_mbar_init();
  }
  __syncthreads();
  double acc = 0.0;
  if (warp == 8) {
    if (lane == 0) {
      unsigned next_static = blockIdx.x;
      for (int it = 0;; ++it) {
        const int s = it % kS;
        mbar_wait(&empty[s], ((it / kS) & 1) ^ 1);
        unsigned t;
        if (mode == 0)
          t = atomicAdd(counter, 1u);
        else {
          t = next_static;
          next_static += gridDim.x;
        }
        if (t >= unsigned(ntiles)) {
          tiles[s] = -1;
          mbar_arrive(&full[s]);
          break;
        }
        tiles[s] = int(t);
        unsigned char* sb = smem + s * kSB;
        mbar_arrive_expect_tx(&full[s], kEB + kCB);
        tma_load_2d(sb, &tm_e, 0, int(t) * 256, &full[s]);
        tma_load_2d(sb + kEB, &tm_c, 0, int(t) * 256, &full[s]);
      }
    }
  } else {
    for (int it = 0;; ++it) {
      const int s = it % kS;
      mbar_wait(&full[s], (it / kS) & 1);
      if (tiles[s] < 0) break;
      const double* e = reinterpret_cast<const double*>(smem + s * kSB);
      acc += e[tid * 8];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  if (acc == 12345.0) sink[0] = acc;
}

__global__ void ldg_kernel(const double2* e, const uint4* c, long long n16, long long nc16,
                           double* sink) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n16;
       i += (long long)gridDim.x * blockDim.x) {
    const double2 v = __ldcs(e + i);
    acc += v.x + v.y;
    if (i < nc16) {
      const uint4 w = __ldcs(c + i);
      acc += w.x;
    }
  }
  if (acc == 12345.0) sink[0] = acc;
}

int main() {
  const long long n = 10000000, ntiles = (n + kTileRows - 1) / kTileRows, npad = ntiles * kTileRows;
  double* e;
  uint32_t* code;
  double* sink;
  unsigned* counter;
  cudaMalloc(&e, npad * 8);
  cudaMalloc(&code, npad * 4);
  cudaMalloc(&sink, 8);
  cudaMalloc(&counter, 4);
  cudaMemset(e, 0, npad * 8);
  cudaMemset(code, 0, npad * 4);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  CUtensorMap tm_e, tm_c;
  cuuint64_t dims[2] = {8, cuuint64_t(npad / 8)};
  cuuint32_t box[2] = {8, 256}, es[2] = {1, 1};
  cuuint64_t st_e[1] = {64}, st_c[1] = {32};
  fn(&tm_e, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, e, dims, st_e, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
     CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  fn(&tm_c, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, code, dims, st_c, box, es,
     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const size_t smem = 1024 + kS * kSB;
  cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tma_kernel, 288, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double bytes = double(npad) * 12.0;
  for (int mode = 0; mode < 3; ++mode) {
    for (int grid : {148, 296}) {
      float best = 1e9;
      for (int rep = 0; rep < 6; ++rep) {
        cudaMemset(counter, 0, 4);
        cudaEventRecord(a);
        if (mode < 2)
          tma_kernel<<<grid, 288, smem>>>(tm_e, tm_c, int(ntiles), counter, mode, sink);
        else
          ldg_kernel<<<grid * 4, 512>>>(reinterpret_cast<double2*>(e), reinterpret_cast<uint4*>(code),
                                        npad / 2, npad / 4, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0 && ms < best) best = ms;
      }
      printf("mode %d grid %d occ %d: %.2f us  %.0f GB/s  err=%s\n", mode, grid, occ, best * 1e3,
             bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
