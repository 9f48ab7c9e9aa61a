// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/shfl_wait tools/micro/shfl_wait.cu
// Does a warp parked in mbarrier.try_wait slow other warps' shuffles / smem ops?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(double* out, long long* cyc, int n, int mode) {
  __shared__ uint64_t bar;
  __shared__ double sm[64];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 64) sm[threadIdx.x] = 1.0;
  __syncthreads();
  if (w >= 1) {  // waiters
    if (mode == 0) return;
    if (mode == 4) {  // parked at a named barrier that warp 0 completes at the end
      asm volatile("bar.sync 9, 544;" ::: "memory");
      return;
    }
    if (lane != 0 && mode != 3) return;
    uint32_t ok = 0;
    while (!ok) {
      if (mode == 1 || mode == 3)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su32(&bar)) : "memory");
      else {
        asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su32(&bar)) : "memory");
        if (!ok) __nanosleep(64);
      }
    }
    return;
  }
  double a = lane;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __shfl_xor_sync(0xffffffffu, a, 1) + 1e-9;
  long long t1 = clock64();
  int idx = lane;
  for (int i = 0; i < n; ++i) { a += sm[idx]; idx = (idx + (a > 0 ? 1 : 0)) & 63; }
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) a = a + 1.0000001;
  long long t3 = clock64();
  out[lane] = a;
  if (lane == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2;
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar)) : "memory");
  }
  if (mode == 4) asm volatile("bar.arrive 9, 544;" ::: "memory");
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 4096 * 8); cudaMallocManaged(&cyc, 64 * 8);
  const char* nm[] = {"no waiters", "16 warps lane0 try_wait", "16 warps lane0 test_wait+nanosleep", "16 warps all-lanes try_wait", "16 warps parked in bar.sync"};
  for (int mode = 0; mode < 5; ++mode) {
    for (int r = 0; r < 2; ++r) { k<<<1, 544>>>(out, cyc, 2000, mode); cudaDeviceSynchronize(); }
    printf("%-38s SHFL+DADD %.1f  LDS+DADD %.1f  DADD %.1f cycles\n", nm[mode], cyc[0] / 2000.0, cyc[1] / 2000.0, cyc[2] / 2000.0);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
