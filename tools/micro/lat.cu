// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/lat tools/micro/lat.cu
// Latency microbenchmark: dependent chains of fp64 ops, shuffles, smem loads
// on one warp (clock64), with and without 16 other busy warps on the SM.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, int n, double x0, int busy) {
  __shared__ double sm[1024];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  __syncthreads();
  if (w > 0) {  // background fp64 + shuffle load (like the consumer scans)
    if (!busy) return;
    double a = x0 + threadIdx.x, b = 1.0;
    for (int i = 0; i < n * 4; ++i) {
      a = a * 1.0000001 + b;
      b = __shfl_xor_sync(0xffffffffu, a, 1) * 0.5;
    }
    out[threadIdx.x + 64] = a + b;
    return;
  }
  double a = x0 + lane;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = a + 1.0000001;
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) a = a * 1.0000001;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, 1.0000001, 1e-9);
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) a = __shfl_xor_sync(0xffffffffu, a, 1) + 1e-9;
  long long t4 = clock64();
  int idx = lane;
  for (int i = 0; i < n; ++i) { a += sm[idx]; idx = (idx + (a > 0 ? 1 : 0)) & 1023; }
  long long t5 = clock64();
  float f = (float)a;
  for (int i = 0; i < n; ++i) f = f * 1.0000001f + 1e-7f;
  long long t6 = clock64();
  for (int i = 0; i < n; ++i) a = __drcp_rn(a) + 1e-9;
  long long t7 = clock64();
  out[lane] = a + f;
  if (lane == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
    cyc[5] = t6 - t5; cyc[6] = t7 - t6;
  }
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 4096 * 8); cudaMallocManaged(&cyc, 64 * 8);
  const int n = 2000;
  const char* nm[] = {"DADD", "DMUL", "DFMA", "SHFL+DADD", "LDS+DADD", "FFMA", "DRCP+DADD"};
  for (int busy = 0; busy < 2; ++busy) {
    lat<<<1, 544, 0>>>(out, cyc, n, 1.0, busy);
    cudaDeviceSynchronize();
    lat<<<1, 544, 0>>>(out, cyc, n, 1.0, busy);
    cudaDeviceSynchronize();
    printf("busy=%d:", busy);
    for (int i = 0; i < 7; ++i) printf(" %s %.1f", nm[i], (double)cyc[i] / n);
    printf("  (cycles per dependent op)\n");
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
