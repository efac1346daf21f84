// Latency of dependent DMMA.8x8x4 chains and throughput vs. independent chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void chain(double* out, long long* cyc, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-3;
  double c[CH][2];
#pragma unroll
  for (int k = 0; k < CH; ++k) c[k][0] = c[k][1] = 0;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CH; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += c[k][0] + c[k][1];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8);
  const int iters = 1000;
  long long h;
#define RUN(CH, WARPS)                                                                   \
  chain<CH><<<1, 32 * WARPS>>>(out, cyc, iters); cudaDeviceSynchronize();               \
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);                                        \
  printf("chains/warp %2d warps/CTA %2d: %.1f cycles per chain step (%.1f cyc/DMMA/SM)\n", CH, WARPS, \
         (double)h / iters, (double)h / iters / (CH * WARPS));
  RUN(1, 1) RUN(2, 1) RUN(3, 1) RUN(4, 1) RUN(6, 1) RUN(8, 1) RUN(12, 1) RUN(16, 1)
  RUN(3, 4) RUN(3, 8) RUN(6, 4) RUN(6, 8) RUN(8, 8) RUN(12, 4)
  return 0;
}
