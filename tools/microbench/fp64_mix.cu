// Do DMMA (tensor FP64) and DFMA (FP64 ALU) run concurrently on one SM? Half the warps of each
// block issue DMMA, the other half DFMA; compare with each alone.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dfma_work(double* out, int iters) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], 1.0000001, 1e-9);
  double s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ void dmma_work(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-3;
  double c[4][2] = {};
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void mixed(double* out, int it_mma, int it_fma, int mode) {
  const int w = threadIdx.x / 32;
  if (mode == 0) dmma_work(out, it_mma);
  else if (mode == 1) dfma_work(out, it_fma);
  else { if (w & 1) dfma_work(out, it_fma); else dmma_work(out, it_mma); }
}
int main() {
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 2, threads = 512;
  const int it_mma = 4000, it_fma = 2000;
  for (int mode = 0; mode < 3; ++mode) {
    mixed<<<blocks, threads>>>(out, 10, 10, mode);
    cudaEventRecord(e0);
    mixed<<<blocks, threads>>>(out, it_mma, it_fma, mode);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warps = blocks * threads / 32.0;
    double fl_mma = 2.0 * 256 * 16 * it_mma * (mode == 2 ? warps / 2 : warps);
    double fl_fma = 2.0 * 64 * it_fma * 32 * (mode == 2 ? warps / 2 : warps);
    if (mode == 0) fl_fma = 0; if (mode == 1) fl_mma = 0;
    printf("mode %d (%s): %.3f ms  dmma %.2f TF  dfma %.2f TF  total %.2f TF\n", mode,
           mode == 0 ? "dmma only" : mode == 1 ? "dfma only" : "half/half", ms,
           fl_mma / ms / 1e9, fl_fma / ms / 1e9, (fl_mma + fl_fma) / ms / 1e9);
  }
  return 0;
}
