// FP64 pipe microbenchmark: DFMA (CUDA cores) vs DMMA (mma.sync .f64 tensor path) on sm_100a.
// Used once to fix the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-3;
  double c[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma16_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1e-4, a2 = a0 + 2e-4, a3 = a0 + 3e-4;
  double b0 = 1.0 - threadIdx.x * 1e-3, b1 = b0 - 1e-4;
  double c[4][4];
#pragma unroll
  for (int k = 0; k < 4; ++k) { c[k][0] = 0; c[k][1] = 0; c[k][2] = 0; c[k][3] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        // m16n8k8: A 16x8 (4 regs), B 8x8 (2 regs), C 16x8 (4 regs)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                     : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("device %s SMs %d clock %d kHz smemOptin %zu\n", p.name, p.multiProcessorCount, p.clockRate, p.sharedMemPerBlockOptin);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int threads : {256, 512, 1024}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps; int iters = 4000;
      dfma_kernel<<<blocks, threads>>>(out, 10, 1.0000001, 1e-9);
      cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 64 * iters * (double)blocks * threads;
      printf("DFMA threads %d blocks %d: %.3f ms  %.2f TFLOP/s\n", threads, blocks, ms, flops / ms / 1e9);
    }
  }
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps; int iters = 2000;
      dmma_kernel<<<blocks, threads>>>(out, 10);
      cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
      double warps = (double)blocks * threads / 32;
      double flops = 2.0 * 8 * 8 * 4 * 32 * iters * warps;
      printf("DMMA m8n8k4 threads %d blocks %d: %.3f ms  %.2f TFLOP/s\n", threads, blocks, ms, flops / ms / 1e9);
      dmma16_kernel<<<blocks, threads>>>(out, 10);
      cudaEventRecord(e0); dmma16_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 16 * 8 * 8 * 16 * iters * warps;
      printf("DMMA m16n8k8 threads %d blocks %d: %.3f ms  %.2f TFLOP/s\n", threads, blocks, ms, flops / ms / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}
