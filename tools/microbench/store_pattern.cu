// Store bandwidth of the epilogue's access pattern: a warp writes 4 segments of 128 B
// (8 columns x 16 B of 4 components) at row offsets a*ncol (16-B aligned, not 128-B aligned).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void pattern(double2* out, int ncomp, int ncol, int n, long long vol, int ncoltiles,
                        int mirror) {
  // one CTA of 256 threads handles a 16-component x 8-column tile; grid-stride over tiles
  const int ntiles = (ncomp / 16) * ncoltiles;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int g = t / ncoltiles, ct = t % ncoltiles;
    const int pair = threadIdx.x % 128, a0 = threadIdx.x / 128;
    const int comp = g * 16 + pair / 8, col = ct * 8 + pair % 8;
    if (col >= ncol) continue;
    double2* o = out + (long long)comp * vol + col;
    double2* om = out + (long long)(comp + ncomp) * vol + col;
    for (int a = a0; a < n; a += 2) {
      o[(long long)a * ncol] = make_double2(a, col);
      if (mirror) om[(long long)a * ncol] = make_double2(col, a);
    }
  }
}
__global__ void contiguous(double2* out, long long count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = make_double2(i, 0);
}
int main() {
  const int n = 33, nb = 17, ncol = n * nb, ncomp = 10592;  // config 2: 10,585 computed
  const long long vol = (long long)n * ncol;
  double2* out;
  const size_t bytes = 2ull * ncomp * vol * 16;
  if (cudaMalloc(&out, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    for (int blocks : {148, 296, 592}) {
      for (int mirror : {0, 1}) {
        cudaEventRecord(e0);
        pattern<<<blocks, 256>>>(out, ncomp, ncol, n, vol, (ncol + 7) / 8, mirror);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        const double b = (mirror ? 2.0 : 1.0) * ncomp * vol * 16;
        if (rep) printf("pattern blocks %d mirror %d: %.3f ms %.1f GB/s\n", blocks, mirror, ms, b / ms / 1e6);
      }
    }
    cudaEventRecord(e0);
    contiguous<<<148 * 8, 256>>>(out, 2ll * ncomp * vol);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("contiguous: %.3f ms %.1f GB/s\n", ms, bytes / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
