// Is 32-B sector alignment of each row segment enough? Rows of the real layout (pitch 561,
// odd); tiles of W written columns per row. "shift" mode: tile ct writes, in row a, the W
// columns starting at C + ((a*ncol + C) & 1), C = ct*W (segments sector-aligned, abutting).
#include <cstdio>
#include <cuda_runtime.h>
template <int W, int SHIFT>
__global__ void pattern(double2* out, int ncomp, int ncol, int n, long long vol) {
  constexpr int MT = 256 / 16;           // 16 comps x 16 lanes per tile row
  const int ncoltiles = (ncol + W - 1) / W;
  const int ntiles = (ncomp / MT) * ncoltiles;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int g = t / ncoltiles, ct = t % ncoltiles;
    const int comp = g * MT + threadIdx.x / 16, j = threadIdx.x % 16;
    if (j >= W) continue;
    const int C = ct * W;
    double2* o = out + (long long)comp * vol;
    for (int a = 0; a < n; ++a) {
      const int s = SHIFT ? C + (int)(((long long)a * ncol + C) & 1) : C;
      const int col = s + j;
      if (col < ncol) o[(long long)a * ncol + col] = make_double2(a, col);
    }
  }
}
int main() {
  const int n = 33, nb = 17, ncol = n * nb, ncomp = 21024;
  const long long vol = (long long)n * ncol;
  double2* out;
  cudaMalloc(&out, ncomp * vol * 16 + (1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const double bytes = (double)ncomp * vol * 16;
  for (int rep = 0; rep < 2; ++rep) {
#define RUN(W, S)                                                                        \
  cudaEventRecord(e0);                                                                   \
  pattern<W, S><<<148 * 2, 256>>>(out, ncomp, ncol, n, vol);                            \
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);      \
  if (rep) printf("W %2d shift %d: %.3f ms %.1f GB/s\n", W, S, ms, bytes / ms / 1e6);
    RUN(8, 0) RUN(8, 1) RUN(14, 0) RUN(14, 1) RUN(16, 0) RUN(16, 1)
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
