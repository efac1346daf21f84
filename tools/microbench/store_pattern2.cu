// Which property of the epilogue store pattern limits bandwidth: run width (NT columns per
// component row) and row alignment. Each CTA writes a (256/NT)-comp x NT-col tile of 33 rows;
// tiles in column-fastest order.
#include <cstdio>
#include <cuda_runtime.h>
template <int NT>
__global__ void pattern(double2* out, int ncomp, int ncol, int rowpitch, int n, long long vol) {
  constexpr int MT = 256 / NT;
  const int ncoltiles = (ncol + NT - 1) / NT;
  const int ntiles = (ncomp / MT) * ncoltiles;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int g = t / ncoltiles, ct = t % ncoltiles;
    const int comp = g * MT + threadIdx.x / NT, col = ct * NT + threadIdx.x % NT;
    if (col >= ncol) continue;
    double2* o = out + (long long)comp * vol + col;
    for (int a = 0; a < n; ++a) o[(long long)a * rowpitch] = make_double2(a, col);
  }
}
int main() {
  const int n = 33, nb = 17, ncol = n * nb, ncomp = 21024;
  double2* out;
  const long long vol_al = (long long)n * ((ncol + 7) / 8 * 8);
  cudaMalloc(&out, ncomp * vol_al * 16 + (1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    for (int aligned : {0, 1}) {
      const int pitch = aligned ? (ncol + 7) / 8 * 8 : ncol;
      const long long vol = (long long)n * pitch;
      const double bytes = (double)ncomp * n * ncol * 16;
#define RUN(NT)                                                                          \
  cudaEventRecord(e0);                                                                   \
  pattern<NT><<<148 * 2, 256>>>(out, ncomp, ncol, pitch, n, vol);                        \
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);      \
  if (rep) printf("NT %3d aligned %d: %.3f ms %.1f GB/s\n", NT, aligned, ms, bytes / ms / 1e6);
      RUN(8) RUN(16) RUN(32) RUN(64) RUN(128)
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
