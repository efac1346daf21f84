// Misaligned 128-B strips (So3Volume rows, pitch 561) with different L2 store policies.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__device__ __forceinline__ void st(double2* p, double2 v, unsigned long long pol) {
  if (MODE == 0) *p = v;
  else if (MODE == 1) __stcs(p, v);
  else if (MODE == 2)
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
  else
    asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};\n" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
template <int MODE, int ORDER>
__global__ void pattern(double2* out, int ncomp, int ncol, int n, long long vol) {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  const int ncoltiles = (ncol + 7) / 8;
  const int ngroups = ncomp / 16;
  const int ntiles = ngroups * ncoltiles;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int g = ORDER ? t % ngroups : t / ncoltiles, ct = ORDER ? t / ngroups : t % ncoltiles;
    const int pair = threadIdx.x % 128, a0 = threadIdx.x / 128;
    const int comp = g * 16 + pair / 8, col = ct * 8 + pair % 8;
    if (col >= ncol) continue;
    double2* o = out + (long long)comp * vol + col;
    for (int a = a0; a < n; a += 2) st<MODE>(o + (long long)a * ncol, make_double2(a, col), pol);
  }
}
int main() {
  const int n = 33, ncol = 561, ncomp = 21024;
  const long long vol = (long long)n * ncol;
  double2* out;
  cudaMalloc(&out, ncomp * vol * 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const double bytes = (double)ncomp * vol * 16;
  const char* names[] = {"default", "st.cs", "evict_last hint", "L1::no_allocate"};
  for (int rep = 0; rep < 2; ++rep) {
#define RUN(M, O)                                                                        \
  cudaEventRecord(e0);                                                                   \
  pattern<M, O><<<148 * 2, 256>>>(out, ncomp, ncol, n, vol);                            \
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);      \
  if (rep) printf("%-16s order %s: %.3f ms %.1f GB/s\n", names[M], O ? "group-fast" : "col-fast", ms, bytes / ms / 1e6);
    RUN(0, 0) RUN(1, 0) RUN(2, 0) RUN(3, 0) RUN(0, 1) RUN(2, 1)
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
