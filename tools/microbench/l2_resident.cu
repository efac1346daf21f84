// Does a write -> read scratch buffer of S MB stay in L2 while the consumer streams its
// results to HBM? (The two-pass coupling's T buffer: k_tgemm writes it, k_qfft reads it and
// writes the same number of bytes of volumes.) A cooperative kernel alternates two phases over
// a scratch of S MB: phase A writes it, phase B reads it and streams the data to a fresh slice
// of a large output (st.cs). Reported: output GB/s. If the scratch stays L2-resident the loop
// runs at the streaming-store rate; if not, at a third of the HBM rate.
//   mode 0: stream-out only (phase B without the scratch read)
//   mode 1: A + B, default stores to the scratch
//   mode 2: A + B, scratch stores / loads with an L2 evict_last policy
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ void st_pol(double2* p, double2 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ double2 ld_pol(const double2* p, unsigned long long pol) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;\n" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol) : "memory");
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(256) loop(double2* scratch, size_t s_elems, double2* out, size_t out_elems,
                                            int iters) {
  cg::grid_group grid = cg::this_grid();
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
  size_t obase = 0;
  for (int it = 0; it < iters; ++it) {
    if (MODE != 0) {
      for (size_t i = tid; i < s_elems; i += nth) {
        const double2 v = make_double2((double)i, (double)it);
        if (MODE == 2) st_pol(scratch + i, v, pol);
        else scratch[i] = v;
      }
      __threadfence();
      grid.sync();
    }
    for (size_t i = tid; i < s_elems; i += nth) {
      double2 v;
      if (MODE == 0) v = make_double2((double)i, (double)it);
      else if (MODE == 2) v = ld_pol(scratch + i, pol);
      else v = __ldcg(scratch + i);
      v.x += 1.0;
      __stcs(out + obase + i, v);
    }
    obase += s_elems;
    if (obase + s_elems > out_elems) obase = 0;
    if (MODE != 0) grid.sync();
  }
}

int main(int argc, char** argv) {
  const size_t out_bytes = 8ull << 30;
  double2 *scratch, *out;
  cudaMalloc(&out, out_bytes);
  cudaMalloc(&scratch, 1ull << 30);
  cudaMemset(out, 0, out_bytes);
  int dev = 0, sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool window = argc > 1 && atoi(argv[1]) == 1;  // persisting access-policy window on the scratch
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int sizes_mb[] = {8, 16, 24, 32, 48, 64, 80, 96, 128, 256, 1024};
  for (int mode = 0; mode < 3; ++mode) {
    void* fn = mode == 0 ? (void*)loop<0> : mode == 1 ? (void*)loop<1> : (void*)loop<2>;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (void (*)(double2*, size_t, double2*, size_t, int))fn, 256, 0);
    for (int smb : sizes_mb) {
      size_t s_elems = ((size_t)smb << 20) / 16;
      if (window) {
        size_t lim = 0;
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 96u << 20);
        cudaDeviceGetLimit(&lim, cudaLimitPersistingL2CacheSize);
        cudaStreamAttrValue av{};
        av.accessPolicyWindow.base_ptr = scratch;
        av.accessPolicyWindow.num_bytes = std::min((size_t)smb << 20, (size_t)128 << 20);
        av.accessPolicyWindow.hitRatio = 1.0f;
        av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &av);
        if (mode == 0 && smb == 8) printf("persisting L2 limit %zu MB\n", lim >> 20);
      }
      size_t out_elems = out_bytes / 16;
      int iters = (int)std::max<size_t>(4, (6ull << 30) / ((size_t)smb << 20));
      void* args[] = {&scratch, &s_elems, &out, &out_elems, &iters};
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0, s);
        cudaLaunchCooperativeKernel(fn, dim3(sms * per), dim3(256), args, 0, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      const double gb = (double)iters * smb * 1048576.0 / 1e9;
      printf("mode %d scratch %5d MB: %8.3f ms  %7.1f GB/s of output  (%.2f us per iteration)%s\n", mode, smb, ms,
             gb / ms * 1e3, ms * 1e3 / iters, window ? " [window]" : "");
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
