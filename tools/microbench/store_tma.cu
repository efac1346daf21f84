// TMA tensor stores (cp.async.bulk.tensor.3d.global.shared::cta) of the epilogue's boxes:
// per component a box of 33 rows (a) x 8 complex (16 doubles) at column offset ct*8 of a
// [slots][33][561 complex] tensor, misaligned rows as in the So3Volume layout.
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int NTC>
__global__ void tma_store(const __grid_constant__ CUtensorMap tmap, int ncomp, int ncoltiles) {
  extern __shared__ __align__(128) double2 buf[];  // [16 comps][33][NTC]
  const int ntiles = (ncomp / 16) * ncoltiles;
  for (int i = threadIdx.x; i < 16 * 33 * NTC; i += blockDim.x) buf[i] = make_double2(i, 1.0);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int g = t / ncoltiles, ct = t % ncoltiles;
    if (threadIdx.x < 16) {
      const int comp = g * 16 + threadIdx.x;
      const double2* src = buf + threadIdx.x * 33 * NTC;
      asm volatile(
          "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(&tmap),
          "r"(ct * NTC * 2), "r"(0), "r"(comp), "r"(smem_u32(src))
          : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    __syncthreads();
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

int main() {
  const int n = 33, ncol = 561, ncomp = 21024;
  const long long vol = (long long)n * ncol;
  double* out;
  cudaMalloc(&out, ncomp * vol * 16);
  PFN_cuTensorMapEncodeTiled_v12000 encode;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const double bytes = (double)ncomp * vol * 16;
  for (int NTC : {8, 16}) {
    CUtensorMap tmap;
    cuuint64_t dims[3] = {(cuuint64_t)ncol * 2, (cuuint64_t)n, (cuuint64_t)ncomp};
    cuuint64_t strides[2] = {(cuuint64_t)ncol * 16, (cuuint64_t)vol * 16};
    cuuint32_t box[3] = {(cuuint32_t)NTC * 2, (cuuint32_t)n, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, out, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    const size_t smem = 16 * 33 * NTC * 16;
    auto k = NTC == 8 ? tma_store<8> : tma_store<16>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k<<<148, 128, smem>>>(tmap, ncomp, (ncol + NTC - 1) / NTC);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("TMA box %d cols x 33 rows: %.3f ms %.1f GB/s\n", NTC, ms, bytes / ms / 1e6);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
