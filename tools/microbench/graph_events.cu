// Does cudaEventElapsedTime work on events recorded by a captured CUDA graph?
#include <cstdio>
__global__ void spin(long long n) { long long t = clock64(); while (clock64() - t < n) {} }
int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  cudaEventRecordWithFlags(e0, s, cudaEventRecordExternal); spin<<<1, 1, 0, s>>>(2000000); cudaEventRecordWithFlags(e1, s, cudaEventRecordExternal);
  cudaGraph_t g; cudaStreamEndCapture(s, &g);
  cudaGraphExec_t x; printf("inst %d\n", (int)cudaGraphInstantiate(&x, g, 0));
  for (int i = 0; i < 3; ++i) {
    printf("launch %d\n", (int)cudaGraphLaunch(x, s));
    printf("sync %d\n", (int)cudaEventSynchronize(e1));
    float ms = -1; cudaError_t r = cudaEventElapsedTime(&ms, e0, e1);
    printf("elapsed rc=%d (%s) ms=%f\n", (int)r, cudaGetErrorString(r), ms);
  }
  return 0;
}
