// Experiment helper: occupy N SMs (one 227 KB CTA each) for a fixed number of
// cycles, to measure how fast a concurrent kernel runs on the remaining SMs.
#include <cuda_runtime.h>
__global__ void blocker_kernel(long long cycles) {
  extern __shared__ unsigned char s[];
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  if (threadIdx.x == 0) s[0] = 1;
}
extern "C" int launch_blocker(int nblocks, long long cycles, void *stream) {
  const int smem = 227 * 1024;
  cudaFuncSetAttribute(blocker_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  blocker_kernel<<<nblocks, 512, smem, (cudaStream_t)stream>>>(cycles);
  return (int)cudaGetLastError();
}
