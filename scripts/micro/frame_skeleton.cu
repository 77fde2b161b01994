// Microbenchmark (debug only): per-iteration cost of the per-frame skeleton
// primitives of fb_chain_kernel with 512 threads: barrier, warp shuffle
// reductions, reciprocal.  Prints cycles per iteration for each variant.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float wsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) skel(float *out, long long *cyc, int iters) {
  __shared__ float part[2][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float acc = tid * 1e-3f, inv = 1.f;
  if (tid < 64) (&part[0][0])[tid] = 1.f;
  __syncthreads();
  long long t0 = clock64();
  for (int k = 0; k < iters; ++k) {
    const int cur = k & 1;
    if (MODE & 1) {  // normaliser: lane_sum over 16 warp partials + reciprocal
      float x = lane < 16 ? part[cur][lane] : 0.f;
      x = wsum(x);
      inv = __frcp_rn(x + 1.f);
    }
    if (MODE & 2) {  // two warp sums + STS of the partials
      float a = wsum(acc * inv), b = wsum(acc + inv);
      if (lane == 0) part[cur ^ 1][warp] = a + b;
    }
    if (MODE & 4) acc = fmaf(acc, 0.999f, inv);
    if (MODE & 8) __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * 512 + tid] = acc + inv;
}

template <int MODE>
void run(const char *name, int iters) {
  float *out; long long *cyc;
  cudaMalloc(&out, 128 * 512 * 4); cudaMalloc(&cyc, 128 * 8);
  skel<MODE><<<128, 512>>>(out, cyc, iters);
  skel<MODE><<<128, 512>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h[128]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0; for (int i = 0; i < 128; ++i) m += h[i] / 128.0;
  printf("%-40s %8.1f cycles/iter\n", name, m / iters);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  const int it = 10000;
  run<8>("barrier only", it);
  run<1>("normaliser (lane_sum + rcp)", it);
  run<2>("2 warp sums + STS", it);
  run<3>("normaliser + 2 warp sums", it);
  run<11>("normaliser + 2 warp sums + barrier", it);
  run<15>("all + fma + barrier", it);
  return 0;
}
