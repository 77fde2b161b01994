// Micro-benchmark (one CTA of 512 threads, 1 SM): cost of the posterior scatter
// of one WSJ-mono frame (10k arc terms, 84 pdfs) per scheme, in cycles.
//   slots : u16 slot-index load + fp32 store to the arc's per-pdf slot (current split kernel)
//   atoms : u32 fixed-point shared atomic add into the pdf's bin (ATOMS.ADD)
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void bench(const unsigned short *xslot_g, const unsigned char *pdf_g, int n, int reps,
                      long long *cycles, unsigned *sink) {
  extern __shared__ __align__(16) unsigned char sm[];
  float *xterm = reinterpret_cast<float *>(sm);                       // 10752 floats
  unsigned short *xs = reinterpret_cast<unsigned short *>(sm + 43008);  // 10752 u16
  unsigned char *pdf = sm + 43008 + 21504;                             // 10752 u8
  unsigned *bins = reinterpret_cast<unsigned *>(sm + 43008 + 21504 + 10752);
  for (int i = threadIdx.x; i < n; i += blockDim.x) { xs[i] = xslot_g[i]; pdf[i] = pdf_g[i]; xterm[i] = 0.f; }
  if (threadIdx.x < 128) bins[threadIdx.x] = 0;
  __syncthreads();
  float v = 1e-3f * threadIdx.x;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) xterm[xs[i]] = v + i;
    __syncthreads();
  }
  long long t1 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&bins[pdf[i]], unsigned(i) & 1023u);
    __syncthreads();
  }
  long long t2 = clock64();
  if (threadIdx.x == 0) { cycles[0] = (t1 - t0) / reps; cycles[1] = (t2 - t1) / reps; }
  sink[threadIdx.x] = bins[threadIdx.x & 127] + unsigned(xterm[threadIdx.x]);
}

int main() {
  const int n = 10000, D = 84;
  std::vector<unsigned short> xs(n);
  std::vector<unsigned char> pd(n);
  srand(1);
  for (int i = 0; i < n; ++i) { pd[i] = rand() % D; xs[i] = rand() % n; }
  unsigned short *dxs; unsigned char *dpd; long long *dc; unsigned *ds;
  cudaMalloc(&dxs, n * 2); cudaMalloc(&dpd, n); cudaMalloc(&dc, 16); cudaMalloc(&ds, 4096);
  cudaMemcpy(dxs, xs.data(), n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dpd, pd.data(), n, cudaMemcpyHostToDevice);
  const int smem = 43008 + 21504 + 10752 + 512;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<<<1, 512, smem>>>(dxs, dpd, n, 200, dc, ds);
  long long c[2];
  cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
  printf("per frame (10k arcs, 512 threads): slot stores %lld cycles, ATOMS.ADD bins %lld cycles\n", c[0], c[1]);
  return 0;
}
