// Latency probes for the single-CTA Cholesky design: dependent chains of DDIV, DSQRT, RSQRT+Newton,
// double SHFL, LDS, generic LD of shared memory, and __syncthreads at 512 threads.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(double* out, long long* cyc, const double* gin, int iters) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double x = 1.0000001 + threadIdx.x * 1e-12;
  long long t0, t1;
  // DDIV chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0000003 / x;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
  // DSQRT chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = sqrt(x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / iters;
  // rsqrt chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = rsqrt(x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / iters;
  // SHFL double chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-9;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / iters;
  // LDS chain (address depends on value)
  int idx = threadIdx.x & 511;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double v = sm[idx];
    idx = (idx + (int)(v > 2.0) + 1) & 511;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / iters;
  // generic LD of shared memory
  const double* gp = (iters > 0) ? sm : gin;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double v = gp[idx];
    idx = (idx + (int)(v > 2.0) + 1) & 511;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0) / iters;
  // __syncthreads
  t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0) / iters;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 0.999999, 1e-9);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[7] = (t1 - t0) / iters;
  // division by a loop-invariant (compiler may hoist reciprocal?)
  double y = x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) y = y / 1.0000001 + 1e-9;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[8] = (t1 - t0) / iters;
  out[threadIdx.x] = x + idx + y;
}

int main() {
  double* out;
  long long* cyc;
  double* g;
  cudaMalloc(&out, 8 * 1024);
  cudaMalloc(&cyc, 8 * 16);
  cudaMalloc(&g, 8 * 1024);
  for (int threads : {32, 512}) {
    probe<<<1, threads>>>(out, cyc, g, 1000);
    cudaDeviceSynchronize();
    long long h[16];
    cudaMemcpy(h, cyc, 8 * 16, cudaMemcpyDeviceToHost);
    printf("threads=%d  DDIV %lld  DSQRT %lld  RSQRT %lld  SHFL.f64 %lld  LDS %lld  LD.generic(smem) %lld  BAR %lld  DFMA %lld  DDIV-by-const %lld cycles\n",
           threads, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8]);
  }
  return 0;
}
