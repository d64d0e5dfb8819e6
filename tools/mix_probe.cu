// FP64 pipe sharing: DMMA.8x8x4 throughput with R independent DFMA per DMMA interleaved
// (TRSM mixes ~1 DFMA per DMMA: the diagonal-block substitution).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int R>
__global__ void probe(double* out, int iters) {
  double c[8][2], f[8];
  const double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = c[i][1] = 0; f[i] = i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      dmma(c[i][0], c[i][1], a, b);
#pragma unroll
      for (int r = 0; r < R; ++r) f[(i + r) & 7] = fma(f[(i + r) & 7], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int R>
void run(double* out) {
  const int iters = 20000, blocks = 148, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  probe<R><<<blocks, threads>>>(out, 100);
  cudaEventRecord(e0);
  probe<R><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double dmma = double(blocks) * threads / 32 * iters * 8;
  const double cyc_per_dmma_smsp = ms * 1e-3 * 1.965e9 / (dmma / (148.0 * 4));
  printf("R=%d DFMA per DMMA: %.3f ms  %.2f cycles per DMMA per SMSP  (DMMA %.1f TF/s)\n", R, ms, cyc_per_dmma_smsp,
         dmma * 512 / (ms * 1e-3) / 1e12);
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 256 * 8);
  run<0>(out); run<1>(out); run<2>(out); run<4>(out);
  return 0;
}
