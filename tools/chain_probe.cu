// Dependent-chain latencies of the TRSM diagonal-block path on one warp (cycles per link):
// DMMA->DMMA (accumulator), DMMA->DFMA (C result consumed by the FP64 ALU), DFMA->DMMA (A operand),
// DMMA->SHFL, SHFL->DFMA, DFMA->DFMA.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void probe(double* out, long long* cyc, int iters) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + lane * 1e-9, b = 0.5 - lane * 1e-9, c0 = 0.1 * lane, c1 = 0.2;
  long long t0, t1;
  int k = 0;
#define TIME(body)                                                   \
  t0 = clock64();                                                    \
  for (int i = 0; i < iters; ++i) { body; }                          \
  t1 = clock64();                                                    \
  if (threadIdx.x == 0) cyc[k] = (t1 - t0) / iters;                  \
  ++k;
  TIME(dmma(c0, c1, a, b));                                                         // 0 DMMA->DMMA (C)
  TIME(dmma(c0, c1, a, b); c0 = fma(c0, 0.999, 1e-9));                              // 1 DMMA->DFMA->DMMA
  TIME(dmma(c0, c1, a, b); a = fma(c0, 1e-3, 1.0));                                 // 2 DMMA->DFMA->A
  TIME(dmma(c0, c1, a, b); c0 = __shfl_xor_sync(0xffffffffu, c0, 2));               // 3 DMMA->SHFL->DMMA
  TIME(c0 = __shfl_xor_sync(0xffffffffu, c0, 2) * 0.999);                           // 4 SHFL->DMUL
  TIME(c0 = fma(c0, 0.999, 1e-9));                                                  // 5 DFMA
  TIME(c0 = fma(__shfl_sync(0xffffffffu, c0, lane ^ 1), 0.999, c1));               // 6 SHFL.IDX->DFMA
  TIME(c0 = (lane & 2) ? fma(c0, 0.999, 1e-9) : c0 * 1.0001);                       // 7 DFMA + FSEL
  out[threadIdx.x] = a + b + c0 + c1;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8 * 1024);
  cudaMalloc(&cyc, 8 * 16);
  probe<<<1, 32>>>(out, cyc, 10);
  cudaDeviceSynchronize();
  probe<<<1, 32>>>(out, cyc, 2000);
  cudaDeviceSynchronize();
  long long h[16];
  cudaMemcpy(h, cyc, 8 * 16, cudaMemcpyDeviceToHost);
  const char* names[] = {"DMMA->DMMA(C)", "DMMA->DFMA->DMMA", "DMMA->DFMA->A", "DMMA->SHFL->DMMA", "SHFL->DMUL",
                         "DFMA", "SHFL.IDX->DFMA", "DFMA+FSEL"};
  for (int i = 0; i < 8; ++i) printf("%-20s %lld cycles\n", names[i], h[i]);
  return 0;
}
