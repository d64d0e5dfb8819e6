// DMMA issue-pattern probe: how do operand sources (register array vs LDS) and the number of
// independent accumulators per warp affect FP64 tensor throughput on B200?
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// MODE 0: A from register array, B constant; 1: A const, B from LDS; 2: both varying (A regs, B LDS)
template <int ACC, int MODE>
__global__ void pat(double* out, int iters) {
  __shared__ double sb[64 * 32];
  for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) sb[i] = 1.0 + i * 1e-9;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double areg[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) areg[i] = 1.0 + (lane + i) * 1e-7;
  double c[ACC][2];
#pragma unroll
  for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = 0.0;
  const double bconst = 0.999 + lane * 1e-9, aconst = 1.001;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const double b = (MODE == 0) ? bconst : sb[((it + k) & 63) * 32 + lane];
      const double a = (MODE == 1) ? aconst : areg[k];
#pragma unroll
      for (int i = 0; i < ACC; ++i) dmma(c[i][0], c[i][1], (MODE == 1) ? a : areg[(k + i) & 31], b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int ACC, int MODE>
void run(int sms, int warps_per_sm, double* out) {
  const int iters = 400;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  pat<ACC, MODE><<<sms, 32 * warps_per_sm>>>(out, 10);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  pat<ACC, MODE><<<sms, 32 * warps_per_sm>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop = 2.0 * 256 * ACC * 32.0 * iters * sms * warps_per_sm;
  printf("mode=%d acc=%d warps/SM=%2d : %.2f TF/s\n", MODE, ACC, warps_per_sm, flop / ms / 1e9);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  for (int w : {4, 8, 12}) {
    run<1, 0>(sms, w, out); run<2, 0>(sms, w, out); run<4, 0>(sms, w, out);
    run<1, 1>(sms, w, out); run<2, 1>(sms, w, out); run<4, 1>(sms, w, out);
    run<1, 2>(sms, w, out); run<2, 2>(sms, w, out); run<4, 2>(sms, w, out);
  }
  return 0;
}
