// FP64 peak probes on B200 (sm_100a): DFMA loop and DMMA (mma.sync f64) loops.
// Used to derive the roofline denominator for the FP64 path (MEASURED_PEAKS.json has no fp64 entry).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i];
  if (s == 12345.0) out[0] = s;
}

template <int ACC>
__global__ void dmma884_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
  double c[ACC][2];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int ACC>
__global__ void dmma16816_loop(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-6;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-6;
  double c[ACC][4];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}

template <typename F>
double time_ms(F f, int reps) {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0)); f(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("device %s sms %d smem/block optin %zu regs/sm %d\n", p.name, sms, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
  double* out; CK(cudaMalloc(&out, 8));
  const int iters = 20000;
  for (int threads : {128, 256, 512, 1024}) {
    for (int bps : {1, 2, 4}) {
      int grid = sms * bps;
      if (threads * bps > 2048) continue;
      double ms = time_ms([&] { dfma_loop<8><<<grid, threads>>>(out, iters, 0.999999, 1e-9); }, 5);
      double flop = 2.0 * 8 * iters * (double)grid * threads;
      printf("DFMA chains=8 threads=%d blocks/sm=%d : %.3f ms  %.2f TFLOP/s\n", threads, bps, ms, flop / ms / 1e9);
    }
  }
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int grid = sms * bps;
      if (threads * bps > 2048) continue;
      double ms = time_ms([&] { dmma884_loop<8><<<grid, threads>>>(out, iters / 4); }, 5);
      double flop = 2.0 * 256 * 8 * (iters / 4) * (double)grid * (threads / 32);
      printf("DMMA m8n8k4 acc=8 threads=%d blocks/sm=%d : %.3f ms  %.2f TFLOP/s\n", threads, bps, ms, flop / ms / 1e9);
      ms = time_ms([&] { dmma884_loop<2><<<grid, threads>>>(out, iters); }, 5);
      flop = 2.0 * 256 * 2 * iters * (double)grid * (threads / 32);
      printf("DMMA m8n8k4 acc=2 threads=%d blocks/sm=%d : %.3f ms  %.2f TFLOP/s\n", threads, bps, ms, flop / ms / 1e9);
      ms = time_ms([&] { dmma16816_loop<4><<<grid, threads>>>(out, iters / 16); }, 5);
      flop = 2.0 * 16 * 8 * 16 * 4 * (iters / 16) * (double)grid * (threads / 32);
      printf("DMMA m16n8k16 acc=4 threads=%d blocks/sm=%d : %.3f ms  %.2f TFLOP/s\n", threads, bps, ms, flop / ms / 1e9);
    }
  }
  // single-warp latency of a dependent DMMA chain
  {
    double ms = time_ms([&] { dmma884_loop<1><<<1, 32>>>(out, iters); }, 3);
    printf("DMMA m8n8k4 dependent-chain latency: %.1f ns/mma\n", ms * 1e6 / iters);
    ms = time_ms([&] { dfma_loop<1><<<1, 32>>>(out, iters * 4, 0.999, 1e-9); }, 3);
    printf("DFMA dependent-chain latency: %.2f ns/fma\n", ms * 1e6 / (iters * 4));
  }
  // sustained: long DMMA run (~3 s)
  {
    int grid = sms * 2, threads = 256;
    double ms1 = time_ms([&] { dmma884_loop<8><<<grid, threads>>>(out, 200000); }, 1);
    double flop = 2.0 * 256 * 8 * 200000.0 * grid * (threads / 32);
    printf("DMMA sustained single launch %.1f ms: %.2f TFLOP/s\n", ms1, flop / ms1 / 1e9);
    double ms2 = time_ms([&] { dfma_loop<8><<<grid, 512>>>(out, 400000, 0.999999, 1e-9); }, 1);
    flop = 2.0 * 8 * 400000.0 * grid * 512;
    printf("DFMA sustained single launch %.1f ms: %.2f TFLOP/s\n", ms2, flop / ms2 / 1e9);
  }
  return 0;
}
