// Shared-memory load throughput for the TRSM access patterns (wavefront cost per warp load):
//   128b_b4: LDS.128, 4 distinct 16-B addresses (lanes with equal t share)  -- D row loads
//   64b_b4 : LDS.64,  4 distinct addresses                                   -- split D loads
//   64b_d  : LDS.64,  32 distinct consecutive doubles                        -- B fragments
//   64b_b1 : LDS.64,  one address (warp-uniform)
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void probe(double* out, int iters) {
  __shared__ __align__(16) double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0.5;
  __syncthreads();
  const int lane = threadIdx.x & 31, t = lane & 3;
  double acc0 = 0, acc1 = 0;
  int base = (threadIdx.x >> 5) * 64;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int o = (base + k * 8) & 4031;
      if (MODE == 0) {
        const double2 v = *reinterpret_cast<const double2*>(s + o + 2 * t);
        acc0 += v.x; acc1 += v.y;
      } else if (MODE == 1) {
        double a, b;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a) : "r"((unsigned)__cvta_generic_to_shared(s + o + 2 * t)));
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(b) : "r"((unsigned)__cvta_generic_to_shared(s + o + 2 * t + 1)));
        acc0 += a; acc1 += b;
      } else if (MODE == 2) {
        double a;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a) : "r"((unsigned)__cvta_generic_to_shared(s + ((o + lane) & 4095))));
        acc0 += a;
      } else if (MODE == 3) {
        double a;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a) : "r"((unsigned)__cvta_generic_to_shared(s + o)));
        acc0 += a;
      } else if (MODE == 4) {  // LDS.128 distinct
        const double2 v = *reinterpret_cast<const double2*>(s + ((o + 2 * lane) & 4094));
        acc0 += v.x; acc1 += v.y;
      } else if (MODE == 5) {  // LDS.128, 8 distinct (lanes (g&1, t))
        const double2 v = *reinterpret_cast<const double2*>(s + o + 2 * (lane & 7));
        acc0 += v.x; acc1 += v.y;
      } else if (MODE == 6) {  // SHFL of a double from lane (lane&~3)|k
        acc0 = __shfl_sync(0xffffffffu, acc0, (lane & ~3) | (k & 3)) + 1.0;
      } else {  // LDS.64 bcast4 with t-major 32B-apart addresses
        double a;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a) : "r"((unsigned)__cvta_generic_to_shared(s + o + 4 * t)));
        acc0 += a;
      }
    }
    base += 16;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1;
}

int main() {
  cudaError_t e0 = cudaFree(0); printf("init %s\n", cudaGetErrorString(e0));
  double* out;
  cudaMalloc(&out, 148 * 4 * 1024 * 8);
  int sms = 148;
  const int iters = 4096;
  const char* names[] = {"LDS.128 bcast4 (D rows)", "2x LDS.64 bcast4", "LDS.64 distinct (B frags)", "LDS.64 uniform", "LDS.128 distinct", "LDS.128 8-distinct", "SHFL.f64 quad", "LDS.64 bcast4 stride4"};
  for (int mode = 0; mode < 8; ++mode) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      switch (mode) {
        case 0: probe<0><<<sms * 2, 512>>>(out, iters); break;
        case 1: probe<1><<<sms * 2, 512>>>(out, iters); break;
        case 2: probe<2><<<sms * 2, 512>>>(out, iters); break;
        case 3: probe<3><<<sms * 2, 512>>>(out, iters); break;
        case 4: probe<4><<<sms * 2, 512>>>(out, iters); break;
        case 5: probe<5><<<sms * 2, 512>>>(out, iters); break;
        case 6: probe<6><<<sms * 2, 512>>>(out, iters); break;
        default: probe<7><<<sms * 2, 512>>>(out, iters); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      { cudaError_t le = cudaGetLastError(); if (le != cudaSuccess) printf("launch error %s\n", cudaGetErrorString(le)); }
    }
    float ms; cudaEventElapsedTime(&ms, a, b);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double warp_loads_per_sm = 2.0 * 16 * iters * 16 * (mode == 1 ? 2 : 1);  // blocks/SM * warps * ...
    const double cycles = ms * 1e-3 * 1.965e9;
    printf("%-28s %.3f ms  %.2f cycles per warp-load per SM\n", names[mode], ms, cycles / warp_loads_per_sm);
  }
  return 0;
}
