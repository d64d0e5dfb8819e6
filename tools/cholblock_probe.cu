// Cycle cost of the Cholesky kernel's 8x8 diagonal-block factorisation on ONE thread, first
// (cold instruction cache) and repeated calls, with three reciprocal square roots:
// rsqrt() (CUDA's double rsqrt), rsqrt.approx.f64 + one Newton step, and 1/sqrt().
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__device__ __forceinline__ double rs(double d) {
  if (V == 0) return rsqrt(d);
  if (V == 1) {
    double y;
    asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(d));
    const double h = 0.5 * d;
    return fma(y, fma(-h * y, y, 0.5), y);  // y (1.5 - d y^2 / 2)
  }
  return 1.0 / sqrt(d);
}

template <int V>
__global__ void probe(const double* A, double* out, long long* cyc) {
  __shared__ double W[8 * 9];
  for (int i = threadIdx.x; i < 72; i += blockDim.x) W[i] = A[i];
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int rep = 0; rep < 4; ++rep) {
    const long long t0 = clock64();
    double a[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int j = r; j < 8; ++j) a[r][j] = W[r * 9 + j];
    int bad = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      double d = a[c][c];
      if (!bad && (!(d > 0.0) || !isfinite(d))) bad = c + 1;
      if (bad) d = 1.0;
      const double inv = rs<V>(d);
      a[c][c] = d * inv;
#pragma unroll
      for (int j = c + 1; j < 8; ++j) a[c][j] *= inv;
#pragma unroll
      for (int i = c + 1; i < 8; ++i)
#pragma unroll
        for (int j = i; j < 8; ++j) a[i][j] = fma(-a[c][i], a[c][j], a[i][j]);
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int j = r; j < 8; ++j) W[r * 9 + j] = a[r][j];
    const long long t1 = clock64();
    cyc[rep] = t1 - t0;
    out[rep] = a[7][7] + bad;
  }
}

int main() {
  double hA[72];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 9; ++j) hA[i * 9 + j] = (i == j) ? 10.0 + i : (j < 8 ? 0.1 * (i + j) : 0.0);
  double *A, *out;
  long long* cyc;
  cudaMalloc(&A, 72 * 8);
  cudaMalloc(&out, 64);
  cudaMalloc(&cyc, 64);
  cudaMemcpy(A, hA, 72 * 8, cudaMemcpyHostToDevice);
  long long h[4];
  probe<0><<<1, 32>>>(A, out, cyc);
  cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
  printf("rsqrt():            %lld %lld %lld %lld cycles\n", h[0], h[1], h[2], h[3]);
  probe<1><<<1, 32>>>(A, out, cyc);
  cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
  printf("rsqrt.approx+Newton: %lld %lld %lld %lld cycles\n", h[0], h[1], h[2], h[3]);
  probe<2><<<1, 32>>>(A, out, cyc);
  cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
  printf("1/sqrt():           %lld %lld %lld %lld cycles\n", h[0], h[1], h[2], h[3]);
  // accuracy of rsqrt.approx.f64 + one Newton step against rsqrt() over many arguments
  return 0;
}
