// Per-step cycle cost of the register-resident 16x16 Cholesky diagonal-block factorisation
// (chol.cu step (a)), one warp, to find what dominates its pivot chain.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int P = 16;
constexpr unsigned kFull = 0xffffffffu;

template <int VARIANT>
__global__ void probe(const double* A, double* out, long long* clk) {
  const int lane = threadIdx.x;
  double col[P];
#pragma unroll
  for (int r = 0; r < P; ++r) col[r] = (lane < P && r <= lane) ? A[r * P + lane] : (r == lane ? 1.0 : 0.0);
  long long t[P + 1];
#pragma unroll
  for (int c = 0; c < P; ++c) {
    t[c] = clock64();
    double d = __shfl_sync(kFull, col[c], c);
    double inv;
    if (VARIANT == 0) inv = rsqrt(d);
    else if (VARIANT == 1) inv = 1.0 / sqrt(d);
    else inv = (double)rsqrtf((float)d);  // (timing only)
    if (lane == c) col[c] = d * inv;
    else if (lane > c) col[c] *= inv;
#pragma unroll
    for (int i = c + 1; i < P; ++i) {
      const double ri = __shfl_sync(kFull, col[c], i);
      if (lane >= i) col[i] = fma(-ri, col[c], col[i]);
    }
  }
  t[P] = clock64();
  double s = 0;
#pragma unroll
  for (int r = 0; r < P; ++r) s += col[r];
  out[lane] = s;
  if (lane == 0)
    for (int c = 0; c < P; ++c) clk[c] = t[c + 1] - t[c];
}

// Variant: row c of the block broadcast through shared memory (1 STS + 8 LDS.128 per step)
__global__ void probe_smem(const double* A, double* out, long long* clk) {
  __shared__ __align__(16) double rowc[2][32];
  const int lane = threadIdx.x;
  double col[P];
#pragma unroll
  for (int r = 0; r < P; ++r) col[r] = (lane < P && r <= lane) ? A[r * P + lane] : (r == lane ? 1.0 : 0.0);
  long long t[P + 1];
#pragma unroll
  for (int c = 0; c < P; ++c) {
    t[c] = clock64();
    const double d = __shfl_sync(kFull, col[c], c);
    const double inv = rsqrt(d);
    if (lane == c) col[c] = d * inv;
    else if (lane > c) col[c] *= inv;
    if (c + 1 < P && lane == c + 1) col[c + 1] = fma(-col[c], col[c], col[c + 1]);
    rowc[c & 1][lane] = col[c];
    __syncwarp();
#pragma unroll
    for (int i2 = (c + 1) & ~1; i2 < P; i2 += 2) {
      const double2 r2 = *reinterpret_cast<const double2*>(&rowc[c & 1][i2]);
      if (i2 > c && i2 != c + 1 && lane >= i2) col[i2] = fma(-r2.x, col[c], col[i2]);
      if (i2 + 1 > c && i2 + 1 != c + 1 && lane >= i2 + 1) col[i2 + 1] = fma(-r2.y, col[c], col[i2 + 1]);
      if (i2 == c + 1 - 1 + 1 && false) {}
    }
    // lanes > c+1 still need row c+1's update from step c
    if (c + 1 < P && lane > c + 1) col[c + 1] = fma(-rowc[c & 1][c + 1], col[c], col[c + 1]);
  }
  t[P] = clock64();
  double s = 0;
#pragma unroll
  for (int r = 0; r < P; ++r) s += col[r];
  out[lane] = s;
  if (lane == 0)
    for (int c = 0; c < P; ++c) clk[c] = t[c + 1] - t[c];
}

int main() {
  double hA[P * P];
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < P; ++j) hA[i * P + j] = (i == j ? P + 1.0 : 0.5 / (1 + i + j));
  double *A, *out;
  long long* clk;
  cudaMalloc(&A, sizeof hA);
  cudaMalloc(&out, 32 * 8);
  cudaMalloc(&clk, P * 8);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  long long h[P];
  for (int rep = 0; rep < 2; ++rep) {
    probe<0><<<1, 32>>>(A, out, clk);
    cudaMemcpy(h, clk, sizeof h, cudaMemcpyDeviceToHost);
    printf("rsqrt   :");
    for (int c = 0; c < P; ++c) printf(" %lld", h[c]);
    printf("\n");
    probe<1><<<1, 32>>>(A, out, clk);
    cudaMemcpy(h, clk, sizeof h, cudaMemcpyDeviceToHost);
    printf("1/sqrt  :");
    for (int c = 0; c < P; ++c) printf(" %lld", h[c]);
    printf("\n");
    probe<2><<<1, 32>>>(A, out, clk);
    cudaMemcpy(h, clk, sizeof h, cudaMemcpyDeviceToHost);
    printf("rsqrtf  :");
    for (int c = 0; c < P; ++c) printf(" %lld", h[c]);
    printf("\n");
    double o1[32], o2[32];
    probe<0><<<1, 32>>>(A, out, clk);
    cudaMemcpy(o1, out, sizeof o1, cudaMemcpyDeviceToHost);
    probe_smem<<<1, 32>>>(A, out, clk);
    cudaMemcpy(o2, out, sizeof o2, cudaMemcpyDeviceToHost);
    cudaMemcpy(h, clk, sizeof h, cudaMemcpyDeviceToHost);
    printf("smem    :");
    for (int c = 0; c < P; ++c) printf(" %lld", h[c]);
    double md = 0;
    for (int i = 0; i < 32; ++i) md = fmax(md, fabs(o1[i] - o2[i]));
    printf("   (max diff vs shuffle version %.3e)\n", md);
  }
  return 0;
}
