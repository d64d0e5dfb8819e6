// zwide.cu -- complex X with n in (256, 512] ("everything carries over to
// complex matrices"; reading D23).
//
// The m x 2n real split matrix S (zchol.cu) is wider than the real kernels' 512 columns, so it is
// taken as two column blocks S = [S1 S2]: S1 = the first 512 columns (complex columns 0..255),
// S2 = the last q = 2n - 512.  Per pass:
//   * Gram  S^T S = [[S1^T S1, C12], [C12^T, S2^T S2]]: the real Gram kernel on each block and
//     the cross block C12 = S1^T S2 by xgram_kernel (split-m partials, then xreduce_kernel sums
//     the chunks in a fixed order -- deterministic, as the real Gram); zcombine_wide_kernel forms
//     A = X^H X from the three pieces.
//   * TRSM  Q M = S with M = [[M11, M12], [0, M22]] (the real upper-triangular image of R~):
//     Q1 = S1 M11^-1 (real TRSM), S2 := S2 - Q1 M12 (xupdate_kernel), Q2 = S2 M22^-1 (real TRSM).
//     This is block back substitution on each row of S, so the row-wise backward error model of
//     the TRSM carries over with the update's inner products.
// The products are DMMA m8n8k4 (fp64 tensor cores) on 64 x 64 output blocks staged through
// shared memory, 8 warps per CTA each owning an 8 x 64 strip.
#include "scqr3.h"
#include "scqr3_dev.cuh"
#include "scqr3_kernels.h"

namespace scqr3 {

namespace {
constexpr int kXThreads = 256;
constexpr int kXRows = 32;      // rows of S per stage (xgram: the contraction index)
constexpr int kXLd = kXRows + 4;  // column stride of a staged block (doubles): conflict-free fragments
constexpr int kUK = 32;         // contraction columns per stage (xupdate)
constexpr int kULd = 64 + 4;    // row-block stride of the staged Q1 slab (doubles)
}  // namespace

// partials[c][i + j p] = sum over the rows of chunk c of S1(r, i) S2(r, j), i < p, j < q.
// Grid: chunks x nbp x nbq CTAs (the blocks of one chunk adjacent, so they share its rows in L2).
__global__ void __launch_bounds__(kXThreads) xgram_kernel(const double* __restrict__ A, long long lda,
                                                          const double* __restrict__ B, long long ldb, long long m,
                                                          int p, int q, long long rows_per_chunk,
                                                          double* __restrict__ partials, PassGate gate) {
  if (SCQR3_GATE_SKIP(gate)) return;
  __shared__ __align__(16) double As[64 * kXLd];
  __shared__ __align__(16) double Bs[64 * kXLd];
  const int nbp = (p + 63) / 64, nbq = (q + 63) / 64;
  const int bj = blockIdx.x % nbq, bi = (blockIdx.x / nbq) % nbp;
  const long long chunk = blockIdx.x / (nbp * nbq);
  const long long r0 = chunk * rows_per_chunk, r1 = min(m, r0 + rows_per_chunk);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int i0 = bi * 64, j0 = bj * 64;
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
  // staging: thread (row lane, columns w + 8 s): 256 contiguous bytes per column per warp
  double av[8], bv[8];
  auto load = [&](long long r) {
    const long long row = r + lane;
    const bool rok = row < r1;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int ci = i0 + w + 8 * s, cj = j0 + w + 8 * s;
      av[s] = rok && ci < p ? __ldg(A + row + ci * lda) : 0.0;
      bv[s] = rok && cj < q ? __ldg(B + row + cj * ldb) : 0.0;
    }
  };
  if (r0 < r1) load(r0);
  for (long long r = r0; r < r1; r += kXRows) {
    __syncthreads();
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      As[(w + 8 * s) * kXLd + lane] = av[s];
      Bs[(w + 8 * s) * kXLd + lane] = bv[s];
    }
    __syncthreads();
    if (r + kXRows < r1) load(r + kXRows);  // next stage in flight during the products
#pragma unroll
    for (int kk = 0; kk < kXRows; kk += 4) {
      const double a = As[(8 * w + g) * kXLd + kk + t];  // A(m = g, k = t) = S1(row kk + t, col 8w + g)
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma(acc[j][0], acc[j][1], a, Bs[(8 * j + g) * kXLd + kk + t]);
    }
  }
  double* out = partials + chunk * static_cast<long long>(p) * q;
  const int i = i0 + 8 * w + g;
  if (i < p) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = j0 + 8 * j + 2 * t + e;
        if (c < q) out[i + static_cast<long long>(c) * p] = acc[j][e];
      }
  }
}

// out[k] = sum_c partials[c][k], c ascending (fixed order: the same bits run to run)
__global__ void xreduce_kernel(const double* __restrict__ partials, int chunks, long long count,
                               double* __restrict__ out, PassGate gate) {
  if (SCQR3_GATE_SKIP(gate)) return;
  for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < count;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < chunks; ++c) s += partials[c * count + k];
    out[k] = s;
  }
}

// S2(i, j) -= sum_{k < p} Q1(i, k) M12(k, j) for i < m, j < q.  Grid: ceil(m / 64) x nbq CTAs
// (the column blocks of one row block adjacent: they share its Q1 rows in L2).
__global__ void __launch_bounds__(kXThreads) xupdate_kernel(const double* __restrict__ Q1, long long ldq,
                                                            const double* __restrict__ M12, long long ldm,
                                                            double* __restrict__ S2, long long lds, long long m,
                                                            int p, int q, PassGate gate) {
  if (SCQR3_GATE_SKIP(gate)) return;
  __shared__ __align__(16) double Qs[kUK * kULd];   // [k][row]
  __shared__ __align__(16) double Ms[64 * kXLd];    // [col][k]
  const int nbq = (q + 63) / 64;
  const int bj = blockIdx.x % nbq;
  const long long rb = blockIdx.x / nbq;
  const long long i0 = rb * 64;
  const int j0 = bj * 64;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
  const int qrow = tid & 63, qk = tid >> 6;  // Q1 staging: row qrow, columns qk + 4 s
  double qv[8], mv[8];
  auto load = [&](int k0) {
    const long long row = i0 + qrow;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int k = k0 + qk + 4 * s;
      qv[s] = row < m && k < p ? __ldg(Q1 + row + k * ldq) : 0.0;
      const int c = j0 + w + 8 * s, km = k0 + lane;
      mv[s] = c < q && km < p ? __ldg(M12 + km + c * ldm) : 0.0;
    }
  };
  load(0);
  for (int k0 = 0; k0 < p; k0 += kUK) {
    __syncthreads();
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      Qs[(qk + 4 * s) * kULd + qrow] = qv[s];
      Ms[(w + 8 * s) * kXLd + lane] = mv[s];
    }
    __syncthreads();
    if (k0 + kUK < p) load(k0 + kUK);
#pragma unroll
    for (int kk = 0; kk < kUK; kk += 4) {
      const double a = Qs[(kk + t) * kULd + 8 * w + g];  // A(m = g, k = t) = Q1(row 8w + g, col kk + t)
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma(acc[j][0], acc[j][1], a, Ms[(8 * j + g) * kXLd + kk + t]);
    }
  }
  const long long i = i0 + 8 * w + g;
  if (i < m) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = j0 + 8 * j + 2 * t + e;
        if (c < q) {
          double* d = S2 + i + static_cast<long long>(c) * lds;
          *d = *d - acc[j][e];
        }
      }
  }
}

// out (nr x nc, column-major, ld nr) = M(r0 : r0 + nr, c0 : c0 + nc) (column-major, ld ldm)
__global__ void zsub_kernel(const double* __restrict__ M, long long ldm, int r0, int c0, int nr, int nc,
                            double* __restrict__ out, PassGate gate) {
  if (SCQR3_GATE_SKIP(gate)) return;
  const long long total = static_cast<long long>(nr) * nc;
  for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(k % nr), j = static_cast<int>(k / nr);
    out[k] = M[(r0 + i) + static_cast<long long>(c0 + j) * ldm];
  }
}

// A = X^H X (n x n complex, column-major interleaved) from the split Gram's pieces: packed upper
// 8 x 8 tiles of S1^T S1 (t1) and S2^T S2 (t2), and C12 = S1^T S2 (h x (2n - h), column-major).
// Split column 2j is Re x_j, 2j + 1 is Im x_j; A_jl = G_2j,2l + G_2j+1,2l+1 + i (G_2j,2l+1 - G_2j+1,2l).
__global__ void zcombine_wide_kernel(const double* __restrict__ t1, const double* __restrict__ t2,
                                     const double* __restrict__ c12, int n, int h, double* __restrict__ A,
                                     const int* last_pass, int pass) {
  if (last_pass && pass > *(volatile const int*)last_pass) return;
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= static_cast<long long>(n) * n) return;
  const int j = static_cast<int>(k % n), l = static_cast<int>(k / n);
  auto tile = [](const double* t, int a, int b) {  // a <= b
    return t[(static_cast<size_t>(b >> 3) * ((b >> 3) + 1) / 2 + (a >> 3)) * 64 + 8 * (a & 7) + (b & 7)];
  };
  auto G = [&](int a, int b) -> double {  // symmetric 2n x 2n entry
    if (a > b) {
      const int s = a;
      a = b;
      b = s;
    }
    if (b < h) return tile(t1, a, b);
    if (a >= h) return tile(t2, a - h, b - h);
    return c12[a + static_cast<size_t>(b - h) * h];
  };
  const int p = j <= l ? j : l, q = j <= l ? l : j;  // the upper entry (p, q); A_lj = conj(A_jl)
  const double re = G(2 * p, 2 * q) + G(2 * p + 1, 2 * q + 1);
  const double im = p == q ? 0.0 : G(2 * p, 2 * q + 1) - G(2 * p + 1, 2 * q);
  A[2 * k] = re;
  A[2 * k + 1] = j <= l ? im : -im;
}

}  // namespace scqr3
