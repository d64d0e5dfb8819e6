// chol.cu -- the per-pass n x n step (a3 norm/shift, a4 shifted Cholesky, a7 pass control) on
// ONE CTA, replicated on every rank (identical input bits after the Gram allreduce give identical
// R~, so no broadcast is needed), plus the R accumulation (a6) kernels that run on a side
// stream, overlapped with the TRSM of the same pass.
//
//   N^2 ~ ||Q||_2^2 by power iteration on the Gram (reading D2), or trace / user bound
//   s = 11{mn+n(n+1)} u N^2              (eq. finds2)
//   s = 11{2m sqrt(mn)+n(n+1)} u N^2 N_B (eq. finds2B, oblique)
//   pass 1: R~ = chol(A + sI)            (Alg. 3 line 4)
//   pass k>1: R~ = chol(A); on breakdown R~ = chol(A + sI)   (Alg. 2 lines 4-7)
//   R := R~ R                              (Alg. 2 line 8)   [trmul_kernel]
//   stop after an unshifted pass with ||A - I||_F <= stop_tol (reading D6)
// Breakdown = first pivot <= 0 or non-finite, in pivot order (reading D9).  The norm estimate is
// only needed when a shift is formed (pass 1, or a pass whose plain Cholesky broke down).
//
// Cholesky: right-looking with 8-column panels on a row-major working copy W of A (leading
// dimension n + 4; shared memory for n <= 157, else an L2-resident global scratch).  Per panel:
// ONE thread factors the 8x8 diagonal block in registers (pivot chain rsqrt -> scale -> FMA, no
// shuffle or barrier in it); the panel's rows of R~ by forward substitution, one thread per
// column; the rank-8 trailing update.  n % 8 == 0: the update as 8x8 tiles on DMMA, and one
// barrier per panel -- warp 1 updates the next row block, warp 0 the next diagonal tile, whose
// block lane 0 factors, warps 0, 1, 4 form the next panel's rows behind a named barrier, while
// warps 2, 3, 5, 6, 7 update the rest (panel k+1 is ready when the barrier releases panel k's
// update).  Otherwise three barriers per panel and scalar 4x4 register tiles.  Outputs for the
// TRSM kernel: -R~ in mma B-fragment order, and for each 8x8 diagonal block the strict upper part
// scaled by its row's reciprocal pivot plus the reciprocal pivots; R~ itself for trmul_kernel.
// n in (128, 256]: pass 1's power iteration runs before this kernel on a cluster of 8 CTAs
// (power_cluster_kernel).
#include <math.h>

#include <type_traits>

#include "scqr3.h"
#include "scqr3_dev.cuh"
#include "scqr3_kernels.h"

namespace scqr3 {

namespace {
constexpr int kThreads = 256;
// 8-column panels: the diagonal block (36 doubles) fits one thread's registers, and the
// unrolled code of a panel step stays resident in the instruction caches.
constexpr int kPanel = 8;
constexpr unsigned kFull = 0xffffffffu;
__device__ long long g_phase[2];  // diagnostics: cycles in panel steps (a) and (b) of the last factor

__device__ __forceinline__ double2 block_sum2(double a, double b, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(kFull, a, o);
    b += __shfl_down_sync(kFull, b, o);
  }
  __syncthreads();  // protect red[] from a previous use
  if (lane == 0) {
    red[warp] = a;
    red[32 + warp] = b;
  }
  __syncthreads();
  double sa = 0.0, sb = 0.0;
  for (int w = 0; w < kThreads / 32; ++w) {  // same order in every thread: deterministic
    sa += red[w];
    sb += red[32 + w];
  }
  return make_double2(sa, sb);
}

__device__ __forceinline__ double gram_entry(const CholParams& p, int i, int j) {
  const int a = i <= j ? i : j, b = i <= j ? j : i;
  if (p.mode == CHOL_ONLY) return p.Afull[a + static_cast<size_t>(b) * p.n];
  const size_t tile = static_cast<size_t>(b >> 3) * ((b >> 3) + 1) / 2 + (a >> 3);
  return p.tiles[tile * 64 + 8 * (a & 7) + (b & 7)];
}

// Packed upper tile index -> tile column TJ (tile (TI, TJ) sits at TJ(TJ+1)/2 + TI).
__device__ __forceinline__ int tile_col(int tile) {
  int TJ = static_cast<int>((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
  while ((TJ + 1) * (TJ + 2) / 2 <= tile) ++TJ;
  while (TJ * (TJ + 1) / 2 > tile) --TJ;
  return TJ;
}

// tiles: packed upper Gram tiles to load (default: the pass's Gram, p.tiles).  With acc set,
// also returns this thread's share of the stop-test sums: sum over all (i, j) of (A_ij - delta_ij)^2
// (off-diagonal entries counted twice, once per triangle) and of the diagonal (the trace).
__device__ __forceinline__ void load_W(const CholParams& p, double* W, int ldw, const double* tiles = nullptr,
                                       double* acc_dev = nullptr, double* acc_tr = nullptr) {
  const int n = p.n;
  if (!tiles) tiles = p.tiles;
  double dv = 0.0, tr = 0.0;
  if (p.mode == CHOL_ONLY) {
    for (int i = threadIdx.x >> 5; i < n; i += kThreads / 32)
      for (int j = threadIdx.x & 31; j < n; j += 32) W[i * ldw + j] = gram_entry(p, i, j);
  } else {
    // read the packed tiles linearly, 16 bytes per load (two columns of one tile row) and eight
    // loads in flight per thread, and place each upper element at (i, j) and (j, i): the same
    // values gram_entry gives, without its scattered reads.  A thread's pair index e2 walks the
    // tiles in order, so its tile column follows from the previous one (no sqrt per element).
    const int ne2 = p.NT * (p.NT + 1) / 2 * 32;  // element pairs
    constexpr int kU = 8;
    // (the oblique plain Gram follows the B-Gram and ||Q||_F^2: 8-byte aligned only)
    const bool al16 = (reinterpret_cast<uintptr_t>(tiles) & 15) == 0;
    int TJ = 0, tbase = 0;  // tile column of the current tile and index of its first tile
    for (int e0 = threadIdx.x; e0 < ne2; e0 += kU * kThreads) {
      double2 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e2 = e0 + u * kThreads;
        if (e2 >= ne2) v[u] = make_double2(0.0, 0.0);
        else if (al16) v[u] = reinterpret_cast<const double2*>(tiles)[e2];
        else v[u] = make_double2(tiles[2 * e2], tiles[2 * e2 + 1]);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e2 = e0 + u * kThreads;
        if (e2 >= ne2) continue;
        const int tile = e2 >> 5, r = (e2 >> 2) & 7, c = 2 * (e2 & 3);
        while (tbase + TJ + 1 <= tile) tbase += ++TJ;  // tiles only grow along a thread's walk
        const int TI = tile - tbase;
        const int i = 8 * TI + r, j0 = 8 * TJ + c;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = j0 + h;
          const double x = h ? v[u].y : v[u].x;
          if (TI == TJ && r > c + h) continue;  // a diagonal tile's upper half serves both triangles
          if (i < n && j < n) {
            W[i * ldw + j] = x;
            W[j * ldw + i] = x;
            if (i == j) {
              tr += x;
              dv = fma(x - 1.0, x - 1.0, dv);
            } else {
              dv = fma(2.0 * x, x, dv);
            }
          }
        }
      }
    }
  }
  if (acc_dev) *acc_dev = dv;
  if (acc_tr) *acc_tr = tr;
  __syncthreads();
}

// Power iteration from the all-ones vector on sc*A (sc = exact power of two with sc*trace <= 1,
// so the unnormalised iterates neither overflow nor need a reduction per step), then the
// Rayleigh quotient.  Same iterate directions as the normalised iteration (reading D2).
// (SMEM: W is the dynamic shared-memory array -- addressed as such so loads are LDS.)
template <bool SMEM>
__device__ __noinline__ double power_lmax(const double* Wg, int ldw, int n, int iters, double trace,
                                          double (*ybuf)[kMaxN + 64], double* red) {
  extern __shared__ double smdyn[];
  const double* W = SMEM ? smdyn : Wg;
  if (!(trace > 0.0) || !isfinite(trace)) return 0.0;
  const double sc = ldexp(1.0, -(ilogb(trace) + 1));
  int tpr = 1;
  while (tpr * 2 <= 32 && tpr * 2 * n <= kThreads) tpr *= 2;
  const int tid = threadIdx.x, part = tid % tpr, rstep = kThreads / tpr;  // rows strided when n > kThreads
  for (int i = tid; i < n; i += kThreads) ybuf[0][i] = 1.0;
  __syncthreads();
  // this thread's share of (W y)_row: four independent FMA chains, eight loads in flight
  auto rowdot = [&](int row, const double* y) -> double {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (row >= n) return 0.0;
    int j = part;
    if (n < 32 * tpr) {  // short rows (n <= 64): one chain is faster (measured)
      for (; j < n; j += tpr) a0 = fma(W[j * ldw + row], y[j], a0);
      return a0;
    }
#pragma unroll 2
    for (; j + 3 * tpr < n; j += 4 * tpr) {
      a0 = fma(W[j * ldw + row], y[j], a0);
      a1 = fma(W[(j + tpr) * ldw + row], y[j + tpr], a1);
      a2 = fma(W[(j + 2 * tpr) * ldw + row], y[j + 2 * tpr], a2);
      a3 = fma(W[(j + 3 * tpr) * ldw + row], y[j + 3 * tpr], a3);
    }
    for (; j < n; j += tpr) a0 = fma(W[j * ldw + row], y[j], a0);
    return (a0 + a1) + (a2 + a3);
  };
  int cur = 0;
  for (int it = 0; it < iters; ++it) {
    for (int r0 = 0; r0 < n; r0 += rstep) {
      const int row = r0 + tid / tpr;
      double acc = rowdot(row, ybuf[cur]);
      for (int o = 1; o < tpr; o <<= 1) acc += __shfl_xor_sync(kFull, acc, o);
      if (part == 0 && row < n) ybuf[cur ^ 1][row] = acc * sc;
    }
    __syncthreads();
    cur ^= 1;
  }
  double num = 0.0, den = 0.0;
  for (int r0 = 0; r0 < n; r0 += rstep) {
    const int row = r0 + tid / tpr;
    double acc = rowdot(row, ybuf[cur]);
    for (int o = 1; o < tpr; o <<= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if (part == 0 && row < n) {
      const double y = ybuf[cur][row];
      num = fma(y, acc, num);
      den = fma(y, y, den);
    }
  }
  const double2 nd = block_sum2(num, den, red);
  return nd.y > 0.0 ? nd.x / nd.y : 0.0;
}

// n <= 128 (W in shared memory): the same iteration with this thread's share of W -- row
// tid / TPR, the CPP contiguous columns part * CPP + k -- held in registers for all iterations,
// so an iteration reads only y: 16-byte loads of consecutive y entries, the TPR parts of a warp
// on different banks (y stored with 2 doubles of skew per part), i.e. one wavefront per load
// (shared-memory wavefronts of the y reads bound the iteration: ~750 cycles with 8-byte loads of
// strided columns at n = 128).  TPR threads per row (the largest power of two <= 32 with
// TPR * n <= 256); CPP >= ceil(n / TPR) a compile-time power of two, so the iteration has no
// branches; columns past n carry zeros.
template <int TPR, int CPP>
__device__ __noinline__ double power_lmax_reg(int ldw, int n, int iters, double trace, double (*ybuf)[kMaxN + 64],
                                              double* red) {
  extern __shared__ double smdyn[];
  const double* W = smdyn;
  if (!(trace > 0.0) || !isfinite(trace)) return 0.0;
  const double sc = ldexp(1.0, -(ilogb(trace) + 1));
  const int tid = threadIdx.x, part = tid % TPR, row = tid / TPR;
  constexpr int kSkew = CPP >= 2 ? 2 : 0;
  auto yix = [](int j) { return j + kSkew * (j / CPP); };  // skewed position of y_j
  double w[CPP];
  const int rc = row < n ? row : n - 1;
#pragma unroll
  for (int k = 0; k < CPP; ++k) {  // (clamped unconditional loads: no branch per element)
    const int j = part * CPP + k;
    const double x = W[(j < n ? j : n - 1) * ldw + rc];
    w[k] = (j < n && row < n) ? x : 0.0;
  }
  for (int i = tid; i < TPR * CPP; i += kThreads) {  // y past n stays 0
    ybuf[0][yix(i)] = i < n ? 1.0 : 0.0;
    ybuf[1][yix(i)] = 0.0;
  }
  __syncthreads();
  auto rowdot = [&](const double* y) -> double {
    constexpr int NC = CPP < 4 ? CPP : 4;  // independent FMA chains
    double a[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) a[c] = 0.0;
    const double* yp = y + part * (CPP + kSkew);
    if constexpr (CPP >= 2) {
#pragma unroll
      for (int k = 0; k < CPP; k += 2) {
        const double2 yy = *reinterpret_cast<const double2*>(yp + k);
        a[k % NC] = fma(w[k], yy.x, a[k % NC]);
        a[(k + 1) % NC] = fma(w[k + 1], yy.y, a[(k + 1) % NC]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < CPP; ++k) a[k % NC] = fma(w[k], yp[k], a[k % NC]);
    }
    double acc = a[0];
#pragma unroll
    for (int c = 1; c < NC; ++c) acc += a[c];
#pragma unroll
    for (int o = 1; o < TPR; o <<= 1) acc += __shfl_xor_sync(kFull, acc, o);
    return acc;
  };
  int cur = 0;
  for (int it = 0; it < iters; ++it) {
    const double acc = rowdot(ybuf[cur]);
    if (part == 0 && row < n) ybuf[cur ^ 1][yix(row)] = acc * sc;
    __syncthreads();
    cur ^= 1;
  }
  double num = 0.0, den = 0.0;
  const double acc = rowdot(ybuf[cur]);
  if (part == 0 && row < n) {
    const double y = ybuf[cur][yix(row)];
    num = fma(y, acc, num);
    den = fma(y, y, den);
  }
  const double2 nd = block_sum2(num, den, red);
  return nd.y > 0.0 ? nd.x / nd.y : 0.0;
}

// lambda_max estimate of the n x n Gram in W (reading D2): register version for n <= 128
template <bool SMEM>
__device__ double power_lmax_any(const double* W, int ldw, int n, int iters, double trace, double (*ybuf)[kMaxN + 64],
                                 double* red) {
  if (SMEM && n <= 128) {
    if (n > 64) return power_lmax_reg<2, 64>(ldw, n, iters, trace, ybuf, red);
    if (n > 32) return power_lmax_reg<4, 16>(ldw, n, iters, trace, ybuf, red);
    if (n > 16) return power_lmax_reg<8, 4>(ldw, n, iters, trace, ybuf, red);
    if (n > 8) return power_lmax_reg<16, 1>(ldw, n, iters, trace, ybuf, red);
    return power_lmax_reg<32, 1>(ldw, n, iters, trace, ybuf, red);
  }
  return power_lmax<SMEM>(W, ldw, n, iters, trace, ybuf, red);
}

// Blocked right-looking Cholesky of W (+ s on the diagonal).  Returns 0, or the 1-based
// breakdown pivot (value in *pv_out).  On success the upper triangle of W holds R~.
// (__noinline__: one copy of this heavily unrolled code instead of one per call site keeps the
//  kernel's instruction footprint small enough for the instruction caches.)
template <bool SMEM>
__device__ __noinline__ int factor(double* Wg, int ldw, int n, double s, bool add_shift, double* pv_out,
                                   int* sflag, double* sval, double* rinv) {
  extern __shared__ double smdyn[];
  double* W = SMEM ? smdyn : Wg;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (add_shift)
    for (int i = tid; i < n; i += kThreads) W[i * ldw + i] = W[i * ldw + i] + s;
  __syncthreads();
  long long t_a = 0, t_b = 0, t0 = 0;
  // (a) diagonal block on ONE thread, entirely in registers (identity beyond kb): the pivot
  // chain is rsqrt -> scale -> one FMA per column, with no shuffle or barrier in it, and the
  // rest of each rank-1 update is independent work that fills the rsqrt latency.
  // (FULL: kb == 8 known at compile time, so the per-entry kb guards vanish from the chain)
  auto diag_block_t = [&](int k0, int kb_rt, auto full_tag) {
    constexpr bool FULL = decltype(full_tag)::value;
    const int kb = FULL ? kPanel : kb_rt;
    {
      double a[kPanel][kPanel];
#pragma unroll
      for (int r = 0; r < kPanel; ++r)
#pragma unroll
        for (int j = r; j < kPanel; ++j)
          a[r][j] = (j < kb) ? W[(k0 + r) * ldw + k0 + j] : (r == j ? 1.0 : 0.0);
      int bad = 0;
      double badv = 0.0;
#pragma unroll
      for (int c = 0; c < kPanel; ++c) {
        double d = a[c][c];
        if (c < kb && !bad && (!(d > 0.0) || !isfinite(d))) {
          bad = c + 1;
          badv = d;
        }
        if (bad) d = 1.0;  // finish harmlessly; the factor is discarded
        const double inv = rsqrt(d);
        a[c][c] = d * inv;  // r_cc
#pragma unroll
        for (int j = c + 1; j < kPanel; ++j) a[c][j] *= inv;  // r_cj
#pragma unroll
        for (int i = c + 1; i < kPanel; ++i)
#pragma unroll
          for (int j = i; j < kPanel; ++j) a[i][j] = fma(-a[c][i], a[c][j], a[i][j]);
        rinv[c] = inv;
      }
      if (!bad) {
#pragma unroll
        for (int r = 0; r < kPanel; ++r)
#pragma unroll
          for (int j = r; j < kPanel; ++j)
            if (j < kb) W[(k0 + r) * ldw + k0 + j] = a[r][j];
      } else {
        *sflag = k0 + bad;
        *sval = badv;
      }
    }
  };
  auto diag_block = [&](int k0, int kb) {
    if (kb == kPanel) diag_block_t(k0, kb, std::integral_constant<bool, true>{});
    else diag_block_t(k0, kb, std::integral_constant<bool, false>{});
  };
  // (b) rows k0..k0+7 of R~ right of the diagonal block: forward substitution per column, for
  // the columns jj = start, start + stride, ... (full 8-column panel)
  // Rows k0..k0+7 of R~ as read by the rank-8 updates: W itself when W is in shared memory;
  // with W in global memory, a shared-memory copy written by panel_rows (two buffers: panel k's
  // rows are read by the trailing update while panel k+1's are formed), so the mma fragment loads
  // of the updates do not go to L2.
  extern __shared__ double smdyn_p[];
  auto prow = [&](int k0, int r) -> double* {
    if constexpr (SMEM) return W + (k0 + r) * ldw;
    else return smdyn_p + (((k0 / kPanel) & 1) * kPanel + r) * ldw;
  };
  auto panel_rows = [&](int k0, int start, int stride) {
    const int ncols = n - k0 - kPanel;
    for (int jj = start; jj < ncols; jj += stride) {
      const int j = k0 + kPanel + jj;
      double w[kPanel];
#pragma unroll
      for (int r = 0; r < kPanel; ++r) w[r] = W[(k0 + r) * ldw + j];
#pragma unroll
      for (int r = 0; r < kPanel; ++r) {
        const double v = w[r] * rinv[r];
        w[r] = v;
#pragma unroll
        for (int l = r + 1; l < kPanel; ++l) w[l] = fma(-W[(k0 + r) * ldw + k0 + l], v, w[l]);
      }
#pragma unroll
      for (int r = 0; r < kPanel; ++r) W[(k0 + r) * ldw + j] = w[r];
      if constexpr (!SMEM) {
#pragma unroll
        for (int r = 0; r < kPanel; ++r) prow(k0, r)[j] = w[r];
      }
    }
  };
  // n a multiple of 8: one barrier per panel.  While warps 1..7 apply panel k's rank-8 update to
  // the trailing tiles below the next row block, warp 0 updates that row block (tiles (k+1, J)),
  // lane 0 factors its diagonal block, and the warp's lanes form its rows of R~ -- so panel k+1
  // is complete when the barrier releases the update by panel k+1.  (Same operations in the
  // same order on every entry as the three-barrier form below.)
  if ((n & 7) == 0) {
    if (tid == 0) diag_block(0, kPanel);
    __syncthreads();
    if (*sflag) {
      *pv_out = *sval;
      return *sflag;
    }
    panel_rows(0, tid, kThreads);
    __syncthreads();
    const int g = lane >> 2, t = lane & 3;
    long long ph[4] = {0, 0, 0, 0}, tq = 0;  // diagnostics (warp 0: diag tile + block, rows; warp 1: row block; warp 2: update)
    // roles per panel (warp w runs on SM sub-partition w % 4): warp 0 (alone on sub-partition 0
    // with the idle warp 4, so no tensor-core work delays its pivot chain) updates the next
    // diagonal tile and lane 0 factors it; warp 1 updates the rest of the next row block; warps
    // 0, 1, 4 then form that row block's rows of R~; warps 2, 3, 5, 6, 7 update the other tiles
    auto update_tile = [&](int k0, int base, int I, int J) {  // C_IJ -= P_I^T P_J (trailing coords)
      double* cp = W + (base + 8 * I + g) * ldw + base + 8 * J + 2 * t;
      double c0 = cp[0], c1 = cp[1], a[2], b[2];
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2) {
        const double* pr = prow(k0, t + 4 * s2) + base;
        a[s2] = pr[8 * I + g];
        b[s2] = -pr[8 * J + g];
      }
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2) dmma(c0, c1, a[s2], b[s2]);
      cp[0] = c0;
      cp[1] = c1;
    };
    for (int k0 = 0; k0 + kPanel < n; k0 += kPanel) {
      const int base = k0 + kPanel, TL = (n - base) >> 3;
      tq = clock64();
      if (warp == 0 || warp == 1 || warp == 4) {
        if (warp == 0) {
          update_tile(k0, base, 0, 0);
          __syncwarp();
          if (lane == 0) diag_block(base, kPanel);
          __syncwarp();
          ph[2] += clock64() - tq;  // (diagnostics: diagonal tile + block, before the wait)
        } else if (warp == 1) {
          // row block tiles (0, J), J >= 1: 4 in flight
          double a[2];
#pragma unroll
          for (int s2 = 0; s2 < 2; ++s2) a[s2] = prow(k0, t + 4 * s2)[base + g];
          for (int J0 = 1; J0 < TL; J0 += 4) {
            double c0[4], c1[4], b[4][2];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int J = min(J0 + u, TL - 1);
              const double* cp = W + (base + g) * ldw + base + 8 * J + 2 * t;
              c0[u] = cp[0];
              c1[u] = cp[1];
#pragma unroll
              for (int s2 = 0; s2 < 2; ++s2) b[u][s2] = -prow(k0, t + 4 * s2)[base + 8 * J + g];
            }
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
              for (int u = 0; u < 4; ++u) dmma(c0[u], c1[u], a[s2], b[u][s2]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (J0 + u < TL) {
                double* cp = W + (base + g) * ldw + base + 8 * (J0 + u) + 2 * t;
                cp[0] = c0[u];
                cp[1] = c1[u];
              }
            }
          }
        }
        asm volatile("bar.sync 1, 96;" ::: "memory");  // warps 0, 1, 4: the row block is updated
        if (warp == 0) ph[0] += clock64() - tq;
        if (warp == 1) ph[1] += clock64() - tq;
        tq = clock64();
        if (!*sflag) panel_rows(base, warp == 0 ? lane : warp == 1 ? 32 + lane : 64 + lane, 96);
      } else {
        // the other trailing tiles (I, J), 1 <= I <= J < TL, J-major; 4 in flight per warp (8
        // with W in global memory: L2 latency)
        constexpr int kU = SMEM ? 4 : 8, kW = 5;
        const int wi = warp < 4 ? warp - 2 : warp - 3;  // 2, 3, 5, 6, 7 -> 0..4
        const int ntiles = TL * (TL - 1) / 2;
        int J = 1, cum = 0;  // tiles of columns < J: cum = J(J-1)/2
        for (int tau0 = wi; tau0 < ntiles; tau0 += kU * kW) {
          double c0[kU], c1[kU], a[kU][2], b[kU][2];
          int off[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int tau = min(tau0 + u * kW, ntiles - 1);
            while (cum + J <= tau) cum += J++;
            const int I = 1 + tau - cum;
            off[u] = (base + 8 * I + g) * ldw + base + 8 * J + 2 * t;
            c0[u] = W[off[u]];
            c1[u] = W[off[u] + 1];
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
              const double* pr = prow(k0, t + 4 * s2) + base;
              a[u][s2] = pr[8 * I + g];
              b[u][s2] = -pr[8 * J + g];
            }
          }
#pragma unroll
          for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
            for (int u = 0; u < kU; ++u) dmma(c0[u], c1[u], a[u][s2], b[u][s2]);
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            if (tau0 + u * kW < ntiles) {
              W[off[u]] = c0[u];
              W[off[u] + 1] = c1[u];
            }
          }
        }
        if (warp == 2) ph[3] += clock64() - tq;
      }
      __syncthreads();
      if (*sflag) {
        *pv_out = *sval;
        return *sflag;
      }
    }
    __shared__ long long sph[4];
    if (threadIdx.x == 0) { sph[0] = ph[0]; sph[2] = ph[2]; }
    if (threadIdx.x == 32) sph[1] = ph[1];
    if (threadIdx.x == 64) sph[3] = ph[3];
    __syncthreads();
    if (threadIdx.x == 0) {
      g_phase[0] = sph[0] + (sph[1] << 32);
      g_phase[1] = sph[3] + (sph[2] << 32);
    }
    return 0;
  }
  // n not a multiple of 8: three barriers per panel, scalar 4x4 register tiles for the update
  for (int k0 = 0; k0 < n; k0 += kPanel) {
    const int kb = min(kPanel, n - k0);
    t0 = clock64();
    if (tid == 0) diag_block(k0, kb);
    __syncthreads();
    t_a += clock64() - t0;
    t0 = clock64();
    if (*sflag) {
      *pv_out = *sval;
      return *sflag;
    }
    const int ncols = n - k0 - kb;
    // (b) rows k0..k0+kb-1 of R~ right of the block: forward substitution per column
    for (int jj = tid; jj < ncols; jj += kThreads) {
      const int j = k0 + kb + jj;
      double w[kPanel];
#pragma unroll
      for (int r = 0; r < kPanel; ++r) w[r] = r < kb ? W[(k0 + r) * ldw + j] : 0.0;
#pragma unroll
      for (int r = 0; r < kPanel; ++r) {
        if (r < kb) {
          const double v = w[r] * rinv[r];
          w[r] = v;
#pragma unroll
          for (int l = r + 1; l < kPanel; ++l)
            if (l < kb) w[l] = fma(-W[(k0 + r) * ldw + k0 + l], v, w[l]);
        }
      }
#pragma unroll
      for (int r = 0; r < kPanel; ++r)
        if (r < kb) W[(k0 + r) * ldw + j] = w[r];
    }
    __syncthreads();
    t_b += clock64() - t0;
    // (c) trailing update W_ij -= sum_r r_ri r_rj over k0+kb <= i <= j.  A warp takes 4 rows
    // (broadcast loads) and 128 columns (lane + 32b: consecutive, conflict-free loads), so each
    // lane keeps a 4x4 register tile.
    const int L = ncols, T4 = (L + 3) >> 2;
    const int base = k0 + kb;
    for (int I = warp; I < T4; I += kThreads / 32) {
      const int i0 = 4 * I;
      for (int jc = i0 & ~31; jc < L; jc += 128) {
        double acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
#pragma unroll
        for (int r = 0; r < kPanel; ++r) {
          if (r < kb) {
            const double* pr = W + (k0 + r) * ldw + base;
            double xi[4], xj[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) xi[a] = (i0 + a < L) ? pr[i0 + a] : 0.0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const int j = jc + lane + 32 * b;
              xj[b] = (j < L) ? pr[j] : 0.0;
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int b = 0; b < 4; ++b) acc[a][b] = fma(xi[a], xj[b], acc[a][b]);
          }
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int i = i0 + a, j = jc + lane + 32 * b;
            if (i < L && j < L && i <= j) W[(base + i) * ldw + base + j] -= acc[a][b];
          }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    g_phase[0] = t_a;
    g_phase[1] = t_b;
  }
  return 0;
}


// Upper-triangular entry (i, j) of R~ padded with the identity past n, read without a branch:
// the (clamped) load is unconditional and the select comes after it, so a loop can keep all its
// loads in flight (a load inside a branch serialises on its latency).
__device__ __forceinline__ double rload(const double* W, int ldw, int n, int i, int j) {
  const int ic = i < n ? i : n - 1, jc = j < n ? j : n - 1;
  const double x = W[ic * ldw + jc];
  return (i < n && j < n) ? (i <= j ? x : 0.0) : (i == j ? 1.0 : 0.0);
}

// Reading D24: the TRSM may apply R~'s 8 x 8 diagonal blocks D_J as products with inverses Y_J
// (one DMMA k-step pair per block on the tensor cores instead of a latency-bound substitution
// chain) when that keeps every row's backward error inside the paper's bound (eq. DeltaRbound,
// P:328-331): ||dR_i||_2 <= gamma_n sqrt(n) ||R~||_2.  Rows of Y_J are computed by substitution
// (y D_J = e_i), so |Y_J D_J - I| <= gamma_8 |Y_J||D_J|, and a row solved as q_J = fl(b_J Y_J)
// satisfies |q_J D_J - b_J| <= 2 gamma_8 |q_J||D_J||Y_J||D_J| (first order): a rank-one
// perturbation of D_J of 2-norm <= 2 gamma_8 mu_J, mu_J = || |D_J||Y_J||D_J| ||_F.  The blocks off
// the diagonal are applied as in substitution (|dR| <= gamma_n |R~_off|).  Hence the guard
//     gamma_n ||R~_off||_F + 2 gamma_8 max_J mu_J  <=  gamma_n sqrt(n) max_j ||R~ e_j||_2
// (the right side <= the paper's bound).  Block-wide (blockDim.x == 256): writes Y_J as DMMA B
// fragments (k-step h, lane l: Y[2(l&3)+h][l>>2]) to dblk + dinv_off(NT) and the flag (1: inverse
// path) to dblk[dflag_off(NT)]; mode SCQR3_TRSM_DIAG_SUBST / _INVERSE forces 0 / 1.
// rp(i, j): R~(i, j) for i <= j < n, 0 below the diagonal, the identity past n.
template <class RP>
__device__ __forceinline__ void trsm_diag_guard(RP rp, int n, int NT, double* dblk, int mode) {
  __shared__ double gred[3][8];
  const int tid = threadIdx.x, lane = tid & 31;
  double mu2max = 0.0;
  for (int x0 = 0; x0 < NT * 8; x0 += 256) {  // thread (J, i): row i of Y_J (uniform trip count)
    const int x = x0 + tid, J = min(x >> 3, NT - 1), i = x & 7;
    double d[8][8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int j = 0; j < 8; ++j) d[k][j] = k <= j ? rp(8 * J + k, 8 * J + j) : 0.0;
    double y[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // y_j = (delta_ij - sum_{i <= l < j} y_l d_lj) / d_jj
      double s = j == i ? 1.0 : 0.0;
#pragma unroll
      for (int l = 0; l < j; ++l) s = l >= i ? fma(-y[l], d[l][j], s) : s;
#ifdef SCQR3_G_RCP
      y[j] = j >= i ? s * (1.0 / d[j][j]) : 0.0;
#else
      y[j] = j >= i ? s / d[j][j] : 0.0;
#endif
    }
    if (x < NT * 8) {
      double* dinv = dblk + dinv_off(NT) + J * 64 + (i & 1) * 32 + (i >> 1);
#pragma unroll
      for (int j = 0; j < 8; ++j) dinv[4 * j] = y[j];
    }
    double tr[8];  // row i of |Y||D|
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double v = 0.0;
#pragma unroll
      for (int k = 0; k <= j; ++k) v += fabs(y[k]) * fabs(d[k][j]);
      tr[j] = v;
    }
    // row i of M = |D| |Y||D| (rows k >= i of |Y||D| from the group's lanes); past n excluded
#ifdef SCQR3_G_NOMU
    if (x < NT * 8) mu2max = fmax(mu2max, tr[7]);
    continue;
#endif
    double di[8];  // row i of |D_J| (a runtime row index into d[][] would go to local memory)
#pragma unroll
    for (int k = 0; k < 8; ++k) di[k] = k >= i ? fabs(rp(8 * J + i, 8 * J + k)) : 0.0;
    double mu2 = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double v = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double tk = __shfl_sync(0xffffffffu, tr[j], (lane & ~7) | k);
        v += di[k] * tk;
      }
      if (8 * J + i < n && 8 * J + j < n) mu2 += v * v;
    }
    mu2 += __shfl_xor_sync(0xffffffffu, mu2, 1);
    mu2 += __shfl_xor_sync(0xffffffffu, mu2, 2);
    mu2 += __shfl_xor_sync(0xffffffffu, mu2, 4);
    if (x < NT * 8) mu2max = fmax(mu2max, mu2);
  }
  // ||R~ e_j||_2^2 per column and ||R~_off||_F^2: warp w sums the rows i = w, w + 8, ... of the
  // columns j = j0 + lane (coalesced for row-major R~, loads independent); the warps' partials of
  // a column are added in warp order (the flag is a deterministic function of R~)
  __shared__ double gpart[8][32];
  const int warp = tid >> 5;
  double off2 = 0.0, col2max = 0.0;
#ifdef SCQR3_G_NOCOL
  for (int j0 = 0; j0 < 0; j0 += 32) {
#else
  for (int j0 = 0; j0 < n; j0 += 32) {
#endif
    const int j = j0 + lane, iend = min(j0 + 32, n);
    double c = 0.0;
#pragma unroll 4
    for (int i = warp; i < iend; i += 8) {
      const double r = (j < n && i <= j) ? rp(i, j) : 0.0;
      c = fma(r, r, c);
      off2 = (i >> 3) != (j >> 3) ? fma(r, r, off2) : off2;
    }
    gpart[warp][lane] = c;
    __syncthreads();
    if (warp == 0) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += gpart[w][lane];
      col2max = fmax(col2max, t);
    }
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mu2max = fmax(mu2max, __shfl_xor_sync(0xffffffffu, mu2max, o));
    off2 += __shfl_xor_sync(0xffffffffu, off2, o);
    col2max = fmax(col2max, __shfl_xor_sync(0xffffffffu, col2max, o));
  }
  if (lane == 0) {
    gred[0][tid >> 5] = mu2max;
    gred[1][tid >> 5] = off2;
    gred[2][tid >> 5] = col2max;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, b = 0.0, c = 0.0;
    for (int w = 0; w < 8; ++w) {
      a = fmax(a, gred[0][w]);
      b += gred[1][w];
      c = fmax(c, gred[2][w]);
    }
    constexpr double u = 1.1102230246251565e-16;  // 2^-53 (D1)
    const double g8 = 8.0 * u / (1.0 - 8.0 * u), gn = n * u / (1.0 - n * u);
    const double lhs = gn * sqrt(b) + 2.0 * g8 * sqrt(a);
    const double rhs = gn * sqrt(static_cast<double>(n)) * sqrt(c);
    const bool ok = lhs <= rhs;  // false on NaN
    dblk[dflag_off(NT)] = mode == SCQR3_TRSM_DIAG_INVERSE ? 1.0 : mode == SCQR3_TRSM_DIAG_SUBST ? 0.0 : (ok ? 1.0 : 0.0);
    dblk[dflag_off(NT) + 1] = lhs / rhs;
  }
  __syncthreads();
}

// Outputs of a pass.  R~ for trmul_kernel and trsm_prep_kernel, row-major (Rt[i n + j], zero
// below the diagonal): consecutive threads read consecutive entries of a row of W (no bank
// conflicts in shared memory, coalesced from L2 when W is global) and store consecutive
// addresses.  The TRSM operands -- B fragments of -R~ and the scaled diagonal blocks, the same
// values trsm_prep_kernel forms -- are written here only when bfrag != null (n <= 32, and the
// unfused n <= 64, where a second launch costs more than it saves); for larger n trsm_prep_kernel forms them on many
// CTAs (on this one CTA they took 13 K cycles at n = 128 and 73 K at n = 256) and runs the D24
// guard.
template <bool SMEM>
__device__ __noinline__ void write_outputs(const double* Wg, int ldw, int n, int NT, double* bfrag, double* dblk,
                                           double* Rt, int diag_mode) {
  (void)diag_mode;  // no inverse-diagonal instance runs for these n (flag 0 below)
  extern __shared__ double smdyn[];
  const double* W = SMEM ? smdyn : Wg;
  constexpr int kU = 8;
#ifdef SCQR3_CHOL_OUTCLK
  long long o0 = clock64();
#endif
  if (bfrag) {
    const int nf = NT * (NT - 1) * 32;  // fragment f = idx / 32: target block J >= 1, k-step s < 2J
    for (int i0 = threadIdx.x; i0 < nf; i0 += kU * kThreads) {
      double v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int idx = min(i0 + u * kThreads, nf - 1);
        const int f = idx >> 5, lane = idx & 31;
        int J = static_cast<int>((1.0f + sqrtf(1.0f + 4.0f * f)) * 0.5f);  // largest J with J(J-1) <= f
        J -= J * (J - 1) > f ? 1 : 0;
        J += (J + 1) * J <= f ? 1 : 0;
        const int s = f - J * (J - 1);
        v[u] = -rload(W, ldw, n, 8 * (s >> 1) + 2 * (lane & 3) + (s & 1), 8 * J + (lane >> 2));
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (i0 + u * kThreads < nf) bfrag[i0 + u * kThreads] = v[u];
    }
    for (int idx = threadIdx.x; idx < NT * 72; idx += kThreads) {
      const int J = idx / 72, w = idx % 72;
      const int c = 8 * J + (w < 64 ? (w >> 3) : w - 64), j = 8 * J + (w < 64 ? (w & 7) : w - 64);
      const double rcj = rload(W, ldw, n, c, j), rcc = rload(W, ldw, n, c, c);
      dblk[idx] = w < 64 ? (j > c ? rcj / rcc : 0.0) : 1.0 / rcc;
    }
    // (called for n <= 32 and the unfused n <= 64, which have no inverse-diagonal TRSM instance:
    //  the D24 flag is 0; trsm_prep_kernel forms the operands and runs the guard otherwise)
    if (threadIdx.x == 0) {
      dblk[dflag_off(NT)] = 0.0;
      dblk[dflag_off(NT) + 1] = 0.0;
    }
  }
#ifdef SCQR3_CHOL_OUTCLK
  long long o1 = clock64();
#endif
  const int nn = n * n;
  for (int i0 = threadIdx.x; i0 < nn; i0 += kU * kThreads) {
    double v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int idx = min(i0 + u * kThreads, nn - 1);
      const int i = idx / n, j = idx - i * n;
      const double x = W[i * ldw + j];
      v[u] = i <= j ? x : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i0 + u * kThreads < nn) Rt[i0 + u * kThreads] = v[u];
  }
#ifdef SCQR3_CHOL_OUTCLK
  if (threadIdx.x == 0) {
    g_phase[0] = o1 - o0;
    g_phase[1] = clock64() - o1;
  }
#endif
}

template <bool SMEM>
__device__ __forceinline__ void chol_body(const CholParams& p, double* smW) {
  // pass number: a kernel parameter, or (CUDA-graph loop body) a device counter
  const int pass = p.pass_dev ? *(volatile const int*)p.pass_dev : p.pass;
  if (p.last_pass && pass > *(volatile const int*)p.last_pass) return;  // a pass after the stop
  __shared__ double red[64];
  __shared__ __align__(16) double ybuf[2][kMaxN + 64];
  __shared__ double rinv[kPanel];
  __shared__ int sflag;
  __shared__ double sval;
  const int n = p.n, tid = threadIdx.x;
  const int ldw = chol_ldw(n);
  double* W = SMEM ? smW : p.W;
  long long clk[8] = {};
  clk[0] = clock64();
  if (tid == 0) sflag = 0;
  double loc = 0.0, tr = 0.0;  // a7 input: ||A - I||_F^2 and trace(A) shares (stop test, reading D6)
  load_W(p, W, ldw, nullptr, &loc, &tr);
  clk[1] = clock64();

  if (p.mode == CHOL_ONLY) {
    double pv = 0.0;
    const int piv = factor<SMEM>(W, ldw, n, p.shift_value, p.shift_value != 0.0, &pv, &sflag, &sval, rinv);
    for (int j = tid >> 5; j < n; j += kThreads / 32)
      for (int i = tid & 31; i < n; i += 32)
        p.R[i + static_cast<size_t>(j) * n] = (piv == 0 && i <= j) ? W[i * ldw + j] : 0.0;
    if (tid == 0) {
      DevStatus st{};
      st.code = piv ? SCQR3_EBREAKDOWN : SCQR3_OK;
      st.breakdown_pivot = piv;
      st.pivot_value = pv;
      st.shift = p.shift_value;
      *p.st_dev = st;
    }
    return;
  }

  const double2 dt = block_sum2(loc, tr, red);
  const double dev = sqrt(dt.x), trace = dt.y;
  clk[2] = clock64();
  if (pass == 1 && !isfinite(trace)) {
    // non-finite entries in X (every NaN / Inf reaches the trace of its Gram): an invalid
    // argument, reported before any factorisation
    if (tid == 0) {
      DevStatus st{};
      st.code = SCQR3_EINVAL;
      st.pass = pass;
      st.dev_F = dev;
      *p.st_dev = st;
      if (p.last_pass) *(volatile int*)p.last_pass = 0;
      if (p.st_host) {
        volatile DevStatus* h = p.st_host;
        h->pass = st.pass;
        h->dev_F = st.dev_F;
        h->code = st.code;
      }
    }
    return;
  }

  // ---- a3: norm estimate and shift, only when a shift is formed
  const double u = 0x1p-53;
  const double mg = p.m_global, nn = static_cast<double>(n);
  bool w_plain = false;  // W holds the plain Gram (oblique norm estimate): reload before factoring
  auto shift_for = [&](double& N2) -> double {
    if (p.oblique) {
      const size_t nout = static_cast<size_t>(p.NT) * (p.NT + 1) / 2 * 64;
      const double fro = p.tiles[nout];  // ||Q||_F^2, accumulated with the B-Gram
      if (pass == 1 && p.norm_mode == SCQR3_NORM_USER) {
        N2 = p.norm2_bound * p.norm2_bound;
      } else if (p.norm_mode == SCQR3_NORM_FROBENIUS) {
        N2 = fro;
      } else if (p.lmax_dev && pass == 1) {  // computed by power_cluster_kernel before this kernel
        N2 = *p.lmax_dev * 1.01;
      } else {  // lambda_max(Q^T Q) x 1.01 from the plain Gram formed alongside (reading D4)
        __syncthreads();
        load_W(p, W, ldw, p.tiles + nout + 1);
        N2 = power_lmax_any<SMEM>(W, ldw, n, p.power_iters, fro, ybuf, red) * 1.01;
        w_plain = true;
      }
    } else if (pass == 1 && p.norm_mode == SCQR3_NORM_USER) {
      N2 = p.norm2_bound * p.norm2_bound;
    } else if (p.norm_mode == SCQR3_NORM_FROBENIUS) {
      N2 = trace;
    } else if (p.lmax_dev && pass == 1) {  // computed by power_cluster_kernel before this kernel
      N2 = *p.lmax_dev * 1.01;
    } else {
      N2 = power_lmax_any<SMEM>(W, ldw, n, p.power_iters, trace, ybuf, red) * 1.01;
    }
    if (p.shift_mode == SCQR3_SHIFT_FIXED && pass == 1) return p.shift_value;
    if (p.oblique) return 11.0 * (2.0 * mg * sqrt(mg * nn) + nn * (nn + 1.0)) * u * N2 * (*p.nb_dev);
    return 11.0 * (mg * nn + nn * (nn + 1.0)) * u * N2;
  };

  // ---- a4: (shifted) Cholesky with breakdown-triggered re-shift.  SAFE / FIXED shift pass 1
  // (Alg. 3 line 4); ADAPTIVE tries every pass unshifted first (Alg. 2); PRACTICAL
  // shifts pass 1 with s_p = u N2 (N_B) (Remark P:1600-1606) and falls back to the safe s when
  // chol(A + s_p I) breaks down (reading D21).
  int shifted = 0, bpiv = 0, piv = 1;
  double bval = 0.0, pv = 0.0, s = 0.0, N2 = 0.0;
  const bool practical = p.shift_mode == SCQR3_SHIFT_PRACTICAL;
  const bool shift_first = pass == 1 && (p.shift_mode == SCQR3_SHIFT_SAFE || p.shift_mode == SCQR3_SHIFT_FIXED ||
                                           practical);
  bool w_dirty = false;
  clk[3] = clock64();
  if (!shift_first) {
    piv = factor<SMEM>(W, ldw, n, 0.0, false, &pv, &sflag, &sval, rinv);
    w_dirty = true;
    if (piv) { bpiv = piv; bval = pv; }
  }
  if (piv && p.shift_mode != SCQR3_SHIFT_NONE) {
    const double s_safe = shift_for(N2);
    if (w_plain) w_dirty = true;
    const double s_p = 0x1p-53 * N2 * (p.oblique ? *p.nb_dev : 1.0);
    clk[3] = clock64();
    for (int attempt = practical ? 0 : 1; attempt < 2 && piv; ++attempt) {
      if (w_dirty) {
        __syncthreads();
        if (tid == 0) sflag = 0;
        load_W(p, W, ldw);
      }
      s = attempt == 0 ? s_p : s_safe;
      shifted = 1;
      piv = factor<SMEM>(W, ldw, n, s, true, &pv, &sflag, &sval, rinv);
      w_dirty = true;
      if (piv) { bpiv = piv; bval = pv; }
    }
  }
  const int code = piv ? SCQR3_EBREAKDOWN : SCQR3_OK;
  clk[4] = clock64();
  if (code == SCQR3_OK) write_outputs<SMEM>(W, ldw, n, p.NT, p.bfrag, p.dblk, p.Rt, p.trsm_diag);
  if (tid == 0) {
    DevStatus st{};
    st.code = code;
    st.stop = (code == SCQR3_OK && !shifted && dev <= p.stop_tol) ? 1 : 0;
    st.pass = pass;
    st.shifted = shifted;
    st.shift = shifted ? s : 0.0;
    st.breakdown_pivot = bpiv;
    st.pivot_value = bval;
    st.norm2_est = N2;
    st.dev_F = dev;
    clk[5] = clock64();
    clk[6] = g_phase[0];
    clk[7] = g_phase[1];
    for (int i = 0; i < 8; ++i) st.clk[i] = clk[i];
    *p.st_dev = st;
    if (p.last_pass) {  // device-side pass control: later (speculative) passes become no-ops
      if (st.code != SCQR3_OK) *(volatile int*)p.last_pass = pass - 1;
      else if (st.stop) *(volatile int*)p.last_pass = pass;
    }
    // (host-mapped status slot: the host reads it only after an event recorded behind this
    // kernel has completed, which orders these writes -- no system-scope fence, which cost
    // ~6 us per pass)
    if (p.st_host) {
      volatile DevStatus* h = p.st_host + (p.mode == CHOL_PASS ? pass - 1 : 0);
      h->stop = st.stop;
      h->pass = st.pass;
      h->shifted = st.shifted;
      h->shift = st.shift;
      h->breakdown_pivot = st.breakdown_pivot;
      h->pivot_value = st.pivot_value;
      h->norm2_est = st.norm2_est;
      h->dev_F = st.dev_F;
      h->code = st.code;
    }
  }
}
}  // namespace

// ---- power iteration for n in (128, 256] on a cluster of 8 CTAs (reading D2): the one-CTA
// kernel keeps W in global memory there (it does not fit one SM's shared memory), and its
// power iteration re-read W from L2 every step (~9 us per step at n = 256).  Here CTA r holds
// rows [32 r, 32 r + 32) of the Gram in its shared memory; each step every CTA forms its rows of
// sc * W y and stores them into every CTA's copy of the next y (distributed shared memory),
// then one cluster barrier.  Same iteration as power_lmax (all-ones start, unnormalised
// iterates scaled by the exact power of two sc, Rayleigh quotient) -- the summation order of
// the dot products differs, so the estimate agrees to rounding.
constexpr int kPowCl = 8, kPowRows = 32, kPowThreads = 256;

__device__ __forceinline__ void st_cluster_f64(double* local_addr, uint32_t cta, double v) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(smem_u32(local_addr)), "r"(cta));
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(remote), "d"(v) : "memory");
}

__global__ void __cluster_dims__(kPowCl, 1, 1) __launch_bounds__(kPowThreads, 1) power_cluster_kernel(PowerParams p) {
  extern __shared__ __align__(16) double psm[];
  const int pass = p.pass_dev ? *(volatile const int*)p.pass_dev : p.pass;
  if (p.last_pass && pass > *(volatile const int*)p.last_pass) return;  // (every CTA of the cluster alike)
  const int n = p.n, tid = threadIdx.x;
  const int ldl = ((n + 7) / 16) * 16 + 8;  // = 8 (mod 16): two rows of 8 parts on distinct banks
  const uint32_t r = cluster_ctarank();
  const int row0 = static_cast<int>(r) * kPowRows;
  double* Wl = psm;                                  // [kPowRows][ldl]
  double* y[2] = {Wl + kPowRows * ldl, Wl + kPowRows * ldl + kMaxN};
  double* slots = y[1] + kMaxN;                      // [2][kPowCl]: per-CTA partial sums
  // my rows of the symmetric Gram from its packed upper tiles
  for (int idx = tid; idx < kPowRows * n; idx += kPowThreads) {
    const int ir = idx / n, c = idx % n, i = row0 + ir;
    double v = 0.0;
    if (i < n) {
      const int a = i <= c ? i : c, b = i <= c ? c : i;
      const size_t tile = static_cast<size_t>(b >> 3) * ((b >> 3) + 1) / 2 + (a >> 3);
      v = p.tiles[tile * 64 + 8 * (a & 7) + (b & 7)];
    }
    Wl[ir * ldl + c] = v;
  }
  for (int c = tid; c < kMaxN; c += kPowThreads) y[0][c] = c < n ? 1.0 : 0.0;
  __syncthreads();
  // trace (for the scale sc): every CTA gets all partials, summed in rank order
  if (tid < 32) {
    double t = 0.0;
    for (int ir = tid; ir < kPowRows; ir += 32)
      if (row0 + ir < n) t += Wl[ir * ldl + row0 + ir];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if (tid == 0)
      for (int j = 0; j < kPowCl; ++j) st_cluster_f64(slots + r, static_cast<uint32_t>(j), t);
  }
  cluster_sync();
  double trace = 0.0;
  for (int j = 0; j < kPowCl; ++j) trace += slots[j];
  const bool ok = trace > 0.0 && isfinite(trace);
  const double sc = ok ? ldexp(1.0, -(ilogb(trace) + 1)) : 1.0;
  const int ir = tid / 8, part = tid % 8, i = row0 + ir;
  auto rowdot = [&](const double* yv) -> double {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const double* w = Wl + ir * ldl;
    int c = part;
    for (; c + 24 < n; c += 32) {
      a0 = fma(w[c], yv[c], a0);
      a1 = fma(w[c + 8], yv[c + 8], a1);
      a2 = fma(w[c + 16], yv[c + 16], a2);
      a3 = fma(w[c + 24], yv[c + 24], a3);
    }
    for (; c < n; c += 8) a0 = fma(w[c], yv[c], a0);
    double acc = (a0 + a1) + (a2 + a3);
    for (int o = 1; o < 8; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    return acc;
  };
  int cur = 0;
  for (int it = 0; it < p.iters; ++it) {
    const double acc = rowdot(y[cur]);
    if (part == 0 && i < n) {
      const double v = acc * sc;
      for (int j = 0; j < kPowCl; ++j) st_cluster_f64(y[cur ^ 1] + i, static_cast<uint32_t>(j), v);
    }
    cluster_sync();  // every CTA's next y is complete (and nobody still reads this one)
    cur ^= 1;
  }
  const double acc = rowdot(y[cur]);
  double num = 0.0, den = 0.0;
  if (part == 0 && i < n) {
    const double yi = y[cur][i];
    num = yi * acc;
    den = yi * yi;
  }
  // CTA partials (fixed order) -> CTA 0, which sums them in rank order
  for (int o = 8; o < 32; o <<= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
  }
  __shared__ double wsum[2][kPowThreads / 32];
  if ((tid & 31) == 0) {
    wsum[0][tid >> 5] = num;
    wsum[1][tid >> 5] = den;
  }
  __syncthreads();
  if (tid == 0) {
    double sn = 0.0, sd = 0.0;
    for (int w = 0; w < kPowThreads / 32; ++w) {
      sn += wsum[0][w];
      sd += wsum[1][w];
    }
    st_cluster_f64(slots + kPowCl + r, 0u, sn);
    st_cluster_f64(slots + 2 * kPowCl + r, 0u, sd);
  }
  cluster_sync();
  if (r == 0 && tid == 0) {
    double sn = 0.0, sd = 0.0;
    for (int j = 0; j < kPowCl; ++j) {
      sn += slots[kPowCl + j];
      sd += slots[2 * kPowCl + j];
    }
    *p.out = (ok && sd > 0.0) ? sn / sd : 0.0;
  }
}

size_t power_cluster_smem(int n) {
  const int ldl = ((n + 7) / 16) * 16 + 8;
  return (static_cast<size_t>(kPowRows) * ldl + 2 * kMaxN + 3 * kPowCl) * sizeof(double);
}

__global__ void __launch_bounds__(kThreads, 1) chol_kernel_smem(CholParams p) {
  extern __shared__ double smW[];
  chol_body<true>(p, smW);
}

// n >= 160: W in an L2-resident global scratch (same code path through the generic pointer)
__global__ void __launch_bounds__(kThreads, 1) chol_kernel_gmem(CholParams p) {
  extern __shared__ double smW[];
  chol_body<false>(p, smW);
}

// a6: Rnew = R~ R (pass > 1) or R~ (pass 1), k ascending like the oracle; off the critical path
// (side stream, overlapped with the TRSM).  Skipped when the pass broke down.
__global__ void trmul_kernel(const double* Rt, const double* R, double* Rnew, int n, int first,
                             const DevStatus* st, PassGate gate) {
  if (SCQR3_GATE_SKIP(gate) || st->code != SCQR3_OK) return;
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= static_cast<long long>(n) * n) return;
  const int i = static_cast<int>(k % n), j = static_cast<int>(k / n);
  double acc = 0.0;
  if (i <= j) {
    // (R~ row-major, see write_outputs; R column-major)
    if (first) acc = Rt[static_cast<size_t>(i) * n + j];
    else
      for (int kk = i; kk <= j; ++kk) acc = fma(Rt[static_cast<size_t>(i) * n + kk], R[kk + static_cast<size_t>(j) * n], acc);
  }
  Rnew[k] = acc;
}

__global__ void copy_kernel(const double* src, double* dst, long long count, const DevStatus* st, PassGate gate) {
  if (SCQR3_GATE_SKIP(gate) || (st && st->code != SCQR3_OK)) return;
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < count) dst[k] = src[k];
}

// R (n x n, upper, positive diagonal; column-major, or row-major as chol_kernel writes R~) ->
// TRSM layout: B fragments of -R (fragment f = idx / 32: target block J >= 1, k-step s < 2J) and
// the 8 x 8 diagonal blocks pre-scaled by their pivots (r_cj / r_cc) with the reciprocal pivots,
// the identity past n.  In a pass it runs after chol_kernel (skipped when that failed or after a
// stop); also used by the kernel-level scqr3_trsm API and the complex path.
__global__ void trsm_prep_kernel(const double* R, int n, int NT, double* bfrag, double* dblk, int rowmajor,
                                 const DevStatus* st, PassGate gate, int diag_mode) {
  if (SCQR3_GATE_SKIP(gate) || (st && st->code != SCQR3_OK)) return;
  auto rp = [&](int i, int j) -> double {
    if (i < n && j < n)
      return i <= j ? R[rowmajor ? static_cast<size_t>(i) * n + j : i + static_cast<size_t>(j) * n] : 0.0;
    return i == j ? 1.0 : 0.0;
  };
  if (blockIdx.x == gridDim.x - 1) {  // the guard CTA (trsm_prep_blocks: launched with 256 threads)
    trsm_diag_guard(rp, n, NT, dblk, diag_mode);
    return;
  }
  const int nf = NT * (NT - 1) * 32;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nf + NT * 72; idx += (gridDim.x - 1) * blockDim.x) {
    if (idx < nf) {
      const int f = idx >> 5, lane = idx & 31;
      int J = 1;
      while ((J + 1) * J <= f) ++J;
      const int s = f - J * (J - 1);
      const int row = 8 * (s >> 1) + 2 * (lane & 3) + (s & 1);
      const int col = 8 * J + (lane >> 2);
      bfrag[idx] = -rp(row, col);
    } else {
      const int k = idx - nf, J = k / 72, w = k % 72;
      if (w < 64) {
        const int c = 8 * J + (w >> 3), j = 8 * J + (w & 7);
        dblk[k] = j > c ? rp(c, j) / rp(c, c) : 0.0;
      } else {
        dblk[k] = 1.0 / rp(8 * J + (w - 64), 8 * J + (w - 64));
      }
    }
  }
}


// WHILE condition after pass k (= *pass_dev): run the body again if k < last_pass and k <
// max_passes, and then advance the counter to the body's pass number k + 1 here (one graph node
// per pass less than a separate advance kernel at the top of the body)
__global__ void pass_loop_cond_kernel(int* pass_dev, const int* last_pass, int max_passes,
                                      cudaGraphConditionalHandle handle) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const int k = *pass_dev;
    const bool more = k < *last_pass && k < max_passes;
    if (more) *pass_dev = k + 1;
    cudaGraphSetConditional(handle, more ? 1u : 0u);
  }
}

}  // namespace scqr3
