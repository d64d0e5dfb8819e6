// chol.cu -- the per-pass n x n step (a3 norm/shift, a4 shifted Cholesky, a6 R accumulation,
// a7 pass control) on ONE CTA; it is replicated on every rank (identical input bits after
// the Gram allreduce give identical R~, so no broadcast is needed).
//
//   N^2 ~ ||Q||_2^2 by power iteration on the Gram (reading D2), or trace / user bound
//   s = 11{mn+n(n+1)} u N^2            (eq. finds2)
//   s = 11{2m sqrt(mn)+n(n+1)} u N^2 N_B (eq. finds2B, oblique)
//   pass 1: R~ = chol(A + sI)         (Alg. 3 line 4)
//   pass k>1: R~ = chol(A); on breakdown R~ = chol(A + sI)   (Alg. 2 lines 4-7)
//   R := R~ R                           (Alg. 2 line 8)
//   stop after an unshifted pass with ||A - I||_F <= stop_tol (reading D6)
// Breakdown = first pivot <= 0 or non-finite (reading D9).  The Cholesky is unblocked
// right-looking, like the oracle, on a row-major working copy W of A (shared memory when
// n*n*8 B fits, else an L2-resident global scratch).  Outputs for the TRSM kernel: negated
// R~ in mma B-fragment order and the 8x8 diagonal blocks with reciprocal pivots.
#include <math.h>

#include "scqr3.h"
#include "scqr3_dev.cuh"
#include "scqr3_kernels.h"

namespace scqr3 {

namespace {
constexpr int kCholThreads = 1024;

__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  __syncthreads();  // protect red[] from a previous use
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double w = lane < (blockDim.x >> 5) ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) w += __shfl_down_sync(0xffffffffu, w, o);
    if (lane == 0) red[32] = w;
  }
  __syncthreads();
  return red[32];
}

__device__ __forceinline__ double gram_entry(const CholParams& p, int i, int j) {
  const int a = i <= j ? i : j, b = i <= j ? j : i;
  if (p.mode == CHOL_ONLY) return p.Afull[a + static_cast<size_t>(b) * p.n];
  const size_t tile = static_cast<size_t>(b >> 3) * ((b >> 3) + 1) / 2 + (a >> 3);
  return p.tiles[tile * 64 + 8 * (a & 7) + (b & 7)];
}

__device__ void load_W(const CholParams& p, double* W) {
  const int n = p.n;
  for (int k = threadIdx.x; k < n * n; k += blockDim.x) W[k] = gram_entry(p, k / n, k % n);
  __syncthreads();
}

// returns 0, or the 1-based breakdown pivot (value in *pv); W upper holds R~ on success
__device__ int factor(double* W, int n, double s, bool add_shift, double* pv_out, int* sflag, double* sval) {
  if (add_shift) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) W[i * n + i] = W[i * n + i] + s;
  }
  __syncthreads();
  for (int kk = 0; kk < n; ++kk) {
    if (threadIdx.x == 0) {
      const double d = W[kk * n + kk];
      if (!(d > 0.0) || !isfinite(d)) {
        *sflag = kk + 1;
        *sval = d;
      } else {
        W[kk * n + kk] = sqrt(d);
      }
    }
    __syncthreads();
    if (*sflag) {
      *pv_out = *sval;
      return *sflag;
    }
    const double rkk = W[kk * n + kk];
    for (int j = kk + 1 + threadIdx.x; j < n; j += blockDim.x) W[kk * n + j] = W[kk * n + j] / rkk;
    __syncthreads();
    const int L = n - kk - 1;
    const double* rk = W + kk * n + kk + 1;
    for (int idx = threadIdx.x; idx < L * L; idx += blockDim.x) {
      const int ii = idx / L, jj = idx - ii * L;
      if (jj >= ii) {
        double* w = W + (kk + 1 + ii) * n + (kk + 1 + jj);
        *w = *w - rk[ii] * rk[jj];
      }
    }
    __syncthreads();
  }
  return 0;
}

__device__ __forceinline__ double rpad(const double* W, int n, int i, int j) {
  if (i < n && j < n) return i <= j ? W[i * n + j] : 0.0;
  return i == j ? 1.0 : 0.0;
}

__device__ void write_trsm_layout(const double* W, int n, int NT, double* bfrag, double* dblk) {
  const int nf = NT * (NT - 1) * 32;
  for (int idx = threadIdx.x; idx < nf; idx += blockDim.x) {
    const int f = idx >> 5, lane = idx & 31;
    int J = 1;
    while ((J + 1) * J <= f) ++J;
    const int s = f - J * (J - 1);
    const int g = lane >> 2, t = lane & 3;
    const int row = 8 * (s >> 1) + 2 * t + (s & 1);
    const int col = 8 * J + g;
    bfrag[idx] = -rpad(W, n, row, col);
  }
  for (int idx = threadIdx.x; idx < NT * 72; idx += blockDim.x) {
    const int J = idx / 72, w = idx % 72;
    if (w < 64) dblk[idx] = rpad(W, n, 8 * J + (w >> 3), 8 * J + (w & 7));
    else dblk[idx] = 1.0 / rpad(W, n, 8 * J + (w - 64), 8 * J + (w - 64));
  }
}
}  // namespace

__global__ void __launch_bounds__(kCholThreads, 1) chol_kernel(CholParams p) {
  extern __shared__ double smW[];
  __shared__ double red[33];
  __shared__ double xv[kMaxN];
  __shared__ int sflag;
  __shared__ double sval;
  const int n = p.n;
  double* W = p.w_in_smem ? smW : p.W;
  if (threadIdx.x == 0) sflag = 0;
  load_W(p, W);

  if (p.mode == CHOL_ONLY) {
    double pv = 0.0;
    const int piv = factor(W, n, p.shift_value, p.shift_value != 0.0, &pv, &sflag, &sval);
    for (int k = threadIdx.x; k < n * n; k += blockDim.x) {
      const int i = k % n, j = k / n;
      p.R[k] = (piv == 0 && i <= j) ? W[i * n + j] : 0.0;
    }
    if (threadIdx.x == 0) {
      DevStatus st{};
      st.code = piv ? SCQR3_EBREAKDOWN : SCQR3_OK;
      st.breakdown_pivot = piv;
      st.pivot_value = pv;
      st.shift = p.shift_value;
      *p.st_dev = st;
    }
    return;
  }

  // ---- a7 input: distance of the Gram from I (stop test, reading D6) and its trace
  double loc = 0.0, tr = 0.0;
  for (int k = threadIdx.x; k < n * n; k += blockDim.x) {
    const int i = k / n, j = k % n;
    const double v = W[k] - (i == j ? 1.0 : 0.0);
    loc += v * v;
    if (i == j) tr += W[k];
  }
  const double dev = sqrt(block_sum(loc, red));
  const double trace = block_sum(tr, red);

  // ---- a3: norm estimate N^2 and shift s
  double N2;
  if (p.oblique) {
    if (p.pass == 1 && p.norm_mode == SCQR3_NORM_USER) N2 = p.norm2_bound * p.norm2_bound;
    else N2 = p.tiles[static_cast<size_t>(p.NT) * (p.NT + 1) / 2 * 64];  // ||Q||_F^2 (reading D4)
  } else if (p.pass == 1 && p.norm_mode == SCQR3_NORM_USER) {
    N2 = p.norm2_bound * p.norm2_bound;
  } else if (p.norm_mode == SCQR3_NORM_FROBENIUS) {
    N2 = trace;
  } else {
    // power iteration on the Gram from the all-ones vector (reading D2); W is symmetric so
    // row i is read as column i (conflict-free)
    const int i = threadIdx.x;
    if (i < n) xv[i] = 1.0 / sqrt(static_cast<double>(n));
    __syncthreads();
    for (int it = 0; it < p.power_iters; ++it) {
      double y = 0.0;
      if (i < n)
        for (int j = 0; j < n; ++j) y = fma(W[j * n + i], xv[j], y);
      const double ny = sqrt(block_sum(i < n ? y * y : 0.0, red));
      if (!(ny > 0.0)) break;
      if (i < n) xv[i] = y / ny;
      __syncthreads();
    }
    double y = 0.0;
    if (i < n)
      for (int j = 0; j < n; ++j) y = fma(W[j * n + i], xv[j], y);
    N2 = block_sum(i < n ? xv[i] * y : 0.0, red) * 1.01;
  }
  const double u = 0x1p-53;
  const double mg = p.m_global, nn = static_cast<double>(n);
  double s;
  if (p.shift_mode == SCQR3_SHIFT_FIXED && p.pass == 1) s = p.shift_value;
  else if (p.oblique) s = 11.0 * (2.0 * mg * sqrt(mg * nn) + nn * (nn + 1.0)) * u * N2 * (*p.nb_dev);
  else s = 11.0 * (mg * nn + nn * (nn + 1.0)) * u * N2;

  // ---- a4: (shifted) Cholesky with breakdown-triggered re-shift
  int shifted = 0, bpiv = 0, piv;
  double bval = 0.0, pv = 0.0;
  if (p.pass == 1 && p.shift_mode != SCQR3_SHIFT_NONE) {
    shifted = 1;
    piv = factor(W, n, s, true, &pv, &sflag, &sval);
    if (piv) { bpiv = piv; bval = pv; }
  } else {
    piv = factor(W, n, 0.0, false, &pv, &sflag, &sval);
    if (piv) {
      bpiv = piv;
      bval = pv;
      if (p.shift_mode != SCQR3_SHIFT_NONE) {
        __syncthreads();
        if (threadIdx.x == 0) sflag = 0;
        load_W(p, W);
        shifted = 1;
        piv = factor(W, n, s, true, &pv, &sflag, &sval);
        if (piv) { bpiv = piv; bval = pv; }
      }
    }
  }
  const int code = piv ? SCQR3_EBREAKDOWN : SCQR3_OK;

  if (code == SCQR3_OK) {
    // ---- outputs for the TRSM kernel
    write_trsm_layout(W, n, p.NT, p.bfrag, p.dblk);
    // ---- a6: R := R~ R  (k ascending, like the oracle)
    if (p.pass == 1) {
      for (int k = threadIdx.x; k < n * n; k += blockDim.x) {
        const int i = k % n, j = k / n;
        p.R[k] = i <= j ? W[i * n + j] : 0.0;
      }
    } else {
      for (int k = threadIdx.x; k < n * n; k += blockDim.x) {
        const int i = k % n, j = k / n;
        double acc = 0.0;
        if (i <= j)
          for (int kk = i; kk <= j; ++kk) acc = fma(W[i * n + kk], p.R[kk + static_cast<size_t>(j) * n], acc);
        p.Rnew[k] = acc;
      }
      __syncthreads();
      for (int k = threadIdx.x; k < n * n; k += blockDim.x) p.R[k] = p.Rnew[k];
    }
  }
  if (threadIdx.x == 0) {
    DevStatus st{};
    st.code = code;
    st.stop = (code == SCQR3_OK && !shifted && dev <= p.stop_tol) ? 1 : 0;
    st.pass = p.pass;
    st.shifted = shifted;
    st.shift = shifted ? s : 0.0;
    st.breakdown_pivot = bpiv;
    st.pivot_value = bval;
    st.norm2_est = N2;
    st.dev_F = dev;
    *p.st_dev = st;
    if (p.st_host) {
      volatile DevStatus* h = p.st_host;
      h->stop = st.stop;
      h->pass = st.pass;
      h->shifted = st.shifted;
      h->shift = st.shift;
      h->breakdown_pivot = st.breakdown_pivot;
      h->pivot_value = st.pivot_value;
      h->norm2_est = st.norm2_est;
      h->dev_F = st.dev_F;
      __threadfence_system();
      h->code = st.code;
      __threadfence_system();
    }
  }
}

// R (n x n col-major, upper, positive diagonal) -> TRSM layout (kernel-level scqr3_trsm API)
__global__ void trsm_prep_kernel(const double* R, int n, int NT, double* bfrag, double* dblk) {
  auto rp = [&](int i, int j) -> double {
    if (i < n && j < n) return i <= j ? R[i + static_cast<size_t>(j) * n] : 0.0;
    return i == j ? 1.0 : 0.0;
  };
  const int nf = NT * (NT - 1) * 32;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nf + NT * 72; idx += gridDim.x * blockDim.x) {
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
      if (w < 64) dblk[k] = rp(8 * J + (w >> 3), 8 * J + (w & 7));
      else dblk[k] = 1.0 / rp(8 * J + (w - 64), 8 * J + (w - 64));
    }
  }
}

}  // namespace scqr3
