// zchol.cu -- complex X ("everything carries over to complex matrices",
// P:124-125; reading D23: ^T -> ^H, u = 2^-53, the shift formula unchanged).
//
// The tall-skinny steps reuse the real kernels on a real m x 2n "split" matrix whose columns are
// (Re x_0, Im x_0, Re x_1, Im x_1, ...):
//   * Gram: X'^T X' (2n x 2n) holds A = X^H X as A_jl = G_2j,2l + G_2j+1,2l+1
//     + i (G_2j,2l+1 - G_2j+1,2l)                                   [zcombine_kernel]
//   * TRSM: with R~ upper and a real diagonal, Q R~ = X is Q' M = X' for the REAL upper-triangular
//     2n x 2n matrix M whose 2x2 block (k, j) is [[Re r_kj, Im r_kj], [-Im r_kj, Re r_kj]], so the
//     real TRSM kernel solves it row by row (row-wise backward stability carries over).
// Only the n x n step is complex: zchol_kernel (norm estimate, shift, Hermitian Cholesky with
// breakdown detection, pass control, and M for the TRSM) and ztrmul_kernel (R := R~ R).
#include <math.h>

#include "scqr3.h"
#include "scqr3_dev.cuh"
#include "scqr3_kernels.h"

namespace scqr3 {

namespace {
constexpr int kZThreads = 256;
constexpr int kZPanel = 16;  // rows of R~ per panel of the blocked factorisation (W in global memory)

__device__ __forceinline__ double2 zsum2(double a, double b, double* red) {
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) {
    red[2 * w] = a;
    red[2 * w + 1] = b;
  }
  __syncthreads();
  double2 r = make_double2(0.0, 0.0);
  for (int i = 0; i < kZThreads / 32; ++i) {  // fixed order
    r.x += red[2 * i];
    r.y += red[2 * i + 1];
  }
  __syncthreads();
  return r;
}
}  // namespace

// X (complex, interleaved, ld) -> X' (m x 2n real, ld2): X'(:, 2j) = Re x_j, X'(:, 2j+1) = Im x_j
__global__ void z2split_kernel(const double* Z, long long ldz, long long m, int n, double* S, long long lds) {
  const long long total = m * n;
  for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = k % m, j = k / m;
    const double2 v = *reinterpret_cast<const double2*>(Z + 2 * (i + j * ldz));
    S[i + (2 * j) * lds] = v.x;
    S[i + (2 * j + 1) * lds] = v.y;
  }
}

__global__ void split2z_kernel(const double* S, long long lds, long long m, int n, double* Z, long long ldz) {
  const long long total = m * n;
  for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = k % m, j = k / m;
    *reinterpret_cast<double2*>(Z + 2 * (i + j * ldz)) = make_double2(S[i + (2 * j) * lds], S[i + (2 * j + 1) * lds]);
  }
}

// packed upper tiles of the 2n x 2n split Gram -> A = X^H X (n x n complex, full, interleaved)
__global__ void zcombine_kernel(const double* tiles, int n, double* A, const int* last_pass, int pass) {
  if (last_pass && pass > *(volatile const int*)last_pass) return;
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= static_cast<long long>(n) * n) return;
  const int j = static_cast<int>(k % n), l = static_cast<int>(k / n);
  auto G = [&](int a, int b) -> double {  // symmetric 2n x 2n Gram entry (upper tiles)
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    return tiles[(static_cast<size_t>(b >> 3) * ((b >> 3) + 1) / 2 + (a >> 3)) * 64 + 8 * (a & 7) + (b & 7)];
  };
  const int p = j <= l ? j : l, q = j <= l ? l : j;  // the upper entry (p, q); A_lj = conj(A_jl)
  const double re = G(2 * p, 2 * q) + G(2 * p + 1, 2 * q + 1);
  const double im = p == q ? 0.0 : G(2 * p, 2 * q + 1) - G(2 * p + 1, 2 * q);
  A[2 * k] = re;
  A[2 * k + 1] = j <= l ? im : -im;
}

// n x n complex step, one CTA: dev / trace, norm estimate and shift (as chol_kernel, ^T -> ^H),
// Hermitian Cholesky (unblocked right-looking; breakdown at the first pivot <= 0 / non-finite),
// status, R~ for ztrmul_kernel, and the real 2n x 2n upper-triangular M for the TRSM.
__global__ void __launch_bounds__(kZThreads, 1) zchol_kernel(ZCholParams p) {
  const int pass = p.pass_dev ? *(volatile const int*)p.pass_dev : p.pass;
  if (p.last_pass && pass > *(volatile const int*)p.last_pass) return;
  __shared__ double red[2 * kZThreads / 32];
  __shared__ double ybuf[2][2 * kMaxN];  // complex power-iteration vector (n <= 512)
  __shared__ double piv_inv;
  __shared__ double rowk[2 * kMaxN];  // row k of R~ (complex, n <= 512)
  __shared__ int sflag;
  __shared__ double sval;
  extern __shared__ double zsm[];
  const int n = p.n, tid = threadIdx.x;
  // working copy of the upper triangle: packed column-major ((i, j), i <= j, at j(j+1)/2 + i) in
  // shared memory when it fits (n <= 128: 132 KB), else the full n x n in global scratch
  const bool packed = p.w_in_smem != 0;
  double* W = packed ? zsm : p.W;
  auto widx = [&](int i, int j) -> size_t {
    return packed ? static_cast<size_t>(j) * (j + 1) / 2 + i : i + static_cast<size_t>(j) * n;
  };
  auto wre = [&](int i, int j) -> double& { return W[2 * widx(i, j)]; };
  auto wim = [&](int i, int j) -> double& { return W[2 * widx(i, j) + 1]; };
  auto are = [&](int i, int j) -> double { return p.A[2 * (i + static_cast<size_t>(j) * n)]; };
  auto aim = [&](int i, int j) -> double { return p.A[2 * (i + static_cast<size_t>(j) * n) + 1]; };
  auto load = [&]() {
    for (int j = tid >> 5; j < n; j += kZThreads / 32)
      for (int i = tid & 31; i <= j; i += 32) {
        wre(i, j) = are(i, j);
        wim(i, j) = aim(i, j);
      }
    __syncthreads();
  };
  load();
  // ---- distance from I (stop test, D6) and the trace
  double loc = 0.0, tr = 0.0;
  for (long long k = tid; k < static_cast<long long>(n) * n; k += kZThreads) {
    const int i = static_cast<int>(k % n), j = static_cast<int>(k / n);
    const double vr = p.A[2 * k] - (i == j ? 1.0 : 0.0), vi = p.A[2 * k + 1];
    loc = fma(vr, vr, fma(vi, vi, loc));
    if (i == j) tr += p.A[2 * k];
  }
  const double2 dt = zsum2(loc, tr, red);
  const double dev = sqrt(dt.x), trace = dt.y;
  auto write_status = [&](int code, int stop, int shifted, double s, int bpiv, double bval, double N2) {
    if (tid != 0) return;
    DevStatus st{};
    st.code = code;
    st.stop = stop;
    st.pass = pass;
    st.shifted = shifted;
    st.shift = shifted ? s : 0.0;
    st.breakdown_pivot = bpiv;
    st.pivot_value = bval;
    st.norm2_est = N2;
    st.dev_F = dev;
    *p.st_dev = st;
    if (p.last_pass) {
      if (code != SCQR3_OK) *(volatile int*)p.last_pass = pass - 1;
      else if (stop) *(volatile int*)p.last_pass = pass;
    }
    if (p.st_host) {
      volatile DevStatus* h = p.st_host + (pass - 1);
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
  };
  if (pass == 1 && !isfinite(trace)) {  // NaN / Inf in X
    write_status(SCQR3_EINVAL, 0, 0, 0.0, 0, 0.0, 0.0);
    return;
  }
  // ---- power iteration on the Hermitian A (as power_lmax: scaled, unnormalised iterates)
  auto lmax = [&]() -> double {
    if (!(trace > 0.0) || !isfinite(trace)) return 0.0;
    const double sc = ldexp(1.0, -(ilogb(trace) + 1));
    for (int i = tid; i < n; i += kZThreads) {
      ybuf[0][2 * i] = 1.0;
      ybuf[0][2 * i + 1] = 0.0;
    }
    __syncthreads();
    int cur = 0;
    for (int it = 0; it < p.power_iters; ++it) {
      for (int row = tid; row < n; row += kZThreads) {
        double vr = 0.0, vi = 0.0;
        for (int j = 0; j < n; ++j) {
          const double a = are(row, j), b = aim(row, j), c = ybuf[cur][2 * j], d = ybuf[cur][2 * j + 1];
          vr = fma(a, c, fma(-b, d, vr));
          vi = fma(a, d, fma(b, c, vi));
        }
        ybuf[cur ^ 1][2 * row] = vr * sc;
        ybuf[cur ^ 1][2 * row + 1] = vi * sc;
      }
      __syncthreads();
      cur ^= 1;
    }
    double num = 0.0, den = 0.0;
    for (int row = tid; row < n; row += kZThreads) {
      double vr = 0.0, vi = 0.0;
      for (int j = 0; j < n; ++j) {
        const double a = are(row, j), b = aim(row, j), c = ybuf[cur][2 * j], d = ybuf[cur][2 * j + 1];
        vr = fma(a, c, fma(-b, d, vr));
        vi = fma(a, d, fma(b, c, vi));
      }
      const double yr = ybuf[cur][2 * row], yi = ybuf[cur][2 * row + 1];
      num = fma(yr, vr, fma(yi, vi, num));  // Re(conj(y) (A y))
      den = fma(yr, yr, fma(yi, yi, den));
    }
    const double2 nd = zsum2(num, den, red);
    return nd.y > 0.0 ? nd.x / nd.y : 0.0;
  };
  const double u = 0x1p-53, mg = p.m_global, nn = static_cast<double>(n);
  auto shift_for = [&](double& N2) -> double {
    if (pass == 1 && p.norm_mode == SCQR3_NORM_USER) N2 = p.norm2_bound * p.norm2_bound;
    else if (p.norm_mode == SCQR3_NORM_FROBENIUS) N2 = trace;
    else N2 = lmax() * 1.01;
    if (p.shift_mode == SCQR3_SHIFT_FIXED && pass == 1) return p.shift_value;
    return 11.0 * (mg * nn + nn * (nn + 1.0)) * u * N2;
  };
  // ---- Hermitian Cholesky of W + sI (W reloaded when shifting after a plain attempt)
  auto factor = [&](double s, bool add_shift, double* pv) -> int {
    if (add_shift) {
      for (int i = tid; i < n; i += kZThreads) wre(i, i) += s;
      __syncthreads();
    }
    if (tid == 0) sflag = 0;
    __syncthreads();
    for (int k = 0; k < n; ++k) {
      if (tid == 0) {
        const double d = wre(k, k);
        if (!(d > 0.0) || !isfinite(d) || !isfinite(wim(k, k))) {
          sflag = k + 1;
          sval = d;
        } else {
          const double r = sqrt(d);
          wre(k, k) = r;
          wim(k, k) = 0.0;
          piv_inv = 1.0 / r;
        }
      }
      __syncthreads();
      if (sflag) {
        *pv = sval;
        return sflag;
      }
      const double ri = piv_inv;
      for (int j = k + 1 + tid; j < n; j += kZThreads) {  // row k of R~ (also cached: rowk)
        const double a = wre(k, j) * ri, b = wim(k, j) * ri;
        wre(k, j) = a;
        wim(k, j) = b;
        rowk[2 * j] = a;
        rowk[2 * j + 1] = b;
      }
      __syncthreads();
      // W_ij -= conj(r_ki) r_kj for k < i <= j: a warp per column j, lanes down the column
      for (int j = k + 1 + (tid >> 5); j < n; j += kZThreads / 32) {
        const double c = rowk[2 * j], d = rowk[2 * j + 1];
        for (int i = k + 1 + (tid & 31); i <= j; i += 32) {
          const double a = rowk[2 * i], b = rowk[2 * i + 1];
          wre(i, j) = wre(i, j) - (a * c + b * d);
          wim(i, j) = wim(i, j) - (a * d - b * c);
        }
      }
      __syncthreads();
    }
    return 0;
  };
  // ---- the same factorisation blocked for W in global memory (n > 128): panels of kZPanel rows
  // of R~ factored in shared memory (dynamic: kZPanel x (n - kb) complex), then one rank-kZPanel
  // update of the trailing upper triangle, so each entry of W is read and written once per panel
  // instead of once per column (n = 512: ~31 ms per pass unblocked).  Same pivots, same breakdown
  // test at the same column; only the order of the updates' roundings differs.
  auto factor_blocked = [&](double s, bool add_shift, double* pv) -> int {
    if (add_shift) {
      for (int i = tid; i < n; i += kZThreads) wre(i, i) += s;
      __syncthreads();
    }
    if (tid == 0) sflag = 0;
    __syncthreads();
    double* P = zsm;
    const int warp = tid >> 5, lane = tid & 31;
    for (int kb = 0; kb < n; kb += kZPanel) {
      const int b = min(kZPanel, n - kb), ldp = n - kb;
      auto pre = [&](int r, int c) -> double& { return P[2 * (r * ldp + c)]; };
      auto pim = [&](int r, int c) -> double& { return P[2 * (r * ldp + c) + 1]; };
      for (int idx = tid; idx < b * ldp; idx += kZThreads) {  // rows kb.., down each column
        const int r = idx % b, c = idx / b;
        if (c >= r) {
          pre(r, c) = wre(kb + r, kb + c);
          pim(r, c) = wim(kb + r, kb + c);
        }
      }
      __syncthreads();
      for (int k = 0; k < b; ++k) {
        if (tid == 0) {
          const double d = pre(k, k);
          if (!(d > 0.0) || !isfinite(d) || !isfinite(pim(k, k))) {
            sflag = kb + k + 1;
            sval = d;
          } else {
            const double r = sqrt(d);
            pre(k, k) = r;
            pim(k, k) = 0.0;
            piv_inv = 1.0 / r;
          }
        }
        __syncthreads();
        if (sflag) {
          *pv = sval;
          return sflag;
        }
        const double ri = piv_inv;
        for (int c = k + 1 + tid; c < ldp; c += kZThreads) {
          pre(k, c) *= ri;
          pim(k, c) *= ri;
        }
        __syncthreads();
        const int rows = b - k - 1;  // panel rows below k: W_ic -= conj(r_ki) r_kc, c >= i
        for (int idx = tid; idx < rows * ldp; idx += kZThreads) {
          const int i = k + 1 + idx % rows, c = idx / rows;
          if (c >= i) {
            const double a = pre(k, i), bb = pim(k, i), cr = pre(k, c), ci = pim(k, c);
            pre(i, c) = pre(i, c) - (a * cr + bb * ci);
            pim(i, c) = pim(i, c) - (a * ci - bb * cr);
          }
        }
        __syncthreads();
      }
      for (int idx = tid; idx < b * ldp; idx += kZThreads) {  // R~ rows kb..kb+b-1 back to W
        const int r = idx % b, c = idx / b;
        if (c >= r) {
          wre(kb + r, kb + c) = pre(r, c);
          wim(kb + r, kb + c) = pim(r, c);
        }
      }
      // trailing update W_ij -= sum_r conj(r_ri) r_rj (i <= j, both >= kb + b): work items are
      // 32 x 32 blocks (row chunk ci <= column chunk sj); a warp per item, lanes down the rows,
      // this lane's panel column in registers, the column's panel entries broadcast from smem
      const int t0 = kb + b;
      const int nch = (n - t0 + 31) / 32;
      const int items = nch * (nch + 1) / 2;
      for (int it = warp; it < items; it += kZThreads / 32) {
        int sj = static_cast<int>((sqrt(8.0 * it + 1.0) - 1.0) * 0.5);
        while (sj * (sj + 1) / 2 > it) --sj;
        while ((sj + 1) * (sj + 2) / 2 <= it) ++sj;
        const int ci = it - sj * (sj + 1) / 2;
        const int i = t0 + 32 * ci + lane;
        const bool iok = i < n;
        double ar[kZPanel], ai[kZPanel];
#pragma unroll
        for (int r = 0; r < kZPanel; ++r) {
          ar[r] = iok && r < b ? pre(r, i - kb) : 0.0;
          ai[r] = iok && r < b ? pim(r, i - kb) : 0.0;
        }
        const int j0 = t0 + 32 * sj, j1 = min(n, j0 + 32);
        for (int j = j0; j < j1; j += 4) {
          double wr[4], wi[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const bool ok = iok && j + u < j1 && i <= j + u;
            wr[u] = ok ? wre(i, j + u) : 0.0;
            wi[u] = ok ? wim(i, j + u) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int jj = min(j + u, j1 - 1) - kb;
            double sr = 0.0, si = 0.0;
#pragma unroll
            for (int r = 0; r < kZPanel; ++r) {
              const double pr = r < b ? pre(r, jj) : 0.0, pi = r < b ? pim(r, jj) : 0.0;
              sr = fma(ar[r], pr, fma(ai[r], pi, sr));
              si = fma(ar[r], pi, fma(-ai[r], pr, si));
            }
            if (iok && j + u < j1 && i <= j + u) {
              wre(i, j + u) = wr[u] - sr;
              wim(i, j + u) = wi[u] - si;
            }
          }
        }
      }
      __syncthreads();
    }
    return 0;
  };
  auto run_factor = [&](double s, bool add_shift, double* pv) -> int {
    return packed ? factor(s, add_shift, pv) : factor_blocked(s, add_shift, pv);
  };
  int shifted = 0, bpiv = 0, piv = 1;
  double bval = 0.0, pv = 0.0, s = 0.0, N2 = 0.0;
  const bool practical = p.shift_mode == SCQR3_SHIFT_PRACTICAL;
  const bool shift_first = pass == 1 && (p.shift_mode == SCQR3_SHIFT_SAFE || p.shift_mode == SCQR3_SHIFT_FIXED ||
                                         practical);
  bool dirty = false;
  if (!shift_first) {
    piv = run_factor(0.0, false, &pv);
    dirty = true;
    if (piv) { bpiv = piv; bval = pv; }
  }
  if (piv && p.shift_mode != SCQR3_SHIFT_NONE) {
    if (dirty) load();
    const double s_safe = shift_for(N2);
    const double s_p = u * N2;
    for (int attempt = practical ? 0 : 1; attempt < 2 && piv; ++attempt) {
      if (dirty) load();
      s = attempt == 0 ? s_p : s_safe;
      shifted = 1;
      piv = run_factor(s, true, &pv);
      dirty = true;
      if (piv) { bpiv = piv; bval = pv; }
    }
  }
  const int code = piv ? SCQR3_EBREAKDOWN : SCQR3_OK;
  if (code == SCQR3_OK) {
    // R~ (complex, column-major, zero strict lower) and M (real 2n x 2n upper, column-major)
    const int n2 = 2 * n;
    for (long long k = tid; k < static_cast<long long>(n) * n; k += kZThreads) {
      const int i = static_cast<int>(k % n), j = static_cast<int>(k / n);
      const bool up = i <= j;
      const double re = up ? wre(i, j) : 0.0, im = up ? wim(i, j) : 0.0;
      p.Rt[2 * k] = re;
      p.Rt[2 * k + 1] = im;
      double* M = p.M;
      M[(2 * i) + static_cast<size_t>(2 * j) * n2] = re;
      M[(2 * i) + static_cast<size_t>(2 * j + 1) * n2] = im;
      M[(2 * i + 1) + static_cast<size_t>(2 * j) * n2] = -im;
      M[(2 * i + 1) + static_cast<size_t>(2 * j + 1) * n2] = re;
    }
  }
  write_status(code, (code == SCQR3_OK && !shifted && dev <= p.stop_tol) ? 1 : 0, shifted, s, bpiv, bval, N2);
}

// R := R~ R for complex upper n x n (column-major interleaved), k ascending; first: R := R~
__global__ void ztrmul_kernel(const double* Rt, const double* R, double* Rnew, int n, int first, const DevStatus* st,
                              PassGate gate) {
  if (SCQR3_GATE_SKIP(gate) || st->code != SCQR3_OK) return;
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= static_cast<long long>(n) * n) return;
  const int i = static_cast<int>(k % n), j = static_cast<int>(k / n);
  double re = 0.0, im = 0.0;
  if (i <= j) {
    if (first) {
      re = Rt[2 * k];
      im = Rt[2 * k + 1];
    } else {
      for (int l = i; l <= j; ++l) {
        const double a = Rt[2 * (i + static_cast<size_t>(l) * n)], b = Rt[2 * (i + static_cast<size_t>(l) * n) + 1];
        const double c = R[2 * (l + static_cast<size_t>(j) * n)], d = R[2 * (l + static_cast<size_t>(j) * n) + 1];
        re = fma(a, c, fma(-b, d, re));
        im = fma(a, d, fma(b, c, im));
      }
    }
  }
  Rnew[2 * k] = re;
  Rnew[2 * k + 1] = im;
}

}  // namespace scqr3
