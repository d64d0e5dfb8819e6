/*
 * scqr3_oracle.c -- plain, slow, obviously-correct CPU oracle for shifted CholeskyQR3.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1809_11085_b200/, libscqr3.so) never links, imports or calls it, and this
 * file shares no code, header, table or constant generator with it.
 *
 * Reference: /root/reference/PAPER.md (Fukaya, Kannan, Nakatsukasa, Yamamoto,
 * Yanagisawa, "Shifted CholeskyQR for computing the QR factorization of
 * ill-conditioned matrices", arXiv:1809.11085).  "P:L" = PAPER.md line L,
 * "S:L" = SPEC.md line L.  Readings of the paper (D1..D20) are listed in DESIGN.md.
 *
 * Arithmetic: IEEE binary64, round-to-nearest, compiled with -ffp-contract=off so
 * every a*b+c is two roundings (the paper's standard model).  Loops are
 * written in the order the paper states the operation; the only parallelism is
 * over independent outputs (rows of Q, entries of A), which never changes the
 * order in which any single output is summed.
 *
 * Parity status of each function (pins live in tests/test_oracle_*.py):
 *   orc_gram              pinned (exact small integer cases, componentwise T1 bound
 *                         against an exact rational/extended reference, symmetry)
 *   orc_gram_oblique      pinned (B=I reduces to orc_gram; exact integer cases;
 *                         brute force dense X^T B X)
 *   orc_gram_oblique_csr  pinned (CSR of the tridiagonal B in the same term order is
 *                         bitwise orc_gram_oblique; CSR identity = orc_gram; exact integer
 *                         cases against int64 arithmetic)
 *   orc_z* (complex, N4)  pinned (a real input reproduces the real functions bit for bit;
 *                         exact Gaussian-integer Gram / Cholesky / TRSM / trmul; numpy complex
 *                         Householder QR; eigvalsh closed forms; CholeskyQR2 breakdown + target)
 *   orc_scqr3_csr         pinned (CSR-tridiagonal equals orc_scqr3 bitwise; 2-D Laplacian
 *                         B: Q^T B Q = I and X = QR within the T9 ceilings)
 *   orc_cholesky          pinned (exact hand cases, S:69 breakdown, T2 backward error)
 *   orc_trsm_rows         pinned (S:78 hand case, T3 row-wise backward error)
 *   orc_trmul             pinned (brute force)
 *   orc_power_lmax        pinned (diagonal / rank-one closed forms, numpy eigvalsh)
 *   orc_shift*            pinned (S:167-168, S:274 values, homogeneity)
 *   orc_scqr3             pinned (exact tiny QR, Householder brute force, invariants,
 *                         paper Tables 1-3 orders of magnitude, CholeskyQR2 breakdown)
 *   orc_orth_F / resid_F  pinned (Dot2 against exact integer cases)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_U 0x1p-53 /* unit roundoff u = 2^-53 (D1) */

/* ------------------------------------------------------------------------- */
/* Gram matrix A = X^T X  (eq. (1); Alg. 1 line 1; Alg. 2 line 3).
 * A_jl = sum_{i=1..m} x_ij x_il, summed over rows i in ascending order,
 * upper triangle computed and mirrored (exactly symmetric).
 * X is m x n column-major with leading dimension ld; A is n x n column-major.
 * Threads own disjoint sets of (j,l) entries; every entry is still summed over
 * i = 0..m-1 ascending, so the result is bit-identical to the serial loop. */
void orc_gram(int64_t m, int64_t n, const double* X, int64_t ld, double* A) {
  const int64_t npairs = n * (n + 1) / 2;
  double* acc = (double*)calloc((size_t)npairs, sizeof(double));
  const int64_t RB = 512; /* rows per block: a cache-friendly loop order only */
#pragma omp parallel
  {
    int nt = 1, tid = 0;
#ifdef _OPENMP
    nt = omp_get_num_threads();
    tid = omp_get_thread_num();
#endif
    /* pair p = (j,l), j<=l, enumerated column-wise over l */
    int64_t p0 = npairs * tid / nt, p1 = npairs * (tid + 1) / nt;
    int64_t* pj = (int64_t*)malloc((size_t)(p1 - p0 + 1) * sizeof(int64_t));
    int64_t* pl = (int64_t*)malloc((size_t)(p1 - p0 + 1) * sizeof(int64_t));
    {
      int64_t p = 0;
      for (int64_t l = 0; l < n; ++l)
        for (int64_t j = 0; j <= l; ++j, ++p)
          if (p >= p0 && p < p1) { pj[p - p0] = j; pl[p - p0] = l; }
    }
    for (int64_t i0 = 0; i0 < m; i0 += RB) {
      int64_t i1 = i0 + RB < m ? i0 + RB : m;
      for (int64_t p = p0; p < p1; ++p) {
        const double* xj = X + pj[p - p0] * ld;
        const double* xl = X + pl[p - p0] * ld;
        double s = acc[p];
        for (int64_t i = i0; i < i1; ++i) s = s + xj[i] * xl[i];
        acc[p] = s;
      }
    }
    free(pj);
    free(pl);
  }
  int64_t p = 0;
  for (int64_t l = 0; l < n; ++l)
    for (int64_t j = 0; j <= l; ++j, ++p) {
      A[j + l * n] = acc[p];
      A[l + j * n] = acc[p];
    }
  free(acc);
}

/* ------------------------------------------------------------------------- */
/* The SPD metric B of the oblique inner product (Alg. 4/5).
 *   tridiagonal: B(i,i) = d[i], B(i,i+1) = B(i+1,i) = e[i] (e[m-1] unused);
 *   CSR: row i holds cv[k] at column ci[k] for
 *   k = rp[i] .. rp[i+1]-1 (0-based global columns, B symmetric).
 * (B x)_i is formed row by row: tridiagonal d_i x_i + e_{i-1} x_{i-1} + e_i x_{i+1} (terms
 * in this order, missing neighbours omitted); CSR sum of cv[k] x[ci[k]] in storage order. */
typedef struct orc_metric {
  const double* d;
  const double* e;
  const int64_t* rp;
  const int32_t* ci;
  const double* cv;
} orc_metric;

static double bx_row(const orc_metric* B, int64_t m, const double* x, int64_t i) {
  if (B->rp) {
    double v = 0.0;
    for (int64_t k = B->rp[i]; k < B->rp[i + 1]; ++k) v = v + B->cv[k] * x[B->ci[k]];
    return v;
  }
  double v = B->d[i] * x[i];
  if (i > 0) v = v + B->e[i - 1] * x[i - 1];
  if (i + 1 < m) v = v + B->e[i] * x[i + 1];
  return v;
}

/* ||B||_inf = max_i sum_k |B_ik| >= ||B||_2 (Gershgorin, reading D4). */
static double metric_norm_inf(const orc_metric* B, int64_t m) {
  double nb = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    double r = 0.0;
    if (B->rp) {
      for (int64_t k = B->rp[i]; k < B->rp[i + 1]; ++k) r = r + fabs(B->cv[k]);
    } else {
      r = B->d[i];
      if (i > 0) r = r + fabs(B->e[i - 1]);
      if (i + 1 < m) r = r + fabs(B->e[i]);
    }
    if (r > nb) nb = r;
  }
  return nb;
}

/* Oblique Gram A = X^T B X (Alg. 4 line 1): Y = B X row by row, then
 * A = X^T Y summed over rows ascending, then symmetrised A <- (A + A^T)/2 because
 * fl(X^T (BX)) is not exactly symmetric.  colsq[j] = sum_i x_ij^2 (= diag(X^T X),
 * for the Frobenius bound, D4). */
static void gram_metric(int64_t m, int64_t n, const double* X, int64_t ld, const orc_metric* B, double* A,
                        double* colsq) {
  double* Y = (double*)malloc((size_t)m * (size_t)n * sizeof(double));
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j) {
    const double* x = X + j * ld;
    double* y = Y + j * m;
    for (int64_t i = 0; i < m; ++i) y[i] = bx_row(B, m, x, i);
  }
  double* G = (double*)malloc((size_t)n * (size_t)n * sizeof(double));
#pragma omp parallel for schedule(dynamic)
  for (int64_t jl = 0; jl < n * n; ++jl) {
    int64_t j = jl % n, l = jl / n;
    const double* xj = X + j * ld;
    const double* yl = Y + l * m;
    double s = 0.0;
    for (int64_t i = 0; i < m; ++i) s = s + xj[i] * yl[i];
    G[j + l * n] = s; /* (X^T Y)_jl */
  }
  for (int64_t l = 0; l < n; ++l)
    for (int64_t j = 0; j < n; ++j) A[j + l * n] = (G[j + l * n] + G[l + j * n]) * 0.5;
  if (colsq) {
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j) {
      const double* x = X + j * ld;
      double s = 0.0;
      for (int64_t i = 0; i < m; ++i) s = s + x[i] * x[i];
      colsq[j] = s;
    }
  }
  free(G);
  free(Y);
}

void orc_gram_oblique(int64_t m, int64_t n, const double* X, int64_t ld, const double* d,
                      const double* e, double* A, double* colsq) {
  const orc_metric B = {d, e, NULL, NULL, NULL};
  gram_metric(m, n, X, ld, &B, A, colsq);
}

void orc_gram_oblique_csr(int64_t m, int64_t n, const double* X, int64_t ld, const int64_t* rp,
                          const int32_t* ci, const double* cv, double* A, double* colsq) {
  const orc_metric B = {NULL, NULL, rp, ci, cv};
  gram_metric(m, n, X, ld, &B, A, colsq);
}

/* ------------------------------------------------------------------------- */
/* Cholesky factorisation R^T R = A + s I (eq. (2); Alg. 1 line 3, P:139;
 * computed-quantity model P:188).  Unblocked right-looking, upper R,
 * n x n column-major output with the strict lower triangle zero.
 * Breakdown (D9): the first pivot k (1-based) whose value before the square root
 * is <= 0 or not finite; returns 1 and reports (k, value); R is then undefined.
 * Returns 0 on success. */
int orc_cholesky(int64_t n, const double* A, double s, double* R, int64_t* piv, double* pivval) {
  double* W = (double*)malloc((size_t)n * (size_t)n * sizeof(double));
  for (int64_t l = 0; l < n; ++l)
    for (int64_t j = 0; j < n; ++j) W[j + l * n] = A[j + l * n];
  for (int64_t j = 0; j < n; ++j) W[j + j * n] = W[j + j * n] + s;
  memset(R, 0, (size_t)n * (size_t)n * sizeof(double));
  int rc = 0;
  for (int64_t k = 0; k < n; ++k) {
    double dkk = W[k + k * n];
    if (!(dkk > 0.0) || !isfinite(dkk)) {
      if (piv) *piv = k + 1;
      if (pivval) *pivval = dkk;
      rc = 1;
      break;
    }
    double rkk = sqrt(dkk);
    R[k + k * n] = rkk;
    for (int64_t j = k + 1; j < n; ++j) R[k + j * n] = W[k + j * n] / rkk;
    /* trailing update of the upper triangle: W_ij -= r_ki r_kj, k < i <= j */
    for (int64_t j = k + 1; j < n; ++j)
      for (int64_t i = k + 1; i <= j; ++i) W[i + j * n] = W[i + j * n] - R[k + i * n] * R[k + j * n];
  }
  if (rc == 0) {
    if (piv) *piv = 0;
    if (pivval) *pivval = 0.0;
  }
  free(W);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* Q = X R^{-1}, row by row (eq. (3); Alg. 1 line 4; per-row model
 * q_i^T = x_i^T (R + dR_i)^{-1}).  Forward substitution with
 * division on each row independently:
 *   q_ij = (x_ij - sum_{l<j} q_il r_lj) / r_jj,  l ascending.
 * Q may alias X when ldq == ldx. */
void orc_trsm_rows(int64_t m, int64_t n, const double* X, int64_t ldx, const double* R, double* Q,
                   int64_t ldq) {
#pragma omp parallel
  {
    double* q = (double*)malloc((size_t)n * sizeof(double));
#pragma omp for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
      for (int64_t j = 0; j < n; ++j) {
        double v = X[i + j * ldx];
        for (int64_t l = 0; l < j; ++l) v = v - q[l] * R[l + j * n];
        q[j] = v / R[j + j * n];
      }
      for (int64_t j = 0; j < n; ++j) Q[i + j * ldq] = q[j];
    }
    free(q);
  }
}

/* ------------------------------------------------------------------------- */
/* R := Rt * R for upper-triangular n x n column-major matrices (Alg. 2 line 8
 * "R := R~R"; Alg. 3 lines 6-7).
 * (Rt R)_ij = sum_{k=i..j} Rt_ik R_kj, k ascending. */
void orc_trmul(int64_t n, const double* Rt, double* R) {
  double* P = (double*)calloc((size_t)n * (size_t)n, sizeof(double));
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i <= j; ++i) {
      double s = 0.0;
      for (int64_t k = i; k <= j; ++k) s = s + Rt[i + k * n] * R[k + j * n];
      P[i + j * n] = s;
    }
  memcpy(R, P, (size_t)n * (size_t)n * sizeof(double));
  free(P);
}

/* ------------------------------------------------------------------------- */
/* Norm estimate ||X||_2^2 ~= lambda_max(A), A = X^T X ("estimate it
 * reliably using a norm estimator e.g. MATLAB's normest"; S:98-106 iterates
 * x -> X^T(X x), here on the already-computed Gram, reading D2).
 * Power iteration from the all-ones vector, `iters` steps, then the Rayleigh
 * quotient x^T A x of the unit iterate.  Returns lambda (no inflation). */
double orc_power_lmax(int64_t n, const double* A, int iters) {
  double* x = (double*)malloc((size_t)n * sizeof(double));
  double* y = (double*)malloc((size_t)n * sizeof(double));
  double nx = sqrt((double)n);
  for (int64_t i = 0; i < n; ++i) x[i] = 1.0 / nx;
  for (int it = 0; it < iters; ++it) {
    double ss = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double v = 0.0;
      for (int64_t j = 0; j < n; ++j) v = v + A[i + j * n] * x[j];
      y[i] = v;
      ss = ss + v * v;
    }
    double ny = sqrt(ss);
    if (!(ny > 0.0)) break;
    for (int64_t i = 0; i < n; ++i) x[i] = y[i] / ny;
  }
  double lam = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double v = 0.0;
    for (int64_t j = 0; j < n; ++j) v = v + A[i + j * n] * x[j];
    lam = lam + x[i] * v;
  }
  free(x);
  free(y);
  return lam;
}

/* Shift s = 11{mn + n(n+1)} u ||X||_2^2  (eq. (finds2)).
 * N2 is the (estimate of) ||X||_2^2. */
double orc_shift(double m, double n, double N2) { return 11.0 * (m * n + n * (n + 1.0)) * ORC_U * N2; }

/* Oblique shift s = 11{2m sqrt(mn) + n(n+1)} u ||X||_2^2 ||B||_2  (eq. (finds2B),
 * P:1303-1306). */
double orc_shift_oblique(double m, double n, double NX2, double NB) {
  return 11.0 * (2.0 * m * sqrt(m * n) + n * (n + 1.0)) * ORC_U * NX2 * NB;
}

/* ------------------------------------------------------------------------- */
/* Error-free transformations and Dot2 (Ogita-Rump-Oishi), used only by the
 * metrics below, which need accuracy beyond the quantities they measure (F6). */
static inline void two_sum(double a, double b, double* s, double* e) {
  double x = a + b, z = x - a;
  *e = (a - (x - z)) + (b - z);
  *s = x;
}
static inline void two_prod(double a, double b, double* p, double* e) {
  double x = a * b;
  *e = fma(a, b, -x);
  *p = x;
}

/* ||Q^T Y - I||_F with compensated (Dot2) accumulation of every entry, Y = B Q (Y == NULL:
 * B = I).  Orthogonality measure of P:1547, P:1633 (Frobenius). */
static double orth_core(int64_t m, int64_t n, const double* Q, int64_t ld, const double* Y) {
  double tot = 0.0;
#pragma omp parallel for schedule(dynamic) reduction(+ : tot)
  for (int64_t jl = 0; jl < n * n; ++jl) {
    int64_t j = jl % n, l = jl / n;
    if (j > l) continue;
    const double* a = Q + j * ld;
    const double* b = Y ? Y + l * m : Q + l * ld;
    double s = 0, c = 0, p, pe, t, te;
    for (int64_t i = 0; i < m; ++i) {
      two_prod(a[i], b[i], &p, &pe);
      two_sum(s, p, &t, &te);
      s = t;
      c += te + pe;
    }
    double v = s + c;
    if (j == l) v = v - 1.0;
    tot += (j == l ? 1.0 : 2.0) * v * v;
  }
  return sqrt(tot);
}

/* ||Q^T B Q - I||_F, B tridiagonal (d, e) or I (d == NULL); y = B q in double-double. */
double orc_orth_F(int64_t m, int64_t n, const double* Q, int64_t ld, const double* d, const double* e) {
  double* Y = NULL;
  if (d) {
    Y = (double*)malloc((size_t)m * (size_t)n * sizeof(double));
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < m; ++i) {
        /* y = B q computed in double-double, rounded once */
        double s = 0, c = 0, p, pe, t, te;
        two_prod(d[i], Q[i + j * ld], &p, &pe);
        two_sum(s, p, &t, &te); s = t; c += te + pe;
        if (i > 0) { two_prod(e[i - 1], Q[i - 1 + j * ld], &p, &pe); two_sum(s, p, &t, &te); s = t; c += te + pe; }
        if (i + 1 < m) { two_prod(e[i], Q[i + 1 + j * ld], &p, &pe); two_sum(s, p, &t, &te); s = t; c += te + pe; }
        Y[i + j * m] = s + c;
      }
  }
  const double r = orth_core(m, n, Q, ld, Y);
  free(Y);
  return r;
}

/* ||Q^T B Q - I||_F for a CSR metric B; y = B q in double-double. */
double orc_orth_F_csr(int64_t m, int64_t n, const double* Q, int64_t ld, const int64_t* rp, const int32_t* ci,
                      const double* cv) {
  double* Y = (double*)malloc((size_t)m * (size_t)n * sizeof(double));
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) {
      double s = 0, c = 0, p, pe, t, te;
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
        two_prod(cv[k], Q[ci[k] + j * ld], &p, &pe);
        two_sum(s, p, &t, &te);
        s = t;
        c += te + pe;
      }
      Y[i + j * m] = s + c;
    }
  const double r = orth_core(m, n, Q, ld, Y);
  free(Y);
  return r;
}

/* ||X - Q R||_F / ||X||_F with compensated row products (D13). */
double orc_resid_F(int64_t m, int64_t n, const double* X, int64_t ldx, const double* Q, int64_t ldq,
                   const double* R) {
  double num = 0.0, den = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : num, den)
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t j = 0; j < n; ++j) {
      double s = -X[i + j * ldx], c = 0, p, pe, t, te;
      for (int64_t l = 0; l <= j; ++l) {
        two_prod(Q[i + l * ldq], R[l + j * n], &p, &pe);
        two_sum(s, p, &t, &te);
        s = t;
        c += te + pe;
      }
      double r = s + c;
      num += r * r;
      den += X[i + j * ldx] * X[i + j * ldx];
    }
  }
  return sqrt(num) / sqrt(den);
}

/* ------------------------------------------------------------------------- */
/* The pass controller (Alg. 3, with Alg. 2's breakdown-triggered
 * re-shift; readings D2-D6, D8 in DESIGN.md).
 *
 *   Q := X, R := I, k := 0
 *   repeat
 *     k := k+1
 *     A := Q^T Q            (oblique: Q^T B Q, all passes -- D8)
 *     N2 := ||Q||_2^2 estimate (norm_mode)
 *     s := 11{mn+n(n+1)} u N2  (oblique: eq. finds2B)
 *     if k == 1: R~ := chol(A + sI)                       (Alg. 3 line 4)
 *     else:      R~ := chol(A); on breakdown R~ := chol(A + sI)   (Alg. 2 lines 4-7)
 *   shift_mode ADAPTIVE (Alg. 2 literal): pass 1 too is tried unshifted first.
 *   shift_mode PRACTICAL (the Remark after eq. finds2B, Fig. 2): every shifted
 *     attempt first uses s_p = u N2 (oblique: u N2 N_B); if chol(A + s_p I) breaks down it
 *     falls back to the safe s (reading D21), so Alg. 3's guarantee is kept.
 *     breakdown with the shift -> status 2
 *     Q := Q R~^{-1},  R := R~ R                           (Alg. 2 line 8)
 *   until (R~ was unshifted and ||A - I||_F <= stop_tol)    (D6)
 *   k == max_passes without stopping -> status 3
 */
typedef struct orc_opts {
  int shift_mode;      /* 0 SAFE (eq. finds2/finds2B), 1 FIXED (shift_value on pass 1), 2 NONE,
                          3 ADAPTIVE (Alg. 2: shift only on breakdown), 4 PRACTICAL (s_p = u N2 first) */
  double shift_value;
  int norm_mode;       /* 0 POWER (lambda_max of the Gram x 1.01), 1 FROBENIUS (trace), 2 USER */
  double norm2_bound;  /* USER: N >= ||X||_2 for pass 1 */
  double bnorm_bound;  /* oblique: bound on ||B||_2 (0 => Gershgorin max_i d_i+|e_{i-1}|+|e_i|) */
  int max_passes;      /* default 8 */
  double stop_tol;     /* default 0.5 */
  int power_iters;     /* default 32 */
  double m_global;     /* m used in the shift formula (0 => m) */
  int nparts;          /* emulate a P-rank Gram: shard Grams summed in rank order (1 = plain) */
} orc_opts;

typedef struct orc_trace {
  double shift;
  int shifted;
  int breakdown_pivot; /* 0 = none (plain attempt), else 1-based pivot of the failed plain attempt */
  double pivot_value;
  double norm2_est;
  double dev_F;        /* ||A_k - I||_F of the pass's input Gram */
} orc_trace;

static void gram_any(int64_t m, int64_t n, const double* Q, int64_t ld, const orc_metric* B,
                     int nparts, double* A, double* colsq) {
  const int d = B != NULL; /* oblique */
  if (nparts <= 1) {
    if (d) gram_metric(m, n, Q, ld, B, A, colsq);
    else orc_gram(m, n, Q, ld, A);
    return;
  }
  /* P-rank emulation: each contiguous shard's Gram, summed in rank order.
   * Oblique shards see their neighbours' boundary rows exactly as the halo would. */
  double* Ap = (double*)malloc((size_t)n * (size_t)n * sizeof(double));
  double* cp = (double*)malloc((size_t)n * sizeof(double));
  memset(A, 0, (size_t)n * (size_t)n * sizeof(double));
  if (colsq) memset(colsq, 0, (size_t)n * sizeof(double));
  for (int p = 0; p < nparts; ++p) {
    int64_t r0 = m * p / nparts, r1 = m * (p + 1) / nparts;
    if (r1 <= r0) continue;
    if (!d) {
      orc_gram(r1 - r0, n, Q + r0, ld, Ap);
    } else {
      /* shard Gram: X_p^T (B X)_p where (B X)_p uses halo rows r0-1 and r1 */
      int64_t mp = r1 - r0;
      double* Y = (double*)malloc((size_t)mp * (size_t)n * sizeof(double));
      for (int64_t j = 0; j < n; ++j)
        for (int64_t i = r0; i < r1; ++i) Y[(i - r0) + j * mp] = bx_row(B, m, Q + j * ld, i);
      for (int64_t l = 0; l < n; ++l)
        for (int64_t j = 0; j < n; ++j) {
          double s = 0.0;
          for (int64_t i = 0; i < mp; ++i) s = s + Q[r0 + i + j * ld] * Y[i + l * mp];
          Ap[j + l * n] = s;
        }
      free(Y);
      for (int64_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (int64_t i = r0; i < r1; ++i) s = s + Q[i + j * ld] * Q[i + j * ld];
        cp[j] = s;
      }
    }
    for (int64_t i = 0; i < n * n; ++i) A[i] = A[i] + Ap[i];
    if (colsq && d)
      for (int64_t j = 0; j < n; ++j) colsq[j] = colsq[j] + cp[j];
  }
  if (d) { /* symmetrise the summed non-symmetric Gram */
    for (int64_t l = 0; l < n; ++l)
      for (int64_t j = 0; j < l; ++j) {
        double v = (A[j + l * n] + A[l + j * n]) * 0.5;
        A[j + l * n] = v;
        A[l + j * n] = v;
      }
  }
  free(Ap);
  free(cp);
}

/* The Gram of one pass as gram_any forms it (exported for pins): nparts contiguous row blocks,
 * each block's (oblique: X_p^T (B X)_p with the neighbours' boundary rows as halo) Gram summed
 * in rank order; oblique results symmetrised after the sum.  d/e (tridiagonal) or rp/ci/cv
 * (CSR, global column indices) select the metric; all NULL = the plain Gram. */
void orc_gram_parts(int64_t m, int64_t n, const double* X, int64_t ld, const double* d, const double* e,
                    const int64_t* rp, const int32_t* ci, const double* cv, int nparts, double* A,
                    double* colsq) {
  const orc_metric B = {d, e, rp, ci, cv};
  const int oblique = d != NULL || rp != NULL;
  gram_any(m, n, X, ld, oblique ? &B : NULL, nparts, A, colsq);
}

/* Returns 0 ok, 2 breakdown even with the shift, 3 not converged, 1 bad argument. */
static int scqr3_impl(int64_t m, int64_t n, const double* X, int64_t ld, const orc_metric* B,
                      double* Q, int64_t ldq, double* R, const orc_opts* o, orc_trace* trace, int trace_cap,
                      int* passes_out) {
  if (m < 1 || n < 1 || ld < m || ldq < m) return 1;
  const int max_passes = o->max_passes > 0 ? o->max_passes : 8;
  const double stop_tol = o->stop_tol > 0 ? o->stop_tol : 0.5;
  const int iters = o->power_iters > 0 ? o->power_iters : 32;
  const double mg = o->m_global > 0 ? o->m_global : (double)m;
  const int oblique = B != NULL;

  double NB = 0.0;
  if (oblique) NB = o->bnorm_bound > 0 ? o->bnorm_bound : metric_norm_inf(B, m); /* (D4) */

  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) Q[i + j * ldq] = X[i + j * ld];
  memset(R, 0, (size_t)n * (size_t)n * sizeof(double));
  for (int64_t j = 0; j < n; ++j) R[j + j * n] = 1.0;

  double* A = (double*)malloc((size_t)n * (size_t)n * sizeof(double));
  double* Rt = (double*)malloc((size_t)n * (size_t)n * sizeof(double));
  double* colsq = (double*)malloc((size_t)n * sizeof(double));
  double* Pg = (double*)malloc((size_t)n * (size_t)n * sizeof(double)); /* oblique: plain Gram for N2 */
  int status = 3, k = 0;
  for (k = 1; k <= max_passes; ++k) {
    gram_any(m, n, Q, ldq, B, o->nparts, A, colsq);
    double dev = 0.0;
    for (int64_t l = 0; l < n; ++l)
      for (int64_t j = 0; j < n; ++j) {
        double v = A[j + l * n] - (j == l ? 1.0 : 0.0);
        dev = dev + v * v;
      }
    dev = sqrt(dev);
    if (k == 1) { /* non-finite X is an invalid argument: it reaches the Gram's diagonal */
      int bad = 0;
      for (int64_t j = 0; j < n; ++j)
        if (!isfinite(A[j + j * n])) bad = 1;
      if (bad) {
        status = 1;
        break;
      }
    }
    /* norm estimate N2 ~ ||Q||_2^2.  Oblique (D4): lambda_max of the plain Gram Q^T Q by power
     * iteration x 1.01 (the norm estimator of P:660, formed alongside the B-Gram), or ||Q||_F^2
     * (FROBENIUS), or the user bound on pass 1 */
    double N2;
    if (oblique) {
      if (k == 1 && o->norm_mode == 2) N2 = o->norm2_bound * o->norm2_bound;
      else if (o->norm_mode == 1) {
        N2 = 0.0;
        for (int64_t j = 0; j < n; ++j) N2 = N2 + colsq[j]; /* ||Q||_F^2 >= ||Q||_2^2 */
      } else {
        gram_any(m, n, Q, ldq, NULL, o->nparts, Pg, NULL);
        N2 = orc_power_lmax(n, Pg, iters) * 1.01;
      }
    } else if (k == 1 && o->norm_mode == 2) {
      N2 = o->norm2_bound * o->norm2_bound;
    } else if (o->norm_mode == 1) {
      N2 = 0.0;
      for (int64_t j = 0; j < n; ++j) N2 = N2 + A[j + j * n];
    } else {
      N2 = orc_power_lmax(n, A, iters) * 1.01;
    }
    double s;
    if (o->shift_mode == 1 && k == 1) s = o->shift_value;
    else if (oblique) s = orc_shift_oblique(mg, (double)n, N2, NB);
    else s = orc_shift(mg, (double)n, N2);

    /* the practical shift of the Remark: u ||X||_2^2 ||B||_2 */
    const double sp = 0x1p-53 * N2 * (oblique ? NB : 1.0);
    const int practical = o->shift_mode == 4;
    int64_t piv = 0;
    double pv = 0.0;
    int shifted = 0, bpiv = 0;
    double bval = 0.0, s_used = 0.0;
    int rc;
    const int shift_first = k == 1 && (o->shift_mode == 0 || o->shift_mode == 1 || practical);
    if (!shift_first) {
      rc = orc_cholesky(n, A, 0.0, Rt, &piv, &pv);
      if (rc) { bpiv = (int)piv; bval = pv; }
    } else {
      rc = 1;
    }
    if (rc && o->shift_mode != 2) {
      /* shifted attempt(s): PRACTICAL tries s_p before the safe s */
      shifted = 1;
      s_used = practical ? sp : s;
      rc = orc_cholesky(n, A, s_used, Rt, &piv, &pv);
      if (rc) { bpiv = (int)piv; bval = pv; }
      if (rc && practical) {
        s_used = s;
        rc = orc_cholesky(n, A, s_used, Rt, &piv, &pv);
        if (rc) { bpiv = (int)piv; bval = pv; }
      }
    }
    if (trace && k - 1 < trace_cap) {
      trace[k - 1].shift = shifted ? s_used : 0.0;
      trace[k - 1].shifted = shifted;
      trace[k - 1].breakdown_pivot = bpiv;
      trace[k - 1].pivot_value = bval;
      trace[k - 1].norm2_est = N2;
      trace[k - 1].dev_F = dev;
    }
    if (rc) {
      status = 2;
      break;
    }
    orc_trsm_rows(m, n, Q, ldq, Rt, Q, ldq);
    orc_trmul(n, Rt, R);
    if (!shifted && dev <= stop_tol) {
      status = 0;
      break;
    }
  }
  if (passes_out) *passes_out = k > max_passes ? max_passes : k;
  free(A);
  free(Rt);
  free(colsq);
  free(Pg);
  return status;
}

int orc_scqr3(int64_t m, int64_t n, const double* X, int64_t ld, const double* d, const double* e,
              double* Q, int64_t ldq, double* R, const orc_opts* o, orc_trace* trace, int trace_cap,
              int* passes_out) {
  const orc_metric B = {d, e, NULL, NULL, NULL};
  return scqr3_impl(m, n, X, ld, d ? &B : NULL, Q, ldq, R, o, trace, trace_cap, passes_out);
}

/* Oblique shifted CholeskyQR3 with a general sparse SPD B in CSR. */
int orc_scqr3_csr(int64_t m, int64_t n, const double* X, int64_t ld, const int64_t* rp, const int32_t* ci,
                  const double* cv, double* Q, int64_t ldq, double* R, const orc_opts* o, orc_trace* trace,
                  int trace_cap, int* passes_out) {
  if (!rp || !ci || !cv) return 1;
  const orc_metric B = {NULL, NULL, rp, ci, cv};
  return scqr3_impl(m, n, X, ld, &B, Q, ldq, R, o, trace, trace_cap, passes_out);
}

/* ========================================================================= */
/* Complex matrices ("everything carries over to complex matrices", P:124-125;
 * reading D23: transposes become conjugate transposes, u = 2^-53, the shift formula unchanged).
 * Storage: column-major interleaved complex, element (i, j) at Z[2(i + j ld)] (re), +1 (im).
 * Complex arithmetic is written out on real parts in a fixed order, so a real input (all
 * imaginary parts 0) reproduces the real functions above bit for bit (a pin). */
#define ZRE(Z, i, j, ld) (Z)[2 * ((i) + (j) * (ld))]
#define ZIM(Z, i, j, ld) (Z)[2 * ((i) + (j) * (ld)) + 1]

/* A = X^H X (n x n, Hermitian, full), rows ascending: A_jl = sum_i conj(x_ij) x_il for j <= l,
 * A_lj = conj(A_jl) (Alg. 1 line 1 with ^T -> ^H). */
void orc_zgram(int64_t m, int64_t n, const double* X, int64_t ld, double* A) {
#pragma omp parallel for schedule(dynamic)
  for (int64_t jl = 0; jl < n * n; ++jl) {
    const int64_t j = jl % n, l = jl / n;
    if (j > l) continue;
    double re = 0.0, im = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      const double a = ZRE(X, i, j, ld), b = ZIM(X, i, j, ld), c = ZRE(X, i, l, ld), d = ZIM(X, i, l, ld);
      re = re + (a * c + b * d); /* conj(a + ib)(c + id) */
      im = im + (a * d - b * c);
    }
    ZRE(A, j, l, n) = re;
    ZIM(A, j, l, n) = j == l ? 0.0 : im;
    ZRE(A, l, j, n) = re;
    ZIM(A, l, j, n) = j == l ? 0.0 : -im;
  }
}

/* R^H R = A + sI (upper R, real positive diagonal), unblocked right-looking; breakdown at the
 * first pivot (real part of the diagonal) <= 0 or non-finite, as orc_cholesky. */
int orc_zcholesky(int64_t n, const double* A, double s, double* R, int64_t* piv, double* pivval) {
  double* W = (double*)malloc((size_t)n * (size_t)n * 2 * sizeof(double));
  memcpy(W, A, (size_t)n * (size_t)n * 2 * sizeof(double));
  for (int64_t j = 0; j < n; ++j) ZRE(W, j, j, n) = ZRE(W, j, j, n) + s;
  memset(R, 0, (size_t)n * (size_t)n * 2 * sizeof(double));
  int rc = 0;
  for (int64_t k = 0; k < n; ++k) {
    const double dkk = ZRE(W, k, k, n);
    if (!(dkk > 0.0) || !isfinite(dkk) || !isfinite(ZIM(W, k, k, n))) {
      if (piv) *piv = k + 1;
      if (pivval) *pivval = dkk;
      rc = 1;
      break;
    }
    const double rkk = sqrt(dkk);
    ZRE(R, k, k, n) = rkk;
    for (int64_t j = k + 1; j < n; ++j) {
      ZRE(R, k, j, n) = ZRE(W, k, j, n) / rkk;
      ZIM(R, k, j, n) = ZIM(W, k, j, n) / rkk;
    }
    /* W_ij -= conj(r_ki) r_kj, k < i <= j */
    for (int64_t j = k + 1; j < n; ++j)
      for (int64_t i = k + 1; i <= j; ++i) {
        const double a = ZRE(R, k, i, n), b = ZIM(R, k, i, n), c = ZRE(R, k, j, n), d = ZIM(R, k, j, n);
        ZRE(W, i, j, n) = ZRE(W, i, j, n) - (a * c + b * d);
        ZIM(W, i, j, n) = ZIM(W, i, j, n) - (a * d - b * c);
      }
  }
  if (rc == 0) {
    if (piv) *piv = 0;
    if (pivval) *pivval = 0.0;
  }
  free(W);
  return rc;
}

/* Q = X R^{-1} row by row: q_ij = (x_ij - sum_{l<j} q_il r_lj) / r_jj (r_jj real). */
void orc_ztrsm_rows(int64_t m, int64_t n, const double* X, int64_t ldx, const double* R, double* Q, int64_t ldq) {
#pragma omp parallel
  {
    double* q = (double*)malloc((size_t)n * 2 * sizeof(double));
#pragma omp for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
      for (int64_t j = 0; j < n; ++j) {
        double vr = ZRE(X, i, j, ldx), vi = ZIM(X, i, j, ldx);
        for (int64_t l = 0; l < j; ++l) {
          const double a = q[2 * l], b = q[2 * l + 1], c = ZRE(R, l, j, n), d = ZIM(R, l, j, n);
          vr = vr - (a * c - b * d); /* (a + ib)(c + id) */
          vi = vi - (a * d + b * c);
        }
        const double rjj = ZRE(R, j, j, n);
        q[2 * j] = vr / rjj;
        q[2 * j + 1] = vi / rjj;
      }
      for (int64_t j = 0; j < n; ++j) {
        ZRE(Q, i, j, ldq) = q[2 * j];
        ZIM(Q, i, j, ldq) = q[2 * j + 1];
      }
    }
    free(q);
  }
}

/* R := Rt R (upper, complex): (Rt R)_ij = sum_{k=i..j} Rt_ik R_kj, k ascending. */
void orc_ztrmul(int64_t n, const double* Rt, double* R) {
  double* P = (double*)calloc((size_t)n * (size_t)n * 2, sizeof(double));
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i <= j; ++i) {
      double re = 0.0, im = 0.0;
      for (int64_t k = i; k <= j; ++k) {
        const double a = ZRE(Rt, i, k, n), b = ZIM(Rt, i, k, n), c = ZRE(R, k, j, n), d = ZIM(R, k, j, n);
        re = re + (a * c - b * d);
        im = im + (a * d + b * c);
      }
      ZRE(P, i, j, n) = re;
      ZIM(P, i, j, n) = im;
    }
  memcpy(R, P, (size_t)n * (size_t)n * 2 * sizeof(double));
  free(P);
}

/* lambda_max of Hermitian A by power iteration from the all-ones vector (as orc_power_lmax),
 * Rayleigh quotient Re(x^H A x). */
double orc_zpower_lmax(int64_t n, const double* A, int iters) {
  double* x = (double*)malloc((size_t)n * 2 * sizeof(double));
  double* y = (double*)malloc((size_t)n * 2 * sizeof(double));
  const double nx = sqrt((double)n);
  for (int64_t i = 0; i < n; ++i) { x[2 * i] = 1.0 / nx; x[2 * i + 1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
    double ss = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double vr = 0.0, vi = 0.0;
      for (int64_t j = 0; j < n; ++j) {
        const double a = ZRE(A, i, j, n), b = ZIM(A, i, j, n), c = x[2 * j], d = x[2 * j + 1];
        vr = vr + (a * c - b * d);
        vi = vi + (a * d + b * c);
      }
      y[2 * i] = vr;
      y[2 * i + 1] = vi;
      ss = ss + (vr * vr + vi * vi);
    }
    const double ny = sqrt(ss);
    if (!(ny > 0.0)) break;
    for (int64_t i = 0; i < 2 * n; ++i) x[i] = y[i] / ny;
  }
  double lam = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double vr = 0.0, vi = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      const double a = ZRE(A, i, j, n), b = ZIM(A, i, j, n), c = x[2 * j], d = x[2 * j + 1];
      vr = vr + (a * c - b * d);
      vi = vi + (a * d + b * c);
    }
    lam = lam + (x[2 * i] * vr + x[2 * i + 1] * vi); /* Re(conj(x_i) v_i) */
  }
  free(x);
  free(y);
  return lam;
}

/* ||Q^H Q - I||_F, every entry accumulated in double-double (Dot2 on real and imaginary parts). */
double orc_zorth_F(int64_t m, int64_t n, const double* Q, int64_t ld) {
  double tot = 0.0;
#pragma omp parallel for schedule(dynamic) reduction(+ : tot)
  for (int64_t jl = 0; jl < n * n; ++jl) {
    const int64_t j = jl % n, l = jl / n;
    if (j > l) continue;
    double sr = 0, cr = 0, si = 0, ci = 0, p, pe, t, te;
    for (int64_t i = 0; i < m; ++i) {
      const double a = ZRE(Q, i, j, ld), b = ZIM(Q, i, j, ld), c = ZRE(Q, i, l, ld), d = ZIM(Q, i, l, ld);
      two_prod(a, c, &p, &pe); two_sum(sr, p, &t, &te); sr = t; cr += te + pe;
      two_prod(b, d, &p, &pe); two_sum(sr, p, &t, &te); sr = t; cr += te + pe;
      two_prod(a, d, &p, &pe); two_sum(si, p, &t, &te); si = t; ci += te + pe;
      two_prod(-b, c, &p, &pe); two_sum(si, p, &t, &te); si = t; ci += te + pe;
    }
    double vr = sr + cr, vi = si + ci;
    if (j == l) vr = vr - 1.0;
    tot += (j == l ? 1.0 : 2.0) * (vr * vr + vi * vi);
  }
  return sqrt(tot);
}

/* ||X - Q R||_F / ||X||_F, compensated row products. */
double orc_zresid_F(int64_t m, int64_t n, const double* X, int64_t ldx, const double* Q, int64_t ldq,
                    const double* R) {
  double num = 0.0, den = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : num, den)
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t j = 0; j < n; ++j) {
      double sr = -ZRE(X, i, j, ldx), si = -ZIM(X, i, j, ldx), cr = 0, ci = 0, p, pe, t, te;
      for (int64_t l = 0; l <= j; ++l) {
        const double a = ZRE(Q, i, l, ldq), b = ZIM(Q, i, l, ldq), c = ZRE(R, l, j, n), d = ZIM(R, l, j, n);
        two_prod(a, c, &p, &pe); two_sum(sr, p, &t, &te); sr = t; cr += te + pe;
        two_prod(-b, d, &p, &pe); two_sum(sr, p, &t, &te); sr = t; cr += te + pe;
        two_prod(a, d, &p, &pe); two_sum(si, p, &t, &te); si = t; ci += te + pe;
        two_prod(b, c, &p, &pe); two_sum(si, p, &t, &te); si = t; ci += te + pe;
      }
      const double rr = sr + cr, ri = si + ci;
      num += rr * rr + ri * ri;
      den += ZRE(X, i, j, ldx) * ZRE(X, i, j, ldx) + ZIM(X, i, j, ldx) * ZIM(X, i, j, ldx);
    }
  }
  return sqrt(num / den);
}

/* Shifted CholeskyQR3 for complex X (standard inner product): the pass controller of
 * scqr3_impl with ^T -> ^H (shift modes, re-shift on breakdown, stop rule D6). */
int orc_zscqr3(int64_t m, int64_t n, const double* X, int64_t ld, double* Q, int64_t ldq, double* R,
               const orc_opts* o, orc_trace* trace, int trace_cap, int* passes_out) {
  if (m < 1 || n < 1 || ld < m || ldq < m) return 1;
  const int max_passes = o->max_passes > 0 ? o->max_passes : 8;
  const double stop_tol = o->stop_tol > 0 ? o->stop_tol : 0.5;
  const int iters = o->power_iters > 0 ? o->power_iters : 32;
  const double mg = o->m_global > 0 ? o->m_global : (double)m;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) {
      ZRE(Q, i, j, ldq) = ZRE(X, i, j, ld);
      ZIM(Q, i, j, ldq) = ZIM(X, i, j, ld);
    }
  memset(R, 0, (size_t)n * (size_t)n * 2 * sizeof(double));
  for (int64_t j = 0; j < n; ++j) ZRE(R, j, j, n) = 1.0;
  double* A = (double*)malloc((size_t)n * (size_t)n * 2 * sizeof(double));
  double* Rt = (double*)malloc((size_t)n * (size_t)n * 2 * sizeof(double));
  int status = 3, k = 0;
  for (k = 1; k <= max_passes; ++k) {
    orc_zgram(m, n, Q, ldq, A);
    double dev = 0.0;
    for (int64_t l = 0; l < n; ++l)
      for (int64_t j = 0; j < n; ++j) {
        const double vr = ZRE(A, j, l, n) - (j == l ? 1.0 : 0.0), vi = ZIM(A, j, l, n);
        dev = dev + (vr * vr + vi * vi);
      }
    dev = sqrt(dev);
    if (k == 1) {
      int bad = 0;
      for (int64_t j = 0; j < n; ++j)
        if (!isfinite(ZRE(A, j, j, n))) bad = 1;
      if (bad) { status = 1; break; }
    }
    double N2;
    if (k == 1 && o->norm_mode == 2) N2 = o->norm2_bound * o->norm2_bound;
    else if (o->norm_mode == 1) {
      N2 = 0.0;
      for (int64_t j = 0; j < n; ++j) N2 = N2 + ZRE(A, j, j, n);
    } else {
      N2 = orc_zpower_lmax(n, A, iters) * 1.01;
    }
    const double s = (o->shift_mode == 1 && k == 1) ? o->shift_value : orc_shift(mg, (double)n, N2);
    const double sp = 0x1p-53 * N2;
    const int practical = o->shift_mode == 4;
    int64_t piv = 0;
    double pv = 0.0, bval = 0.0, s_used = 0.0;
    int shifted = 0, bpiv = 0, rc;
    const int shift_first = k == 1 && (o->shift_mode == 0 || o->shift_mode == 1 || practical);
    if (!shift_first) {
      rc = orc_zcholesky(n, A, 0.0, Rt, &piv, &pv);
      if (rc) { bpiv = (int)piv; bval = pv; }
    } else {
      rc = 1;
    }
    if (rc && o->shift_mode != 2) {
      shifted = 1;
      s_used = practical ? sp : s;
      rc = orc_zcholesky(n, A, s_used, Rt, &piv, &pv);
      if (rc) { bpiv = (int)piv; bval = pv; }
      if (rc && practical) {
        s_used = s;
        rc = orc_zcholesky(n, A, s_used, Rt, &piv, &pv);
        if (rc) { bpiv = (int)piv; bval = pv; }
      }
    }
    if (trace && k - 1 < trace_cap) {
      trace[k - 1].shift = shifted ? s_used : 0.0;
      trace[k - 1].shifted = shifted;
      trace[k - 1].breakdown_pivot = bpiv;
      trace[k - 1].pivot_value = bval;
      trace[k - 1].norm2_est = N2;
      trace[k - 1].dev_F = dev;
    }
    if (rc) { status = 2; break; }
    orc_ztrsm_rows(m, n, Q, ldq, Rt, Q, ldq);
    orc_ztrmul(n, Rt, R);
    if (!shifted && dev <= stop_tol) { status = 0; break; }
  }
  if (passes_out) *passes_out = k > max_passes ? max_passes : k;
  free(A);
  free(Rt);
  return status;
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void orc_set_num_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}
