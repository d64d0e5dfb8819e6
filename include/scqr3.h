/*
 * scqr3.h -- C ABI of libscqr3.so: shifted CholeskyQR3 for tall-skinny fp64 matrices on
 * NVIDIA B200 (sm_100a).
 *
 * Method: Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa, "Shifted CholeskyQR for
 * computing the QR factorization of ill-conditioned matrices" (arXiv:1809.11085).
 * Citations "P:L" are lines of the paper's text; readings "Dn" are listed in
 * DESIGN.md.  Everything is IEEE binary64 (u = 2^-53).
 *
 * Conventions common to every entry point
 *   - Matrices are COLUMN-MAJOR.  X, Q are m x n with leading dimensions ld, ldq >= m.
 *     R is n x n with leading dimension n; on success its strict lower triangle is zero
 *     and its diagonal is positive, so it is the unique R factor.
 *   - Pointers are DEVICE pointers unless the name ends in _host.  The caller owns all
 *     memory (allocated e.g. with torch); the library allocates nothing per call on the
 *     device (it keeps a small pinned host status block and two events per thread).
 *   - TMA requirements: X, Q 16-byte aligned and ld, ldq even (8*ld % 16 == 0).
 *   - Supported sizes: 1 <= n <= 512 (SURVEY 8(b) contract), m_global >= n, m >= 0 on
 *     every rank (an oblique metric across ranks needs m >= its halo rows on every rank).
 *     n in (128, 512] is padded to the next compiled width (192, 256 or 512) and its TRSM runs
 *     as block-column launches: columns 0..127 by the register-resident kernel, then the
 *     targets 16..31 (16..23 for n <= 192), then for n > 256 up to five launches for the
 *     targets 32..40, 40..48, 48..56, 56..60, 60..64 (8-column tiles), each skipped when its
 *     targets lie wholly past n.
 *   - With opts->comm, argument errors are agreed collectively: if any rank's arguments are
 *     invalid, every rank returns SCQR3_EINVAL before the first exchange.
 *   - All device work is ordered on opts->stream; every call returns only after that
 *     work has finished (the pass count is data dependent).
 *   - Return codes: SCQR3_OK; SCQR3_EINVAL (bad argument -- including NaN/Inf entries in X,
 *     detected from the pass-1 Gram -- CUDA or NCCL error; detail in
 *     scqr3_last_error()); SCQR3_EBREAKDOWN (Cholesky broke down even with the shift:
 *     out of the method's regime or rank deficient); SCQR3_ENOCONV (no stop
 *     within max_passes).  On a non-OK return Q and R are unspecified; the trace is valid.
 */
#ifndef SCQR3_H
#define SCQR3_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCQR3_ABI_VERSION 2

enum { SCQR3_OK = 0, SCQR3_EINVAL = 1, SCQR3_EBREAKDOWN = 2, SCQR3_ENOCONV = 3 };

/* Shift policy.  SAFE: s = 11{mn+n(n+1)} u N^2 (eq. finds2) or the
 * oblique 11{2m sqrt(mn)+n(n+1)} u N^2 ||B|| (eq. finds2B) on pass 1 and on any
 * later pass whose plain Cholesky breaks down (Alg. 2 lines 4-7).
 * FIXED: shift_value on pass 1 (kernel-level parity tests), SAFE on breakdown.
 * NONE: no shift ever (plain iterated CholeskyQR, for tests; breakdown is final).
 * ADAPTIVE: Alg. 2 literally -- pass 1 is also tried unshifted and shifted only
 *   when its Cholesky breaks down: CholeskyQR2 (2 passes) for kappa(X) up to ~u^-1/2.
 * PRACTICAL: pass 1 (and any breakdown) first shifted by s_p = u N^2 (oblique: u N^2 ||B||),
 *   the Remark's smaller shift (Fig. 2); if chol(A + s_p I) breaks down the SAFE
 *   shift follows (reading D21), keeping Alg. 3's guarantee. */
enum { SCQR3_SHIFT_SAFE = 0, SCQR3_SHIFT_FIXED = 1, SCQR3_SHIFT_NONE = 2, SCQR3_SHIFT_ADAPTIVE = 3,
       SCQR3_SHIFT_PRACTICAL = 4 };

/* Estimate N^2 of ||Q||_2^2 for the shift (reading D2/D4).
 * POWER: 1.01 * Rayleigh quotient after power_iters steps on the computed n x n Gram.
 * FROBENIUS: trace of the Gram = ||Q||_F^2 (paper-sanctioned conservative choice).
 * USER: norm2_bound^2 on pass 1 (POWER afterwards).  Oblique (D4): the same choices for X, with
 * POWER iterating on the plain Gram Q^T Q that the oblique Gram kernel forms alongside the
 * B-Gram; ||B||_2 is bnorm_bound, else the Gershgorin bound. */
enum { SCQR3_NORM_POWER = 0, SCQR3_NORM_FROBENIUS = 1, SCQR3_NORM_USER = 2 };

/* How the TRSM Q := Q R~^{-1} solves its 8 x 8 diagonal blocks D_J (reading D24).
 * AUTO (default): per pass, the Cholesky step inverts every D_J by substitution (Y_J, rows of
 *   Y_J D_J = I) and checks that multiplying by Y_J keeps each row's backward error inside the
 *   paper's bound ||dR_i||_2 <= gamma_n sqrt(n) ||R~||_2 (eq. DeltaRbound):
 *   gamma_n ||R~_off||_F + 2 gamma_8 max_J || |D_J| |Y_J| |D_J| ||_F <= gamma_n sqrt(n) max_j ||R~ e_j||_2
 *   (R~_off: R~ without its diagonal blocks).  If it holds, the diagonal blocks are applied as
 *   products with Y_J on the FP64 tensor cores (every TRSM instance with 16-row warps: n in
 *   (32, 128] and all block-column launches of n > 128); otherwise by substitution.
 * SUBST: always substitution (the paper's row-wise forward substitution).
 * INVERSE: always the Y_J products where built (tests; no guard). */
enum { SCQR3_TRSM_DIAG_AUTO = 0, SCQR3_TRSM_DIAG_SUBST = 1, SCQR3_TRSM_DIAG_INVERSE = 2 };

typedef struct scqr3_pass_trace {
  double shift;            /* shift added on this pass (0 if none)                     */
  int32_t shifted;         /* 1 if chol(A + sI) was used                               */
  int32_t breakdown_pivot; /* 1-based pivot of the failed plain attempt, 0 if none     */
  double pivot_value;      /* value of that pivot before the square root               */
  double norm2_est;        /* N^2 used in the shift formula                            */
  double dev_F;            /* ||A_k - I||_F of this pass's input Gram (stop test, D6)  */
} scqr3_pass_trace;

/* Optional per-kernel device time, accumulated over calls (caller zeroes it).  Measured with
 * CUDA events recorded on opts->stream around each launch, so it adds two event records per
 * launch and is meant for benchmarks. */
typedef struct scqr3_prof {
  double gram_ms;          /* gram_tma_kernel (Q^T Q or Q^T B Q partial tiles)            */
  int64_t gram_launches;
  double reduce_ms;        /* gram_reduce_kernel (+ the B*Q kernel for the oblique Gram)   */
  int64_t reduce_launches;
  double chol_ms;          /* chol_kernel                                                  */
  int64_t chol_launches;
  double trsm_ms;          /* trsm_kernel                                                  */
  int64_t trsm_launches;
  double comm_ms;          /* NCCL allreduce / halo exchange                               */
  int64_t comm_calls;
  double trmul_ms;         /* R := R~ R on the side stream (overlaps the TRSM)             */
  int64_t trmul_launches;
} scqr3_prof;

typedef struct scqr3_opts {
  int32_t abi_version;     /* = SCQR3_ABI_VERSION                                      */
  int32_t shift_mode;      /* SCQR3_SHIFT_*                                            */
  double shift_value;      /* for SCQR3_SHIFT_FIXED                                    */
  int32_t norm_mode;       /* SCQR3_NORM_*                                             */
  int32_t power_iters;     /* default 32                                               */
  double norm2_bound;      /* USER: N >= ||X||_2                                       */
  double bnorm_bound;      /* oblique: N_B >= ||B||_2 (0 => Gershgorin)                */
  int32_t max_passes;      /* default 8                                        */
  int32_t deterministic;   /* with comm: 1 = allgather the Gram and sum it in rank order: bitwise reproducible whatever NCCL algorithm runs; up to >= 22 ranks at every n (Gram slots of the workspace), else SCQR3_EINVAL */
  double stop_tol;         /* stop after a plain pass with ||A_k - I||_F <= stop_tol (D6); default 0.5 */
  int64_t m_global;        /* rows over all ranks (shift uses the global m); 0 => sum over ranks */
  void* stream;            /* cudaStream_t; NULL = legacy default stream                */
  void* comm;              /* from scqr3_comm_init; NULL = single GPU                   */
  void* workspace;         /* device memory of >= scqr3_workspace_size() bytes, 256-B aligned */
  size_t workspace_bytes;
  scqr3_pass_trace* trace; /* host array of trace_cap entries (may be NULL)            */
  int32_t trace_cap;
  int32_t* passes_out;     /* host; number of passes executed (may be NULL)            */
  scqr3_prof* prof;        /* host; per-kernel device time (may be NULL)                */
  int32_t trsm_diag;       /* SCQR3_TRSM_DIAG_* (default AUTO; ABI version 2)           */
} scqr3_opts;

/* Fills *o with the defaults above (abi_version, SAFE, POWER, 32 iterations, 8 passes,
 * stop_tol 0.5, everything else zero). */
void scqr3_default_opts(scqr3_opts* o);

/* Device workspace bytes for scqr3_factor / scqr3_factor_oblique on this rank's m x n
 * shard (independent of the data; oblique needs an extra m x n buffer for B*Q). */
size_t scqr3_workspace_size(int64_t m, int64_t n, int32_t oblique);

/* Shifted CholeskyQR3 X = QR (Alg. 3, with Alg. 2's breakdown re-shift,
 * P:672-688; pass control D5/D6).  Per pass: Gram A = Q^T Q (one NCCL allreduce of
 * the packed n x n Gram when opts->comm is set), norm estimate and shift,
 * Cholesky R~ (replicated on every rank), Q := Q R~^{-1} row by row, and
 * R := R~ R.  Q may alias X (then ldq == ld).  With opts->comm, X/Q/m are this
 * rank's contiguous row block and R is identical on every rank. */
int scqr3_factor(int64_t m, int64_t n, const double* X, int64_t ld, double* Q, int64_t ldq,
                 double* R, const scqr3_opts* opts);

/* Oblique inner product (Alg. 5; B-Gram in every pass, reading D8):
 * X = QR with Q^T B Q = I for the SPD tridiagonal B with B(i,i) = b_diag[i] and
 * B(i,i+1) = B(i+1,i) = b_off[i] (b_off[m-1] couples this rank's last row to the next
 * rank's first row; ignored on the last rank).  Bands are sharded with the rows; the
 * one-row halo is exchanged with NCCL send/recv when opts->comm is set. */
int scqr3_factor_oblique(int64_t m, int64_t n, const double* X, int64_t ld, const double* b_diag,
                         const double* b_off, double* Q, int64_t ldq, double* R,
                         const scqr3_opts* opts);

/* General sparse SPD metric B in CSR (the paper's sparse-B experiments,
 * P:1876-1888).  All arrays are DEVICE arrays owned by the caller and hold this
 * rank's rows of B:
 *   row_ptr[m+1]  int64, row_ptr[0] = 0, non-decreasing;
 *   col_idx[nnz]  int32 column indices RELATIVE to this rank's first row: a value c in
 *                 [0, m) is a local row of Q, c in [-halo, 0) a row of the previous rank
 *                 (its last halo rows), c in [m, m + halo) one of the next rank's first
 *                 halo rows;
 *   vals[nnz]     float64, B symmetric positive definite (not checked).
 * halo: rows exchanged with each neighbouring rank per pass (NCCL send/recv, like the
 * tridiagonal halo); 0 on one GPU (required without opts->comm).  Each rank must own at
 * least halo rows.  Index and row_ptr violations are detected on the device -> EINVAL.
 *
 * halo == SCQR3_CSR_GHOSTS: rows of other ranks by the sparsity pattern (any B, not only a
 * banded one; the distributed sparse matrix-vector product's ghost-row plan):
 *   col_idx  a value c in [0, m) is a local row of Q, c in [m, m + nghost) ghost row c - m;
 *   ghost rows are grouped by the rank that owns them, in rank order: the recv_counts[r] rows
 *   from rank r follow those of ranks < r, in the order rank r lists them in its send list;
 *   nghost       total ghost rows of this rank (sum of recv_counts);
 *   recv_counts  HOST int64[nranks]: ghost rows received from each rank (0 for this rank);
 *   send_counts  HOST int64[nranks]: rows of this rank sent to each rank (0 for itself);
 *   send_rows    DEVICE int64[sum send_counts]: the local rows (in [0, m)) sent, grouped by
 *                destination rank in rank order.
 * Per pass the listed rows of Q are gathered and exchanged (NCCL grouped send/recv with every
 * rank that has a nonzero count).  Rank r's send_counts[p] must equal rank p's recv_counts[r]
 * (checked collectively once per call); send_rows and col_idx are checked on the device.
 * Without opts->comm, nghost must be 0.  The fields after halo are ignored when halo >= 0. */
#define SCQR3_CSR_GHOSTS (-1)
typedef struct scqr3_csr {
  const int64_t* row_ptr;
  const int32_t* col_idx;
  const double* vals;
  int64_t halo;
  int64_t nghost;               /* ghost plan (halo == SCQR3_CSR_GHOSTS; ABI version 2) */
  const int64_t* recv_counts;
  const int64_t* send_counts;
  const int64_t* send_rows;
} scqr3_csr;

/* Workspace bytes for the CSR-metric calls (the halo buffers scale with halo * n). */
size_t scqr3_workspace_size_csr(int64_t m, int64_t n, int64_t halo);
/* Workspace bytes for a ghost-plan CSR metric: nghost received and nsend sent rows per pass. */
size_t scqr3_workspace_size_csr_ghosts(int64_t m, int64_t n, int64_t nghost, int64_t nsend);

/* Oblique shifted CholeskyQR3 (Alg. 5 with the B-Gram in all passes, D8) for a CSR metric:
 * Y = B Q by csr_y_tile_kernel, then the same Gram / shift / Cholesky / TRSM path; the shift's
 * ||B||_2 bound is opts->bnorm_bound or the Gershgorin max_i sum_k |B_ik| (allreduce-max
 * over ranks).  Target Q^T B Q = I, X = QR. */
int scqr3_factor_oblique_csr(int64_t m, int64_t n, const double* X, int64_t ld, const scqr3_csr* B,
                             double* Q, int64_t ldq, double* R, const scqr3_opts* opts);

/* Complex X ("everything carries over to complex matrices";
 * reading D23: X^H X, R~^H R~ = A + sI with a real positive diagonal, the same shift formula).
 * X, Q: m x n complex double (C99 double complex / cuDoubleComplex: interleaved re, im),
 * column-major with leading dimensions ld, ldq >= m counted in complex elements, 16-byte
 * aligned; R: n x n complex, column-major, leading dimension n, upper with a real positive
 * diagonal.  1 <= n <= 512.  The tall-skinny steps run the real Gram and TRSM kernels on the
 * m x 2n real "split" matrix (Re x_0, Im x_0, Re x_1, ...), the n x n step is complex; for
 * n > 256 the split matrix is taken as two column blocks [S1 S2] (512 and 2n - 512 columns):
 * the real kernels on each block plus a cross Gram S1^T S2 and the block update S2 -= Q1 M12
 * (zwide.cu; deterministic mode: up to 8 ranks fit the workspace's gather slots).  Same
 * options, statuses and trace as scqr3_factor; opts->workspace must hold
 * scqr3_workspace_size_complex(m, n) bytes. */
size_t scqr3_workspace_size_complex(int64_t m, int64_t n);
int scqr3_factor_complex(int64_t m, int64_t n, const double* X, int64_t ld, double* Q, int64_t ldq, double* R,
                         const scqr3_opts* opts);

/* Host-memory variant of scqr3_factor (the end-to-end call): copies X_host to the device
 * (pinned host memory recommended), factors in place, copies Q and R back.  opts->workspace
 * must hold scqr3_host_workspace_size(m, n) bytes. */
size_t scqr3_host_workspace_size(int64_t m, int64_t n);
int scqr3_factor_host(int64_t m, int64_t n, const double* X_host, int64_t ld, double* Q_host,
                      int64_t ldq, double* R_host, const scqr3_opts* opts);

/* Streaming variant of scqr3_factor_host for `count` independent m x n host matrices (a serving
 * loop): X_hosts[i] (ld) -> Q_hosts[i] (ldq), R_hosts[i] (n x n), statuses[i] (SCQR3_OK /
 * _EBREAKDOWN / _ENOCONV; Q and R written on OK only).  Three device staging buffers rotate, so
 * matrix i+1's upload and matrix i-1's download run on the two PCIe directions (library streams)
 * while matrix i is factored on opts->stream -- each matrix still goes host -> device -> host.
 * Host buffers: pinned for full bandwidth; an X_hosts entry must not alias a Q_hosts / R_hosts
 * entry of another matrix in the batch (repeating the same X, or the same Q / R, is fine).
 * opts->workspace: scqr3_host_batch_workspace_size(m, n) bytes.  Returns SCQR3_OK once every
 * matrix is done (statuses per matrix), or SCQR3_EINVAL.  Single GPU or one rank per GPU
 * (every rank calls it with the same count). */
size_t scqr3_host_batch_workspace_size(int64_t m, int64_t n);
int scqr3_factor_host_batch(int64_t count, int64_t m, int64_t n, const double* const* X_hosts, int64_t ld,
                            double* const* Q_hosts, int64_t ldq, double* const* R_hosts, int32_t* statuses,
                            const scqr3_opts* opts);

/* ---- kernel-level entry points (parity tests call these through the same library) ---- */
/* A = Q^T Q (n x n, column-major, both triangles) -- one Gram kernel + reduction. */
int scqr3_gram(int64_t m, int64_t n, const double* X, int64_t ld, double* A, const scqr3_opts* opts);
/* A = sym(X^T B X) for the tridiagonal B above; *colsq = ||X||_F^2 (D4). */
int scqr3_gram_oblique(int64_t m, int64_t n, const double* X, int64_t ld, const double* b_diag,
                       const double* b_off, double* A, double* colsq, const scqr3_opts* opts);
/* A = sym(X^T B X) for a CSR metric (B->halo must be 0; single GPU), *colsq = ||X||_F^2.
 * Workspace: scqr3_workspace_size_csr(m, n, 0). */
int scqr3_gram_oblique_csr(int64_t m, int64_t n, const double* X, int64_t ld, const scqr3_csr* B,
                           double* A, double* colsq, const scqr3_opts* opts);
/* R~ = chol(A + sI) (upper, n x n column-major) with breakdown detection (D9).
 * Returns SCQR3_EBREAKDOWN with *pivot (1-based) and *pivot_value on a pivot <= 0 or
 * non-finite, else SCQR3_OK with *pivot = 0. */
int scqr3_cholesky(int64_t n, const double* A, double s, double* R, int32_t* pivot,
                   double* pivot_value, const scqr3_opts* opts);
/* Q = X R^{-1} for upper-triangular R with positive diagonal. */
int scqr3_trsm(int64_t m, int64_t n, const double* X, int64_t ld, const double* R, double* Q,
               int64_t ldq, const scqr3_opts* opts);

/* ---- multi-GPU (one process per GPU; NCCL over NVLink) ---- */
#define SCQR3_COMM_ID_BYTES 128
/* Writes an NCCL unique id (SCQR3_COMM_ID_BYTES bytes) to id_out; call on rank 0 and
 * broadcast the bytes (e.g. with torch.distributed). */
int scqr3_comm_unique_id(void* id_out);
/* Creates this rank's communicator on the current CUDA device; *comm_out is passed in
 * scqr3_opts.comm.  Collective over all nranks. */
int scqr3_comm_init(void** comm_out, int32_t nranks, const void* id, int32_t rank);
/* In-process "loopback" communicator group (validation of the multi-rank protocol on one GPU):
 * writes nranks handles to comms_out[0..nranks-1], 1 <= nranks <= 16.  Rank r's handle is
 * passed in scqr3_opts.comm by the host thread that drives rank r; the nranks threads call the
 * same entry point concurrently, each on its own stream and rows, on the SAME current device.
 * The exchanges run the same protocol as NCCL (Gram sum, halo rows, b_off coupling, global m,
 * ||B|| bound): a rank publishes a device buffer and an event, a host barrier, then each rank's
 * stream waits on its peers' events and reads their buffers with its own copies / kernels
 * (rank-ordered sum, so R is bitwise identical on every rank).  No kernel waits on another.
 * If a rank fails after the exchanges began, the group is marked failed and its peers return
 * SCQR3_EINVAL; a group whose ranks stop calling times out after 600 s.  Every handle is
 * released with scqr3_comm_destroy (the shared state with the last one). */
int scqr3_comm_init_loopback(void** comms_out, int32_t nranks);
/* Releases a communicator (NCCL or loopback). */
int scqr3_comm_destroy(void* comm);

/* Thread-local description of the last SCQR3_EINVAL. */
const char* scqr3_last_error(void);
/* Number of kernel launches issued by this thread since the last reset (bench evidence). */
int64_t scqr3_launch_count(int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* SCQR3_H */
