// scqr3_comm.h -- the exchanges of the row-block-parallel method behind one interface
// (internal; the public ABI is include/scqr3.h).
//
// The method's one exchange per pass is the sum of the per-rank Grams ("the reduction operator
// is addition"); the oblique variant also swaps halo rows of Q with each neighbour
// (Y = BQ needs the neighbours' rows) and, once, the coupling entry b_off and the
// max of the per-rank ||B|| bounds.  Two backends:
//   NCCL      one process per GPU over NVLink / NVSwitch (production).
//   LOOPBACK  P ranks = P host threads of one process sharing the current device, each with its
//             own stream (validation of the multi-rank protocol where only one GPU exists).  A
//             rank publishes a device buffer and records an event; after a host barrier every
//             rank's stream waits on the peers' events and reads the published buffers with its
//             own copies / kernels; a second barrier orders the next overwrite after those
//             reads.  Dependencies are stream-order only: no kernel ever waits on another.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <stddef.h>
#include <stdint.h>

namespace scqr3 {

// Sets the thread's scqr3_last_error() text and returns SCQR3_EINVAL (scqr3_host.cu).
int set_error(const char* fmt, ...);

enum CommKind { COMM_NCCL = 0, COMM_LOOPBACK = 1 };
enum CommOp { COMM_SUM = 0, COMM_MIN = 1, COMM_MAX = 2 };

struct LoopGroup;
struct Comm {
  int kind = COMM_NCCL;
  int rank = 0, nranks = 1;
  ncclComm_t nccl = nullptr;
  int64_t* dscratch = nullptr;  // NCCL: a few int64 of device scratch for host-level reductions
  int64_t* hscratch = nullptr;  // NCCL: pinned host staging of those values (async copies)
  LoopGroup* lg = nullptr;      // LOOPBACK: shared by the group's ranks
};

constexpr int kMaxLoopRanks = 16;

int comm_create_loopback(Comm** out, int nranks);  // nranks handles, one per rank
int comm_destroy(Comm* c);

// Host-level reduction of one int64 per rank (sizes, validity flags); synchronous.
int comm_host_allreduce(Comm* c, int64_t v, int op, int64_t* out, cudaStream_t st);
// All ranks agree that every rank's arguments are valid (ok = local validity).  Returns
// SCQR3_OK when all are; else SCQR3_EINVAL with a message naming the first failing rank.
int comm_agree(Comm* c, bool ok, cudaStream_t st);

// buf[0:count] := sum over ranks (in place, on st).  deterministic: NCCL allgathers into
// `gather` (count * nranks doubles, capacity gather_cap) and sums in rank order; the loopback
// backend always sums in rank order (same bits on every rank, every run).
int comm_allreduce_sum(Comm* c, double* buf, size_t count, bool deterministic, double* gather, size_t gather_cap,
                       cudaStream_t st);
// *buf := max over ranks of one double (device scalar).
int comm_allreduce_max1(Comm* c, double* buf, cudaStream_t st);
// Halo exchange of h rows of the m x n block Q (ld): halo holds four h x n blocks (ld h):
// [0] my first h rows, [1] my last h rows (packed here), [2] <- the previous rank's last h rows,
// [3] <- the next rank's first h rows.  Requires m >= h (checked collectively by the caller).
int comm_halo(Comm* c, const double* Q, int64_t ld, int64_t m, int n, int64_t h, double* halo, cudaStream_t st);
// All ranks' host int64[cnt] arrays: out[r * cnt + i] = rank r's v[i] (synchronous; the NCCL
// backend stages through dscratch, device memory of nranks * cnt int64).
int comm_host_allgather(Comm* c, const int64_t* v, int cnt, int64_t* out, int64_t* dscratch, cudaStream_t st);
// Ghost-row exchange of a sparsity-pattern plan (scqr3_csr with SCQR3_CSR_GHOSTS): the rows
// send_rows[0:nsend] of Q are packed row-major into sendbuf (nsend x n) and sent, grouped by
// destination in rank order (send_counts, host); ghost (row-major) receives recv_counts[p] rows
// from each rank p, in rank order.
int comm_ghosts(Comm* c, const double* Q, int64_t ld, int n, const int64_t* send_rows, const int64_t* send_counts,
                const int64_t* recv_counts, int64_t nsend, double* sendbuf, double* ghost, cudaStream_t st);
// One double to the next rank: send[0] := *src (0 if src is null); recv[0] <- previous rank's
// send[0] (untouched on rank 0).
int comm_shift_right1(Comm* c, const double* src, double* send, double* recv, cudaStream_t st);
// Marks a loopback group failed (a rank returns an error mid-call): the peers' barriers return
// SCQR3_EINVAL instead of waiting for it.  No-op for NCCL.
void comm_abort(Comm* c, const char* why);

}  // namespace scqr3
