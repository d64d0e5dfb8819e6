// comm.cu -- NCCL and loopback backends of the per-pass exchanges (scqr3_comm.h).
//
// The method's exchange: each rank forms the Gram of its row block, the Grams are
// summed, and every rank factors the same sum.  The loopback backend runs the same protocol
// with P host threads on one GPU, so the library's multi-rank code paths (halo branches,
// e_prev exchange, global m, rank-ordered sum) execute and can be compared with the oracle's
// P-part emulation where only one GPU exists.
#include <algorithm>
#include <condition_variable>
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "scqr3.h"
#include "scqr3_comm.h"

namespace scqr3 {

#define CTRY(expr)                                                                                      \
  do {                                                                                                  \
    cudaError_t e_ = (expr);                                                                            \
    if (e_ != cudaSuccess) return set_error("%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)
#define NTRY(expr)                                                                      \
  do {                                                                                  \
    ncclResult_t r_ = (expr);                                                           \
    if (r_ != ncclSuccess) return set_error("%s: %s", #expr, ncclGetErrorString(r_));  \
  } while (0)
#define RTRY(expr)                   \
  do {                               \
    int rc_ = (expr);                \
    if (rc_ != SCQR3_OK) return rc_; \
  } while (0)

struct LoopGroup {
  int nranks = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  bool aborted = false;
  std::string why;
  int refs = 0;
  const double* pub[kMaxLoopRanks] = {};     // published device buffer of each rank
  cudaEvent_t ev_write[kMaxLoopRanks] = {};  // rank's published buffer written (its stream)
  cudaEvent_t ev_read[kMaxLoopRanks] = {};   // rank finished reading the peers' buffers
  double* stage[kMaxLoopRanks] = {};         // per-rank staging of allreduce contributions
  size_t stage_cap = 0;                      // doubles per rank
  int64_t hval[kMaxLoopRanks] = {};
  const int64_t* hvec[kMaxLoopRanks] = {};     // published host arrays (allgather, ghost-plan counts)
};

// Staging per rank: the largest exchanged Gram is the oblique one at n = 512 (two sets of
// NT(NT+1)/2 = 2080 packed tiles of 64 doubles, + 1).
constexpr size_t kStageDoubles = 2 * 2080 * 64 + 64;

struct PtrPack {
  const double* p[kMaxLoopRanks];
};

// out[i] = op over ranks r = 0, 1, ..., P-1 (in that order) of part_r[i]; the same bits on
// every rank (each computes the same ordered sum of the same inputs).
__global__ void lb_reduce_kernel(PtrPack parts, int nparts, long long count, int op, double* out) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    double s = parts.p[0][i];
    for (int r = 1; r < nparts; ++r) {
      const double v = parts.p[r][i];
      s = op == COMM_MAX ? fmax(s, v) : s + v;
    }
    out[i] = s;
  }
}

namespace {

// Host barrier of a loopback group.  A rank that fails mid-call aborts the group so that its
// peers return an error instead of waiting; a 600 s timeout guards against a rank that never
// arrives (e.g. a caller that did not start all P threads).
int lb_barrier(LoopGroup* g) {
  std::unique_lock<std::mutex> lk(g->mu);
  if (g->aborted) return set_error("loopback group aborted: %s", g->why.c_str());
  const long long my = g->gen;
  if (++g->arrived == g->nranks) {
    g->arrived = 0;
    ++g->gen;
    g->cv.notify_all();
    return SCQR3_OK;
  }
  const bool ok = g->cv.wait_for(lk, std::chrono::seconds(600), [&] { return g->gen != my || g->aborted; });
  if (g->gen != my) return SCQR3_OK;
  if (!ok) {
    g->aborted = true;
    g->why = "barrier timed out (600 s): a rank did not take part in the collective";
    g->cv.notify_all();
  }
  return set_error("loopback group aborted: %s", g->why.c_str());
}

// One loopback collective: [barrier A] wait until the peers have read what this rank published
// last time -> pack (writes the buffer to publish) -> publish + record -> [barrier B] -> wait
// for the peers' writes -> read (copies / kernels on this rank's stream) -> record.
template <class Pack, class Read>
int lb_collective(Comm* c, cudaStream_t st, const double* pub, Pack pack, Read read) {
  LoopGroup* g = c->lg;
  RTRY(lb_barrier(g));
  for (int j = 0; j < g->nranks; ++j)
    if (j != c->rank) CTRY(cudaStreamWaitEvent(st, g->ev_read[j], 0));
  RTRY(pack());
  g->pub[c->rank] = pub;
  CTRY(cudaEventRecord(g->ev_write[c->rank], st));
  RTRY(lb_barrier(g));
  for (int j = 0; j < g->nranks; ++j)
    if (j != c->rank) CTRY(cudaStreamWaitEvent(st, g->ev_write[j], 0));
  RTRY(read(g->pub));
  CTRY(cudaEventRecord(g->ev_read[c->rank], st));
  return SCQR3_OK;
}

int lb_reduce(Comm* c, const double* const* pub, long long count, int op, double* out, cudaStream_t st) {
  PtrPack pp{};
  for (int r = 0; r < c->nranks; ++r) pp.p[r] = pub[r];
  const long long blocks = std::max<long long>(1, std::min<long long>((count + 255) / 256, 1024));
  lb_reduce_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(pp, c->nranks, count, op, out);
  CTRY(cudaGetLastError());
  return SCQR3_OK;
}

}  // namespace

int comm_create_loopback(Comm** out, int nranks) {
  if (!out) return set_error("comms is NULL");
  if (nranks < 1 || nranks > kMaxLoopRanks) return set_error("loopback nranks %d outside [1, %d]", nranks, kMaxLoopRanks);
  LoopGroup* g = new LoopGroup{};
  g->nranks = nranks;
  g->stage_cap = kStageDoubles;
  for (int r = 0; r < nranks; ++r) {
    if (cudaEventCreateWithFlags(&g->ev_write[r], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->ev_read[r], cudaEventDisableTiming) != cudaSuccess ||
        cudaMalloc(&g->stage[r], kStageDoubles * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return set_error("loopback group: CUDA allocation failed");
    }
  }
  for (int r = 0; r < nranks; ++r) {
    Comm* c = new Comm{};
    c->kind = COMM_LOOPBACK;
    c->rank = r;
    c->nranks = nranks;
    c->lg = g;
    out[r] = c;
  }
  g->refs = nranks;
  return SCQR3_OK;
}

int comm_destroy(Comm* c) {
  if (!c) return SCQR3_OK;
  if (c->kind == COMM_NCCL) {
    if (c->nccl) ncclCommDestroy(c->nccl);
    if (c->dscratch) cudaFree(c->dscratch);
    if (c->hscratch) cudaFreeHost(c->hscratch);
  } else {
    LoopGroup* g = c->lg;
    bool last = false;
    {
      std::lock_guard<std::mutex> lk(g->mu);
      last = --g->refs == 0;
    }
    if (last) {
      for (int r = 0; r < g->nranks; ++r) {
        cudaEventDestroy(g->ev_write[r]);
        cudaEventDestroy(g->ev_read[r]);
        cudaFree(g->stage[r]);
      }
      delete g;
    }
  }
  delete c;
  return SCQR3_OK;
}

void comm_abort(Comm* c, const char* why) {
  if (!c || c->kind != COMM_LOOPBACK) return;
  std::lock_guard<std::mutex> lk(c->lg->mu);
  if (!c->lg->aborted) {
    c->lg->aborted = true;
    c->lg->why = std::string("rank ") + std::to_string(c->rank) + ": " + (why ? why : "error");
  }
  c->lg->cv.notify_all();
}

int comm_host_allreduce(Comm* c, int64_t v, int op, int64_t* out, cudaStream_t st) {
  if (c->kind == COMM_NCCL) {
    const ncclRedOp_t nop = op == COMM_SUM ? ncclSum : op == COMM_MIN ? ncclMin : ncclMax;
    // (pinned staging: both copies stay asynchronous, one stream synchronisation in total)
    c->hscratch[0] = v;
    CTRY(cudaMemcpyAsync(c->dscratch, c->hscratch, 8, cudaMemcpyHostToDevice, st));
    NTRY(ncclAllReduce(c->dscratch, c->dscratch, 1, ncclInt64, nop, c->nccl, st));
    CTRY(cudaMemcpyAsync(c->hscratch + 1, c->dscratch, 8, cudaMemcpyDeviceToHost, st));
    CTRY(cudaStreamSynchronize(st));
    *out = c->hscratch[1];
    return SCQR3_OK;
  }
  LoopGroup* g = c->lg;
  g->hval[c->rank] = v;
  RTRY(lb_barrier(g));
  int64_t s = g->hval[0];
  for (int r = 1; r < g->nranks; ++r) {
    const int64_t x = g->hval[r];
    s = op == COMM_SUM ? s + x : op == COMM_MIN ? std::min(s, x) : std::max(s, x);
  }
  RTRY(lb_barrier(g));  // nobody overwrites hval before every rank has read it
  *out = s;
  return SCQR3_OK;
}

int comm_agree(Comm* c, bool ok, cudaStream_t st) {
  // min over ranks of (ok ? nranks : rank): >= nranks iff every rank is fine, else the first bad rank
  int64_t r = 0;
  const int rc = comm_host_allreduce(c, ok ? c->nranks : c->rank, COMM_MIN, &r, st);
  if (rc != SCQR3_OK) return rc;
  if (r >= c->nranks) return SCQR3_OK;
  if (!ok) return SCQR3_EINVAL;  // keep this rank's own message
  return set_error("rank %lld rejected its arguments (see that rank's scqr3_last_error)", static_cast<long long>(r));
}

int comm_allreduce_sum(Comm* c, double* buf, size_t count, bool deterministic, double* gather, size_t gather_cap,
                       cudaStream_t st) {
  if (c->kind == COMM_NCCL) {
    if (deterministic) {
      // every rank's buffer side by side, then one fixed-order sum: the same bits on every
      // rank and every run whatever algorithm NCCL picks
      if (static_cast<unsigned long long>(c->nranks) * count > gather_cap)
        return set_error("deterministic mode: %d ranks exceed the workspace's Gram slots", c->nranks);
      NTRY(ncclAllGather(buf, gather, count, ncclDouble, c->nccl, st));
      std::vector<const double*> ptrs(c->nranks);
      if (c->nranks > kMaxLoopRanks) {
        // more ranks than one pointer pack: sum in rank order in chunks of kMaxLoopRanks
        CTRY(cudaMemcpyAsync(buf, gather, count * 8, cudaMemcpyDeviceToDevice, st));
        for (int r0 = 1; r0 < c->nranks; r0 += kMaxLoopRanks - 1) {
          PtrPack pp{};
          pp.p[0] = buf;
          int k = 1;
          for (int r = r0; r < c->nranks && k < kMaxLoopRanks; ++r, ++k) pp.p[k] = gather + static_cast<size_t>(r) * count;
          const long long blocks = std::max<long long>(1, std::min<long long>((count + 255) / 256, 1024));
          lb_reduce_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(pp, k, static_cast<long long>(count), COMM_SUM, buf);
          CTRY(cudaGetLastError());
        }
        return SCQR3_OK;
      }
      for (int r = 0; r < c->nranks; ++r) ptrs[r] = gather + static_cast<size_t>(r) * count;
      return lb_reduce(c, ptrs.data(), static_cast<long long>(count), COMM_SUM, buf, st);
    }
    NTRY(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, c->nccl, st));
    return SCQR3_OK;
  }
  LoopGroup* g = c->lg;
  if (count > g->stage_cap) return set_error("loopback allreduce of %zu doubles exceeds the staging", count);
  double* mine = g->stage[c->rank];
  return lb_collective(
      c, st, mine,
      [&]() -> int {
        CTRY(cudaMemcpyAsync(mine, buf, count * 8, cudaMemcpyDeviceToDevice, st));
        return SCQR3_OK;
      },
      [&](const double* const* pub) -> int { return lb_reduce(c, pub, static_cast<long long>(count), COMM_SUM, buf, st); });
}

int comm_allreduce_max1(Comm* c, double* buf, cudaStream_t st) {
  if (c->kind == COMM_NCCL) {
    NTRY(ncclAllReduce(buf, buf, 1, ncclDouble, ncclMax, c->nccl, st));
    return SCQR3_OK;
  }
  double* mine = c->lg->stage[c->rank];
  return lb_collective(
      c, st, mine,
      [&]() -> int {
        CTRY(cudaMemcpyAsync(mine, buf, 8, cudaMemcpyDeviceToDevice, st));
        return SCQR3_OK;
      },
      [&](const double* const* pub) -> int { return lb_reduce(c, pub, 1, COMM_MAX, buf, st); });
}

int comm_halo(Comm* c, const double* Q, int64_t ld, int64_t m, int n, int64_t h, double* halo, cudaStream_t st) {
  if (h <= 0) return SCQR3_OK;
  if (m < h) return set_error("halo of %lld rows exceeds this rank's %lld rows", (long long)h, (long long)m);
  const size_t blk = static_cast<size_t>(h) * n;
  auto pack = [&]() -> int {
    CTRY(cudaMemcpy2DAsync(halo, h * 8, Q, ld * 8, h * 8, n, cudaMemcpyDeviceToDevice, st));
    CTRY(cudaMemcpy2DAsync(halo + blk, h * 8, Q + (m - h), ld * 8, h * 8, n, cudaMemcpyDeviceToDevice, st));
    return SCQR3_OK;
  };
  if (c->kind == COMM_NCCL) {
    RTRY(pack());
    NTRY(ncclGroupStart());
    if (c->rank > 0) {
      NTRY(ncclSend(halo, blk, ncclDouble, c->rank - 1, c->nccl, st));
      NTRY(ncclRecv(halo + 2 * blk, blk, ncclDouble, c->rank - 1, c->nccl, st));
    }
    if (c->rank + 1 < c->nranks) {
      NTRY(ncclSend(halo + blk, blk, ncclDouble, c->rank + 1, c->nccl, st));
      NTRY(ncclRecv(halo + 3 * blk, blk, ncclDouble, c->rank + 1, c->nccl, st));
    }
    NTRY(ncclGroupEnd());
    return SCQR3_OK;
  }
  return lb_collective(c, st, halo, pack, [&](const double* const* pub) -> int {
    if (c->rank > 0)
      CTRY(cudaMemcpyAsync(halo + 2 * blk, pub[c->rank - 1] + blk, blk * 8, cudaMemcpyDeviceToDevice, st));
    if (c->rank + 1 < c->nranks)
      CTRY(cudaMemcpyAsync(halo + 3 * blk, pub[c->rank + 1], blk * 8, cudaMemcpyDeviceToDevice, st));
    return SCQR3_OK;
  });
}

int comm_host_allgather(Comm* c, const int64_t* v, int cnt, int64_t* out, int64_t* dscratch, cudaStream_t st) {
  if (c->kind == COMM_NCCL) {
    CTRY(cudaMemcpyAsync(dscratch + static_cast<size_t>(c->rank) * cnt, v, cnt * 8, cudaMemcpyHostToDevice, st));
    NTRY(ncclAllGather(dscratch + static_cast<size_t>(c->rank) * cnt, dscratch, cnt, ncclInt64, c->nccl, st));
    CTRY(cudaMemcpyAsync(out, dscratch, static_cast<size_t>(c->nranks) * cnt * 8, cudaMemcpyDeviceToHost, st));
    CTRY(cudaStreamSynchronize(st));
    return SCQR3_OK;
  }
  LoopGroup* g = c->lg;
  g->hvec[c->rank] = v;
  RTRY(lb_barrier(g));
  for (int r = 0; r < g->nranks; ++r) std::memcpy(out + static_cast<size_t>(r) * cnt, g->hvec[r], cnt * 8);
  RTRY(lb_barrier(g));  // nobody changes its array before every rank has read it
  return SCQR3_OK;
}

// sendbuf[k][j] = Q[send_rows[k] + j ld] (row-major; consecutive threads write consecutive j)
__global__ void ghost_pack_kernel(const double* Q, long long ld, int n, const int64_t* rows, long long nsend,
                                  double* sendbuf) {
  const long long total = nsend * n;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long k = i / n;
    const int j = static_cast<int>(i - k * n);
    sendbuf[i] = Q[rows[k] + j * ld];
  }
}

int comm_ghosts(Comm* c, const double* Q, int64_t ld, int n, const int64_t* send_rows, const int64_t* send_counts,
                const int64_t* recv_counts, int64_t nsend, double* sendbuf, double* ghost, cudaStream_t st) {
  auto pack = [&]() -> int {
    if (nsend > 0) {
      const long long total = nsend * n;
      const long long blocks = std::max<long long>(1, std::min<long long>((total + 255) / 256, 2048));
      ghost_pack_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(Q, ld, n, send_rows, nsend, sendbuf);
      CTRY(cudaGetLastError());
    }
    return SCQR3_OK;
  };
  if (c->kind == COMM_NCCL) {
    RTRY(pack());
    NTRY(ncclGroupStart());
    int64_t so = 0, ro = 0;
    for (int p = 0; p < c->nranks; ++p) {
      if (send_counts[p] > 0) NTRY(ncclSend(sendbuf + so * n, send_counts[p] * n, ncclDouble, p, c->nccl, st));
      if (recv_counts[p] > 0) NTRY(ncclRecv(ghost + ro * n, recv_counts[p] * n, ncclDouble, p, c->nccl, st));
      so += send_counts[p];
      ro += recv_counts[p];
    }
    NTRY(ncclGroupEnd());
    return SCQR3_OK;
  }
  LoopGroup* g = c->lg;
  return lb_collective(
      c, st, sendbuf,
      [&]() -> int {
        g->hvec[c->rank] = send_counts;  // (read by the peers between the two barriers)
        return pack();
      },
      [&](const double* const* pub) -> int {
        int64_t ro = 0;
        for (int p = 0; p < c->nranks; ++p) {
          if (recv_counts[p] > 0) {
            int64_t off = 0;  // rows rank p sends to ranks before this one
            for (int q = 0; q < c->rank; ++q) off += g->hvec[p][q];
            CTRY(cudaMemcpyAsync(ghost + ro * n, pub[p] + off * n, recv_counts[p] * n * 8, cudaMemcpyDeviceToDevice, st));
          }
          ro += recv_counts[p];
        }
        return SCQR3_OK;
      });
}

int comm_shift_right1(Comm* c, const double* src, double* send, double* recv, cudaStream_t st) {
  auto pack = [&]() -> int {
    if (src) CTRY(cudaMemcpyAsync(send, src, 8, cudaMemcpyDeviceToDevice, st));
    else CTRY(cudaMemsetAsync(send, 0, 8, st));
    return SCQR3_OK;
  };
  if (c->kind == COMM_NCCL) {
    RTRY(pack());
    NTRY(ncclGroupStart());
    if (c->rank + 1 < c->nranks) NTRY(ncclSend(send, 1, ncclDouble, c->rank + 1, c->nccl, st));
    if (c->rank > 0) NTRY(ncclRecv(recv, 1, ncclDouble, c->rank - 1, c->nccl, st));
    NTRY(ncclGroupEnd());
    return SCQR3_OK;
  }
  return lb_collective(c, st, send, pack, [&](const double* const* pub) -> int {
    if (c->rank > 0) CTRY(cudaMemcpyAsync(recv, pub[c->rank - 1], 8, cudaMemcpyDeviceToDevice, st));
    return SCQR3_OK;
  });
}

}  // namespace scqr3
