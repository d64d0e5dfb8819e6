// scqr3_host.cu -- the C ABI of libscqr3.so (include/scqr3.h): argument checking, workspace
// carving, the pass controller (Alg. 3 P:698-711 + Alg. 2 re-shift P:672-688, readings D5/D6)
// and the NCCL plumbing (one allreduce of the packed Gram per pass; one-row halo for
// the tridiagonal oblique metric).  All arithmetic runs in the kernels of gram.cu, chol.cu
// and trsm.cu; this file only launches them.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX ranges (no-ops unless a profiler is attached)

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "scqr3.h"
#include "scqr3_comm.h"
#include "scqr3_dev.cuh"
#include "scqr3_kernels.h"

using namespace scqr3;

namespace {
thread_local std::string g_err;
thread_local int64_t g_launches = 0;
}  // namespace

namespace scqr3 {
int set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return SCQR3_EINVAL;
}
}  // namespace scqr3

namespace {

#define fail set_error

#define CUDA_TRY(expr)                                                                      \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) return fail("%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)
#define NCCL_TRY(expr)                                                                      \
  do {                                                                                      \
    ncclResult_t r_ = (expr);                                                               \
    if (r_ != ncclSuccess) return fail("%s: %s", #expr, ncclGetErrorString(r_));           \
  } while (0)
#define TRY(expr)              \
  do {                         \
    int rc_ = (expr);          \
    if (rc_ != SCQR3_OK) return rc_; \
  } while (0)

struct GraphKey;
struct GraphPlan {
  alignas(16) unsigned char key[1024] = {};  // GraphKey bytes
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int64_t launches_first = 0, launches_body = 0;
  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
  }
};

struct Ctx {
  bool init = false;
  int device = -1;
  int num_sms = 0;
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static constexpr int kSlots = 16;  // passes with a status slot (max_passes <= kSlots)
  DevStatus* st_host = nullptr;      // pinned, mapped: one slot per pass
  DevStatus* st_host_dev = nullptr;  // device alias of st_host
  cudaEvent_t ev = nullptr;
  cudaEvent_t ev_pass[kSlots] = {};  // chol of pass k done (its status slot is readable)
  int cur_pass = 0;                  // pass being enqueued (tags the profiling events)
  static constexpr int kPlans = 4;   // cached CUDA-graph pass loops (single GPU), one per argument set
  GraphPlan plans[kPlans];           //   (scqr3_factor_host_batch rotates three staging buffers)
  int plan_next = 0;                 // replacement cursor
  bool plan_failed = false;          // capture not supported here: the host loop from now on
  // scqr3_factor_host_batch: upload / download streams and per-staging-buffer events
  cudaStream_t up = nullptr, down = nullptr;
  cudaEvent_t ev_up[3] = {}, ev_fact[3] = {}, ev_down[3] = {}, ev_start = nullptr;
  cudaStream_t side = nullptr;     // R accumulation, overlapped with the TRSM
  cudaStream_t cap = nullptr;      // graph capture (the caller's stream may be the legacy default)
  cudaEvent_t ev_chol = nullptr;   // chol done (st) -> side may start
  cudaEvent_t ev_side = nullptr;   // side done -> st may reuse the R~ buffer
  // profiling: event pairs recorded around launches when opts->prof is set
  static constexpr int kMaxEv = 128;
  cudaEvent_t ev_a[kMaxEv] = {}, ev_b[kMaxEv] = {};
  int ev_kind[kMaxEv] = {};
  int ev_tag[kMaxEv] = {};
  int ev_used = 0;
  scqr3_prof* prof = nullptr;
  cudaStream_t prof_stream = nullptr;
};
thread_local Ctx g_ctx[16];

enum ProfKind { PK_GRAM = 0, PK_REDUCE = 1, PK_CHOL = 2, PK_TRSM = 3, PK_COMM = 4, PK_TRMUL = 5 };

// Opens a timed region on the stream (no-op unless profiling); returns the slot or -1.
int prof_begin(Ctx* c, int kind) {
  if (!c->prof || c->ev_used >= Ctx::kMaxEv) return -1;
  const int i = c->ev_used++;
  if (!c->ev_a[i]) {
    cudaEventCreate(&c->ev_a[i]);
    cudaEventCreate(&c->ev_b[i]);
  }
  c->ev_kind[i] = kind;
  c->ev_tag[i] = c->cur_pass;
  cudaEventRecord(c->ev_a[i], kind == PK_TRMUL ? c->side : c->prof_stream);
  return i;
}
void prof_end(Ctx* c, int slot) {
  if (slot >= 0) cudaEventRecord(c->ev_b[slot], c->ev_kind[slot] == PK_TRMUL ? c->side : c->prof_stream);
}
// After the stream has been synchronised: fold the recorded pairs into *prof (launches of
// speculative passes beyond the last executed one are left out).
void prof_flush(Ctx* c, int last_pass = 1 << 30) {
  if (!c->prof) return;
  for (int i = 0; i < c->ev_used; ++i) {
    if (c->ev_tag[i] > last_pass) continue;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->ev_a[i], c->ev_b[i]) != cudaSuccess) continue;
    switch (c->ev_kind[i]) {
      case PK_GRAM: c->prof->gram_ms += ms; c->prof->gram_launches++; break;
      case PK_REDUCE: c->prof->reduce_ms += ms; c->prof->reduce_launches++; break;
      case PK_CHOL: c->prof->chol_ms += ms; c->prof->chol_launches++; break;
      case PK_TRSM: c->prof->trsm_ms += ms; c->prof->trsm_launches++; break;
      case PK_TRMUL: c->prof->trmul_ms += ms; c->prof->trmul_launches++; break;
      default: c->prof->comm_ms += ms; c->prof->comm_calls++; break;
    }
  }
  c->ev_used = 0;
}

int get_ctx(Ctx** out) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 16) return fail("device index %d out of range", dev);
  Ctx& c = g_ctx[dev];
  if (!c.init) {
    c.device = dev;
    CUDA_TRY(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, dev));
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return fail("cuTensorMapEncodeTiled not available");
    c.encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&c.st_host), sizeof(DevStatus) * Ctx::kSlots, cudaHostAllocMapped));
    for (int i = 0; i < Ctx::kSlots; ++i) CUDA_TRY(cudaEventCreateWithFlags(&c.ev_pass[i], cudaEventDisableTiming));
    CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c.st_host_dev), c.st_host, 0));
    CUDA_TRY(cudaEventCreateWithFlags(&c.ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c.ev_chol, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c.ev_side, cudaEventDisableTiming));
    CUDA_TRY(cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&c.cap, cudaStreamNonBlocking));
    c.init = true;
  }
  *out = &c;
  return SCQR3_OK;
}

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

int max_chunks_for_device() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return std::max(sms, 1) * 4;
}

struct Layout {
  int n, npad, NT;
  long long tiles_sym;     // NT(NT+1)/2
  long long tiles_part;    // per partial
  int max_chunks;
  long long ldy;
  // offsets (bytes)
  size_t st, partials, tiles, W, Rnew, Rt, bfrag, dblk, misc, colsq, y, halo, end;
};

Layout make_layout(int64_t m, int64_t n, int oblique, int64_t halo = 1) {
  Layout L{};
  L.n = static_cast<int>(n);
  L.npad = npad_for(L.n);
  L.NT = L.npad / 8;
  L.tiles_sym = static_cast<long long>(L.NT) * (L.NT + 1) / 2;
  L.tiles_part = oblique ? 2 * L.tiles_sym : L.tiles_sym;  // oblique: [Q^T Y][Q^T Q] upper tiles (D22, D4)
  {
    // CTAs per row chunk = job groups (assign_gram_jobs); fewer chunks fit on the GPU when there are more
    const long long nb = (L.NT + kJobTiles - 1) / kJobTiles;
    const long long codes = 2 * (nb * (nb + 1) / 2) * (oblique ? 2 : 1);
    const int groups_hi = static_cast<int>(std::max<long long>(1, (codes + kMaxConsumers - 1) / kMaxConsumers));
    L.max_chunks = std::max(1, max_chunks_for_device() / groups_hi);
  }
  L.ldy = std::max<long long>(2, (m + 1) & ~1LL);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return o;
  };
  L.st = take(sizeof(DevStatus));
  L.partials = take(static_cast<size_t>(L.max_chunks) * L.tiles_part * 64 * 8);
  L.tiles = take(static_cast<size_t>(L.tiles_sym * 64 * (oblique ? 2 : 1) + 64) * 8);
  L.W = take(static_cast<size_t>(n) * chol_ldw(static_cast<int>(n)) * 8);
  L.Rnew = take(static_cast<size_t>(n) * n * 8);
  L.Rt = take(static_cast<size_t>(n) * n * 8);
  L.bfrag = take(static_cast<size_t>(L.NT) * (L.NT - 1) * 32 * 8 + 8);
  L.dblk = take(static_cast<size_t>(dblk_doubles(L.NT)) * 8);
  L.misc = take(64 * 8);  // [0] nb, [1] e_prev, [2] m_global (int64), ...
  L.colsq = oblique ? take(4096 * 8) : off;
  L.y = oblique ? take(static_cast<size_t>(L.ldy) * n * 8) : off;
  L.halo = oblique ? take(static_cast<size_t>(4 * std::max<int64_t>(halo, 1) * n) * 8) : off;
  L.end = off;
  return L;
}

struct WS {
  DevStatus* st;
  double *partials, *tiles, *W, *Rnew, *Rt, *bfrag, *dblk, *misc, *colsq, *y, *halo;
};

int carve(const Layout& L, const scqr3_opts* o, WS* w) {
  if (!o->workspace) return fail("opts->workspace is NULL");
  if (o->workspace_bytes < L.end) return fail("workspace too small: %zu < %zu bytes", o->workspace_bytes, L.end);
  if (reinterpret_cast<uintptr_t>(o->workspace) % 256) return fail("workspace must be 256-byte aligned");
  char* b = static_cast<char*>(o->workspace);
  w->st = reinterpret_cast<DevStatus*>(b + L.st);
  w->partials = reinterpret_cast<double*>(b + L.partials);
  w->tiles = reinterpret_cast<double*>(b + L.tiles);
  w->W = reinterpret_cast<double*>(b + L.W);
  w->Rnew = reinterpret_cast<double*>(b + L.Rnew);
  w->Rt = reinterpret_cast<double*>(b + L.Rt);
  w->bfrag = reinterpret_cast<double*>(b + L.bfrag);
  w->dblk = reinterpret_cast<double*>(b + L.dblk);
  w->misc = reinterpret_cast<double*>(b + L.misc);
  w->colsq = reinterpret_cast<double*>(b + L.colsq);
  w->y = reinterpret_cast<double*>(b + L.y);
  w->halo = reinterpret_cast<double*>(b + L.halo);
  return SCQR3_OK;
}

int check_opts(const scqr3_opts* o) {
  if (!o) return fail("opts is NULL");
  if (o->abi_version != SCQR3_ABI_VERSION) return fail("abi_version %d != %d", o->abi_version, SCQR3_ABI_VERSION);
  if (o->shift_mode < 0 || o->shift_mode > 4) return fail("bad shift_mode %d", o->shift_mode);
  if (o->norm_mode < 0 || o->norm_mode > 2) return fail("bad norm_mode %d", o->norm_mode);
  if (o->trsm_diag < 0 || o->trsm_diag > 2) return fail("bad trsm_diag %d", o->trsm_diag);
  if (o->norm_mode == SCQR3_NORM_USER && !(o->norm2_bound > 0)) return fail("NORM_USER needs norm2_bound > 0");
  if (o->shift_mode == SCQR3_SHIFT_FIXED && !(o->shift_value >= 0)) return fail("SHIFT_FIXED needs shift_value >= 0");
  return SCQR3_OK;
}

int check_matrix(const char* name, const double* p, int64_t m, int64_t ld) {
  if (m > 0 && !p) return fail("%s is NULL", name);
  if (ld < std::max<int64_t>(m, 1)) return fail("%s: leading dimension %lld < m=%lld", name, (long long)ld, (long long)m);
  if (ld % 2) return fail("%s: leading dimension must be even (TMA needs 16-byte row pitch)", name);
  if (reinterpret_cast<uintptr_t>(p) % 16) return fail("%s must be 16-byte aligned", name);
  return SCQR3_OK;
}

int encode_map(Ctx* c, CUtensorMap* map, const double* base, int64_t m, int64_t n, int64_t ld, int npad) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(n)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kGramStageRows), static_cast<cuuint32_t>(std::min(npad, kTmaBoxCols))};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = c->encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail("cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return SCQR3_OK;
}

// 3-D view of a column-major m x n block for 32-row Gram stages (m % 32 == 0): dims {16 rows,
// m / 16 row blocks, n columns}, box {16, 2, box_cols}, SWIZZLE_128B per 128-B line (gram.cu, RB)
int encode_map3(Ctx* c, CUtensorMap* map, const double* base, int64_t m, int64_t n, int64_t ld, int box_cols) {
  cuuint64_t dims[3] = {16, static_cast<cuuint64_t>(m / 16), static_cast<cuuint64_t>(n)};
  cuuint64_t strides[2] = {128, static_cast<cuuint64_t>(ld) * 8};
  cuuint32_t box[3] = {16, 2, static_cast<cuuint32_t>(box_cols)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = c->encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail("cuTensorMapEncodeTiled (3-D) failed (%d)", static_cast<int>(r));
  return SCQR3_OK;
}

const bool g_gram_debug = std::getenv("SCQR3_GRAM_DEBUG") != nullptr;
const bool g_gram_rb2 = [] {  // 32-row stages (SCQR3_GRAM_RB=1: 16-row stages only, A/B)
  const char* v = std::getenv("SCQR3_GRAM_RB");
  return !(v && v[0] == '1');
}();
const int g_gram_force_groups = std::getenv("SCQR3_GRAM_GROUPS") ? std::atoi(std::getenv("SCQR3_GRAM_GROUPS")) : 0;
const bool g_gram_mc = [] {
  const char* v = std::getenv("SCQR3_GRAM_MC");
  return !(v && v[0] == '0');
}();

// Gram jobs for the consumer warps.  Job codes: 2*block + part.  Three kernel variants:
//   0: JR = 2, <= 20 consumers -- a job is a part (tile rows 2*part, 2*part+1 of a 4x4-tile
//      block: 8 tiles off the diagonal, 7 / 3 on it);
//   1: JR = 4, <= 18 consumers (96 registers) -- a job is a whole block (16 / 10 tiles);
//   2: JR = 4, <= 15 consumers (128 registers).
// Within a variant, jobs are split over `groups` CTAs sharing each row chunk and assigned
// longest first to the least-loaded SM sub-partition (warp w of the CTA runs on sub-partition
// w % 4; consumer c is warp c + 1).  Each SM runs one CTA and a chunk has total/chunks =
// total*groups/SMs stages, so the variant with the least
//     groups x max(64 cycles x (max sub-partition DMMA tiles per stage), stage bytes / 16 B)
// is taken: 4 k-steps of 16 cycles per tile, and ~16 B/cycle/SM of L2 -> shared memory when every
// CTA of a chunk streams its own copy (fit to measured times of all three variants, forced, at
// n = 96, 128, 192, 256, 384, 512 and the oblique n = 64, 128: the model picks the fastest --
// 0 up to n = 128, a whole-block variant above: 1 at n = 192 (2 within 1 %), 2 at 256, 1 at 512).
// Returns the number of groups; sets *ncons_out and *variant_out.
int assign_gram_jobs(GramParams& gp, bool oblique, bool dual, int* ncons_out, int* variant_out) {
  const long long load_cycles = static_cast<long long>(gp.npad) * 128 * (oblique ? 2 : 1) / 16;
  // upper blocks only, also for the oblique Gram (reading D22); the oblique Gram adds the plain
  // Gram's blocks (job codes past 2 * nsym) for its norm estimate (reading D4)
  const int nsym = gp.NB * (gp.NB + 1) / 2;
  const int nblocks = dual ? 2 * nsym : nsym;
  auto coords = [&](int j, int& bi, int& bj) {
    if (j >= nsym) j -= nsym;
    int c = 0;
    while ((c + 1) * (c + 2) / 2 <= j) ++c;
    bj = c;
    bi = j - c * (c + 1) / 2;
  };
  auto weight = [&](int code, int jr) {
    int bi, bj;
    coords(code >> 1, bi, bj);
    const int r0 = 2 * (code & 1);
    int w = 0;
    for (int a = r0; a < r0 + jr; ++a)
      for (int b = 0; b < kJobTiles; ++b)
        if (bi * kJobTiles + a < gp.NT && bj * kJobTiles + b < gp.NT && (bi != bj || a <= b)) ++w;
    return w;
  };
  static const int kVariant[3][2] = {{2, kMaxConsumers}, {4, kMaxConsumersWhole}, {4, kMaxConsumersWhole2}};
  long long best_cost = -1;
  int best = 0, best_groups = 1, best_ncons = 0;
  std::vector<short> best_job;
  for (int v = 0; v < 3; ++v) {
    const int jr = kVariant[v][0], maxc = kVariant[v][1];
    std::vector<int> codes;
    for (int j = 0; j < nblocks; ++j)
      for (int part = 0; part < (jr == 2 ? 2 : 1); ++part)
        if (weight(2 * j + part, jr) > 0) codes.push_back(2 * j + part);
    const int jobs = static_cast<int>(codes.size());
    const int groups = std::max(1, (jobs + maxc - 1) / maxc);
    if (groups > kMaxGroups || (g_gram_force_groups > 0 && groups != g_gram_force_groups)) continue;
    int ncons = 0;
    for (int g = 0; g < groups; ++g) ncons = std::max(ncons, jobs * (g + 1) / groups - jobs * g / groups);
    std::vector<short> job(kMaxGroups * kMaxConsumers, -1);
    int maxload = 0;
    for (int g = 0; g < groups; ++g) {
      const int j0 = jobs * g / groups, j1 = jobs * (g + 1) / groups;
      std::vector<int> order(codes.begin() + j0, codes.begin() + j1);
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return weight(x, jr) > weight(y, jr); });
      int load[4] = {0, 0, 0, 0};
      bool used[kMaxConsumers] = {};
      for (int code : order) {
        int bw = -1;
        for (int w = 0; w < ncons; ++w) {
          if (used[w]) continue;
          if (bw < 0 || load[(w + 1) & 3] < load[(bw + 1) & 3]) bw = w;
        }
        used[bw] = true;
        load[(bw + 1) & 3] += weight(code, jr);
        job[g * kMaxConsumers + bw] = static_cast<short>(code);
      }
      for (int q = 0; q < 4; ++q) maxload = std::max(maxload, load[q]);
    }
    // (parts load 6 fragments per 8 DMMA against 8 per 16 for whole blocks: 69 instead of 64
    //  cycles per tile and k-step, fitted so n = 192 takes a whole-block variant, measured 4 % faster)
    const long long tile_cycles = jr == 2 ? 69 : 64;
    const long long cost = static_cast<long long>(groups) * std::max<long long>(tile_cycles * maxload, load_cycles);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = v;
      best_groups = groups;
      best_ncons = ncons;
      best_job = job;
    }
  }
  for (int i = 0; i < kMaxGroups * kMaxConsumers; ++i) gp.warp_job[i] = best_job[i];
  *ncons_out = best_ncons;
  *variant_out = best;
  return best_groups;
}

// Sum `chunks` partials (per-CTA packed upper tiles) into w.tiles in chunk order.
int launch_gram_reduce(Ctx* c, const Layout& L, const WS& w, int chunks, bool oblique, bool dual, int colsq_count,
                       cudaStream_t st, PassGate gate, int NTc = 0) {
  GramReduceParams rp{};
  rp.gate = gate;
  rp.partials = w.partials;
  rp.tiles = w.tiles;
  rp.chunks = chunks;
  rp.tiles_per_partial = static_cast<int>(L.tiles_part);
  rp.NT = L.NT;
  rp.NTc = NTc > 0 ? NTc : L.NT;
  rp.oblique = oblique ? 1 : 0;
  rp.colsq_partials = oblique ? w.colsq : nullptr;
  rp.colsq_count = colsq_count;
  rp.dual = dual ? 1 : 0;
  const long long nblocks = (L.tiles_sym * 64 * (dual ? 2 : 1) + 31) / 32;  // 32 outputs x 8 chunk classes
  const int pr = prof_begin(c, PK_REDUCE);
  gram_reduce_kernel<<<static_cast<unsigned>(nblocks), 256, 0, st>>>(rp);
  prof_end(c, pr);
  ++g_launches;
  CUDA_TRY(cudaGetLastError());
  return SCQR3_OK;
}

// Gram of the m x n block at src into w.tiles (packed upper tiles; oblique: sym(Q^T Y) and ||Q||_F^2,
// dual: then the plain Gram Q^T Q for the norm estimate of reading D4)
int run_gram(Ctx* c, const Layout& L, const WS& w, const double* src, int64_t ld, int64_t m, bool oblique,
             const ObliqueYParams* yp, cudaStream_t st, PassGate gate = PassGate{}, bool dual = false) {
  if (m == 0) {
    // an empty shard contributes zeros to every summed entry: the (B-)Gram, ||Q||_F^2 and, for
    // the oblique layout, the plain Gram behind them
    const long long nout = L.tiles_sym * 64 * (oblique ? 2 : 1) + 1;
    CUDA_TRY(cudaMemsetAsync(w.tiles, 0, static_cast<size_t>(nout) * 8, st));
    return SCQR3_OK;
  }
  int colsq_count = 0;
  if (oblique) {
    ObliqueYParams p = *yp;
    p.gate = gate;
    const long long total = m * static_cast<long long>(L.n);
    long long blocks = std::min<long long>((total + 255) / 256, 4096);
    colsq_count = static_cast<int>(std::max<long long>(blocks, 1));
    p.colsq_partials = w.colsq;
    const int ps = prof_begin(c, PK_REDUCE);
    if (p.rp) {
      // SCQR3_CSR_Y=0 selects the round-1 kernel (one thread per row and 16-column chunk; A/B
      // measurement); the default is the 256-row tile kernel with the CSR arrays staged in shared memory
      static const bool tile = [] {
        const char* v = std::getenv("SCQR3_CSR_Y");
        return !(v && v[0] == '0');
      }();
      if (tile && p.csr_tile) {
        colsq_count = static_cast<int>(std::min<long long>((m + kCsrTileRows - 1) / kCsrTileRows, 4096));
        csr_y_tile_kernel<<<colsq_count, kCsrTileRows, 0, st>>>(p);
      } else {
        csr_y_kernel<<<colsq_count, 256, 0, st>>>(p);
      }
    } else {
      colsq_count = static_cast<int>(std::max<long long>(1, std::min<long long>((m + 255) / 256, 4096)));
      p.colsq_partials = w.colsq;
      oblique_y_kernel<<<colsq_count, 256, 0, st>>>(p);
    }
    prof_end(c, ps);
    ++g_launches;
    CUDA_TRY(cudaGetLastError());
  }
  GramParams gp{};
  gp.gate = gate;
  // only the tiles of the n columns: L.npad rounds n up to a TRSM instance (n = 144 -> 192), whose
  // zero columns the Gram need not stream or multiply; the partials keep the L.NT layout
  const int NTc = (L.n + 7) / 8;
  gp.NT = NTc;
  gp.NTl = L.NT;
  gp.NB = (NTc + kJobTiles - 1) / kJobTiles;
  gp.npad = 8 * NTc;
  gp.oblique = oblique ? 1 : 0;
  gp.dual = dual ? 1 : 0;
  gp.tiles_per_partial = static_cast<int>(L.tiles_part);
  int ncons = 0, variant = 0;
  const int groups = assign_gram_jobs(gp, oblique, dual, &ncons, &variant);
  if (groups > kMaxGroups) return fail("internal: too many Gram job groups");
  gp.groups = groups;
  const int threads = 32 * (1 + ncons);
  const int nsrc = oblique ? 2 : 1;
  const size_t stage_bytes = static_cast<size_t>(gp.npad) * 128;
  // 2..8 stages within ~96 KB; a single (serialising) stage only where two do not fit (oblique, npad 512)
  const size_t max_stages = (kGramSmemCap - 2048) / (stage_bytes * nsrc);
  gp.stages = static_cast<int>(std::min<size_t>(std::min<size_t>(8, max_stages), std::max<size_t>(2, 98304 / (stage_bytes * nsrc))));
  size_t smem = gp.stages * nsrc * stage_bytes + 2 * gp.stages * 8 + 1024;
  int occ = 1;
  CUDA_TRY(gram_tma_config(variant, false, smem, threads, &occ));
  occ = std::max(occ, 1);
  gp.total_stages = (m + kGramStageRows - 1) / kGramStageRows;
  long long chunks = std::min<long long>((gp.total_stages + 3) / 4, static_cast<long long>(c->num_sms) * occ / groups);
  chunks = std::max<long long>(1, std::min<long long>(chunks, L.max_chunks));
  // Several CTAs per row chunk (n > 128): make them a thread-block cluster and multicast each
  // stage (one L2 read per stage instead of one per CTA: DRAM reads 8mn instead of ~2x), with a
  // deeper stage ring (a cluster advances at the pace of its slowest CTA).  Taken only when as
  // many clusters fit at once as there are row chunks -- GPC granularity can leave SMs idle
  // (n = 256: 45 clusters of 3 against 49 chunks, 10 % slower).  n = 192: 5.56 ms either way at
  // m = 4e6 with half the DRAM traffic.  SCQR3_GRAM_MC=0 turns it off (A/B measurement).
  gp.mc = 1;
  int ncl = 0;
  if (groups > 1 && groups <= 8 && gp.npad % 32 == 0 && g_gram_mc) {
    const int st_mc = static_cast<int>(std::min<size_t>(8, max_stages));
    const size_t smem_mc = st_mc * nsrc * stage_bytes + 2 * st_mc * 8 + 1024;
    int occ_mc = 0;
    CUDA_TRY(gram_tma_config(variant, true, smem_mc, threads, &occ_mc));
    CUDA_TRY(gram_tma_max_clusters(variant, smem_mc, threads, groups, &ncl));
    if (ncl >= chunks) {
      gp.mc = groups;
      gp.stages = st_mc;
      smem = smem_mc;
    }
  }
  // 32-row stages through a 3-D view (two 128-B lines per column and box: TMA reads at 7.3
  // instead of 4.6 TB/s, tools/tma_probe.cu) when the rows tile into them, with the same ring
  // bytes.  Measured at m = 1e7 / 4e6 / 2e6: n = 128 5.13 -> 5.02 ms, n = 64 1.758 -> 1.713 ms;
  // slower for n = 96 (1.351 -> 1.393), n = 256 (4.15 -> 4.18) and the oblique dual Gram at
  // n = 64 (0.582 -> 0.605 ms), which keep 16-row stages
  gp.rb = 1;
  if (gp.mc == 1 && m % 32 == 0 && g_gram_rb2 && !oblique && (gp.npad == 64 || gp.npad == 128)) {
    const size_t sb2 = 2 * stage_bytes;
    const size_t max2 = (kGramSmemCap - 2048) / (sb2 * nsrc);
    if (max2 >= 2) {
      gp.rb = 2;
      // the same ring bytes as the 16-row plan (so as many CTAs fit per SM), at least two stages
      gp.stages = static_cast<int>(std::min<size_t>(max2, std::max(2, gp.stages / 2)));
      smem = gp.stages * nsrc * sb2 + 2 * gp.stages * 8 + 1024;
      CUDA_TRY(gram_tma_config(variant, false, smem, threads, &occ, 2));
      occ = std::max(occ, 1);
      gp.total_stages = m / 32;
      chunks = std::min<long long>((gp.total_stages + 3) / 4, static_cast<long long>(c->num_sms) * occ / groups);
      chunks = std::max<long long>(1, std::min<long long>(chunks, L.max_chunks));
    }
  }
  if (g_gram_debug)
    fprintf(stderr, "gram: n=%d variant=%d groups=%d ncons=%d stages=%d smem=%zu occ=%d mc=%d clusters=%d chunks=%lld rb=%d\n",
            L.n, variant, groups, ncons, gp.stages, smem, occ, gp.mc, ncl, chunks, gp.rb);
  // (equal TMA boxes of <= kTmaBoxCols columns that tile the stage exactly)
  gp.box_cols = gp.mc > 1 ? 32 : gp.npad / ((gp.npad + kTmaBoxCols - 1) / kTmaBoxCols);
  CUtensorMap mq, my;
  if (gp.rb == 2) {
    TRY(encode_map3(c, &mq, src, m, L.n, ld, gp.box_cols));
    if (oblique) TRY(encode_map3(c, &my, w.y, m, L.n, L.ldy, gp.box_cols));
    else my = mq;
  } else {
    TRY(encode_map(c, &mq, src, m, L.n, ld, gp.box_cols));
    if (oblique) TRY(encode_map(c, &my, w.y, m, L.n, L.ldy, gp.box_cols));
    else my = mq;
  }
  gp.chunks = static_cast<int>(chunks);
  gp.partials = w.partials;
  const int pg = prof_begin(c, PK_GRAM);
  const cudaError_t le = launch_gram_tma(variant, static_cast<unsigned>(chunks * groups), threads, smem, st, mq, my, gp);
  prof_end(c, pg);
  ++g_launches;
  CUDA_TRY(le);

  return launch_gram_reduce(c, L, w, gp.chunks, oblique, dual, colsq_count, st, gate, NTc);
}

int launch_chol(const CholParams& p, cudaStream_t st) {
  if (p.w_in_smem) {
    const size_t smem = static_cast<size_t>(p.n) * chol_ldw(p.n) * 8;
    static thread_local LaunchCfgCache chol_cfg;
    CUDA_TRY(cached_launch_cfg(chol_cfg, chol_kernel_smem, smem, 256, nullptr));
    chol_kernel_smem<<<1, 256, smem, st>>>(p);
  } else {
    // (W in global memory; shared memory holds two copies of the panel rows, chol.cu)
    const size_t smem = static_cast<size_t>(2 * 8) * chol_ldw(p.n) * 8;
    static thread_local LaunchCfgCache chol_cfg_g;
    CUDA_TRY(cached_launch_cfg(chol_cfg_g, chol_kernel_gmem, smem, 256, nullptr));
    chol_kernel_gmem<<<1, 256, smem, st>>>(p);
  }
  ++g_launches;
  CUDA_TRY(cudaGetLastError());
  return SCQR3_OK;
}

// a6 on the side stream: R := R~ R once this pass's chol_kernel is done; the main stream only
// waits for it before the next chol_kernel overwrites R~ (by then the TRSM has long finished).
int launch_trmul(Ctx* c, const double* Rt, double* R, double* Rnew, int n, int first, const DevStatus* st_dev,
                 cudaStream_t st, PassGate gate) {
  CUDA_TRY(cudaEventRecord(c->ev_chol, st));
  CUDA_TRY(cudaStreamWaitEvent(c->side, c->ev_chol, 0));
  const long long nn = static_cast<long long>(n) * n;
  const unsigned blocks = static_cast<unsigned>((nn + 127) / 128);
  const int pt = prof_begin(c, PK_TRMUL);
  trmul_kernel<<<blocks, 128, 0, c->side>>>(Rt, R, Rnew, n, first, st_dev, gate);
  copy_kernel<<<blocks, 128, 0, c->side>>>(Rnew, R, nn, st_dev, gate);
  prof_end(c, pt);
  g_launches += 2;
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaEventRecord(c->ev_side, c->side));
  return SCQR3_OK;
}

bool w_fits_smem(int n) { return static_cast<size_t>(n) * chol_ldw(n) * 8 <= 200 * 1024; }

// ---- CUDA-graph pass loop (device-side pass control)
// SCQR3_GRAPH=0 selects the host-driven loop for single-GPU calls too (A/B measurement).
// SCQR3_FUSE_TG=0 selects the unfused TRSM + Gram pair for n <= 64 (A/B measurement).
const bool g_fuse_tg = [] {
  const char* v = std::getenv("SCQR3_FUSE_TG");
  return !(v && v[0] == '0');
}();
const bool g_use_graph = [] {
  const char* v = std::getenv("SCQR3_GRAPH");
  return !(v && v[0] == '0');
}();

// Everything a captured pass loop bakes in (pointers, sizes, kernel parameter blocks).
struct GraphKey {
  const double* X;
  const double* Q;
  double* R;
  int64_t ld, ldq, m, n;
  void* ws;
  cudaStream_t st;
  int max_passes;
  CholParams cp;
  TrsmParams tp;
  ObliqueYParams yp;
};

// Graph: [control init, pass 1, loop condition] -> WHILE (cond) { pass k = ++counter; condition }
template <class Init, class Enq>
int capture_pass_loop(Ctx* c, cudaStream_t st, int max_passes, int* last_pass, int* pass_dev, Init& init,
                      Enq& enqueue, GraphPlan* out) {
  cudaGraph_t g = nullptr;
  CUDA_TRY(cudaGraphCreate(&g, 0));
  auto bail = [&](int rc) {
    cudaStreamCaptureStatus cs;
    if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
      cudaGraph_t tmp = nullptr;
      cudaStreamEndCapture(st, &tmp);
    }
    cudaGetLastError();
    cudaGraphDestroy(g);
    return rc;
  };
  cudaGraphConditionalHandle h;
  if (cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault) != cudaSuccess)
    return bail(fail("cudaGraphConditionalHandleCreate failed"));
  const int64_t l0 = g_launches;
  // segment A
  if (cudaStreamBeginCaptureToGraph(st, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) != cudaSuccess)
    return bail(fail("cudaStreamBeginCaptureToGraph failed"));
  int rc = init();
  if (rc == SCQR3_OK) rc = enqueue(1);
  if (rc != SCQR3_OK) return bail(rc);
  if (cudaStreamWaitEvent(st, c->ev_side, 0) != cudaSuccess) return bail(fail("join failed"));
  pass_loop_cond_kernel<<<1, 32, 0, st>>>(pass_dev, last_pass, max_passes, h);
  if (cudaGetLastError() != cudaSuccess) return bail(fail("loop condition launch failed"));
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  if (cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &ndeps) != cudaSuccess)
    return bail(fail("cudaStreamGetCaptureInfo failed"));
  std::vector<cudaGraphNode_t> dep(deps, deps + ndeps);
  cudaGraph_t gA = nullptr;
  if (cudaStreamEndCapture(st, &gA) != cudaSuccess) return bail(fail("capture of pass 1 failed"));
  const int64_t l1 = g_launches;
  // the WHILE node and its body (one generic pass)
  cudaGraphNodeParams np{};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t wnode;
  if (cudaGraphAddNode(&wnode, g, dep.data(), dep.size(), &np) != cudaSuccess)
    return bail(fail("adding the WHILE node failed"));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  if (cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) != cudaSuccess)
    return bail(fail("capture of the loop body failed to start"));
  rc = enqueue(0);
  if (rc != SCQR3_OK) return bail(rc);
  if (cudaStreamWaitEvent(st, c->ev_side, 0) != cudaSuccess) return bail(fail("join failed"));
  pass_loop_cond_kernel<<<1, 32, 0, st>>>(pass_dev, last_pass, max_passes, h);
  if (cudaGetLastError() != cudaSuccess) return bail(fail("loop condition launch failed"));
  cudaGraph_t gB = nullptr;
  if (cudaStreamEndCapture(st, &gB) != cudaSuccess) return bail(fail("capture of the loop body failed"));
  const int64_t l2 = g_launches;
  cudaGraphExec_t exec = nullptr;
  if (cudaGraphInstantiate(&exec, g, 0) != cudaSuccess) return bail(fail("cudaGraphInstantiate failed"));
  g_launches = l0;  // capture launched nothing; replays are counted per executed pass
  out->graph = g;
  out->exec = exec;
  out->launches_first = l1 - l0 + 1;
  out->launches_body = l2 - l1 + 1;
  return SCQR3_OK;
}

// The oblique metric of a factorisation: none (standard), tridiagonal bands, or CSR.
struct Metric {
  const double* d = nullptr;
  const double* e = nullptr;
  const scqr3_csr* csr = nullptr;
  bool oblique() const { return d != nullptr || csr != nullptr; }
  // ghost-row plan by sparsity pattern (scqr3_csr.halo == SCQR3_CSR_GHOSTS)
  bool ghosts() const { return csr && csr->halo == SCQR3_CSR_GHOSTS; }
  int64_t nsend(int nranks) const {
    int64_t s = 0;
    if (ghosts() && csr->send_counts)
      for (int r = 0; r < nranks; ++r) s += csr->send_counts[r];
    return s;
  }
  // rows of the workspace's halo region (4 blocks of halo x n): the ghost plan keeps its
  // nghost received and nsend packed rows there
  int64_t halo(int nranks = 1) const {
    if (ghosts()) return std::max<int64_t>(1, (csr->nghost + nsend(nranks) + 3) / 4);
    return csr ? csr->halo : 1;
  }
};

// Local argument checks of factor_impl (everything that can fail before the first exchange).
int factor_checks(int64_t m, int64_t n, const double* X, int64_t ld, const Metric& B, const double* Q, int64_t ldq,
                  const double* R, const scqr3_opts* o, Ctx** c, Layout* L, WS* w) {
  const Comm* cm = static_cast<const Comm*>(o->comm);
  TRY(check_opts(o));
  if (n < 1 || n > kMaxN) return fail("n=%lld outside [1, %d]", (long long)n, kMaxN);
  if (m < 0) return fail("m < 0");
  TRY(check_matrix("X", X, m, ld));
  TRY(check_matrix("Q", Q, m, ldq));
  if (!R) return fail("R is NULL");
  if (B.d && m > 0 && !B.e) return fail("b_off is NULL");
  const int nranks = cm ? cm->nranks : 1;
  if (B.csr) {
    if (m > 0 && (!B.csr->row_ptr || !B.csr->col_idx || !B.csr->vals)) return fail("CSR metric has a NULL array");
    if (B.ghosts()) {
      const scqr3_csr& g = *B.csr;
      if (g.nghost < 0) return fail("CSR ghost plan: nghost < 0");
      if (!cm) {
        if (g.nghost != 0) return fail("CSR ghost plan: nghost must be 0 without a communicator");
      } else {
        if (!g.recv_counts || !g.send_counts) return fail("CSR ghost plan: NULL recv_counts / send_counts");
        int64_t nr = 0, ns = 0;
        for (int r = 0; r < nranks; ++r) {
          if (g.recv_counts[r] < 0 || g.send_counts[r] < 0) return fail("CSR ghost plan: negative count");
          nr += g.recv_counts[r];
          ns += g.send_counts[r];
        }
        if (g.recv_counts[cm->rank] != 0 || g.send_counts[cm->rank] != 0)
          return fail("CSR ghost plan: a rank does not exchange rows with itself");
        if (nr != g.nghost) return fail("CSR ghost plan: sum of recv_counts %lld != nghost %lld", (long long)nr,
                                        (long long)g.nghost);
        if (ns > 0 && !g.send_rows) return fail("CSR ghost plan: send_rows is NULL");
      }
    } else {
      if (B.csr->halo < 0) return fail("CSR halo < 0");
      if (!cm && B.csr->halo != 0) return fail("CSR halo must be 0 without a communicator");
    }
  }
  // a rank of an oblique factorisation must own at least its halo rows (its neighbours read them)
  if (cm && B.oblique() && !B.ghosts() && cm->nranks > 1 && m < std::max<int64_t>(B.halo(), 1))
    return fail("oblique metric across ranks: this rank owns %lld rows, fewer than the halo (%lld)", (long long)m,
                (long long)std::max<int64_t>(B.halo(), 1));
  const int max_passes = o->max_passes > 0 ? o->max_passes : 8;
  if (max_passes > Ctx::kSlots) return fail("max_passes %d > %d", max_passes, Ctx::kSlots);
  TRY(get_ctx(c));
  *L = make_layout(m, n, B.oblique(), B.halo(nranks));
  TRY(carve(*L, o, w));
  return SCQR3_OK;
}

int factor_body(int64_t m, int64_t n, const double* X, int64_t ld, const Metric& B, double* Q, int64_t ldq,
                double* R, const scqr3_opts* o, bool* in_protocol) {
  if (!o) return fail("opts is NULL");
  Comm* cm = static_cast<Comm*>(o->comm);
  cudaStream_t st = static_cast<cudaStream_t>(o->stream);
  Ctx* c = nullptr;
  Layout L{};
  WS w{};
  const int rc_local = factor_checks(m, n, X, ld, B, Q, ldq, R, o, &c, &L, &w);
  // every rank returns SCQR3_EINVAL together when any rank's arguments are bad (no rank is left
  // waiting in an exchange)
  if (cm) TRY(comm_agree(cm, rc_local == SCQR3_OK, st));
  else TRY(rc_local);
  *in_protocol = cm != nullptr;
  const bool oblique = B.oblique();
  const double* bd = B.d;
  const double* be = B.e;
  c->prof = o->prof;
  c->prof_stream = st;
  c->ev_used = 0;
  const int max_passes = o->max_passes > 0 ? o->max_passes : 8;
  const double stop_tol = o->stop_tol > 0 ? o->stop_tol : 0.5;
  const int iters = o->power_iters > 0 ? o->power_iters : 32;

  // global m (the shift uses the global m)
  int64_t mg = o->m_global;
  if (mg <= 0) {
    if (cm) TRY(comm_host_allreduce(cm, m, COMM_SUM, &mg, st));
    else mg = m;
  }
  if (mg < n) {
    *in_protocol = false;  // the same decision on every rank
    return fail("m_global=%lld < n=%lld", (long long)mg, (long long)n);
  }

  ObliqueYParams yp{};
  double* nb_dev = w.misc;
  if (oblique) {
    const bool multi = cm != nullptr;
    const int rank = multi ? cm->rank : 0, nranks = multi ? cm->nranks : 1;
    yp.d = bd;
    yp.e = be;
    yp.Y = w.y;
    yp.ldy = L.ldy;
    yp.m = m;
    yp.n = static_cast<int>(n);
    yp.has_prev = rank > 0;
    yp.has_next = rank + 1 < nranks;
    const int64_t hb = B.halo() * n;  // one halo block (halo x n)
    yp.halo_prev = w.halo + 2 * hb;
    yp.halo_next = w.halo + 3 * hb;
    if (B.csr) {
      yp.rp = reinterpret_cast<const long long*>(B.csr->row_ptr);
      yp.ci = B.csr->col_idx;
      yp.cv = B.csr->vals;
      yp.halo = B.csr->halo;
      const bool gh = B.ghosts();
      if (gh) {  // ghost rows (row-major, nghost x n) at the start of the halo region
        yp.ghosts = 1;
        yp.ghost = w.halo;
        yp.halo = B.csr->nghost;
      }
      // argument check on the device: row_ptr monotone from 0, indices inside this rank's rows
      // plus the halo rows that exist (none before rank 0, none after the last rank; the ghost
      // plan: [0, m + nghost)) and the ghost plan's send rows inside [0, m)
      int hbad = 0;
      const int64_t nsend = gh && cm ? B.nsend(cm->nranks) : 0;
      if (m > 0 || nsend > 0) {
        int* bad = reinterpret_cast<int*>(w.misc + 12);
        CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), st));
        if (m > 0) {
          const int blocks = static_cast<int>(std::max<long long>(1, std::min<long long>((m + 255) / 256, 1024)));
          csr_check_kernel<<<blocks, 256, 0, st>>>(yp.rp, yp.ci, m, yp.halo, gh ? 0 : yp.has_prev,
                                                   gh ? 1 : yp.has_next, bad);
          ++g_launches;
          CUDA_TRY(cudaGetLastError());
        }
        if (nsend > 0) {
          const int blocks = static_cast<int>(std::max<long long>(1, std::min<long long>((nsend + 255) / 256, 1024)));
          index_check_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const long long*>(B.csr->send_rows), nsend, 0, m,
                                                     bad);
          ++g_launches;
          CUDA_TRY(cudaGetLastError());
        }
        CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
        long long hnnz = 0;  // row_ptr[m]: picks the Y = BQ kernel (tile kernel up to 12 nonzeros per row)
        if (m > 0) CUDA_TRY(cudaMemcpyAsync(&hnnz, yp.rp + m, sizeof(long long), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        yp.csr_tile = hnnz <= static_cast<long long>(kCsrTileNnzPerRow) * m ? 1 : 0;
        if (hbad) fail("CSR metric: row_ptr not monotone from 0, a column index outside this rank's rows and halo / "
                       "ghosts, or a send row outside [0, m)");
      }
      if (cm && gh && hbad == 0) {
        // rank r's send_counts[p] must equal rank p's recv_counts[r]
        std::vector<int64_t> all(static_cast<size_t>(cm->nranks) * cm->nranks);
        int64_t* dscr = reinterpret_cast<int64_t*>(w.partials);
        TRY(comm_host_allgather(cm, B.csr->send_counts, cm->nranks, all.data(), dscr, st));
        for (int r = 0; r < cm->nranks; ++r)
          if (all[static_cast<size_t>(r) * cm->nranks + cm->rank] != B.csr->recv_counts[r]) {
            hbad = 1;
            fail("CSR ghost plan: rank %d sends %lld rows to rank %d, which expects %lld", r,
                 (long long)all[static_cast<size_t>(r) * cm->nranks + cm->rank], cm->rank,
                 (long long)B.csr->recv_counts[r]);
            break;
          }
      }
      if (cm) {
        const int rc = comm_agree(cm, hbad == 0, st);
        if (rc != SCQR3_OK) *in_protocol = false;  // every rank returns EINVAL together
        TRY(rc);
      } else if (hbad) {
        return SCQR3_EINVAL;
      }
    }
    // e_prev = previous rank's b_off[m_prev - 1]
    double e_prev = 0.0;
    if (multi && B.d) {
      double* ebuf = w.misc + 8;  // [8] send, [9] recv
      TRY(comm_shift_right1(cm, m > 0 ? be + (m - 1) : nullptr, ebuf, ebuf + 1, st));
      CUDA_TRY(cudaMemcpyAsync(&e_prev, ebuf + 1, 8, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      if (rank == 0) e_prev = 0.0;
    }
    yp.e_prev = e_prev;
    if (o->bnorm_bound > 0) {
      CUDA_TRY(cudaMemcpyAsync(nb_dev, &o->bnorm_bound, 8, cudaMemcpyHostToDevice, st));
    } else {
      double* part = w.colsq;
      const int blocks = static_cast<int>(std::max<long long>(1, std::min<long long>((m + 255) / 256, 1024)));
      if (m > 0) {
        if (B.csr) csr_gershgorin_kernel<<<blocks, 256, 0, st>>>(yp.rp, yp.cv, m, part);
        else gershgorin_kernel<<<blocks, 256, 0, st>>>(bd, be, m, yp.has_prev, e_prev, yp.has_next, part);
        ++g_launches;
        CUDA_TRY(cudaGetLastError());
      } else {
        CUDA_TRY(cudaMemsetAsync(part, 0, 8, st));
      }
      max_reduce_kernel<<<1, 32, 0, st>>>(part, m > 0 ? blocks : 1, nb_dev);
      ++g_launches;
      CUDA_TRY(cudaGetLastError());
      if (multi) TRY(comm_allreduce_max1(cm, nb_dev, st));
    }
  }

  CholParams cp{};
  cp.tiles = w.tiles;
  cp.n = static_cast<int>(n);
  cp.NT = L.NT;
  cp.npad = L.npad;
  cp.mode = CHOL_PASS;
  cp.oblique = oblique ? 1 : 0;
  cp.shift_mode = o->shift_mode;
  cp.shift_value = o->shift_value;
  cp.norm_mode = o->norm_mode;
  cp.norm2_bound = o->norm2_bound;
  cp.power_iters = iters;
  cp.m_global = static_cast<double>(mg);
  cp.nb_dev = nb_dev;
  cp.stop_tol = stop_tol;
  cp.W = w.W;
  cp.w_in_smem = w_fits_smem(static_cast<int>(n)) ? 1 : 0;
  cp.Rt = w.Rt;
  // the TRSM operands: written by chol_kernel for n <= 32, else by trsm_prep_kernel (many CTAs;
  // its last CTA runs the D24 guard -- inside the one Cholesky CTA, the guard's once-executed
  // unrolled code cost 31 K cycles at n = 64, mostly cold instruction fetch)
  // (n in (33, 64]: only the fused TRSM + Gram has an inverse-diagonal instance; the others keep
  //  the in-kernel operands, measured 7 us per pass cheaper than the extra launch)
  const bool fuse_tg = g_fuse_tg && !oblique && trsm_fuses_gram(L.NT) && m > 0;
  const bool prep_launch = n > 64 || (n > 32 && fuse_tg && o->trsm_diag != SCQR3_TRSM_DIAG_SUBST);
  cp.bfrag = prep_launch ? nullptr : w.bfrag;
  cp.dblk = prep_launch ? nullptr : w.dblk;
  cp.trsm_diag = o->trsm_diag;
  cp.st_dev = w.st;
  cp.st_host = c->st_host_dev;

  TrsmParams tp{};
  tp.m = m;
  tp.n = static_cast<int>(n);
  tp.bfrag = w.bfrag;
  tp.dblk = w.dblk;
  tp.dinv = w.dblk + dinv_off(L.NT);
  tp.inv_flag = o->trsm_diag == SCQR3_TRSM_DIAG_SUBST ? nullptr : w.dblk + dflag_off(L.NT);  // reading D24
  tp.st = w.st;
  tp.Q = Q;
  tp.ldq = ldq;

  // Device-side pass control: the Cholesky of pass k lowers *last_pass when it stops (or
  // fails), and every kernel of a later pass exits at once (PassGate).  Two drivers use it:
  //  * the CUDA-graph loop (single GPU, no profiling): pass 1, then a conditional WHILE node
  //    whose body is one pass reading its number from a device counter -- no host round trip
  //    between passes;
  //  * the host loop (multi-GPU / profiled calls): the host reads pass k's status (recorded
  //    right after chol_k, while the GPU runs TRSM_k) before enqueueing pass k+1.  (Enqueueing
  //    pass k+1 speculatively first was measured slower: PR1 0.25 -> 0.30 ms.)
  int* last_pass = reinterpret_cast<int*>(w.misc + 14);
  int* pass_dev = reinterpret_cast<int*>(w.misc + 15);
  cp.last_pass = last_pass;
  // n <= 64, standard inner product: TRSM_k also accumulates Gram_{k+1} (fuse_tg
  // above)
  int fused_chunks = 0;
  // k >= 1: pass k with host-known number; k == 0: the generic loop-body pass (number on device)
  auto enqueue = [&](int k) -> int {
    const bool generic = k == 0;
    const double* src = k == 1 ? X : Q;
    const int64_t ldsrc = k == 1 ? ld : ldq;
    const PassGate gate{last_pass, k, generic ? pass_dev : nullptr};
    c->cur_pass = k;
    char nvtx_name[32];
    std::snprintf(nvtx_name, sizeof nvtx_name, generic ? "scqr3 pass (graph body)" : "scqr3 pass %d", k);
    nvtxRangePushA(nvtx_name);
    struct NvtxPop { ~NvtxPop() { nvtxRangePop(); } } nvtx_pop;
    // (the generic body's pass number was advanced by the loop-condition kernel that let it run)
    if (oblique) {
      if (cm) {
        const int ph = prof_begin(c, PK_COMM);
        if (B.ghosts()) {
          const int64_t nsend = B.nsend(cm->nranks);
          TRY(comm_ghosts(cm, src, ldsrc, static_cast<int>(n), B.csr->send_rows, B.csr->send_counts,
                          B.csr->recv_counts, nsend, w.halo + B.csr->nghost * n, w.halo, st));
        } else {
          TRY(comm_halo(cm, src, ldsrc, m, static_cast<int>(n), B.halo(), w.halo, st));
        }
        prof_end(c, ph);
      }
      yp.Q = src;
      yp.ldq = ldsrc;
    }
    if (k == 1 || !fuse_tg) {
      TRY(run_gram(c, L, w, src, ldsrc, m, oblique, &yp, st, gate, oblique));
    } else {
      // this pass's Gram was accumulated by the previous pass's fused TRSM (per-CTA partials)
      TRY(launch_gram_reduce(c, L, w, fused_chunks, false, false, 0, st, gate));
    }
    if (cm) {
      // B-Gram (+ ||Q||_F^2 and the plain Gram for the norm estimate when oblique)
      const size_t cnt = static_cast<size_t>(L.tiles_sym * 64 + (oblique ? 1 + L.tiles_sym * 64 : 0));
      const int pa = prof_begin(c, PK_COMM);
      // (deterministic NCCL mode gathers into the partials area, free once gram_reduce ran)
      TRY(comm_allreduce_sum(cm, w.tiles, cnt, o->deterministic != 0, w.partials,
                             static_cast<size_t>(L.max_chunks) * L.tiles_part * 64, st));
      prof_end(c, pa);
    }
    cp.pass = k;
    cp.pass_dev = generic ? pass_dev : nullptr;
    // previous R~ consumed (a graph segment joins the side stream at its end instead)
    if (k > 1) CUDA_TRY(cudaStreamWaitEvent(st, c->ev_side, 0));
    const int pc = prof_begin(c, PK_CHOL);
    // pass 1's norm estimate for n in (128, 256] (W does not fit one SM's shared memory): the
    // power iteration runs on a cluster of 8 CTAs first (reading D2 / D4)
    const bool pow_needs = k == 1 && n > 128 && n <= 256 && o->norm_mode == SCQR3_NORM_POWER &&
                           (o->shift_mode == SCQR3_SHIFT_SAFE || o->shift_mode == SCQR3_SHIFT_PRACTICAL);
    cp.lmax_dev = nullptr;
    if (pow_needs) {
      PowerParams pp{};
      pp.tiles = oblique ? w.tiles + L.tiles_sym * 64 + 1 : w.tiles;
      pp.n = static_cast<int>(n);
      pp.iters = iters;
      pp.out = w.misc + 24;
      pp.pass = 1;
      pp.last_pass = last_pass;
      const size_t psmem = power_cluster_smem(static_cast<int>(n));
      static thread_local int pow_dev = -1;  // (a cluster kernel: only the shared-memory attribute)
      if (pow_dev != c->device) {
        CUDA_TRY(cudaFuncSetAttribute(power_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(power_cluster_smem(256))));
        pow_dev = c->device;
      }
      power_cluster_kernel<<<8, 256, psmem, st>>>(pp);
      ++g_launches;
      CUDA_TRY(cudaGetLastError());
      cp.lmax_dev = w.misc + 24;
    }
    TRY(launch_chol(cp, st));
    if (prep_launch) {  // R~ (row-major) -> the TRSM's B fragments and scaled diagonal blocks, on many CTAs
      trsm_prep_kernel<<<trsm_prep_blocks(L.NT), 256, 0, st>>>(w.Rt, static_cast<int>(n), L.NT, w.bfrag, w.dblk, 1,
                                                                w.st, gate, o->trsm_diag);
      ++g_launches;
      CUDA_TRY(cudaGetLastError());
    }
    prof_end(c, pc);
    if (!generic) CUDA_TRY(cudaEventRecord(c->ev_pass[k - 1], st));
    TRY(launch_trmul(c, w.Rt, R, w.Rnew, static_cast<int>(n), k == 1, w.st, st, gate));
    tp.X = src;
    tp.ldx = ldsrc;
    tp.gate = gate;
    tp.gram_partials = fuse_tg ? w.partials : nullptr;
    if (m > 0) {
      CUtensorMap mx;
      const bool use_tma = L.NT <= 16 || L.NT >= 24;
      // (NT >= 24: the map of the first 128 columns, for the split TRSM.  A 3-D view with one
      //  32-row box per A = 4 warp slot was measured slower for the unfused n = 64: C5 TRSM 0.423
      //  -> 0.440 ms)
      if (use_tma) TRY(encode_map(c, &mx, src, m, L.NT >= 24 ? 128 : n, ldsrc, trsm_x_box_cols(L.NT)));
      CUtensorMap mq;  // fused TRSM + Gram: bulk stores of Q
      if (fuse_tg) TRY(encode_map(c, &mq, Q, m, n, ldq, L.npad));
      const int pt = prof_begin(c, PK_TRSM);
      CUDA_TRY(launch_trsm(tp, use_tma ? &mx : nullptr, c->num_sms, st, &fused_chunks, fuse_tg ? &mq : nullptr));
      prof_end(c, pt);
      g_launches += trsm_launch_count(tp, use_tma);
    }
    return SCQR3_OK;
  };
  auto init_control = [&]() -> int {
    CUDA_TRY(cudaMemsetAsync(last_pass, 0, sizeof(int), st));
    CUDA_TRY(cudaMemsetAsync(pass_dev, 0, sizeof(int), st));
    CUDA_TRY(cudaMemsetAsync(last_pass, max_passes, 1, st));       // little-endian int = max_passes (<= 16)
    CUDA_TRY(cudaMemsetAsync(pass_dev, 1, 1, st));                  // pass 1 is the unrolled one
    return SCQR3_OK;
  };
  // Read back the per-pass status slots; returns the status, sets *kdone.
  auto collect = [&](int upto, int* kdone) -> int {
    int status = SCQR3_ENOCONV;
    *kdone = 0;
    for (int k = 1; k <= upto; ++k) {
      const volatile DevStatus* h = c->st_host + (k - 1);
      if (h->code < 0) break;
      *kdone = k;
      if (o->trace && k - 1 < o->trace_cap) {
        scqr3_pass_trace& t = o->trace[k - 1];
        t.shift = h->shift;
        t.shifted = h->shifted;
        t.breakdown_pivot = h->breakdown_pivot;
        t.pivot_value = h->pivot_value;
        t.norm2_est = h->norm2_est;
        t.dev_F = h->dev_F;
      }
      if (h->code == SCQR3_EINVAL) return fail("non-finite entries in X (the trace of the pass-1 Gram is not finite)");
      if (h->code != SCQR3_OK) return h->code;
      if (h->stop) return SCQR3_OK;
    }
    if (*kdone == 0) return fail("status block not written by the Cholesky kernel");
    return status;
  };
  for (int k = 0; k < max_passes; ++k) c->st_host[k].code = -1;

  int status = SCQR3_ENOCONV, k = 0;
  const bool use_graph = g_use_graph && !cm && !o->prof && m > 0 && !c->plan_failed;
  bool done = false;
  if (use_graph) {
    // ---- CUDA-graph pass loop, captured once per argument set and replayed
    GraphKey key{};
    key.X = X; key.Q = Q; key.R = R; key.ld = ld; key.ldq = ldq; key.m = m; key.n = n;
    key.ws = o->workspace; key.st = st; key.max_passes = max_passes; key.cp = cp; key.tp = tp; key.yp = yp;
    static_assert(sizeof(GraphKey) <= sizeof(GraphPlan::key), "graph key buffer too small");
    GraphPlan* hit = nullptr;
    for (GraphPlan& p : c->plans)
      if (p.exec && std::memcmp(p.key, &key, sizeof key) == 0) hit = &p;
    GraphPlan& gpn = hit ? *hit : c->plans[c->plan_next++ % Ctx::kPlans];
    if (!hit) {
      gpn.reset();
      const cudaStream_t user_st = st;
      st = c->cap;  // the enqueue lambdas capture on the internal stream
      const int rc = capture_pass_loop(c, st, max_passes, last_pass, pass_dev, init_control, enqueue, &gpn);
      st = user_st;
      if (rc == SCQR3_OK) {
        std::memcpy(gpn.key, &key, sizeof key);
      } else {
        gpn.reset();  // fall through to the host loop (same kernels), and stop trying
        c->plan_failed = true;
      }
    }
    if (gpn.exec) {
      CUDA_TRY(cudaGraphLaunch(gpn.exec, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      status = collect(max_passes, &k);
      g_launches += gpn.launches_first + gpn.launches_body * std::max(0, k - 1);
      done = true;
    }
  }
  if (!done) {
    TRY(init_control());
    TRY(enqueue(1));
    for (k = 1;; ++k) {
      CUDA_TRY(cudaEventSynchronize(c->ev_pass[k - 1]));
      const volatile DevStatus* h = c->st_host + (k - 1);
      if (h->code < 0) return fail("status block not written by the Cholesky kernel");
      if (h->code != SCQR3_OK || h->stop || k == max_passes) break;
      TRY(enqueue(k + 1));
    }
    int kd = 0;
    status = collect(k, &kd);
    k = kd;
  }
  if (o->passes_out) *o->passes_out = k;
  if (!done) CUDA_TRY(cudaStreamWaitEvent(st, c->ev_side, 0));  // R complete (the graph joins itself)
  CUDA_TRY(cudaStreamSynchronize(st));
  prof_flush(c, k);
  c->prof = nullptr;
  return status;
}

int factor_impl(int64_t m, int64_t n, const double* X, int64_t ld, const Metric& B, double* Q, int64_t ldq,
                double* R, const scqr3_opts* o) {
  bool in_protocol = false;
  nvtxRangePushA(B.csr ? "scqr3_factor_oblique_csr" : B.d ? "scqr3_factor_oblique" : "scqr3_factor");
  const int rc = factor_body(m, n, X, ld, B, Q, ldq, R, o, &in_protocol);
  nvtxRangePop();
  // an error after the ranks started exchanging (CUDA / NCCL failure on this rank): a loopback
  // group is marked failed so that the peers return instead of waiting at the next exchange
  if (rc == SCQR3_EINVAL && in_protocol) comm_abort(static_cast<Comm*>(o->comm), g_err.c_str());
  return rc;
}

// ---- complex X (reading D23): real kernels on the m x 2n split matrix, complex
// n x n step (zchol.cu).  Host-driven pass loop (as the multi-GPU path).
struct ZLayout {
  Layout L;        // real layout for the 2n-column split matrix (wide: its first kMaxN columns)
  Layout L2;       // wide (2n > kMaxN, zwide.cu): the last q = 2n - kMaxN columns
  bool wide;
  int64_t lds;     // split matrix leading dimension (even, >= m)
  size_t S, A, Rtz, end;
  // wide only: G = [S1^T S1 tiles | S2^T S2 tiles | C12 = S1^T S2], complex scratch W, the
  // 2n x 2n M, its diagonal blocks M11, M22, complex R scratch, and one partials / gather buffer
  size_t G, Wz, M, M11, M22, Rnz, P;
  long long g_off2, g_offc, g_count, p_cap;
  int q, xchunks_max;
};

constexpr int kXChunksMax = 32;  // row chunks of the wide cross Gram (partials: chunks x 512 x q)

ZLayout make_zlayout(int64_t m, int64_t n) {
  ZLayout Z{};
  Z.wide = 2 * n > kMaxN;
  Z.L = make_layout(m, Z.wide ? kMaxN : 2 * n, 0);
  Z.lds = std::max<int64_t>(2, (m + 1) & ~1LL);
  size_t off = Z.L.end;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return o;
  };
  Z.S = take(static_cast<size_t>(Z.lds) * 2 * n * 8);
  Z.A = take(static_cast<size_t>(n) * n * 16);
  Z.Rtz = take(static_cast<size_t>(n) * n * 16);
  if (Z.wide) {
    Z.q = static_cast<int>(2 * n - kMaxN);
    Z.L2 = make_layout(m, Z.q, 0);
    Z.g_off2 = Z.L.tiles_sym * 64 + 64;
    Z.g_offc = Z.g_off2 + Z.L2.tiles_sym * 64 + 64;
    Z.g_count = Z.g_offc + static_cast<long long>(kMaxN) * Z.q;
    Z.xchunks_max = kXChunksMax;
    Z.p_cap = std::max({Z.L.max_chunks * Z.L.tiles_part * 64, Z.L2.max_chunks * Z.L2.tiles_part * 64,
                        static_cast<long long>(kXChunksMax) * kMaxN * Z.q, 8 * Z.g_count});
    Z.G = take(static_cast<size_t>(Z.g_count) * 8);
    Z.Wz = take(static_cast<size_t>(n) * n * 16);
    Z.M = take(static_cast<size_t>(4 * n) * n * 8);
    Z.M11 = take(static_cast<size_t>(kMaxN) * kMaxN * 8);
    Z.M22 = take(static_cast<size_t>(Z.q) * Z.q * 8);
    Z.Rnz = take(static_cast<size_t>(n) * n * 16);
    Z.P = take(static_cast<size_t>(Z.p_cap) * 8);
  }
  Z.end = off;
  return Z;
}

int zfactor_checks(int64_t m, int64_t n, const double* X, int64_t ld, const double* Q, int64_t ldq, const double* R,
                   const scqr3_opts* o, Ctx** c, ZLayout* Z, WS* w) {
  TRY(check_opts(o));
  if (n < 1 || n > kMaxN) return fail("complex n=%lld outside [1, %d]", (long long)n, kMaxN);
  if (m < 0) return fail("m < 0");
  if (m > 0 && (!X || !Q)) return fail("X or Q is NULL");
  if (ld < std::max<int64_t>(m, 1) || ldq < std::max<int64_t>(m, 1)) return fail("leading dimension < m");
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Q)) % 16) return fail("X, Q must be 16-byte aligned");
  if (!R) return fail("R is NULL");
  const int max_passes = o->max_passes > 0 ? o->max_passes : 8;
  if (max_passes > Ctx::kSlots) return fail("max_passes %d > %d", max_passes, Ctx::kSlots);
  TRY(get_ctx(c));
  *Z = make_zlayout(m, n);
  if (!o->workspace || o->workspace_bytes < Z->end) return fail("workspace too small: %zu < %zu bytes", o->workspace_bytes, Z->end);
  if (reinterpret_cast<uintptr_t>(o->workspace) % 256) return fail("workspace must be 256-byte aligned");
  TRY(carve(Z->L, o, w));
  return SCQR3_OK;
}

// Wide complex Gram (n > 256, zwide.cu): S1^T S1 and S2^T S2 by the real Gram kernel, the cross
// block C12 = S1^T S2 by xgram_kernel + xreduce_kernel, one allreduce of all three across ranks,
// then A = X^H X.
int zwide_gram(Ctx* c, const ZLayout& Z, const WS& w1, const WS& w2, const double* S, int64_t m, Comm* cm, bool det,
               int n, double* Az, const int* last_pass, int k, cudaStream_t st, PassGate gate) {
  TRY(run_gram(c, Z.L, w1, S, Z.lds, m, false, nullptr, st, gate));
  TRY(run_gram(c, Z.L2, w2, S + kMaxN * Z.lds, Z.lds, m, false, nullptr, st, gate));
  double* G = w1.tiles;
  double* C12 = G + Z.g_offc;
  const long long cnt = static_cast<long long>(kMaxN) * Z.q;
  if (m == 0) {
    CUDA_TRY(cudaMemsetAsync(C12, 0, static_cast<size_t>(cnt) * 8, st));
  } else {
    const int nbp = kMaxN / 64, nbq = (Z.q + 63) / 64;
    long long chunks = (4LL * c->num_sms + nbp * nbq - 1) / (nbp * nbq);
    chunks = std::max<long long>(1, std::min<long long>({chunks, Z.xchunks_max, (m + 31) / 32}));
    const long long rpc = ((m + chunks - 1) / chunks + 31) / 32 * 32;
    chunks = (m + rpc - 1) / rpc;
    const int pg = prof_begin(c, PK_GRAM);
    xgram_kernel<<<static_cast<unsigned>(chunks * nbp * nbq), 256, 0, st>>>(S, Z.lds, S + kMaxN * Z.lds, Z.lds, m, kMaxN,
                                                                            Z.q, rpc, w1.partials, gate);
    xreduce_kernel<<<static_cast<unsigned>(std::min<long long>(1024, (cnt + 255) / 256)), 256, 0, st>>>(
        w1.partials, static_cast<int>(chunks), cnt, C12, gate);
    prof_end(c, pg);
    g_launches += 2;
    CUDA_TRY(cudaGetLastError());
  }
  if (cm) {
    const int pa = prof_begin(c, PK_COMM);
    TRY(comm_allreduce_sum(cm, G, static_cast<size_t>(Z.g_count), det, w1.partials, static_cast<size_t>(Z.p_cap), st));
    prof_end(c, pa);
  }
  const long long nn = static_cast<long long>(n) * n;
  zcombine_wide_kernel<<<static_cast<unsigned>((nn + 255) / 256), 256, 0, st>>>(G, G + Z.g_off2, C12, n, kMaxN, Az,
                                                                                  last_pass, k);
  ++g_launches;
  CUDA_TRY(cudaGetLastError());
  return SCQR3_OK;
}

// Wide complex TRSM (n > 256, zwide.cu): Q1 = S1 M11^-1, S2 -= Q1 M12, Q2 = S2 M22^-1, in place.
int zwide_trsm(Ctx* c, const ZLayout& Z, const WS& w, double* S, const double* M11, const double* M22,
               const double* Mz, int64_t m, int trsm_diag, cudaStream_t st, PassGate gate) {
  const int n2 = kMaxN + Z.q;
  for (int h = 0; h < 2; ++h) {
    const int nh = h ? Z.q : kMaxN;
    const Layout& Lh = h ? Z.L2 : Z.L;
    double* Sh = S + (h ? kMaxN * Z.lds : 0);
    const int pt = prof_begin(c, PK_TRSM);
    if (h == 1) {
      const int nbq = (Z.q + 63) / 64;
      xupdate_kernel<<<static_cast<unsigned>((m + 63) / 64 * nbq), 256, 0, st>>>(
          S, Z.lds, Mz + static_cast<size_t>(kMaxN) * n2, n2, Sh, Z.lds, m, kMaxN, Z.q, gate);
      ++g_launches;
      CUDA_TRY(cudaGetLastError());
    }
    trsm_prep_kernel<<<trsm_prep_blocks(Lh.NT), 256, 0, st>>>(h ? M22 : M11, nh, Lh.NT, w.bfrag, w.dblk, 0, nullptr,
                                                               gate, trsm_diag);
    ++g_launches;
    CUDA_TRY(cudaGetLastError());
    TrsmParams tp{};
    tp.m = m;
    tp.n = nh;
    tp.bfrag = w.bfrag;
    tp.dblk = w.dblk;
    tp.dinv = w.dblk + dinv_off(Lh.NT);
    tp.inv_flag = trsm_diag == SCQR3_TRSM_DIAG_SUBST ? nullptr : w.dblk + dflag_off(Lh.NT);
    tp.st = w.st;
    tp.X = Sh;
    tp.ldx = Z.lds;
    tp.Q = Sh;
    tp.ldq = Z.lds;
    tp.gate = gate;
    CUtensorMap mx;
    const bool use_tma = Lh.NT <= 16 || Lh.NT >= 24;
    if (use_tma) TRY(encode_map(c, &mx, Sh, m, Lh.NT >= 24 ? 128 : nh, Z.lds, trsm_x_box_cols(Lh.NT)));
    int grid = 0;
    CUDA_TRY(launch_trsm(tp, use_tma ? &mx : nullptr, c->num_sms, st, &grid, nullptr));
    prof_end(c, pt);
    g_launches += trsm_launch_count(tp, use_tma);
  }
  return SCQR3_OK;
}

int zfactor_impl(int64_t m, int64_t n, const double* X, int64_t ld, double* Q, int64_t ldq, double* R,
                 const scqr3_opts* o) {
  if (!o) return fail("opts is NULL");
  cudaStream_t st = static_cast<cudaStream_t>(o->stream);
  Comm* cm = static_cast<Comm*>(o->comm);
  Ctx* c = nullptr;
  ZLayout Z{};
  WS w{};
  const int rc_local = zfactor_checks(m, n, X, ld, Q, ldq, R, o, &c, &Z, &w);
  if (cm) TRY(comm_agree(cm, rc_local == SCQR3_OK, st));
  else TRY(rc_local);
  const Layout& L = Z.L;
  char* wb = static_cast<char*>(o->workspace);
  double* S = reinterpret_cast<double*>(wb + Z.S);
  double* Az = reinterpret_cast<double*>(wb + Z.A);
  double* Rtz = reinterpret_cast<double*>(wb + Z.Rtz);
  c->prof = o->prof;
  c->prof_stream = st;
  c->ev_used = 0;
  const int max_passes = o->max_passes > 0 ? o->max_passes : 8;
  int64_t mg = o->m_global;
  if (mg <= 0) {
    if (cm) TRY(comm_host_allreduce(cm, m, COMM_SUM, &mg, st));
    else mg = m;
  }
  if (mg < n) return fail("m_global=%lld < n=%lld", (long long)mg, (long long)n);
  const int n2 = static_cast<int>(2 * n);
  if (m > 0) {
    const long long blocks = std::max<long long>(1, std::min<long long>((m * n + 255) / 256, 8192));
    z2split_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(X, ld, m, static_cast<int>(n), S, Z.lds);
    ++g_launches;
    CUDA_TRY(cudaGetLastError());
  }
  int* last_pass = reinterpret_cast<int*>(w.misc + 14);
  CUDA_TRY(cudaMemsetAsync(last_pass, 0, sizeof(int), st));
  CUDA_TRY(cudaMemsetAsync(last_pass, max_passes, 1, st));
  ZCholParams zp{};
  zp.A = Az;
  zp.W = w.W;  // the real layout's 2n(2n+1) doubles hold the n x n complex scratch
  zp.n = static_cast<int>(n);
  zp.last_pass = last_pass;
  zp.shift_mode = o->shift_mode;
  zp.shift_value = o->shift_value;
  zp.norm_mode = o->norm_mode;
  zp.norm2_bound = o->norm2_bound;
  zp.power_iters = o->power_iters > 0 ? o->power_iters : 32;
  zp.m_global = static_cast<double>(mg);
  zp.stop_tol = o->stop_tol > 0 ? o->stop_tol : 0.5;
  zp.Rt = Rtz;
  zp.M = w.Rt;  // real 2n x 2n
  zp.st_dev = w.st;
  zp.st_host = c->st_host_dev;
  zp.w_in_smem = n <= 128 ? 1 : 0;
  // wide (n > 256): the split matrix as [S1 S2] (zwide.cu); their own scratch past the real layout
  double* G = nullptr;
  double* Mz = nullptr;
  double* M11 = nullptr;
  double* M22 = nullptr;
  double* Rnew = w.Rnew;
  WS w1 = w, w2 = w;
  if (Z.wide) {
    G = reinterpret_cast<double*>(wb + Z.G);
    Mz = reinterpret_cast<double*>(wb + Z.M);
    M11 = reinterpret_cast<double*>(wb + Z.M11);
    M22 = reinterpret_cast<double*>(wb + Z.M22);
    Rnew = reinterpret_cast<double*>(wb + Z.Rnz);
    zp.W = reinterpret_cast<double*>(wb + Z.Wz);
    zp.M = Mz;
    w1.partials = w2.partials = reinterpret_cast<double*>(wb + Z.P);
    w1.tiles = G;
    w2.tiles = G + Z.g_off2;
  }
  TrsmParams tp{};
  tp.m = m;
  tp.n = n2;
  tp.bfrag = w.bfrag;
  tp.dblk = w.dblk;
  tp.dinv = w.dblk + dinv_off(L.NT);
  tp.inv_flag = o->trsm_diag == SCQR3_TRSM_DIAG_SUBST ? nullptr : w.dblk + dflag_off(L.NT);  // guard on M (D24)
  tp.st = w.st;
  tp.X = S;
  tp.ldx = Z.lds;
  tp.Q = S;  // in place on the split matrix
  tp.ldq = Z.lds;
  const bool fuse_tg = g_fuse_tg && trsm_fuses_gram(L.NT) && m > 0 && !Z.wide;
  int fused_chunks = 0;
  for (int k = 0; k < max_passes; ++k) c->st_host[k].code = -1;
  int status = SCQR3_ENOCONV, k;
  for (k = 1; k <= max_passes; ++k) {
    const PassGate gate{last_pass, k, nullptr};
    c->cur_pass = k;
    const long long nn = n * n;
    if (Z.wide) {
      TRY(zwide_gram(c, Z, w1, w2, S, m, cm, o->deterministic != 0, static_cast<int>(n), Az, last_pass, k, st, gate));
    } else {
    if (k == 1 || !fuse_tg) TRY(run_gram(c, L, w, S, Z.lds, m, false, nullptr, st, gate));
    else TRY(launch_gram_reduce(c, L, w, fused_chunks, false, false, 0, st, gate));
    if (cm) {
      const int pa = prof_begin(c, PK_COMM);
      TRY(comm_allreduce_sum(cm, w.tiles, static_cast<size_t>(L.tiles_sym * 64), o->deterministic != 0, w.partials,
                             static_cast<size_t>(L.max_chunks) * L.tiles_part * 64, st));
      prof_end(c, pa);
    }
    zcombine_kernel<<<static_cast<unsigned>((nn + 255) / 256), 256, 0, st>>>(w.tiles, static_cast<int>(n), Az,
                                                                              last_pass, k);
    ++g_launches;
    CUDA_TRY(cudaGetLastError());
    }
    zp.pass = k;
    if (k > 1) CUDA_TRY(cudaStreamWaitEvent(st, c->ev_side, 0));
    const int pc = prof_begin(c, PK_CHOL);
    {
      // packed upper W in shared memory (n <= 128), else the panel of the blocked factorisation
      // (zchol.cu: 16 rows of R~ x n complex)
      const size_t zsmem = zp.w_in_smem ? static_cast<size_t>(n) * (n + 1) / 2 * 16 : static_cast<size_t>(16) * n * 16;
      static thread_local LaunchCfgCache zcfg;
      CUDA_TRY(cached_launch_cfg(zcfg, zchol_kernel, zsmem, 256, nullptr));
      zchol_kernel<<<1, 256, zsmem, st>>>(zp);
    }
    ++g_launches;
    CUDA_TRY(cudaGetLastError());
    if (Z.wide) {  // the diagonal blocks of M as contiguous operands for trsm_prep_kernel (zwide_trsm)
      zsub_kernel<<<256, 256, 0, st>>>(Mz, n2, 0, 0, kMaxN, kMaxN, M11, gate);
      zsub_kernel<<<256, 256, 0, st>>>(Mz, n2, kMaxN, kMaxN, Z.q, Z.q, M22, gate);
      g_launches += 2;
    } else {
      trsm_prep_kernel<<<trsm_prep_blocks(L.NT), 256, 0, st>>>(w.Rt, n2, L.NT, w.bfrag, w.dblk, 0, nullptr, gate,
                                                                o->trsm_diag);  // M -> TRSM operands
      ++g_launches;
    }
    CUDA_TRY(cudaGetLastError());
    prof_end(c, pc);
    CUDA_TRY(cudaEventRecord(c->ev_pass[k - 1], st));
    // R := R~ R on the side stream
    CUDA_TRY(cudaEventRecord(c->ev_chol, st));
    CUDA_TRY(cudaStreamWaitEvent(c->side, c->ev_chol, 0));
    ztrmul_kernel<<<static_cast<unsigned>((nn + 127) / 128), 128, 0, c->side>>>(Rtz, R, Rnew, static_cast<int>(n),
                                                                                 k == 1, w.st, gate);
    copy_kernel<<<static_cast<unsigned>((2 * nn + 127) / 128), 128, 0, c->side>>>(Rnew, R, 2 * nn, w.st, gate);
    g_launches += 2;
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(c->ev_side, c->side));
    tp.gate = gate;
    tp.gram_partials = fuse_tg ? w.partials : nullptr;
    if (Z.wide) {
      if (m > 0) TRY(zwide_trsm(c, Z, w, S, M11, M22, Mz, m, o->trsm_diag, st, gate));
    } else if (m > 0) {
      CUtensorMap mx;
      const bool use_tma = L.NT <= 16 || L.NT >= 24;
      if (use_tma) TRY(encode_map(c, &mx, S, m, L.NT >= 24 ? 128 : n2, Z.lds, trsm_x_box_cols(L.NT)));
      const int pt = prof_begin(c, PK_TRSM);
      // (in place on the split matrix: the bulk stores of Q use the same descriptor)
      CUDA_TRY(launch_trsm(tp, use_tma ? &mx : nullptr, c->num_sms, st, &fused_chunks,
                           fuse_tg && use_tma ? &mx : nullptr));
      prof_end(c, pt);
      g_launches += trsm_launch_count(tp, use_tma);
    }
    CUDA_TRY(cudaEventSynchronize(c->ev_pass[k - 1]));
    const volatile DevStatus* h = c->st_host + (k - 1);
    if (h->code < 0) return fail("status block not written by the complex Cholesky kernel");
    if (o->trace && k - 1 < o->trace_cap) {
      scqr3_pass_trace& t = o->trace[k - 1];
      t.shift = h->shift;
      t.shifted = h->shifted;
      t.breakdown_pivot = h->breakdown_pivot;
      t.pivot_value = h->pivot_value;
      t.norm2_est = h->norm2_est;
      t.dev_F = h->dev_F;
    }
    if (h->code == SCQR3_EINVAL) {
      status = fail("non-finite entries in X (the trace of the pass-1 Gram is not finite)");
      break;
    }
    if (h->code != SCQR3_OK) {
      status = h->code;
      break;
    }
    if (h->stop) {
      status = SCQR3_OK;
      break;
    }
  }
  if (k > max_passes) k = max_passes;
  if (o->passes_out) *o->passes_out = k;
  CUDA_TRY(cudaStreamWaitEvent(st, c->ev_side, 0));
  if (status == SCQR3_OK && m > 0) {
    const long long blocks = std::max<long long>(1, std::min<long long>((m * n + 255) / 256, 8192));
    split2z_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(S, Z.lds, m, static_cast<int>(n), Q, ldq);
    ++g_launches;
    CUDA_TRY(cudaGetLastError());
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  prof_flush(c, k);
  c->prof = nullptr;
  return status;
}

}  // namespace

extern "C" {

void scqr3_default_opts(scqr3_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->abi_version = SCQR3_ABI_VERSION;
  o->shift_mode = SCQR3_SHIFT_SAFE;
  o->norm_mode = SCQR3_NORM_POWER;
  o->power_iters = 32;
  o->max_passes = 8;
  o->stop_tol = 0.5;
}

size_t scqr3_workspace_size(int64_t m, int64_t n, int32_t oblique) {
  if (n < 1 || n > kMaxN || m < 0) return 0;
  return make_layout(m, n, oblique).end;
}

int scqr3_factor(int64_t m, int64_t n, const double* X, int64_t ld, double* Q, int64_t ldq, double* R,
                 const scqr3_opts* opts) {
  return factor_impl(m, n, X, ld, Metric{}, Q, ldq, R, opts);
}

int scqr3_factor_oblique(int64_t m, int64_t n, const double* X, int64_t ld, const double* b_diag,
                         const double* b_off, double* Q, int64_t ldq, double* R, const scqr3_opts* opts) {
  if (!b_diag && m > 0) return fail("b_diag is NULL");
  static const double dummy = 0.0;
  Metric B;
  B.d = b_diag ? b_diag : &dummy;
  B.e = b_off;
  return factor_impl(m, n, X, ld, B, Q, ldq, R, opts);
}

size_t scqr3_workspace_size_csr(int64_t m, int64_t n, int64_t halo) {
  if (n < 1 || n > kMaxN || m < 0 || halo < 0) return 0;
  return make_layout(m, n, 1, halo).end;
}

size_t scqr3_workspace_size_csr_ghosts(int64_t m, int64_t n, int64_t nghost, int64_t nsend) {
  if (n < 1 || n > kMaxN || m < 0 || nghost < 0 || nsend < 0) return 0;
  return make_layout(m, n, 1, std::max<int64_t>(1, (nghost + nsend + 3) / 4)).end;  // (Metric::halo)
}

int scqr3_factor_oblique_csr(int64_t m, int64_t n, const double* X, int64_t ld, const scqr3_csr* B_csr, double* Q,
                             int64_t ldq, double* R, const scqr3_opts* opts) {
  if (!B_csr) return fail("CSR metric is NULL");
  Metric B;
  B.csr = B_csr;
  return factor_impl(m, n, X, ld, B, Q, ldq, R, opts);
}

size_t scqr3_host_workspace_size(int64_t m, int64_t n) {
  if (n < 1 || n > kMaxN || m < 0) return 0;
  const int64_t ldd = std::max<int64_t>(2, (m + 1) & ~1LL);
  return align256(static_cast<size_t>(ldd) * n * 8) + align256(static_cast<size_t>(n) * n * 8) +
         make_layout(m, n, 0).end;
}

int scqr3_factor_host(int64_t m, int64_t n, const double* X_host, int64_t ld, double* Q_host, int64_t ldq,
                      double* R_host, const scqr3_opts* opts) {
  TRY(check_opts(opts));
  if (n < 1 || n > kMaxN || m < 0) return fail("bad sizes m=%lld n=%lld", (long long)m, (long long)n);
  if (!X_host || !Q_host || !R_host) return fail("host pointer is NULL");
  if (ld < m || ldq < m) return fail("leading dimension < m");
  if (!opts->workspace || opts->workspace_bytes < scqr3_host_workspace_size(m, n))
    return fail("workspace too small for scqr3_factor_host");
  const int64_t ldd = std::max<int64_t>(2, (m + 1) & ~1LL);
  char* b = static_cast<char*>(opts->workspace);
  double* D = reinterpret_cast<double*>(b);
  double* Rd = reinterpret_cast<double*>(b + align256(static_cast<size_t>(ldd) * n * 8));
  scqr3_opts o2 = *opts;
  o2.workspace = b + align256(static_cast<size_t>(ldd) * n * 8) + align256(static_cast<size_t>(n) * n * 8);
  o2.workspace_bytes = opts->workspace_bytes - (static_cast<char*>(o2.workspace) - b);
  cudaStream_t st = static_cast<cudaStream_t>(opts->stream);
  if (m > 0)
    CUDA_TRY(cudaMemcpy2DAsync(D, ldd * 8, X_host, ld * 8, m * 8, n, cudaMemcpyHostToDevice, st));
  int rc = factor_impl(m, n, D, ldd, Metric{}, D, ldd, Rd, &o2);
  if (rc != SCQR3_OK) return rc;
  if (m > 0)
    CUDA_TRY(cudaMemcpy2DAsync(Q_host, ldq * 8, D, ldd * 8, m * 8, n, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(R_host, Rd, static_cast<size_t>(n) * n * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return SCQR3_OK;
}

size_t scqr3_host_batch_workspace_size(int64_t m, int64_t n) {
  if (n < 1 || n > kMaxN || m < 0) return 0;
  const int64_t ldd = std::max<int64_t>(2, (m + 1) & ~1LL);
  return 3 * (align256(static_cast<size_t>(ldd) * n * 8) + align256(static_cast<size_t>(n) * n * 8)) +
         make_layout(m, n, 0).end;
}

// Streaming end-to-end factorisation of independent host matrices: three device staging buffers
// rotate; matrix i+1 uploads (stream `up`) and matrix i-1 downloads (stream `down`) on the two
// PCIe directions while matrix i is factored on opts->stream (factor_impl, synchronous).
int scqr3_factor_host_batch(int64_t count, int64_t m, int64_t n, const double* const* X_hosts, int64_t ld,
                            double* const* Q_hosts, int64_t ldq, double* const* R_hosts, int32_t* statuses,
                            const scqr3_opts* opts) {
  TRY(check_opts(opts));
  if (count < 0) return fail("count < 0");
  if (n < 1 || n > kMaxN || m < 0) return fail("bad sizes m=%lld n=%lld", (long long)m, (long long)n);
  if (count > 0 && (!X_hosts || !Q_hosts || !R_hosts || !statuses)) return fail("NULL pointer array");
  for (int64_t i = 0; i < count; ++i)
    if ((m > 0 && (!X_hosts[i] || !Q_hosts[i])) || !R_hosts[i]) return fail("host pointer %lld is NULL", (long long)i);
  if (ld < m || ldq < m) return fail("leading dimension < m");
  if (!opts->workspace || opts->workspace_bytes < scqr3_host_batch_workspace_size(m, n))
    return fail("workspace too small for scqr3_factor_host_batch");
  Ctx* c;
  TRY(get_ctx(&c));
  if (!c->up) {
    CUDA_TRY(cudaStreamCreateWithFlags(&c->up, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->down, cudaStreamNonBlocking));
    for (int b = 0; b < 3; ++b) {
      CUDA_TRY(cudaEventCreateWithFlags(&c->ev_up[b], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&c->ev_fact[b], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&c->ev_down[b], cudaEventDisableTiming));
    }
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
  }
  const int64_t ldd = std::max<int64_t>(2, (m + 1) & ~1LL);
  const size_t dbytes = align256(static_cast<size_t>(ldd) * n * 8), rbytes = align256(static_cast<size_t>(n) * n * 8);
  char* b0 = static_cast<char*>(opts->workspace);
  double* D[3];
  double* Rd[3];
  for (int b = 0; b < 3; ++b) {
    D[b] = reinterpret_cast<double*>(b0 + b * (dbytes + rbytes));
    Rd[b] = reinterpret_cast<double*>(b0 + b * (dbytes + rbytes) + dbytes);
  }
  scqr3_opts o2 = *opts;
  o2.workspace = b0 + 3 * (dbytes + rbytes);
  o2.workspace_bytes = opts->workspace_bytes - 3 * (dbytes + rbytes);
  cudaStream_t st = static_cast<cudaStream_t>(opts->stream);
  // the copies follow the work already on opts->stream (and its timing events)
  CUDA_TRY(cudaEventRecord(c->ev_start, st));
  CUDA_TRY(cudaStreamWaitEvent(c->up, c->ev_start, 0));
  CUDA_TRY(cudaStreamWaitEvent(c->down, c->ev_start, 0));
  bool used[3] = {false, false, false};
  auto upload = [&](int64_t i) -> int {
    const int b = static_cast<int>(i % 3);
    if (used[b]) CUDA_TRY(cudaStreamWaitEvent(c->up, c->ev_down[b], 0));  // its previous matrix is down
    used[b] = true;
    if (m > 0)
      CUDA_TRY(cudaMemcpy2DAsync(D[b], ldd * 8, X_hosts[i], ld * 8, m * 8, n, cudaMemcpyHostToDevice, c->up));
    CUDA_TRY(cudaEventRecord(c->ev_up[b], c->up));
    return SCQR3_OK;
  };
  if (count > 0) TRY(upload(0));
  if (count > 1) TRY(upload(1));
  for (int64_t i = 0; i < count; ++i) {
    const int b = static_cast<int>(i % 3);
    CUDA_TRY(cudaStreamWaitEvent(st, c->ev_up[b], 0));
    const int rc = factor_impl(m, n, D[b], ldd, Metric{}, D[b], ldd, Rd[b], &o2);
    if (rc == SCQR3_EINVAL) {
      cudaStreamSynchronize(c->up);
      cudaStreamSynchronize(c->down);
      return rc;
    }
    statuses[i] = rc;
    CUDA_TRY(cudaEventRecord(c->ev_fact[b], st));
    CUDA_TRY(cudaStreamWaitEvent(c->down, c->ev_fact[b], 0));
    if (rc == SCQR3_OK) {  // (Q and R are written only on success, as scqr3_factor's)
      if (m > 0)
        CUDA_TRY(cudaMemcpy2DAsync(Q_hosts[i], ldq * 8, D[b], ldd * 8, m * 8, n, cudaMemcpyDeviceToHost, c->down));
      CUDA_TRY(cudaMemcpyAsync(R_hosts[i], Rd[b], static_cast<size_t>(n) * n * 8, cudaMemcpyDeviceToHost, c->down));
    }
    CUDA_TRY(cudaEventRecord(c->ev_down[b], c->down));
    if (i + 2 < count) TRY(upload(i + 2));
  }
  // opts->stream continues after the last download (timing events recorded on it see all copies)
  CUDA_TRY(cudaEventRecord(c->ev_start, c->down));
  CUDA_TRY(cudaStreamWaitEvent(st, c->ev_start, 0));
  CUDA_TRY(cudaStreamSynchronize(c->down));
  CUDA_TRY(cudaStreamSynchronize(st));
  return SCQR3_OK;
}

int scqr3_gram(int64_t m, int64_t n, const double* X, int64_t ld, double* A, const scqr3_opts* opts) {
  TRY(check_opts(opts));
  if (n < 1 || n > kMaxN || m < 0) return fail("bad sizes");
  TRY(check_matrix("X", X, m, ld));
  Ctx* c;
  TRY(get_ctx(&c));
  const Layout L = make_layout(m, n, 0);
  WS w;
  TRY(carve(L, opts, &w));
  cudaStream_t st = static_cast<cudaStream_t>(opts->stream);
  TRY(run_gram(c, L, w, X, ld, m, false, nullptr, st));
  Comm* cm = static_cast<Comm*>(opts->comm);
  if (cm)
    TRY(comm_allreduce_sum(cm, w.tiles, static_cast<size_t>(L.tiles_sym * 64), opts->deterministic != 0, w.partials,
                           static_cast<size_t>(L.max_chunks) * L.tiles_part * 64, st));
  const long long nn = n * n;
  tiles_to_full_kernel<<<static_cast<unsigned>((nn + 255) / 256), 256, 0, st>>>(w.tiles, static_cast<int>(n), A);
  ++g_launches;
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));
  return SCQR3_OK;
}

int scqr3_gram_oblique(int64_t m, int64_t n, const double* X, int64_t ld, const double* b_diag, const double* b_off,
                       double* A, double* colsq, const scqr3_opts* opts) {
  TRY(check_opts(opts));
  if (n < 1 || n > kMaxN || m < 1) return fail("bad sizes");
  TRY(check_matrix("X", X, m, ld));
  Ctx* c;
  TRY(get_ctx(&c));
  const Layout L = make_layout(m, n, 1);
  WS w;
  TRY(carve(L, opts, &w));
  cudaStream_t st = static_cast<cudaStream_t>(opts->stream);
  ObliqueYParams yp{};
  yp.Q = X;
  yp.ldq = ld;
  yp.d = b_diag;
  yp.e = b_off;
  yp.Y = w.y;
  yp.ldy = L.ldy;
  yp.m = m;
  yp.n = static_cast<int>(n);
  TRY(run_gram(c, L, w, X, ld, m, true, &yp, st));
  const long long nn = n * n;
  tiles_to_full_kernel<<<static_cast<unsigned>((nn + 255) / 256), 256, 0, st>>>(w.tiles, static_cast<int>(n), A);
  ++g_launches;
  CUDA_TRY(cudaGetLastError());
  if (colsq) CUDA_TRY(cudaMemcpyAsync(colsq, w.tiles + L.tiles_sym * 64, 8, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return SCQR3_OK;
}

int scqr3_gram_oblique_csr(int64_t m, int64_t n, const double* X, int64_t ld, const scqr3_csr* B, double* A,
                           double* colsq, const scqr3_opts* opts) {
  TRY(check_opts(opts));
  if (n < 1 || n > kMaxN || m < 1) return fail("bad sizes");
  TRY(check_matrix("X", X, m, ld));
  if (!B || !B->row_ptr || !B->col_idx || !B->vals) return fail("CSR metric has a NULL array");
  if (B->halo != 0) return fail("kernel-level CSR Gram takes no halo (halo must be 0)");
  Ctx* c;
  TRY(get_ctx(&c));
  const Layout L = make_layout(m, n, 1, 0);
  WS w;
  TRY(carve(L, opts, &w));
  cudaStream_t st = static_cast<cudaStream_t>(opts->stream);
  ObliqueYParams yp{};
  yp.Q = X;
  yp.ldq = ld;
  yp.Y = w.y;
  yp.ldy = L.ldy;
  yp.m = m;
  yp.n = static_cast<int>(n);
  yp.rp = reinterpret_cast<const long long*>(B->row_ptr);
  yp.ci = B->col_idx;
  yp.cv = B->vals;
  yp.halo = 0;
  long long hnnz = 0;
  CUDA_TRY(cudaMemcpyAsync(&hnnz, yp.rp + m, sizeof(long long), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  yp.csr_tile = hnnz >= 0 && hnnz <= static_cast<long long>(kCsrTileNnzPerRow) * m ? 1 : 0;
  TRY(run_gram(c, L, w, X, ld, m, true, &yp, st));
  const long long nn = n * n;
  tiles_to_full_kernel<<<static_cast<unsigned>((nn + 255) / 256), 256, 0, st>>>(w.tiles, static_cast<int>(n), A);
  ++g_launches;
  CUDA_TRY(cudaGetLastError());
  if (colsq) CUDA_TRY(cudaMemcpyAsync(colsq, w.tiles + L.tiles_sym * 64, 8, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return SCQR3_OK;
}

int scqr3_cholesky(int64_t n, const double* A, double s, double* R, int32_t* pivot, double* pivot_value,
                   const scqr3_opts* opts) {
  TRY(check_opts(opts));
  if (n < 1 || n > kMaxN) return fail("bad n");
  if (!A || !R) return fail("NULL matrix");
  Ctx* c;
  TRY(get_ctx(&c));
  const Layout L = make_layout(n, n, 0);
  WS w;
  TRY(carve(L, opts, &w));
  cudaStream_t st = static_cast<cudaStream_t>(opts->stream);
  CholParams cp{};
  cp.Afull = A;
  cp.n = static_cast<int>(n);
  cp.NT = L.NT;
  cp.npad = L.npad;
  cp.mode = CHOL_ONLY;
  cp.shift_value = s;
  cp.W = w.W;
  cp.w_in_smem = w_fits_smem(static_cast<int>(n)) ? 1 : 0;
  cp.R = R;
  cp.st_dev = w.st;
  TRY(launch_chol(cp, st));
  DevStatus hs;
  CUDA_TRY(cudaMemcpyAsync(&hs, w.st, sizeof hs, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (pivot) *pivot = hs.breakdown_pivot;
  if (pivot_value) *pivot_value = hs.pivot_value;
  return hs.code;
}

int scqr3_trsm(int64_t m, int64_t n, const double* X, int64_t ld, const double* R, double* Q, int64_t ldq,
               const scqr3_opts* opts) {
  TRY(check_opts(opts));
  if (n < 1 || n > kMaxN || m < 0) return fail("bad sizes");
  TRY(check_matrix("X", X, m, ld));
  TRY(check_matrix("Q", Q, m, ldq));
  if (!R) return fail("R is NULL");
  Ctx* c;
  TRY(get_ctx(&c));
  const Layout L = make_layout(m, n, 0);
  WS w;
  TRY(carve(L, opts, &w));
  cudaStream_t st = static_cast<cudaStream_t>(opts->stream);
  trsm_prep_kernel<<<trsm_prep_blocks(L.NT), 256, 0, st>>>(R, static_cast<int>(n), L.NT, w.bfrag, w.dblk, 0, nullptr,
                                                          PassGate{}, opts->trsm_diag);
  ++g_launches;
  CUDA_TRY(cudaGetLastError());
  TrsmParams tp{};
  tp.X = X;
  tp.ldx = ld;
  tp.Q = Q;
  tp.ldq = ldq;
  tp.m = m;
  tp.n = static_cast<int>(n);
  tp.bfrag = w.bfrag;
  tp.dblk = w.dblk;
  tp.dinv = w.dblk + dinv_off(L.NT);
  tp.inv_flag = opts->trsm_diag == SCQR3_TRSM_DIAG_SUBST ? nullptr : w.dblk + dflag_off(L.NT);  // reading D24
  tp.st = nullptr;
  if (m > 0) {
    CUtensorMap mx;
    const bool use_tma = L.NT <= 16 || L.NT >= 24;
    if (use_tma) TRY(encode_map(c, &mx, X, m, L.NT >= 24 ? 128 : n, ld, trsm_x_box_cols(L.NT)));
    CUDA_TRY(launch_trsm(tp, use_tma ? &mx : nullptr, c->num_sms, st));
    g_launches += trsm_launch_count(tp, use_tma);
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  return SCQR3_OK;
}

int scqr3_comm_unique_id(void* id_out) {
  if (!id_out) return fail("id_out is NULL");
  static_assert(sizeof(ncclUniqueId) == SCQR3_COMM_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof id);
  return SCQR3_OK;
}

int scqr3_comm_init(void** comm_out, int32_t nranks, const void* id, int32_t rank) {
  if (!comm_out || !id) return fail("NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail("bad rank %d / nranks %d", rank, nranks);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  Comm* c = new Comm{};
  c->kind = COMM_NCCL;
  c->rank = rank;
  c->nranks = nranks;
  if (cudaMalloc(&c->dscratch, 64) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&c->hscratch), 64, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    if (c->dscratch) cudaFree(c->dscratch);
    delete c;
    return fail("allocation of the communicator scratch failed");
  }
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, uid, rank);
  if (r != ncclSuccess) {
    cudaFree(c->dscratch);
    cudaFreeHost(c->hscratch);
    delete c;
    return fail("ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  *comm_out = c;
  return SCQR3_OK;
}

int scqr3_comm_init_loopback(void** comms_out, int32_t nranks) {
  if (!comms_out) return fail("comms_out is NULL");
  std::vector<Comm*> cs(std::max(nranks, 1));
  TRY(comm_create_loopback(cs.data(), nranks));
  for (int r = 0; r < nranks; ++r) comms_out[r] = cs[r];
  return SCQR3_OK;
}

int scqr3_comm_destroy(void* comm) { return comm_destroy(static_cast<Comm*>(comm)); }

const char* scqr3_last_error(void) { return g_err.c_str(); }

size_t scqr3_workspace_size_complex(int64_t m, int64_t n) {
  if (n < 1 || n > kMaxN || m < 0) return 0;
  return make_zlayout(m, n).end;
}

int scqr3_factor_complex(int64_t m, int64_t n, const double* X, int64_t ld, double* Q, int64_t ldq, double* R,
                         const scqr3_opts* opts) {
  return zfactor_impl(m, n, X, ld, Q, ldq, R, opts);
}

int64_t scqr3_launch_count(int32_t reset) {
  int64_t v = g_launches;
  if (reset) g_launches = 0;
  return v;
}

}  // extern "C"
