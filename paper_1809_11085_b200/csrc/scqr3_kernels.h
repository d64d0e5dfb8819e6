// scqr3_kernels.h -- parameter blocks and kernel declarations shared by the .cu files of
// libscqr3 (internal; the public ABI is include/scqr3.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace scqr3 {

struct DevStatus;

constexpr int kMaxConsumers = 20;   // consumer warps per Gram CTA (+1 producer = 672 threads)
constexpr int kMaxConsumersWhole = 18;   // whole-block Gram jobs, 19 warps x 96 registers
constexpr int kMaxConsumersWhole2 = 15;  // whole-block Gram jobs, 16 warps x 128 registers
constexpr int kMaxGroups = 32;      // job groups (CTAs sharing one row chunk)

// Device-side pass control (speculative enqueue, scqr3_host.cu): the kernels of pass `pass` exit
// at once when the Cholesky of an earlier pass has set *last_pass below it (stop or error).
struct PassGate {
  const int* last_pass = nullptr;  // null: always run (kernel-level API)
  int pass = 0;
  const int* pass_dev = nullptr;   // CUDA-graph loop body: the pass number lives on the device
};
// (scalar arguments: passing or calling on the struct inside a kernel-parameter block makes the
//  compiler copy the whole block -- 2.6 KB for GramParams -- to local memory; measured)
__device__ __forceinline__ bool gate_skip3(const int* last_pass, int pass, const int* pass_dev) {
  if (!last_pass) return false;
  const int k = pass_dev ? *(volatile const int*)pass_dev : pass;
  return k > *(volatile const int*)last_pass;
}
#define SCQR3_GATE_SKIP(g) gate_skip3((g).last_pass, (g).pass, (g).pass_dev)

struct GramParams {
  PassGate gate;
  double* partials;          // [chunks][tiles_per_partial][64]
  long long total_stages;    // ceil(m / 16)
  int chunks;                // row chunks (CTAs per group)
  int groups;                // job groups (CTAs per chunk)
  int stages;                // pipeline depth
  int npad;                  // padded column count (multiple of 8, TMA box width)
  int NT;                    // npad / 8 tiles per side computed (ceil(n / 8))
  int NTl;                   // tiles per side of the partial layout (n padded to a TRSM instance)
  int NB;                    // ceil(NT / 4) blocks per side
  int oblique;               // 1 = Q^T Y (upper tiles, reading D22)
  int dual;                  // oblique: also the plain Gram Q^T Q (its norm estimate, reading D4)
  int tiles_per_partial;     // NT(NT+1)/2, doubled when dual or NT^2
  int mc;                    // > 1: the `groups` CTAs of a row chunk form a cluster and each stage
                             //   is multicast to all of them (each CTA loads 1 / mc of its boxes)
  int box_cols;              // columns per TMA box of the stage (the map's box width)
  int rb;                    // 16-row blocks per stage: 1 (2-D map) or 2 (3-D map, m % 32 == 0, no multicast)
  // job of consumer warp w in group g: warp_job[g * kMaxConsumers + w] (-1 = idle); the host
  // balances the DMMA work of each group over the SM's four sub-partitions (warp % 4)
  short warp_job[kMaxGroups * kMaxConsumers];  // codes <= 2 * 136 (n <= 512)
};

struct GramReduceParams {
  PassGate gate;
  int dual;                  // partials hold [Q^T Y tiles][Q^T Q tiles]: output [B-Gram][||Q||_F^2][plain]
  const double* partials;
  double* tiles;             // packed upper tiles (+1 double: ||Q||_F^2 for oblique)
  int chunks;
  int tiles_per_partial;
  int NT;                    // tiles per side of the layout
  int NTc;                   // tile columns computed (later ones are written as zeros)
  int oblique;
  const double* colsq_partials;
  int colsq_count;
};

struct ObliqueYParams {
  PassGate gate;
  const double* Q;
  long long ldq;
  const double* d;
  const double* e;
  double* Y;
  long long ldy;
  long long m;
  int n;
  int has_prev, has_next;
  double e_prev;
  const double* halo_prev;   // halo x n (ld halo): previous rank's last rows of Q
  const double* halo_next;   // halo x n (ld halo): next rank's first rows of Q
  double* colsq_partials;    // one per block
  // general sparse metric in CSR (rp != nullptr): column indices relative to
  // this rank's first row, in [-halo, m + halo)
  const long long* rp;
  const int* ci;
  const double* cv;
  long long halo;
  // ghost-row plan (scqr3_csr.halo == SCQR3_CSR_GHOSTS): indices in [m, m + nghost) read ghost
  // row (index - m) of `ghost` (row-major, nghost x n); halo then holds nghost
  int ghosts;
  const double* ghost;
  // host's choice of the Y = BQ kernel: 1 = csr_y_tile_kernel (nnz <= kCsrTileNnzPerRow * m, so the
  // tiles' CSR arrays fit its shared-memory stage), 0 = csr_y_kernel (denser metrics: measured
  // faster there, profiles/csr_y_r02e.md)
  int csr_tile;
};

enum CholMode { CHOL_PASS = 0, CHOL_ONLY = 1 };

// Leading dimension of the Cholesky kernel's working copy W (row-major n x n): n + 4 puts the
// mma fragment loads of the panel rows (lanes t, g -> W[(k + t) * ldw + 8 I + g]) on 16 distinct
// bank pairs per half-warp (n + 1 gave 4-way conflicts: the trailing update was bound by
// shared-memory wavefronts).
inline __host__ __device__ int chol_ldw(int n) { return n + 4; }

struct CholParams {
  const double* tiles;       // packed upper tiles of the Gram (CHOL_PASS)
  const double* Afull;       // or a full column-major n x n matrix (CHOL_ONLY)
  int n, NT, npad;
  int mode;
  int pass;                  // 1-based
  int oblique;
  int shift_mode;
  double shift_value;
  int norm_mode;
  double norm2_bound;
  int power_iters;
  double m_global;
  const double* nb_dev;      // oblique: ||B||_2 bound (device scalar)
  const double* lmax_dev;    // pass 1: lambda_max estimate from power_cluster_kernel (null: in-kernel)
  double stop_tol;
  double* W;                 // n x n scratch (global) when it does not fit in shared memory
  int w_in_smem;
  double* R;                 // CHOL_ONLY output (n x n col-major)
  double* Rt;                // CHOL_PASS: R~ of this pass (n x n row-major) for trmul_kernel, trsm_prep_kernel
  double* bfrag;             // TRSM B fragments (negated R~), NT(NT-1) x 32, written here when
  double* dblk;              //   non-null (n <= 64), else by trsm_prep_kernel; diagonal-block data (dblk_doubles)
  int trsm_diag;             // SCQR3_TRSM_DIAG_*: how the diagonal-block guard flag is set (reading D24)
  DevStatus* st_dev;
  DevStatus* st_host;        // host-mapped per-pass slots (st_host[pass-1]; may be null)
  int* last_pass;            // device-side pass control (may be null): written on stop / error
  const int* pass_dev;       // CUDA-graph loop body: pass number on the device (else `pass`)
};

// power iteration on a cluster of 8 CTAs (n in (128, 256]): Rayleigh quotient -> *out
struct PowerParams {
  const double* tiles;       // packed upper tiles of the Gram to iterate on
  int n;
  int iters;
  double* out;
  int pass;                  // gate as the chol kernel's: skipped after a stop
  const int* pass_dev;
  const int* last_pass;
};
__global__ void power_cluster_kernel(PowerParams p);
size_t power_cluster_smem(int n);

// complex n x n step (zchol.cu)
struct ZCholParams {
  const double* A;           // A = X^H X, n x n complex (column-major interleaved)
  double* W;                 // n x n complex scratch
  int n;
  int pass;
  const int* pass_dev;
  int* last_pass;
  int shift_mode;
  double shift_value;
  int norm_mode;
  double norm2_bound;
  int power_iters;
  double m_global;
  double stop_tol;
  double* Rt;                // R~ (n x n complex) for ztrmul_kernel
  double* M;                 // real 2n x 2n upper-triangular image of R~ for the TRSM (column-major)
  int w_in_smem;             // packed upper working copy in dynamic shared memory (n <= 128)
  DevStatus* st_dev;
  DevStatus* st_host;
};

struct TrsmParams {
  PassGate gate;
  const double* X;
  long long ldx;
  double* Q;
  long long ldq;
  long long m;
  int n;
  const double* bfrag;
  const double* dblk;        // substitution tables of this launch's diagonal blocks (72 doubles each)
  const double* dinv;        // B fragments of the inverted diagonal blocks (64 doubles each; reading D24)
  const double* inv_flag;    // null: substitution only; else *inv_flag > 0 selects the inverse
                             // instance (trsm_kernel<..., INV = true>), 0 the substitution one
  const DevStatus* st;       // skip when st->code != 0 (may be null)
  double* gram_partials;     // fused next-pass Gram (n <= 64): one NT(NT+1)/2-tile partial per CTA
};

// gram_tma_kernel<JR, MAXC> (gram.cu): JR = tile rows per consumer-warp job, 2 (half 4x4-tile
// blocks) or 4 (whole blocks); MAXC = consumer warps it is compiled for.  Variant v of
// assign_gram_jobs: 0 = <2, 20>, 1 = <4, 18>, 2 = <4, 15>.
cudaError_t gram_tma_config(int variant, bool mc, size_t smem, int threads, int* occ, int rb = 1);  // smem attribute + occupancy (cached)
// clusters of mc CTAs that fit at once (multicast launch)
cudaError_t gram_tma_max_clusters(int variant, size_t smem, int threads, int mc, int* nclusters);
cudaError_t launch_gram_tma(int variant, unsigned grid, int threads, size_t smem, cudaStream_t stream,
                            const CUtensorMap& mapQ, const CUtensorMap& mapY, const GramParams& p);
__global__ void gram_reduce_kernel(GramReduceParams p);
__global__ void csr_y_kernel(ObliqueYParams p);
constexpr int kCsrTileRows = 256;       // rows (= threads) per CTA of csr_y_tile_kernel
constexpr int kCsrTileNnzPerRow = 12;   // staged nonzeros per tile row (36 KB of shared memory)
__global__ void csr_y_tile_kernel(ObliqueYParams p);
__global__ void csr_gershgorin_kernel(const long long* rp, const double* cv, long long m, double* partial);
__global__ void index_check_kernel(const long long* v, long long cnt, long long lo, long long hi, int* bad);
__global__ void csr_check_kernel(const long long* rp, const int* ci, long long m, long long halo, int has_prev,
                                 int has_next, int* bad);
__global__ void rank_sum_kernel(const double* parts, int nparts, long long count, double* out);
__global__ void oblique_y_kernel(ObliqueYParams p);
__global__ void gershgorin_kernel(const double* d, const double* e, long long m, int has_prev, double e_prev,
                                  int has_next, double* partial);
__global__ void max_reduce_kernel(const double* partial, int count, double* out);
__global__ void tiles_to_full_kernel(const double* tiles, int n, double* A);
__global__ void chol_kernel_smem(CholParams p);
__global__ void chol_kernel_gmem(CholParams p);
__global__ void trmul_kernel(const double* Rt, const double* R, double* Rnew, int n, int first, const DevStatus* st,
                             PassGate gate);
__global__ void copy_kernel(const double* src, double* dst, long long count, const DevStatus* st, PassGate gate);
__global__ void trsm_prep_kernel(const double* R, int n, int NT, double* bfrag, double* dblk, int rowmajor,
                                 const DevStatus* st, PassGate gate, int diag_mode);  // grid: trsm_prep_blocks(NT) x 256
__global__ void z2split_kernel(const double* Z, long long ldz, long long m, int n, double* S, long long lds);
__global__ void split2z_kernel(const double* S, long long lds, long long m, int n, double* Z, long long ldz);
__global__ void zcombine_kernel(const double* tiles, int n, double* A, const int* last_pass, int pass);
__global__ void zchol_kernel(ZCholParams p);
// complex n in (256, 512]: the split matrix in two column blocks (zwide.cu)
__global__ void xgram_kernel(const double* A, long long lda, const double* B, long long ldb, long long m, int p, int q,
                             long long rows_per_chunk, double* partials, PassGate gate);  // grid chunks*nbp*nbq x 256
__global__ void xreduce_kernel(const double* partials, int chunks, long long count, double* out, PassGate gate);
__global__ void xupdate_kernel(const double* Q1, long long ldq, const double* M12, long long ldm, double* S2,
                               long long lds, long long m, int p, int q, PassGate gate);  // grid ceil(m/64)*nbq x 256
__global__ void zsub_kernel(const double* M, long long ldm, int r0, int c0, int nr, int nc, double* out, PassGate gate);
__global__ void zcombine_wide_kernel(const double* t1, const double* t2, const double* c12, int n, int h, double* A,
                                     const int* last_pass, int pass);
__global__ void ztrmul_kernel(const double* Rt, const double* R, double* Rnew, int n, int first, const DevStatus* st,
                              PassGate gate);
// CUDA-graph pass loop (device-side pass control): the loop-condition kernel
// advances the counter when it lets the body run again; the loop continues while the Cholesky has not stopped it.
__global__ void pass_loop_cond_kernel(int* pass_dev, const int* last_pass, int max_passes,
                                      cudaGraphConditionalHandle handle);  // (also advances the counter)

// Per-call-site cache of cudaFuncSetAttribute(max dynamic smem) + the occupancy query, so a
// pass does not repeat these host API calls (small problems are launch-bound on the host).
struct LaunchCfgCache {
  int dev = -1;
  size_t smem = 0;
  int threads = 0;
  int occ = 0;
};
// The dynamic shared-memory limit is a process-wide attribute of the kernel while this cache is
// per thread, and the host threads of a loopback group (or of any multi-threaded caller) launch
// the same kernel with different sizes (e.g. Gram ring depths that depend on the rank's m): so
// the limit is raised once to the most the kernel can take, never set to one call's size -- a
// later, smaller setting by another thread would make this thread's launch fail.
template <class K>
inline cudaError_t cached_launch_cfg(LaunchCfgCache& cc, K kernel, size_t smem, int threads, int* occ) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (cc.dev != dev || cc.smem != smem || cc.threads != threads) {
    cudaFuncAttributes fa{};
    e = cudaFuncGetAttributes(&fa, kernel);
    if (e != cudaSuccess) return e;
    int optin = 0;
    e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    const int lim = optin - static_cast<int>(fa.sharedSizeBytes);
    if (static_cast<size_t>(lim) < smem) return cudaErrorInvalidValue;
    if (fa.maxDynamicSharedSizeBytes != lim) {
      e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
      if (e != cudaSuccess) return e;
    }
    int o = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kernel, threads, smem);
    if (e != cudaSuccess) return e;
    cc.dev = dev;
    cc.smem = smem;
    cc.threads = threads;
    cc.occ = o;
  }
  if (occ) *occ = cc.occ;
  return cudaSuccess;
}

// TRSM launcher (chooses the template instance for n)
// With p.gram_partials set (n <= 64 only, see trsm_fuses_gram) the launch also writes the next
// pass's Gram partials; *grid_out = the number of partials (CTAs).  mapQ (required then): TMA
// descriptor of Q (same box as map) for the bulk stores of the solved rows.
cudaError_t launch_trsm(const TrsmParams& p, const CUtensorMap* map, int num_sms, cudaStream_t stream,
                        int* grid_out = nullptr, const CUtensorMap* mapQ = nullptr);
inline bool trsm_fuses_gram(int NT) { return NT <= 8; }
int trsm_launch_count(const TrsmParams& p, bool tma);
// width of the TMA box of X the TRSM launcher expects (the map of the first 128 columns for
// NT >= 24; a narrower box where the kernel reads the later columns from global memory)
int trsm_x_box_cols(int NT);

// Diagonal-block data of the TRSM (workspace region dblk, NT = npad / 8 blocks):
//   [NT x 72]  substitution tables: strict upper r_cj / r_cc (64) + reciprocal pivots (8)
//   [NT x 64]  B fragments of the inverted blocks Y_J = D_J^{-1} (k-step h, lane l: Y[2(l&3)+h][l>>2])
//   [1]        guard flag (1: every Y_J keeps the row-wise backward error within eq. (DeltaRbound),
//              reading D24; 0: substitution); [1] the guard's ratio (diagnostics)
__host__ __device__ constexpr int dinv_off(int NT) { return NT * 72; }
__host__ __device__ constexpr int dflag_off(int NT) { return NT * 136; }
__host__ __device__ constexpr int dblk_doubles(int NT) { return NT * 136 + 8; }
// trsm_prep_kernel grid: the operand CTAs plus one guard CTA (last block)
inline int trsm_prep_blocks(int NT) { return (NT * (NT - 1) * 32 + NT * 72 + 255) / 256 + 1; }

inline int npad_for(int n) {
  // tile counts with a compiled TRSM instance
  static const int nts[] = {1, 2, 4, 8, 12, 16, 24, 32, 64};
  int nt = (n + 7) / 8;
  for (int v : nts)
    if (v >= nt) return v * 8;
  return -1;
}

}  // namespace scqr3
