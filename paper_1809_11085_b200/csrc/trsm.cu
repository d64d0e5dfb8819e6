// trsm.cu -- tall-skinny triangular solve Q = X R~^{-1} (step a5; eq. (3); Alg. 1 line 4
// P:140; Alg. 2 line 8 P:685).  The paper's per-row model q_i^T = x_i^T (R + dR_i)^{-1} (P:189,
// P:323-334) holds because every row is solved by (blocked) forward substitution -- no
// explicit inverse of R~ is formed (reading D11).
//
// Design: rows are independent, so each warp owns 8*A rows and keeps
// them in registers for the whole solve, as m8n8k4 C fragments (lane g,t holds row g, columns
// 2t and 2t+1 of each 8-column block).  For column block J the update
//     C_J = X_J - Q_{<J} R~_{<J,J}
// runs on the FP64 tensor cores: the A operand of k-step s is the warp's own C fragment of
// block s/2, element s%2 (the k-index of the step is mapped to columns {8(s/2)+2t+(s%2)}), so
// the solved rows never leave the registers; the B operand (-R~ rows in fragment order,
// written by chol_kernel) is read from shared memory, conflict free.  The 8x8 diagonal block
// is then solved by right-looking substitution inside each quad (shuffle of each pivot
// column, multiply by the reciprocal pivot).  X is read once and Q written once per pass.
#include "scqr3_dev.cuh"
#include "scqr3_kernels.h"

namespace scqr3 {

template <int NT, int A, bool SMEM_B, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) trsm_kernel(TrsmParams p) {
  extern __shared__ double sm[];
  if (p.st && p.st->code != 0) return;
  constexpr int NF = NT * (NT - 1);
  const double* bf;
  const double* db;
  if (SMEM_B) {
    for (int i = threadIdx.x; i < NF * 32 + NT * 72; i += THREADS)
      sm[i] = i < NF * 32 ? p.bfrag[i] : p.dblk[i - NF * 32];
    bf = sm;
    db = sm + NF * 32;
  } else {
    for (int i = threadIdx.x; i < NT * 72; i += THREADS) sm[i] = p.dblk[i];
    bf = p.bfrag;
    db = sm;
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  constexpr int WPB = THREADS / 32;
  const long long m = p.m;
  const int n = p.n;
  const long long ngroups = (m + 8 * A - 1) / (8 * A);
  for (long long rg = static_cast<long long>(blockIdx.x) * WPB + warp; rg < ngroups;
       rg += static_cast<long long>(gridDim.x) * WPB) {
    const long long r0 = rg * 8 * A;
    double q[A][NT][2];
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const long long row = r0 + 8 * a + g;
      const bool rok = row < m;
#pragma unroll
      for (int J = 0; J < NT; ++J)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 8 * J + 2 * t + h;
          q[a][J][h] = (rok && col < n) ? __ldcs(p.X + row + static_cast<long long>(col) * p.ldx) : 0.0;
        }
    }
#pragma unroll
    for (int J = 0; J < NT; ++J) {
      // ---- GEMM part on the tensor cores: C_J += Q_{<J} (-R~_{<J,J})
#pragma unroll
      for (int s = 0; s < 2 * J; ++s) {
        const double b = SMEM_B ? bf[(J * (J - 1) + s) * 32 + lane] : __ldg(bf + (J * (J - 1) + s) * 32 + lane);
#pragma unroll
        for (int a = 0; a < A; ++a) dmma(q[a][J][0], q[a][J][1], q[a][s >> 1][s & 1], b);
      }
      // ---- 8x8 diagonal block: right-looking substitution inside each quad
      const double* D = db + J * 72;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double rinv = D[64 + c];
        const double2 rc = *reinterpret_cast<const double2*>(D + c * 8 + 2 * t);
        const int owner = (lane & ~3) | (c >> 1);
#pragma unroll
        for (int a = 0; a < A; ++a) {
          const double mine = (c & 1) ? q[a][J][1] : q[a][J][0];
          const double qc = __shfl_sync(0xffffffffu, mine * rinv, owner);
          if (t == (c >> 1)) {
            if (c & 1) q[a][J][1] = qc;
            else q[a][J][0] = qc;
          }
          if (2 * t > c) q[a][J][0] = fma(-qc, rc.x, q[a][J][0]);
          if (2 * t + 1 > c) q[a][J][1] = fma(-qc, rc.y, q[a][J][1]);
        }
      }
    }
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const long long row = r0 + 8 * a + g;
      if (row < m) {
#pragma unroll
        for (int J = 0; J < NT; ++J)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int col = 8 * J + 2 * t + h;
            if (col < n) __stcs(p.Q + row + static_cast<long long>(col) * p.ldq, q[a][J][h]);
          }
      }
    }
  }
}

template <int NT, int A, bool SMEM_B, int THREADS>
static cudaError_t launch_one(const TrsmParams& p, int num_sms, cudaStream_t stream) {
  constexpr int NF = NT * (NT - 1);
  const size_t smem = SMEM_B ? static_cast<size_t>(NF * 32 + NT * 72) * 8 : static_cast<size_t>(NT * 72) * 8;
  auto k = trsm_kernel<NT, A, SMEM_B, THREADS>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const long long groups = (p.m + 8 * A - 1) / (8 * A);
  long long grid = static_cast<long long>(num_sms) * per_sm;
  const long long need = (groups + THREADS / 32 - 1) / (THREADS / 32);
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  k<<<static_cast<unsigned>(grid), THREADS, smem, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_trsm(const TrsmParams& p, int num_sms, cudaStream_t stream) {
  const int NT = npad_for(p.n) / 8;
  switch (NT) {
    case 1: return launch_one<1, 4, true, 256>(p, num_sms, stream);
    case 2: return launch_one<2, 4, true, 256>(p, num_sms, stream);
    case 4: return launch_one<4, 4, true, 256>(p, num_sms, stream);
    case 8: return launch_one<8, 4, true, 256>(p, num_sms, stream);
    case 12: return launch_one<12, 2, true, 256>(p, num_sms, stream);
    case 16: return launch_one<16, 2, true, 256>(p, num_sms, stream);
    case 24: return launch_one<24, 1, true, 256>(p, num_sms, stream);
    case 32: return launch_one<32, 1, false, 256>(p, num_sms, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace scqr3
