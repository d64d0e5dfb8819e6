// trsm.cu -- tall-skinny triangular solve Q = X R~^{-1} (step a5; eq. (3); Alg. 1 line 4
// P:140; Alg. 2 line 8 P:685).  The paper's per-row model q_i^T = x_i^T (R + dR_i)^{-1} (P:189,
// P:323-334) holds because every row is solved by blocked forward substitution (reading D11) --
// or, where a per-pass guard proves it keeps ||dR_i||_2 <= gamma_n sqrt(n) ||R~||_2 (eq.
// DeltaRbound), with the 8x8 diagonal blocks applied as products with their inverses
// on the tensor cores (INV instances, reading D24).  No inverse of R~ itself is ever formed.
//
// Design: rows are independent, so each warp owns 8*A rows and keeps
// them in registers for the whole solve, as m8n8k4 C fragments (lane g,t holds row g, columns
// 2t and 2t+1 of each 8-column block).  For column block J the update
//     C_J = X_J - Q_{<J} R~_{<J,J}
// runs on the FP64 tensor cores: the A operand of k-step s is the warp's own C fragment of
// block s/2, element s%2 (the k-index of the step is mapped to columns {8(s/2)+2t+(s%2)}), so
// the solved rows never leave the registers; the B operand (-R~ rows in fragment order,
// written by chol_kernel) is read from shared memory, conflict free.  The 8x8 diagonal block
// is then solved by right-looking substitution inside each quad; with two fragments (rows g and
// g+8) the quad's lanes first swap halves so that each lane holds four columns of one row, and
// each step issues only the DFMAs whose column can still change (18 per pair instead of 28).
// The loop is software-pipelined: the (latency-bound) diagonal solve of block J is interleaved
// with block J-1's tensor-core updates to the later blocks.
// X is read once (TMA into a per-warp shared-memory slot, one row group ahead, so the HBM
// latency is off the critical path) and Q written once per pass.  Block-column launches
// (trsm_wide_kernel below) for n > 128.
#include "scqr3_dev.cuh"
#include "scqr3_kernels.h"
#ifdef SCQR3_TRSM_CLOCK
#include <cstdio>
#endif

namespace scqr3 {

#ifndef SCQR3_TRSM_PIPE
#define SCQR3_TRSM_PIPE 1  // 0: both k-steps of each later target back to back (A/B builds)
#endif

// Which updates C_K += Q_S (-R~_{S,K}) run during the diagonal chain of block J (S <= J - 1 <
// J + 1 <= K; the last one, S = J - 1, K = J, runs before the chain).  Right-looking (CAP >= NT)
// hosts exactly the updates from S = J - 1, so the early chains carry most of the tensor-core
// work and the late ones almost none.  With CAP < NT a chain hosts at most CAP updates: those
// due now (K = J + 1) first, then the fresh source S = J - 1, then the earliest deadlines, and
// the rest wait for a later chain -- always in ascending S for each target, so every target
// still receives its updates in the same order (the same rounding).
template <int NT>
struct TrsmSched {
  int cnt[NT > 0 ? NT : 1];
  int S[NT > 0 ? NT : 1][NT > 0 ? NT : 1];
  int K[NT > 0 ? NT : 1][NT > 0 ? NT : 1];
};
template <int NT, int CAP>
constexpr TrsmSched<NT> make_trsm_sched() {
  TrsmSched<NT> r{};
  bool done[NT > 0 ? NT : 1][NT > 0 ? NT : 1] = {};
  for (int K = 0; K < NT; ++K)
    for (int S = 0; S < NT; ++S) done[S][K] = !(S + 1 < K);  // pending: S <= K - 2
  for (int J = 1; J < NT; ++J) {
    int c = 0;
    auto next_of = [&](int K) {  // smallest pending S of target K (ascending order), or -1
      for (int S = 0; S < K - 1; ++S)
        if (!done[S][K]) return S;
      return -1;
    };
    // pass 0: due now (K = J + 1); pass 1: fresh source S = J - 1; pass 2: earliest deadline
    for (int pass = 0; pass < 3; ++pass)
      for (int K = J + 1; K < NT; ++K)
        for (;;) {
          const int S = next_of(K);
          if (S < 0 || S > J - 1) break;
          const bool take = pass == 0 ? K == J + 1 : c < CAP && (pass == 2 || S == J - 1);
          if (!take) break;
          r.S[J][c] = S;
          r.K[J][c] = K;
          ++c;
          done[S][K] = true;
          if (pass == 1) break;
        }
    r.cnt[J] = c;
  }
  return r;
}
#ifndef SCQR3_INV_K0
#define SCQR3_INV_K0 2  // chain slots of the two inverse k-steps (INV instances)
#endif
#ifndef SCQR3_INV_K1
#define SCQR3_INV_K1 5
#endif
#ifndef SCQR3_TRSM_CAP
#define SCQR3_TRSM_CAP 8  // updates per diagonal chain for NT = 16 (>= 1000: right-looking)
#endif
template <int NT, int CAP>
constexpr bool trsm_sched_ok() {
  constexpr auto r = make_trsm_sched<NT, CAP>();
  int total = 0;
  for (int J = 1; J < NT; ++J) {
    total += r.cnt[J];
    for (int i = 0; i < r.cnt[J]; ++i)
      for (int j = i + 1; j < r.cnt[J]; ++j)
        if (r.K[J][i] == r.K[J][j] && i * 8 / r.cnt[J] == j * 8 / r.cnt[J]) return false;
  }
  return total == (NT - 1) * (NT - 2) / 2;  // every update hosted exactly once
}
#if SCQR3_TRSM_CAP < 1000
static_assert(trsm_sched_ok<16, SCQR3_TRSM_CAP>(), "TRSM update schedule");
#endif

// GRAM (n <= 64): also accumulate the next pass's Gram Q_k^T Q_k from the
// solved rows, so the next pass does not read Q from HBM again.  Each warp writes its 16 finished
// rows to a private swizzled stage and accumulates their Gram (all upper 8x8 tiles) in registers;
// at the end the CTA sums its warps in a fixed order and writes one partial (gram_reduce_kernel
// sums the partials of all CTAs, as after gram_tma_kernel).  Skipped when this pass stops.
// INV (reading D24): the diagonal blocks are applied as products with their inverses Y_J (two
// DMMA k-steps per block, B fragments from chol / trsm_prep) instead of the substitution chain;
// launched beside the substitution instance, each exits unless *p.inv_flag selects it.
template <int NT, int A, bool SMEM_B, int THREADS, bool TMA, bool GRAM = false, bool INV = false>
__global__ void __launch_bounds__(THREADS, 1) trsm_kernel(const __grid_constant__ CUtensorMap mapX,
                                                          const __grid_constant__ CUtensorMap mapQ, TrsmParams p) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  if (SCQR3_GATE_SKIP(p.gate) || (p.st && p.st->code != 0)) return;
  static_assert(!INV || A % 2 == 0, "inverse diagonal blocks: paired fragments");
  if (INV ? !(p.inv_flag && *p.inv_flag > 0.0) : (p.inv_flag && *p.inv_flag > 0.0)) return;
  static_assert(!GRAM || (A == 2 && TMA), "fused Gram: 16-row groups per warp");
  constexpr int NTS = NT * (NT + 1) / 2;  // upper 8x8 tiles of the Gram
  const bool do_gram = GRAM && p.gram_partials && !(p.st && p.st->stop);
  // fused Gram: the solved rows go through the per-warp stage anyway, so Q leaves by one bulk
  // tensor store per 16 rows instead of 8-byte stores from the registers
  const bool bulk_q = GRAM && do_gram;
  constexpr int NF = NT * (NT - 1);
  constexpr int WPB = THREADS / 32;
  constexpr int NPAD = NT * 8;
  constexpr int RS = 8 * A;                                // rows per warp slot (multiple of 16)
  constexpr uint32_t kBoxBytes = 16u * NPAD * 8u;         // one 16-row TMA box
  constexpr uint32_t kSlotBytes = kBoxBytes * (RS / 16);
  static_assert(!TMA || RS % 16 == 0, "TMA slots hold whole 16-row boxes");
  // layout: [TMA slots (1024-aligned)] [B fragments] [diagonal blocks] [mbarriers]
  // (pointer arithmetic on the shared array itself keeps the shared address space -> LDS)
  unsigned char* base = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  unsigned char* slots = base;
  unsigned char* ostage = base + (TMA ? WPB * kSlotBytes : 0);  // GRAM: per-warp Q stages
  double* sm = reinterpret_cast<double*>(ostage + (GRAM ? WPB * kBoxBytes : 0));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (SMEM_B ? NF * 32 : 0) + NT * 72);
  const double* bf;
  const double* db;
  const double* dsrc = INV ? p.dinv : p.dblk;  // (INV: 64 of the 72 slots per block)
  if (SMEM_B) {
    for (int i = threadIdx.x; i < NF * 32 + NT * 72; i += THREADS)
      sm[i] = i < NF * 32 ? p.bfrag[i] : (INV && i - NF * 32 >= NT * 64 ? 0.0 : dsrc[i - NF * 32]);
    bf = sm;
    db = sm + NF * 32;
  } else {
    for (int i = threadIdx.x; i < NT * 72; i += THREADS) sm[i] = INV && i >= NT * 64 ? 0.0 : dsrc[i];
    bf = p.bfrag;
    db = sm;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  if (TMA && threadIdx.x == 0) {
    for (int w = 0; w < WPB; ++w) mbar_init(&bars[w], 1);
    fence_barrier_init();
  }
  __syncthreads();

  const long long m = p.m;
  const int n = p.n;
  // work unit = one row group of RS = 8A rows per warp
  const long long ngroups = (m + RS - 1) / RS;
  const long long stride = static_cast<long long>(gridDim.x) * WPB;
  unsigned char* slot = slots + warp * kSlotBytes;
  uint64_t* bar = bars + warp;
  uint32_t phase = 0;
  auto issue = [&](long long rg) {  // elected lane: TMA of slot group rg into this slot
    if (TMA && lane == 0 && rg < ngroups) {
      fence_proxy_async();
      mbar_arrive_expect_tx(bar, kSlotBytes);
#pragma unroll
      for (int b = 0; b < RS / 16; ++b)
        tma_load_2d(slot + b * kBoxBytes, &mapX, static_cast<int>(rg * RS + 16 * b), 0, bar);
    }
  };
  const long long rg0 = static_cast<long long>(blockIdx.x) * WPB + warp;
  if (TMA) {
    if (lane == 0) tma_prefetch_desc(&mapX);
    issue(rg0);
  }

  double gacc[GRAM ? NTS : 1][2];  // GRAM: this warp's Gram tiles (C fragments)
#pragma unroll
  for (int T = 0; T < (GRAM ? NTS : 1); ++T) gacc[T][0] = gacc[T][1] = 0.0;
  for (long long rg = rg0; rg < ngroups; rg += stride) {
    const long long r0 = rg * RS;
    double q[A][NT][2];
    auto store_block = [&](double (&qq)[A][NT][2], int J) {
#pragma unroll
      for (int a = 0; a < A; ++a) {
        const long long row = r0 + 8 * a + g;
        if (row < m) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int col = 8 * J + 2 * t + h;
            if (col < n) __stcs(p.Q + row + static_cast<long long>(col) * p.ldq, qq[a][J][h]);
          }
        }
      }
    };
    if (TMA) {
      mbar_wait(bar, phase);
      phase ^= 1u;
#pragma unroll
      for (int a = 0; a < A; ++a) {
        const int r = 8 * a + g;  // row inside the slot
        const unsigned char* box = slot + (r >> 4) * kBoxBytes;
#pragma unroll
        for (int J = 0; J < NT; ++J)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            q[a][J][h] = *reinterpret_cast<const double*>(box + swz128_offset(r & 15, 8 * J + 2 * t + h));
      }
    } else {
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
    }
    // Software pipeline over column blocks: iteration J gives block J its last update (from
    // block J-1), then solves block J's diagonal block (a latency-bound shuffle chain)
    // interleaved with block J-1's updates to the later blocks, which do not depend on it.
    // (Right-looking order: block K receives one k-step pair per iteration, so no DMMA
    //  accumulator chain is longer than two, and the updates from block J-1 to blocks > J are
    //  independent MMAs that fill the pipe while block J's shuffle chain runs.)
    auto bfrag = [&](int K, int s) -> double {  // -R~ fragment of k-step s for target block K
      return SMEM_B ? bf[(K * (K - 1) + s) * 32 + lane] : __ldg(bf + (K * (K - 1) + s) * 32 + lane);
    };
#ifdef SCQR3_TRSM_CLOCK
    long long tclk[NT + 1];
#endif
#pragma unroll
    for (int J = 0; J < NT; ++J) {
#ifdef SCQR3_TRSM_CLOCK
      tclk[J] = clock64();
#endif
      if (TMA && J == (NT > 1 ? 1 : 0)) {
        // every lane's slot reads have been consumed by now: refill the slot with the next group
        __syncwarp();
        issue(rg + stride);
      }
      // (i) block J's last update, from block J-1 (final since the previous iteration)
      if (J >= 1) {
#pragma unroll
        for (int s = 2 * (J - 1); s < 2 * J; ++s) {
          const double b = bfrag(J, s);
#pragma unroll
          for (int a = 0; a < A; ++a) dmma(q[a][J][0], q[a][J][1], q[a][J - 1][s & 1], b);
        }
      }
      // (ii) diagonal block J: right-looking substitution on the unscaled values v
      // (v_j -= v_c * (r_cj / r_cc), strict upper only, zeros elsewhere), interleaved with the
      // updates C_K += Q_{J-1} (-R~_{J-1,K}) of the later blocks K = J+1..NT-1
      const int nup = J >= 1 ? NT - 1 - J : 0;
#if !SCQR3_TRSM_PIPE
      int u = 0;
#endif
      const double* D = db + J * 72;
      auto upd = [&](int K, int s) {
        const double b = bfrag(K, s);
#pragma unroll
        for (int a = 0; a < A; ++a) dmma(q[a][K][0], q[a][K][1], q[a][J - 1][s & 1], b);
      };
      // The two k-steps of a target's update are a dependent DMMA pair; step c of the chain
      // issues the first k-step of its targets and the second k-step of step c-1's, so that
      // the dependent DMMAs sit a whole chain step apart (adjacent dependent DMMAs get a NOP
      // and a fixed-latency wait in between).
      auto later_updates = [&](int c) {
#if SCQR3_TRSM_CAP < 1000
       // (INV: no chain latency to hide; right-looking measured best, 5.25 -> 5.20 ms at C3)
       if constexpr (NT == 16 && !INV) {
        // the chain hosts the schedule's updates: update i's first k-step in chain step
        // i * 8 / cnt, its second one step later, issued before that step's first k-steps (a
        // target's updates therefore keep their order; trsm_sched_ok checks that no two
        // updates of one target share a step)
        constexpr auto sch = make_trsm_sched<NT, SCQR3_TRSM_CAP>();
        const int cnt = sch.cnt[J];
        auto upd2 = [&](int S, int K, int s) {
          const double b = bfrag(K, s);
#pragma unroll
          for (int a = 0; a < A; ++a) dmma(q[a][K][0], q[a][K][1], q[a][S][s & 1], b);
        };
        if (c >= 1) {
#pragma unroll
          for (int i = 0; i < NT; ++i)
            if (i < cnt && i * 8 / cnt == c - 1) upd2(sch.S[J][i], sch.K[J][i], 2 * sch.S[J][i] + 1);
        }
#pragma unroll
        for (int i = 0; i < NT; ++i)
          if (i < cnt && i * 8 / cnt == c) upd2(sch.S[J][i], sch.K[J][i], 2 * sch.S[J][i]);
        if (c == 7) {
#pragma unroll
          for (int i = 0; i < NT; ++i)
            if (i < cnt && i * 8 / cnt == 7) upd2(sch.S[J][i], sch.K[J][i], 2 * sch.S[J][i] + 1);
        }
        return;
       }
#endif
#if SCQR3_TRSM_PIPE
#pragma unroll
        for (int v = nup * c / 8; v < nup * (c + 1) / 8; ++v) upd(J + 1 + v, 2 * (J - 1));
        if (c >= 1) {
#pragma unroll
          for (int v = nup * (c - 1) / 8; v < nup * c / 8; ++v) upd(J + 1 + v, 2 * J - 1);
        }
        if (c == 7) {
#pragma unroll
          for (int v = nup * 7 / 8; v < nup; ++v) upd(J + 1 + v, 2 * J - 1);
        }
#else
#pragma unroll
        for (; u < nup * (c + 1) / 8; ++u) {
          const int K = J + 1 + u;
#pragma unroll
          for (int s = 2 * (J - 1); s < 2 * J; ++s) upd(K, s);
        }
#endif
      };
      if constexpr (INV) {
        // q_J = b_J Y_J: k-step h takes the C fragment's element h as the A operand (columns
        // 2t + h), Y_J's rows 2t + h as B; between the k-steps and after them, the later updates
        const double* Y = db + J * 64;
        const double y0 = Y[lane], y1 = Y[32 + lane];
        double acc[A][2];
#pragma unroll
        for (int a = 0; a < A; ++a) acc[a][0] = acc[a][1] = 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c == SCQR3_INV_K0) {
#pragma unroll
            for (int a = 0; a < A; ++a) dmma(acc[a][0], acc[a][1], q[a][J][0], y0);
          }
          if (c == SCQR3_INV_K1) {
#pragma unroll
            for (int a = 0; a < A; ++a) dmma(acc[a][0], acc[a][1], q[a][J][1], y1);
          }
          later_updates(c);
        }
#pragma unroll
        for (int a = 0; a < A; ++a) {
          q[a][J][0] = acc[a][0];
          q[a][J][1] = acc[a][1];
        }
      } else if constexpr (A % 2 == 0) {
        // Fragment pairs (a, a+1) = rows g and g+8 of the quad.  Lanes t^2 swap halves so that
        // lanes t = 0,1 hold row g and lanes t = 2,3 row g+8, four columns each: lane u = t&1
        // holds columns {2u, 2u+1, 2u+4, 2u+5} (V[0..3]).  Step c then updates only the
        // registers whose column can exceed c for some lane: 18 DFMA per pair instead of 28, and
        // the pivot comes from the partner lane (same substitution order, same rounding).
        const int uu = t & 1;
        const bool lo = t < 2;
        double V[A / 2][4];
#pragma unroll
        for (int a = 0; a < A; a += 2) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double snd = lo ? q[a + 1][J][h] : q[a][J][h];
            const double rcv = __shfl_xor_sync(0xffffffffu, snd, 2);
            V[a / 2][h] = lo ? q[a][J][h] : rcv;
            V[a / 2][2 + h] = lo ? rcv : q[a + 1][J][h];
          }
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c < 7) {
            const double2 r01 = *reinterpret_cast<const double2*>(D + c * 8 + 2 * uu);
            const double2 r23 = *reinterpret_cast<const double2*>(D + c * 8 + 4 + 2 * uu);
            const int owner = (lane & ~1) | ((c >> 1) & 1);
            constexpr int kmax[4] = {2, 3, 6, 7};  // register k can still change while c < kmax[k]
#pragma unroll
            for (int b = 0; b < A / 2; ++b) {
              const double vc = __shfl_sync(0xffffffffu, V[b][(c & 1) + 2 * (c >> 2)], owner);
              if (c < kmax[0]) V[b][0] = fma(-vc, r01.x, V[b][0]);
              if (c < kmax[1]) V[b][1] = fma(-vc, r01.y, V[b][1]);
              if (c < kmax[2]) V[b][2] = fma(-vc, r23.x, V[b][2]);
              if (c < kmax[3]) V[b][3] = fma(-vc, r23.y, V[b][3]);
            }
          }
          later_updates(c);
        }
        // (iii) q_j = v_j / r_jj as a multiply by the reciprocal (reading D11), then back to
        // the C-fragment layout
        const double2 i01 = *reinterpret_cast<const double2*>(D + 64 + 2 * uu);
        const double2 i23 = *reinterpret_cast<const double2*>(D + 64 + 4 + 2 * uu);
#pragma unroll
        for (int a = 0; a < A; a += 2) {
          double* Vb = V[a / 2];
          Vb[0] *= i01.x;
          Vb[1] *= i01.y;
          Vb[2] *= i23.x;
          Vb[3] *= i23.y;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double snd = lo ? Vb[2 + h] : Vb[h];
            const double rcv = __shfl_xor_sync(0xffffffffu, snd, 2);
            q[a][J][h] = lo ? Vb[h] : rcv;
            q[a + 1][J][h] = lo ? rcv : Vb[2 + h];
          }
        }
      } else {
        // (odd A: inside each quad, lane t holds columns 2t, 2t+1 of its row)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          // (column 7 of a block updates nothing inside it: its substitution step is skipped)
          if (c < 7) {
            const double2 rc = *reinterpret_cast<const double2*>(D + c * 8 + 2 * t);
            const int owner = (lane & ~3) | (c >> 1);
#pragma unroll
            for (int a = 0; a < A; ++a) {
              const double vc = __shfl_sync(0xffffffffu, q[a][J][c & 1], owner);
              q[a][J][0] = fma(-vc, rc.x, q[a][J][0]);
              q[a][J][1] = fma(-vc, rc.y, q[a][J][1]);
            }
          }
          later_updates(c);
        }
        // (iii) q_j = v_j / r_jj as a multiply by the reciprocal (reading D11)
        const double2 ri = *reinterpret_cast<const double2*>(D + 64 + 2 * t);
#pragma unroll
        for (int a = 0; a < A; ++a) {
          q[a][J][0] *= ri.x;
          q[a][J][1] *= ri.y;
        }
      }
      // block J-1 had its last use above: store it now (spreads the stores over the solve
      // instead of one burst per row group that fills the LSU queue)
      if (J >= 1 && !bulk_q) store_block(q, J - 1);
    }
    if (!bulk_q) store_block(q, NT - 1);
#ifdef SCQR3_TRSM_CLOCK
    tclk[NT] = clock64();
    if (lane == 0 && blockIdx.x == 7 && (warp == 1 || warp == 5) && rg / stride == 2) {
      long long d[16] = {};
      for (int J = 0; J < NT && J < 16; ++J) d[J] = tclk[J + 1] - tclk[J];
      printf("w%d %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld tot %lld\n", warp,
             d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7], d[8], d[9], d[10], d[11], d[12], d[13], d[14], d[15],
             tclk[NT] - tclk[0]);
    }
#endif
    if (TMA && NT <= 1) {
      __syncwarp();
      issue(rg + stride);
    }
    if constexpr (GRAM) {
      if (do_gram) {
        // the 16 solved rows (rows past m and padded columns are exact zeros) -> swizzled stage,
        // then k-steps over row quads {2s, 2s+1, 2s+8, 2s+9} as in gram_tma_kernel: one
        // fragment per column block serves as both MMA operands
        unsigned char* os = ostage + warp * kBoxBytes;
        if (lane == 0) bulk_wait_read_all();  // the previous group's bulk store has read the stage
        __syncwarp();
#pragma unroll
        for (int a = 0; a < A; ++a)
#pragma unroll
          for (int J = 0; J < NT; ++J)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              *reinterpret_cast<double*>(os + swz128_offset(8 * a + g, 8 * J + 2 * t + h)) = q[a][J][h];
        fence_proxy_async();  // the stage writes, visible to the bulk copy
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&mapQ, static_cast<int>(r0), 0, os);  // rows past m / columns past n are clipped
          bulk_commit();
        }
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const uint32_t inner = ((((s + 4 * (t >> 1)) ^ g) & 7u) << 4) + ((t & 1) << 3);
          double f[NT];
#pragma unroll
          for (int J = 0; J < NT; ++J) f[J] = *reinterpret_cast<const double*>(os + (8 * J + g) * 128u + inner);
#pragma unroll
          for (int J = 0; J < NT; ++J)
#pragma unroll
            for (int I = 0; I <= J; ++I) dmma(gacc[J * (J + 1) / 2 + I][0], gacc[J * (J + 1) / 2 + I][1], f[I], f[J]);
        }
        __syncwarp();
      }
    }
  }
  if constexpr (GRAM) {
    if (do_gram) {
      // CTA partial: warps add their tiles in warp order into shared memory (fixed order); the
      // stages become the reduction buffer once every warp's last bulk store has read its stage
      if (lane == 0) bulk_wait_read_all();
      __syncthreads();
      double* red = reinterpret_cast<double*>(ostage);  // NTS * 64 doubles <= WPB * kBoxBytes
      for (int w = 0; w < WPB; ++w) {
        if (warp == w) {
#pragma unroll
          for (int T = 0; T < NTS; ++T) {
            double2* dst = reinterpret_cast<double2*>(red + T * 64 + 8 * g + 2 * t);
            const double2 old = w == 0 ? make_double2(0.0, 0.0) : *dst;
            *dst = make_double2(old.x + gacc[T][0], old.y + gacc[T][1]);
          }
        }
        __syncthreads();
      }
      double* outp = p.gram_partials + static_cast<size_t>(blockIdx.x) * NTS * 64;
      for (int i = threadIdx.x; i < NTS * 64; i += THREADS) outp[i] = red[i];
      if (lane == 0) bulk_wait_all();  // this warp's bulk stores of Q complete before the CTA exits
    }
  }
}

template <int NT, int A, bool SMEM_B, int THREADS, bool TMA, bool GRAM = false, bool INV = false>
static cudaError_t launch_one(const TrsmParams& p, const CUtensorMap* map, int num_sms, cudaStream_t stream,
                              int* grid_out = nullptr, const CUtensorMap* mapQ = nullptr) {
  constexpr int NF = NT * (NT - 1);
  constexpr int WPB = THREADS / 32;
  constexpr int RS = 8 * A;
  constexpr size_t kSlot = 16u * NT * 8 * 8 * (RS / 16 > 0 ? RS / 16 : 1);
  const size_t smem = 1024 + (TMA ? WPB * kSlot : 0) + (GRAM ? WPB * 16u * NT * 8 * 8 : 0) +
                      static_cast<size_t>((SMEM_B ? NF * 32 : 0) + NT * 72) * 8 + WPB * 8;
  auto k = trsm_kernel<NT, A, SMEM_B, THREADS, TMA, GRAM, INV>;
  static thread_local LaunchCfgCache cfg;
  int per_sm = 0;
  cudaError_t e = cached_launch_cfg(cfg, k, smem, THREADS, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const long long groups = (p.m + RS - 1) / RS;
  long long grid = static_cast<long long>(num_sms) * per_sm;
  const long long need = (groups + WPB - 1) / WPB;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  CUtensorMap dummy{};
  k<<<static_cast<unsigned>(grid), THREADS, smem, stream>>>(map ? *map : dummy, mapQ ? *mapQ : dummy, p);
  if (grid_out) *grid_out = static_cast<int>(grid);
  return cudaGetLastError();
}

// Reading D24: with p.inv_flag set, the inverse-diagonal instance and the substitution instance
// are both enqueued; the guard flag (written on the device by chol / trsm_prep) lets one run and
// the other exit at entry (no host round trip; also inside the CUDA-graph pass loop).
template <int NT, int A, bool SMEM_B, int THREADS, bool TMA, bool GRAM = false>
static cudaError_t launch_pair(const TrsmParams& p, const CUtensorMap* map, int num_sms, cudaStream_t stream,
                               int* grid_out = nullptr, const CUtensorMap* mapQ = nullptr) {
  if (p.inv_flag) {
    cudaError_t e = launch_one<NT, A, SMEM_B, THREADS, TMA, GRAM, true>(p, map, num_sms, stream, grid_out, mapQ);
    if (e != cudaSuccess) return e;
  }
  return launch_one<NT, A, SMEM_B, THREADS, TMA, GRAM, false>(p, map, num_sms, stream, grid_out, mapQ);
}

// ------------------------------------------------------------------------------------------
// Wide TRSM (n in (192, 512]): -R~'s B fragments (254 KB at n=256, 1 MB at n=512) do not fit
// shared memory, so the target column blocks are processed in phases whose fragments do; the
// next phase's fragments stream into the second buffer with cp.async while the current phase
// computes.  Each warp owns 8 rows and 32 target blocks in registers (q: 64 doubles).  Per
// phase [K0, K1): (i) the updates of its targets from all earlier blocks (a dependency-free
// DMMA stream, targets interleaved), then (ii) the right-looking triangular part inside the
// phase, as in trsm_kernel.  n > 128 runs as block-column launches (launch_trsm below): columns
// 0..127 by trsm_kernel, targets 16..31 (16..23 for n <= 192) with resident fragments, and for
// n > 256 up to five resident launches for targets 32..40, 40..48, 48..56, 56..60, 60..64 (each
// reads the finished Q columns back; launches wholly past n are skipped).  The phased form
// (fragments re-streamed per row group) remains for the targets 0..31 / 32..63 fallbacks.
constexpr int phase_frags(int k0, int k1) { return k1 * (k1 - 1) - k0 * (k0 - 1); }
template <int TB, int TE> struct WidePhases;  // targets TB..TE-1
template <> struct WidePhases<0, 32> {  // targets 0..31
  static constexpr int P = 4, MAXF = 290;
  __host__ __device__ static constexpr int b(int i) { return i == 0 ? 0 : i == 1 ? 16 : i == 2 ? 22 : i == 3 ? 27 : 32; }
};
template <> struct WidePhases<16, 24> {  // targets 16..23 after a 128-column first launch (n <= 192)
  static constexpr int P = 1, MAXF = 312;  // resident (78 KB)
  __host__ __device__ static constexpr int b(int i) { return i == 0 ? 16 : 24; }
};
template <> struct WidePhases<16, 32> {  // targets 16..31 after a 128-column first launch
  // one resident phase: the 752 fragments (188 KB) stay in shared memory for the whole launch,
  // instead of four phases re-streamed from L2 for every row group (n=256: 13.46 -> 11.96 ms)
  static constexpr int P = 1, MAXF = 752;
  __host__ __device__ static constexpr int b(int i) { return i == 0 ? 16 : 32; }
};
// n in (256, 512]: targets 32..63 in launches whose fragments stay resident (<= 206 KB each)
#define SCQR3_RESIDENT_RANGE(B0, B1)                                                            \
  template <> struct WidePhases<B0, B1> {                                                       \
    static constexpr int P = 1, MAXF = B1 * (B1 - 1) - B0 * (B0 - 1);                           \
    __host__ __device__ static constexpr int b(int i) { return i == 0 ? B0 : B1; }              \
  };
// targets 16..17 / 16..19 / 16..21 (n <= 144 / 160 / 176) and 16..27 (n in (192, 224]): only the
// blocks below n
SCQR3_RESIDENT_RANGE(16, 18)
SCQR3_RESIDENT_RANGE(16, 20)
SCQR3_RESIDENT_RANGE(16, 22)
SCQR3_RESIDENT_RANGE(16, 28)
SCQR3_RESIDENT_RANGE(32, 40)
SCQR3_RESIDENT_RANGE(40, 48)
SCQR3_RESIDENT_RANGE(48, 56)
SCQR3_RESIDENT_RANGE(56, 60)
SCQR3_RESIDENT_RANGE(60, 64)
#undef SCQR3_RESIDENT_RANGE
template <> struct WidePhases<32, 64> {  // targets 32..63 (greedy, <= MAXF fragments per phase)
  static constexpr int P = 10, MAXF = 370;
  __host__ __device__ static constexpr int b(int i) {
    return i == 0 ? 32 : i == 1 ? 37 : i == 2 ? 41 : i == 3 ? 45 : i == 4 ? 48 : i == 5 ? 51
         : i == 6 ? 54 : i == 7 ? 57 : i == 8 ? 60 : i == 9 ? 62 : 64;
  }
};
template <int TB, int TE> constexpr bool phases_ok(int i = 0) {
  using W = WidePhases<TB, TE>;
  return i == W::P || (phase_frags(W::b(i), W::b(i + 1)) <= W::MAXF && W::b(W::P) == TE && phases_ok<TB, TE>(i + 1));
}
static_assert(phases_ok<0, 32>() && phases_ok<16, 24>() && phases_ok<16, 32>() && phases_ok<32, 64>() &&
                  phases_ok<16, 18>() && phases_ok<16, 20>() && phases_ok<16, 22>() && phases_ok<16, 28>() &&
                  phases_ok<32, 40>() && phases_ok<40, 48>() && phases_ok<48, 56>() && phases_ok<56, 60>() &&
                  phases_ok<60, 64>(),
              "phase fragment counts exceed the buffers");

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// One phase of the wide TRSM for one warp's 8A rows (fragment a: rows 8a + g); every register
// index is compile-time.  q[a][k] holds target block TB + k; qe[a] points at this lane's row of
// the finished Q (blocks < TB).
template <int TB, int TE, int PH, int A, bool INV>
__device__ __forceinline__ void wide_phase(double (&q)[A][TE - TB][2], const double* __restrict__ cur,
                                           const double* __restrict__ db, int lane, int t, const bool (&rok)[A],
                                           const long long (&row)[A], const double* const (&qe)[A],
                                           const TrsmParams& p) {
  constexpr int K0 = WidePhases<TB, TE>::b(PH), K1 = WidePhases<TB, TE>::b(PH + 1);
  auto frag = [&](int K, int s) { return cur[(K * (K - 1) - K0 * (K0 - 1) + s) * 32 + lane]; };
  // (i-a) updates from the blocks of the previous launch (finished Q columns, read back)
  if (TB > 0) {
    double av[A][8];
#pragma unroll
    for (int a = 0; a < A; ++a)
#pragma unroll
      for (int i = 0; i < 8; ++i)
        av[a][i] = __ldg(qe[a] + static_cast<long long>(8 * (i >> 1) + 2 * t + (i & 1)) * p.ldq);
#pragma unroll 1
    for (int sb = 0; sb < 2 * TB; sb += 8) {
      double bv[A][8];
      const int sn = sb + 8 < 2 * TB ? sb + 8 : sb;  // (last batch reloads itself, harmless)
#pragma unroll
      for (int a = 0; a < A; ++a)
#pragma unroll
        for (int i = 0; i < 8; ++i)
          bv[a][i] = __ldg(qe[a] + static_cast<long long>(8 * ((sn + i) >> 1) + 2 * t + (i & 1)) * p.ldq);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int K = K0; K < K1; ++K) {
          const double b = frag(K, sb + i);
#pragma unroll
          for (int a = 0; a < A; ++a) dmma(q[a][K - TB][0], q[a][K - TB][1], av[a][i], b);
        }
#pragma unroll
      for (int a = 0; a < A; ++a)
#pragma unroll
        for (int i = 0; i < 8; ++i) av[a][i] = bv[a][i];
    }
  }
  auto upd = [&](int K, int src, int s) {  // C_K += Q_src(k-step s) (-R~ fragment), all fragments
    const double b = frag(K, s);
#pragma unroll
    for (int a = 0; a < A; ++a) dmma(q[a][K - TB][0], q[a][K - TB][1], q[a][src - TB][s & 1], b);
  };
  // (i-b) updates from the blocks of earlier phases of this launch: target K0's here; target
  // J+1's run inside block J's diagonal chain below (a dependency-free DMMA stream that hides the
  // chain's shuffle / DFMA latency; one accumulator chain per warp keeps the pipe ~94 % busy at
  // two warps per sub-partition, tools/dmma_pattern.cu)
  constexpr int NS = 2 * (K0 - TB);  // k-steps per target from earlier phases
#pragma unroll
  for (int s = 2 * TB; s < 2 * K0; ++s) upd(K0, s >> 1, s);
  // (ii) triangular part inside the phase (right-looking, as in trsm_kernel)
#pragma unroll
  for (int J = K0; J < K1; ++J) {
    if (J > K0) {
#pragma unroll
      for (int s = 2 * (J - 1); s < 2 * J; ++s) upd(J, J - 1, s);
    }
    const int nup = J > K0 ? K1 - 1 - J : 0;
    const double* D = db + (J - TB) * (INV ? 64 : 72);
    auto interleave = [&](int c) {
#pragma unroll
      for (int u = nup * c / 8; u < nup * (c + 1) / 8; ++u) {
#pragma unroll
        for (int s = 2 * (J - 1); s < 2 * J; ++s) upd(J + 1 + u, J - 1, s);
      }
      if (J + 1 < K1) {
#pragma unroll
        for (int v = 2 * TB + NS * c / 8; v < 2 * TB + NS * (c + 1) / 8; ++v) upd(J + 1, v >> 1, v);
      }
    };
    if constexpr (INV) {
      // reading D24: q_J = b_J Y_J, two DMMA k-steps (as in trsm_kernel), between the updates
      static_assert(!INV || A == 2, "wide inverse instances: A = 2");
      const double y0 = D[lane], y1 = D[32 + lane];
      double acc[A][2];
#pragma unroll
      for (int a = 0; a < A; ++a) acc[a][0] = acc[a][1] = 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c == SCQR3_INV_K0) {
#pragma unroll
          for (int a = 0; a < A; ++a) dmma(acc[a][0], acc[a][1], q[a][J - TB][0], y0);
        }
        if (c == SCQR3_INV_K1) {
#pragma unroll
          for (int a = 0; a < A; ++a) dmma(acc[a][0], acc[a][1], q[a][J - TB][1], y1);
        }
        interleave(c);
      }
#pragma unroll
      for (int a = 0; a < A; ++a) {
        q[a][J - TB][0] = acc[a][0];
        q[a][J - TB][1] = acc[a][1];
      }
    } else if constexpr (A == 2) {
      // rows g and g+8: the pair swap of trsm_kernel (lane u = t&1 of each half-quad holds
      // columns {2u, 2u+1, 2u+4, 2u+5} of one row; 18 DFMA per block instead of 28)
      const int uu = t & 1;
      const bool lo = t < 2;
      double V[4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double snd = lo ? q[1][J - TB][h] : q[0][J - TB][h];
        const double rcv = __shfl_xor_sync(0xffffffffu, snd, 2);
        V[h] = lo ? q[0][J - TB][h] : rcv;
        V[2 + h] = lo ? rcv : q[1][J - TB][h];
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < 7) {
          const double2 r01 = *reinterpret_cast<const double2*>(D + c * 8 + 2 * uu);
          const double2 r23 = *reinterpret_cast<const double2*>(D + c * 8 + 4 + 2 * uu);
          const double vc = __shfl_sync(0xffffffffu, V[(c & 1) + 2 * (c >> 2)], (lane & ~1) | ((c >> 1) & 1));
          if (c < 2) V[0] = fma(-vc, r01.x, V[0]);
          if (c < 3) V[1] = fma(-vc, r01.y, V[1]);
          if (c < 6) V[2] = fma(-vc, r23.x, V[2]);
          V[3] = fma(-vc, r23.y, V[3]);
        }
        interleave(c);
      }
      const double2 i01 = *reinterpret_cast<const double2*>(D + 64 + 2 * uu);
      const double2 i23 = *reinterpret_cast<const double2*>(D + 64 + 4 + 2 * uu);
      V[0] *= i01.x;
      V[1] *= i01.y;
      V[2] *= i23.x;
      V[3] *= i23.y;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double snd = lo ? V[2 + h] : V[h];
        const double rcv = __shfl_xor_sync(0xffffffffu, snd, 2);
        q[0][J - TB][h] = lo ? V[h] : rcv;
        q[1][J - TB][h] = lo ? rcv : V[2 + h];
      }
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < 7) {  // (column 7 updates nothing inside its block)
          const double2 rc = *reinterpret_cast<const double2*>(D + c * 8 + 2 * t);
          const double vc = __shfl_sync(0xffffffffu, q[0][J - TB][c & 1], (lane & ~3) | (c >> 1));
          q[0][J - TB][0] = fma(-vc, rc.x, q[0][J - TB][0]);
          q[0][J - TB][1] = fma(-vc, rc.y, q[0][J - TB][1]);
        }
        interleave(c);
      }
      const double2 ri = *reinterpret_cast<const double2*>(D + 64 + 2 * t);
      q[0][J - TB][0] *= ri.x;
      q[0][J - TB][1] *= ri.y;
    }
#pragma unroll
    for (int a = 0; a < A; ++a) {
      if (rok[a]) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 8 * J + 2 * t + h;
          if (col < p.n) __stcs(p.Q + row[a] + static_cast<long long>(col) * p.ldq, q[a][J - TB][h]);
        }
      }
    }
  }
}

// Phases PH.. of one row group: phase PH computes from buffer PH&1 while phase PH+1 (or, after
// the last phase, the next row group's phase 0) streams into the other one.
template <int TB, int TE, int PH, int A, bool INV, typename Stage>
__device__ __forceinline__ void wide_phases(double (&q)[A][TE - TB][2], double* const (&buf)[2],
                                            const double* db, int lane, int t, bool act, const bool (&rok)[A],
                                            const long long (&row)[A], const double* const (&qe)[A],
                                            const TrsmParams& p, bool more, Stage& stage) {
  constexpr int P = WidePhases<TB, TE>::P;
  if constexpr (P == 1) {  // resident fragments (staged once per launch): no staging, no barrier
    if (act) wide_phase<TB, TE, 0, A, INV>(q, buf[0], db, lane, t, rok, row, qe, p);
    return;
  }
  if constexpr (PH + 1 < P) stage(PH + 1, buf[(PH + 1) & 1]);
  else if ((P - 1) & 1) { if (more) stage(0, buf[0]); }  // buf[0] is free during an odd last phase
  if (act) wide_phase<TB, TE, PH, A, INV>(q, buf[PH & 1], db, lane, t, rok, row, qe, p);
  cp_async_wait_all();
  __syncthreads();
  if constexpr (PH + 1 < P) {
    wide_phases<TB, TE, PH + 1, A, INV>(q, buf, db, lane, t, act, rok, row, qe, p, more, stage);
  } else if (!((P - 1) & 1)) {  // even last phase used buf[0]: stage the next phase 0 now
    if (more) {
      stage(0, buf[0]);
      cp_async_wait_all();
      __syncthreads();
    }
  }
}

template <int TB, int TE, int THREADS, int A, bool INV = false>
__global__ void __launch_bounds__(THREADS, 1) trsm_wide_kernel(TrsmParams p) {
  constexpr int NTT = TE - TB, WPB = THREADS / 32, MAXF = WidePhases<TB, TE>::MAXF;
  extern __shared__ __align__(16) double smp[];
  if (SCQR3_GATE_SKIP(p.gate) || (p.st && p.st->code != 0)) return;
  if (INV ? !(p.inv_flag && *p.inv_flag > 0.0) : (p.inv_flag && *p.inv_flag > 0.0)) return;  // reading D24
  constexpr int NBUF = WidePhases<TB, TE>::P == 1 ? 1 : 2;
  double* const buf[2] = {smp, smp + (NBUF - 1) * MAXF * 32};
  double* const db = smp + NBUF * MAXF * 32;
  if (INV) {
    for (int i = threadIdx.x; i < NTT * 64; i += THREADS) db[i] = p.dinv[TB * 64 + i];
  } else {
    for (int i = threadIdx.x; i < NTT * 72; i += THREADS) db[i] = p.dblk[TB * 72 + i];
  }
  auto stage = [&](int ph, double* dst) {  // cooperative cp.async of phase ph's fragments
    const int k0 = WidePhases<TB, TE>::b(ph), k1 = WidePhases<TB, TE>::b(ph + 1);
    const double* src = p.bfrag + static_cast<size_t>(k0) * (k0 - 1) * 32;
    const int chunks = phase_frags(k0, k1) * 32 / 2;  // 16-byte chunks
    for (int c = threadIdx.x; c < chunks; c += THREADS) cp_async16(dst + 2 * c, src + 2 * c);
    cp_async_commit();
  };
  stage(0, buf[0]);
  cp_async_wait_all();
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const long long m = p.m;
  const int n = p.n;
  const long long ngroups = (m + 8 * A - 1) / (8 * A);
  const long long stride = static_cast<long long>(gridDim.x) * WPB;
  for (long long base = static_cast<long long>(blockIdx.x) * WPB; base < ngroups; base += stride) {
    const long long rg = base + warp;
    const bool act = rg < ngroups;
    long long row[A];
    bool rok[A];
    const double* qe[A];
#pragma unroll
    for (int a = 0; a < A; ++a) {
      row[a] = rg * 8 * A + 8 * a + g;
      rok[a] = act && row[a] < m;
      qe[a] = p.Q + (rok[a] ? row[a] : 0);
    }
    double q[A][NTT][2];
#pragma unroll
    for (int a = 0; a < A; ++a)
#pragma unroll
      for (int J = 0; J < NTT; ++J)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 8 * (TB + J) + 2 * t + h;
          q[a][J][h] = (rok[a] && col < n) ? __ldcs(p.X + row[a] + static_cast<long long>(col) * p.ldx) : 0.0;
        }
    wide_phases<TB, TE, 0, A, INV>(q, buf, db, lane, t, act, rok, row, qe, p, base + stride < ngroups, stage);
  }
}

template <int TB, int TE, int THREADS, int A = 1, bool INV = false>
static cudaError_t launch_wide1(const TrsmParams& p, int num_sms, cudaStream_t stream) {
  const size_t smem =
      static_cast<size_t>((WidePhases<TB, TE>::P == 1 ? 1 : 2) * WidePhases<TB, TE>::MAXF * 32 + (TE - TB) * 72) * 8;
  auto k = trsm_wide_kernel<TB, TE, THREADS, A, INV>;
  static thread_local LaunchCfgCache cfg;
  cudaError_t e = cached_launch_cfg(cfg, k, smem, THREADS, nullptr);
  if (e != cudaSuccess) return e;
  const long long groups = (p.m + 8 * A - 1) / (8 * A);
  long long grid = num_sms;
  const long long need = (groups + THREADS / 32 - 1) / (THREADS / 32);
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  k<<<static_cast<unsigned>(grid), THREADS, smem, stream>>>(p);
  return cudaGetLastError();
}

// A = 2 instances launch an inverse-diagonal twin when p.inv_flag is set (reading D24)
template <int TB, int TE, int THREADS, int A = 1>
static cudaError_t launch_wide(const TrsmParams& p, int num_sms, cudaStream_t stream) {
  if constexpr (A == 2) {
    if (p.inv_flag) {
      cudaError_t e = launch_wide1<TB, TE, THREADS, A, true>(p, num_sms, stream);
      if (e != cudaSuccess) return e;
    }
    return launch_wide1<TB, TE, THREADS, A, false>(p, num_sms, stream);
  } else {
    TrsmParams ps = p;
    ps.inv_flag = nullptr;
    return launch_wide1<TB, TE, THREADS, A, false>(ps, num_sms, stream);
  }
}

// Width of the TMA box of X that launch_trsm expects for NT column tiles (host: encode_map).
int trsm_x_box_cols(int NT) { return NT >= 24 ? 128 : NT * 8; }

// Kernel launches launch_trsm issues for p (the inverse-diagonal instance counts as a launch
// even when the guard lets it exit at entry).
int trsm_launch_count(const TrsmParams& p, bool tma) {
  const int NT = npad_for(p.n) / 8;
  const int k = p.inv_flag ? 2 : 1;  // an A = 2 / TMA instance launches with its inverse twin
  if (p.gram_partials) return NT == 8 ? k : 1;
  switch (NT) {
    case 8: return 1;
    case 12: case 16: return tma ? k : 1;
    case 24: case 32: return tma ? 2 * k : 1;
    case 64: {
      const int first = tma ? 2 * k : 1;  // columns 0..255
#ifdef SCQR3_WIDE512_PHASED
      return first + 1;
#else
      const int nb = (p.n + 7) / 8;
      return first + k * (1 + (nb > 40) + (nb > 48) + (nb > 56) + (nb > 60));
#endif
    }
    default: return 1;
  }
}

// map: TMA descriptor of X with a {16 rows, npad columns} SWIZZLE_128B box (instances with
// NT <= 16 use it when map != nullptr; NT >= 24: a {16, 128} box of the first 128 columns); the
// others read X with plain coalesced loads.
cudaError_t launch_trsm(const TrsmParams& p, const CUtensorMap* map, int num_sms, cudaStream_t stream,
                        int* grid_out, const CUtensorMap* mapQ) {
  const int NT = npad_for(p.n) / 8;
  const bool tma = map != nullptr;
  // instances with inverse diagonal blocks (reading D24): n in (32, 128] through the TMA path and
  // the first 128 columns of n > 128; everything else substitutes
  TrsmParams ps = p;
  ps.inv_flag = nullptr;
  if (p.gram_partials) {  // fused TRSM + next-pass Gram (A = 2, TMA)
    if (!tma || !mapQ) return cudaErrorInvalidValue;
    switch (NT) {
      case 1: return launch_one<1, 2, true, 256, true, true>(ps, map, num_sms, stream, grid_out, mapQ);
      case 2: return launch_one<2, 2, true, 256, true, true>(ps, map, num_sms, stream, grid_out, mapQ);
      case 4: return launch_one<4, 2, true, 256, true, true>(ps, map, num_sms, stream, grid_out, mapQ);
      case 8: return launch_pair<8, 2, true, 256, true, true>(p, map, num_sms, stream, grid_out, mapQ);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (NT) {
    case 1: return launch_one<1, 4, true, 256, false>(ps, nullptr, num_sms, stream);
    case 2: return tma ? launch_one<2, 4, true, 256, true>(ps, map, num_sms, stream)
                       : launch_one<2, 4, true, 256, false>(ps, nullptr, num_sms, stream);
    case 4: return tma ? launch_one<4, 4, true, 256, true>(ps, map, num_sms, stream)
                       : launch_one<4, 4, true, 256, false>(ps, nullptr, num_sms, stream);
    // (n in (32, 64] unfused -- the oblique n = 64 -- substitutes: its A = 4 inverse twin measured
    //  slower, C5 TRSM 0.424 -> 0.435 ms; the fused n <= 64 instance above has one)
    case 8: return tma ? launch_one<8, 4, true, 256, true>(ps, map, num_sms, stream)
                       : launch_one<8, 4, true, 256, false>(ps, nullptr, num_sms, stream);
    case 12: return tma ? launch_pair<12, 2, true, 256, true>(p, map, num_sms, stream)
                        : launch_one<12, 2, true, 256, false>(ps, nullptr, num_sms, stream);
    case 16: return tma ? launch_pair<16, 2, true, 256, true>(p, map, num_sms, stream)
                        : launch_one<16, 2, true, 256, false>(ps, nullptr, num_sms, stream);
    case 24: {
      // split as for NT = 32: columns 0..127, then targets 16..23 (A = 2)
      if (!map) return launch_one<24, 1, true, 256, false>(ps, nullptr, num_sms, stream);
      TrsmParams p1 = p;
      p1.n = 128;
      cudaError_t e = launch_pair<16, 2, true, 256, true>(p1, map, num_sms, stream);
      if (e != cudaSuccess) return e;
      // only the target blocks below n (n = 136: one of the eight)
      const int nb = (p.n + 7) / 8;
      if (nb <= 18) return launch_wide<16, 18, 256, 2>(p, num_sms, stream);
      if (nb <= 20) return launch_wide<16, 20, 256, 2>(p, num_sms, stream);
      if (nb <= 22) return launch_wide<16, 22, 256, 2>(p, num_sms, stream);
      return launch_wide<16, 24, 256, 2>(p, num_sms, stream);
    }
    case 32: {
      // block-column split: columns 0..127 by the register-resident kernel (map: a 128-column
      // box), then targets 16..31 by the wide kernel with 16 rows per warp (A = 2: 16 target
      // blocks x 2 fragments in registers, the pair-swap diagonal solve), its updates from
      // Q(:, 0:128) read back.  n = 256 at m = 5e6: 13.45 ms, against 13.84 ms with A = 1 at 16
      // warps and 14.3 ms for one wide launch over all 32 targets.
      if (!map) return launch_wide<0, 32, 256>(p, num_sms, stream);
      TrsmParams p1 = p;
      p1.n = 128;
      cudaError_t e = launch_pair<16, 2, true, 256, true>(p1, map, num_sms, stream);
      if (e != cudaSuccess) return e;
      if ((p.n + 7) / 8 <= 28) return launch_wide<16, 28, 256, 2>(p, num_sms, stream);
      return launch_wide<16, 32, 256, 2>(p, num_sms, stream);
    }
    case 64: {
      // block-column TRSM: Q(:, 0:256) first (split as for NT = 32); the last launch reads it
      // back for its updates
      cudaError_t e;
      if (map) {
        TrsmParams p1 = p;
        p1.n = 128;
        e = launch_pair<16, 2, true, 256, true>(p1, map, num_sms, stream);
        if (e != cudaSuccess) return e;
        e = launch_wide<16, 32, 256, 2>(p, num_sms, stream);
      } else {
        e = launch_wide<0, 32, 256>(p, num_sms, stream);
      }
      if (e != cudaSuccess) return e;
#ifdef SCQR3_WIDE512_PHASED
      return launch_wide<32, 64, 256>(p, num_sms, stream);
#else
      // targets 32..63 in five launches with resident fragments, each reading Q(:, 0:8 TB) back;
      // launches whose targets lie wholly in the padding past n are skipped (so every column
      // read back is < n: TB < ceil(n / 8) gives 8 TB < n)
      const int nb = (p.n + 7) / 8;
      if ((e = launch_wide<32, 40, 256, 2>(p, num_sms, stream)) != cudaSuccess) return e;
      if (nb > 40 && (e = launch_wide<40, 48, 256, 2>(p, num_sms, stream)) != cudaSuccess) return e;
      if (nb > 48 && (e = launch_wide<48, 56, 256, 2>(p, num_sms, stream)) != cudaSuccess) return e;
      if (nb > 56 && (e = launch_wide<56, 60, 256, 2>(p, num_sms, stream)) != cudaSuccess) return e;
      if (nb > 60) return launch_wide<60, 64, 256, 2>(p, num_sms, stream);
      return cudaSuccess;
#endif
    }
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace scqr3
