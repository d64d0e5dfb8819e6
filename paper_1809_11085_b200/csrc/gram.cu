// gram.cu -- Gram matrix kernels (step a1 / a1b of the hot path).
//
//   A = Q^T Q            (eq. (1); Alg. 1 line 1 P:137; Alg. 2 line 3 P:678; Alg. 3)
//   A = sym(Q^T (B Q))   (Alg. 4 line 1 P:878; symmetrised as in S:262; every pass, reading D8)
//
// Design: split-m persistent CTAs.  One producer warp streams 16-row
// x npad-column stages of Q (and of Y = BQ for the oblique Gram) from HBM into shared memory
// with 2-D TMA (SWIZZLE_128B, mbarrier pipeline).  Each consumer warp owns one 32x32 block
// ("job", 4x4 tiles of 8x8) of the upper triangle of A (all blocks for the oblique Gram) and
// accumulates it in registers with FP64 tensor-core MMA (mma.sync m8n8k4 f64 = SASS DMMA).
// The k-index of each m8n8k4 step is mapped to rows {2s, 2s+1, 2s+8, 2s+9} of the stage so
// that fragment loads from the swizzled stage are bank-conflict free.  Each CTA writes its
// partial tiles to the workspace; gram_reduce sums the partials in CTA order, so the result
// is bitwise deterministic run to run for a fixed GPU model and grid (reading D10).
#include <type_traits>
#include "scqr3_dev.cuh"
#include "scqr3_kernels.h"

namespace scqr3 {

// Job j -> (bi, bj) block coordinates.  Symmetric: upper blocks enumerated column by column
// (bi <= bj).  Full (oblique): row-major over NB x NB.
__device__ __forceinline__ void decode_job(int j, int NB, bool full, int& bi, int& bj) {
  if (full) {
    bi = j / NB;
    bj = j % NB;
    return;
  }
  int c = 0;
  while ((c + 1) * (c + 2) / 2 <= j) ++c;
  bj = c;
  bi = j - c * (c + 1) / 2;
}

// Whole-block jobs (JR = 4): one stage loop per job kind, so only that kind's state is live
// (18 consumer warps fit 96 registers).  Fragment address of k-step s: the lane's 16-byte chunk
// is (s + 4*(t>>1)) ^ g = s ^ G, i.e. offset ^ (s << 4) on a 128-byte aligned row base; the
// block's tile rows / columns sit 8 x 128 B apart (immediate offsets).
template <bool MC, int RB>
__device__ __forceinline__ void gram_whole_jobs(const GramParams& p, const unsigned char* stages, uint32_t stage_bytes,
                                                int nsrc, uint64_t* full_bar, uint64_t* empty_bar, int nst, int kind,
                                                bool b_from_y, bool full, int bi, int bj, bool diag,
                                                double (&acc)[4][kJobTiles][2], const uint32_t (&offA)[4],
                                                const uint32_t (&offB)[kJobTiles], const uint32_t (&innerR)[RB][4]) {
  const int lane = threadIdx.x & 31;
  constexpr uint32_t TS = 1024u * RB;  // bytes between tile rows / columns (8 columns x RB lines)
  auto release = [&](uint64_t* bar) {  // this stage consumed: in every CTA of the cluster (multicast)
    if constexpr (MC) {
      for (int j = 0; j < p.mc; ++j) mbar_arrive_cluster(bar, static_cast<uint32_t>(j));
    } else {
      mbar_arrive(bar);
    }
  };
  auto frag = [&](uint32_t off) { return *reinterpret_cast<const double*>(stages + off); };
  // each stage holds RB 16-row blocks (line rb of a column at +rb*128); lane_chunk(rb): chunk G
  // << 4 plus the 8-byte half of this lane's k slot for that block's swizzle key
  uint32_t lane_chunk;
  auto stage_loop = [&](auto body) {
    int st = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nst; ++i) {
      mbar_wait(&full_bar[st], ph);
      const uint32_t oA = static_cast<uint32_t>(st) * nsrc * stage_bytes;
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) {
        lane_chunk = innerR[rb][0];
        body(oA + rb * 128u, (b_from_y ? oA + stage_bytes : oA) + rb * 128u);
      }
      __syncwarp();
      if (lane == 0) release(&empty_bar[st]);
      if (++st == p.stages) {
        st = 0;
        ph ^= 1u;
      }
    }
  };
  if (kind == 0) {
    // 4 x 4 tiles of an off-diagonal block: 8 fragment loads, 16 DMMA per k-step
    stage_loop([&](uint32_t oA, uint32_t oB) {
      const uint32_t a0 = offA[0] + lane_chunk, b0 = offB[0] + lane_chunk;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const uint32_t xa = (oA + a0) ^ (s << 4), xb = (oB + b0) ^ (s << 4);
        double fb[kJobTiles];
#pragma unroll
        for (int b = 0; b < kJobTiles; ++b) fb[b] = frag(xb + b * TS);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const double fa = frag(xa + a * TS);
#pragma unroll
          for (int b = 0; b < kJobTiles; ++b) dmma(acc[a][b][0], acc[a][b][1], fa, fb[b]);
        }
      }
    });
  } else if (kind == 1) {
    // diagonal block: its 10 upper tiles (A fragments = B fragments for Q^T Q; from Q for Q^T Y)
    stage_loop([&](uint32_t oA, uint32_t oB) {
      const uint32_t b0 = offB[0] + lane_chunk;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const uint32_t xa = (oA + b0) ^ (s << 4), xb = (oB + b0) ^ (s << 4);
        double fb[kJobTiles], fa[4];
#pragma unroll
        for (int b = 0; b < kJobTiles; ++b) fb[b] = frag(xb + b * TS);
#pragma unroll
        for (int a = 0; a < 4; ++a) fa[a] = full ? frag(xa + a * TS) : fb[a];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = a; b < kJobTiles; ++b) dmma(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
      }
    });
  } else if (kind == 3) {
    // a block of the last block column when NT % 4 != 0: cb = NT - 4 bj < 4 valid tile columns
    // (an off-diagonal edge block has all four tile rows, the diagonal one a <= b < cb).
    // Specialised on cb so that no DMMA is issued for a padded tile -- predicated-off DMMAs
    // still take their issue slots (n = 144 ran 25 % slower than n = 160 that way)
    auto edge = [&](auto cbc) {
      constexpr int CB = decltype(cbc)::value;
      if (diag) {
        stage_loop([&](uint32_t oA, uint32_t oB) {
          const uint32_t a0 = offA[0] + lane_chunk, b0 = offB[0] + lane_chunk;
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const uint32_t xa = (oA + a0) ^ (s << 4), xb = (oB + b0) ^ (s << 4);
            double fb[CB], fa[CB];
#pragma unroll
            for (int b = 0; b < CB; ++b) fb[b] = frag(xb + b * TS);
#pragma unroll
            for (int a = 0; a < CB; ++a) fa[a] = full ? frag(xa + a * TS) : fb[a];
#pragma unroll
            for (int a = 0; a < CB; ++a)
#pragma unroll
              for (int b = a; b < CB; ++b) dmma(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
          }
        });
      } else {
        stage_loop([&](uint32_t oA, uint32_t oB) {
          const uint32_t a0 = offA[0] + lane_chunk, b0 = offB[0] + lane_chunk;
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const uint32_t xa = (oA + a0) ^ (s << 4), xb = (oB + b0) ^ (s << 4);
            double fb[CB];
#pragma unroll
            for (int b = 0; b < CB; ++b) fb[b] = frag(xb + b * TS);
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              const double fa = frag(xa + a * TS);
#pragma unroll
              for (int b = 0; b < CB; ++b) dmma(acc[a][b][0], acc[a][b][1], fa, fb[b]);
            }
          }
        });
      }
    };
    const int cb = p.NT - bj * kJobTiles;
    if (cb == 1) edge(std::integral_constant<int, 1>{});
    else if (cb == 2) edge(std::integral_constant<int, 2>{});
    else edge(std::integral_constant<int, 3>{});
  } else {
    stage_loop([&](uint32_t, uint32_t) {});  // idle warp: release the stages
  }
}

// RB: 16-row blocks per stage.  RB = 2 streams 32-row stages through a 3-D view of Q
// (16 rows, 16-row blocks, columns): one box fetches 256 contiguous bytes per column while each
// 128-B line keeps the SWIZZLE_128B layout -- 7.3 TB/s of TMA reads against 4.6 TB/s for 16-row
// 2-D boxes (tools/tma_probe.cu); taken for m % 32 == 0 without multicast.
template <int JR, int MAXC, bool MC, int RB = 1>
__global__ void __launch_bounds__(32 * (MAXC + 1), 1)
    gram_tma_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapY,
                    GramParams p) {
  static_assert(RB == 1 || !MC, "32-row stages: unclustered only");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  if (SCQR3_GATE_SKIP(p.gate)) return;  // speculative pass after a stop / error (device-side pass control)
  // 1024-B alignment for SWIZZLE_128B
  // (pointer arithmetic on the shared array itself keeps the shared address space -> LDS)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncons = blockDim.x / 32 - 1;
  const int group = blockIdx.x % p.groups;
  const int chunk = blockIdx.x / p.groups;
  const bool full = p.oblique != 0;
  const int nsrc = full ? 2 : 1;
  const uint32_t stage_bytes = static_cast<uint32_t>(p.npad) * 128u * RB;   // 16 RB rows x npad cols x 8 B
  unsigned char* stages = smem;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(p.stages) * nsrc * stage_bytes);
  uint64_t* empty_bar = full_bar + p.stages;

  // contiguous row range of this chunk, in 16-row stages
  const long long s_begin = (long long)p.total_stages * chunk / p.chunks;
  const long long s_end = (long long)p.total_stages * (chunk + 1) / p.chunks;
  const int nst = static_cast<int>(s_end - s_begin);

  // multicast (p.mc > 1): the CTAs of a chunk form a cluster; every stage lands in all of them
  // from one L2 read (each CTA issues 1 / mc of the stage's boxes to the whole cluster), and a
  // stage is refilled only after the consumers of every CTA released it (remote arrivals)
  constexpr bool mc = MC;  // (a template parameter: the runtime branches cost 2-7 % unclustered)
  const uint32_t crank = mc ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < p.stages; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], ncons * (mc ? p.mc : 1));
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (mc) cluster_sync();  // every CTA's barriers are initialised before any remote use

  if (warp == 0) {
    // ---------------- producer: TMA stream of this chunk's rows
    if (lane == 0) {
      tma_prefetch_desc(&mapQ);
      if (full) tma_prefetch_desc(&mapY);
      const uint16_t mask = static_cast<uint16_t>((1u << p.mc) - 1u);
      int st = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nst; ++i, ++st) {
        if (st == p.stages) {
          st = 0;
          ph ^= 1u;
        }
        if (i >= p.stages) {
          if (mc) mbar_wait_cluster(&empty_bar[st], ph ^ 1);
          else mbar_wait(&empty_bar[st], ph ^ 1);
        }
        mbar_arrive_expect_tx(&full_bar[st], stage_bytes * nsrc);
        const int row = static_cast<int>((s_begin + i) * kGramStageRows * RB);
        unsigned char* dst = stages + static_cast<size_t>(st) * nsrc * stage_bytes;
        if constexpr (RB > 1) {  // 3-D boxes {16 rows, RB blocks, box_cols}: [column][block][16 rows]
          for (int c0 = 0; c0 < p.npad; c0 += p.box_cols) {
            tma_load_3d(dst + c0 * 128u * RB, &mapQ, 0, row / 16, c0, &full_bar[st]);
            if (full) tma_load_3d(dst + stage_bytes + c0 * 128u * RB, &mapY, 0, row / 16, c0, &full_bar[st]);
          }
          continue;
        }
        // a TMA box spans at most 256 columns: wider stages take several boxes (npad 512)
        if (mc) {
          for (int c0 = static_cast<int>(crank) * p.box_cols; c0 < p.npad; c0 += p.mc * p.box_cols) {
            tma_load_2d_multicast(dst + c0 * 128u, &mapQ, row, c0, &full_bar[st], mask);
            if (full) tma_load_2d_multicast(dst + stage_bytes + c0 * 128u, &mapY, row, c0, &full_bar[st], mask);
          }
        } else {
          for (int c0 = 0; c0 < p.npad; c0 += p.box_cols) {
            tma_load_2d(dst + c0 * 128u, &mapQ, row, c0, &full_bar[st]);
            if (full) tma_load_2d(dst + stage_bytes + c0 * 128u, &mapY, row, c0, &full_bar[st]);
          }
        }
      }
    }
    if (mc) {
      __syncwarp();
      cluster_sync();  // (matches the consumers' final cluster barrier)
    }
    return;
  }

  // ---------------- consumers (job table: host-balanced over the four SM sub-partitions)
  // JR = 2: every job is one "part": two tile rows (rows 2*part, 2*part+1 of the 4x4-tile block)
  // by the block's four tile columns -- 8 DMMA per k-step for an off-diagonal block, 7 (top) or
  // 3 (bottom) for a diagonal block of the symmetric Gram.  Small parts keep the accumulators at
  // 32 registers and let the host balance the sub-partitions exactly.
  // JR = 4 (more blocks than one CTA's warps hold as parts, n > 128): every job is a whole
  // block -- 16 DMMA per 8 fragment loads off the diagonal, 10 on it -- so half as many CTAs
  // share (and re-read) each row chunk.
  const int cw = warp - 1;
  const int code = p.warp_job[group * kMaxConsumers + cw];  // 2 * block + part, -1 = idle
  const bool active = code >= 0;
  const int part = active ? (code & 1) : 0;
  int bi = 0, bj = 0;
  // the oblique Gram is also computed on the upper blocks only: A = upper(Q^T (BQ)), mirrored
  // (reading D22); its diagonal tiles take the A fragments from Q and the B fragments from Y
  // dual (oblique): jobs past the B-Gram's blocks form the plain Gram Q^T Q (B operand from Q)
  const int nblk = p.NB * (p.NB + 1) / 2;
  const bool plainjob = full && p.dual && active && (code >> 1) >= nblk;
  if (active) decode_job((code >> 1) - (plainjob ? nblk : 0), p.NB, false, bi, bj);
  const bool diag = bi == bj;
  const int NT = p.NT;
  const bool edge = (bi + 1) * kJobTiles > NT || (bj + 1) * kJobTiles > NT;
  const int rr0 = JR == 2 ? 2 * part : 0;  // first tile row of the job within the block
  const int g = lane >> 2, t = lane & 3;

  double acc[JR][kJobTiles][2];
#pragma unroll
  for (int a = 0; a < JR; ++a)
#pragma unroll
    for (int b = 0; b < kJobTiles; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  // per-lane smem offsets (without the k-step part) of the job's tile rows / the block's columns
  uint32_t offA[JR], offB[kJobTiles];
#pragma unroll
  for (int a = 0; a < JR; ++a) offA[a] = static_cast<uint32_t>(8 * min(bi * kJobTiles + rr0 + a, NT - 1) + g) * 128u * RB;
#pragma unroll
  for (int b = 0; b < kJobTiles; ++b) offB[b] = static_cast<uint32_t>(8 * min(bj * kJobTiles + b, NT - 1) + g) * 128u * RB;
  // 16-byte chunk of this lane's k slot per k-step s: rows {2s, 2s+1, 2s+8, 2s+9}[t] -> the
  // chunk index (row>>1) = s + 4*(t>>1) XOR (line & 7) (SWIZZLE_128B), conflict free; the line of
  // block rb of column 8 T + g is RB (8 T + g) + rb, so the key is (RB g + rb) & 7
  uint32_t innerR[RB][4];
#pragma unroll
  for (int rb = 0; rb < RB; ++rb)
#pragma unroll
    for (int s = 0; s < 4; ++s)
      innerR[rb][s] = ((((s + 4 * (t >> 1)) ^ ((RB * g + rb) & 7)) & 7u) << 4) + ((t & 1) << 3);
  // 0 off-diagonal interior, 1 diagonal top part (JR = 4: the whole diagonal block), 2 diagonal
  // bottom part, 3 edge, 4 idle
  const int kind = !active ? 4 : edge ? 3 : diag ? 1 + part : 0;

  if constexpr (JR == 4) {
    gram_whole_jobs<MC, RB>(p, stages, stage_bytes, nsrc, full_bar, empty_bar, nst, kind, full && !plainjob, full,
                            bi, bj, diag, acc, offA, offB, innerR);
  } else {
  int st = 0;
  uint32_t ph = 0;
  for (int i = 0; i < nst; ++i) {
    mbar_wait(&full_bar[st], ph);
    const unsigned char* stA = stages + static_cast<size_t>(st) * nsrc * stage_bytes;
    const unsigned char* stB = (full && !plainjob) ? stA + stage_bytes : stA;
#pragma unroll
    for (int rb = 0; rb < RB; ++rb) {  // the stage's 16-row blocks, in row order
    const unsigned char* srcA = stA + rb * 128u;
    const unsigned char* srcB = stB + rb * 128u;
    const uint32_t* inner = innerR[rb];
    if (kind == 0) {
      // 2 x 4 tiles of an off-diagonal block: 6 fragment loads, 8 DMMA per k-step
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        double fa[2], fb[kJobTiles];
#pragma unroll
        for (int a = 0; a < 2; ++a) fa[a] = *reinterpret_cast<const double*>(srcA + offA[a] + inner[s]);
#pragma unroll
        for (int b = 0; b < kJobTiles; ++b) fb[b] = *reinterpret_cast<const double*>(srcB + offB[b] + inner[s]);
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < kJobTiles; ++b) dmma(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
      }
    } else if (kind == 1) {
      // diagonal block, tile rows 0-1: tiles (0,0..3), (1,1..3); for Q^T Q the A fragments are
      // B fragments, for Q^T Y they come from the Q stage
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        double fb[kJobTiles], fa[2];
#pragma unroll
        for (int b = 0; b < kJobTiles; ++b) fb[b] = *reinterpret_cast<const double*>(srcB + offB[b] + inner[s]);
#pragma unroll
        for (int a = 0; a < 2; ++a) fa[a] = full ? *reinterpret_cast<const double*>(srcA + offB[a] + inner[s]) : fb[a];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = a; b < kJobTiles; ++b) dmma(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
      }
    } else if (kind == 2) {
      // diagonal block, tile rows 2-3: tiles (2,2), (2,3), (3,3)
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const double f2 = *reinterpret_cast<const double*>(srcB + offB[2] + inner[s]);
        const double f3 = *reinterpret_cast<const double*>(srcB + offB[3] + inner[s]);
        const double a2 = full ? *reinterpret_cast<const double*>(srcA + offB[2] + inner[s]) : f2;
        const double a3 = full ? *reinterpret_cast<const double*>(srcA + offB[3] + inner[s]) : f3;
        dmma(acc[0][2][0], acc[0][2][1], a2, f2);
        dmma(acc[0][3][0], acc[0][3][1], a2, f3);
        dmma(acc[1][3][0], acc[1][3][1], a3, f3);
      }
    } else if (kind == 3) {
      // part of a block of the last block column (NT % 4 != 0): cb valid tile columns, no DMMA
      // issued for a padded tile off the diagonal (see gram_whole_jobs); the diagonal edge block
      // keeps per-tile validity
      auto edge = [&](auto cbc) {
        constexpr int CB = decltype(cbc)::value;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          double fa[2], fb[CB];
#pragma unroll
          for (int a = 0; a < 2; ++a) fa[a] = *reinterpret_cast<const double*>(srcA + offA[a] + inner[s]);
#pragma unroll
          for (int b = 0; b < CB; ++b) fb[b] = *reinterpret_cast<const double*>(srcB + offB[b] + inner[s]);
          if (diag) {
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
              for (int b = 0; b < CB; ++b)
                if (rr0 + a <= b) dmma(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
          } else {
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
              for (int b = 0; b < CB; ++b) dmma(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
          }
        }
      };
      const int cb = NT - bj * kJobTiles;
      if (cb == 1) edge(std::integral_constant<int, 1>{});
      else if (cb == 2) edge(std::integral_constant<int, 2>{});
      else edge(std::integral_constant<int, 3>{});
    }
    }  // rb
    __syncwarp();
    if (lane == 0) {
      if (mc) {
        for (int j = 0; j < p.mc; ++j) mbar_arrive_cluster(&empty_bar[st], static_cast<uint32_t>(j));
      } else {
        mbar_arrive(&empty_bar[st]);
      }
    }
    if (++st == p.stages) {
      st = 0;
      ph ^= 1u;
    }
  }

  }  // JR == 2

  // no CTA of a cluster exits while a peer may still arrive on its barriers
  if (mc) cluster_sync();
  if (!active) return;
  // ---------------- write this CTA's partial tiles (8x8 row-major per tile)
  double* out = p.partials + static_cast<size_t>(chunk) * p.tiles_per_partial * 64;
#pragma unroll
  for (int a = 0; a < JR; ++a)
#pragma unroll
    for (int b = 0; b < kJobTiles; ++b) {
      const int TI = bi * kJobTiles + rr0 + a, TJ = bj * kJobTiles + b;
      const bool valid = (TI < NT) && (TJ < NT) && (!diag || rr0 + a <= b);
      if (!valid) continue;
      const size_t tid = static_cast<size_t>(TJ) * (TJ + 1) / 2 + TI + (plainjob ? static_cast<size_t>(p.NTl) * (p.NTl + 1) / 2 : 0);
      double2 v = make_double2(acc[a][b][0], acc[a][b][1]);
      *reinterpret_cast<double2*>(out + tid * 64 + 8 * g + 2 * t) = v;
    }
}

cudaError_t gram_tma_config(int variant, bool mc, size_t smem, int threads, int* occ, int rb) {
  static thread_local LaunchCfgCache cfg[9];
  if (rb == 2) {
    switch (variant) {
      case 0: return cached_launch_cfg(cfg[6], gram_tma_kernel<2, kMaxConsumers, false, 2>, smem, threads, occ);
      case 1: return cached_launch_cfg(cfg[7], gram_tma_kernel<4, kMaxConsumersWhole, false, 2>, smem, threads, occ);
      case 2: return cached_launch_cfg(cfg[8], gram_tma_kernel<4, kMaxConsumersWhole2, false, 2>, smem, threads, occ);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (variant + (mc ? 3 : 0)) {
    case 0: return cached_launch_cfg(cfg[0], gram_tma_kernel<2, kMaxConsumers, false>, smem, threads, occ);
    case 1: return cached_launch_cfg(cfg[1], gram_tma_kernel<4, kMaxConsumersWhole, false>, smem, threads, occ);
    case 2: return cached_launch_cfg(cfg[2], gram_tma_kernel<4, kMaxConsumersWhole2, false>, smem, threads, occ);
    case 3: return cached_launch_cfg(cfg[3], gram_tma_kernel<2, kMaxConsumers, true>, smem, threads, occ);
    case 4: return cached_launch_cfg(cfg[4], gram_tma_kernel<4, kMaxConsumersWhole, true>, smem, threads, occ);
    case 5: return cached_launch_cfg(cfg[5], gram_tma_kernel<4, kMaxConsumersWhole2, true>, smem, threads, occ);
    default: return cudaErrorInvalidValue;
  }
}

template <class K>
static cudaError_t launch_cluster(K kernel, unsigned grid, int threads, size_t smem, cudaStream_t stream, int mc,
                                  const CUtensorMap& mapQ, const CUtensorMap& mapY, const GramParams& p) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = mc;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, mapQ, mapY, p);
}

cudaError_t gram_tma_max_clusters(int variant, size_t smem, int threads, int mc, int* nclusters) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(mc);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = mc;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  switch (variant) {
    case 0: return cudaOccupancyMaxActiveClusters(nclusters, gram_tma_kernel<2, kMaxConsumers, true>, &cfg);
    case 1: return cudaOccupancyMaxActiveClusters(nclusters, gram_tma_kernel<4, kMaxConsumersWhole, true>, &cfg);
    case 2: return cudaOccupancyMaxActiveClusters(nclusters, gram_tma_kernel<4, kMaxConsumersWhole2, true>, &cfg);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gram_tma(int variant, unsigned grid, int threads, size_t smem, cudaStream_t stream,
                            const CUtensorMap& mapQ, const CUtensorMap& mapY, const GramParams& p) {
  if (p.mc > 1) {
    switch (variant) {
      case 0: return launch_cluster(gram_tma_kernel<2, kMaxConsumers, true>, grid, threads, smem, stream, p.mc, mapQ, mapY, p);
      case 1: return launch_cluster(gram_tma_kernel<4, kMaxConsumersWhole, true>, grid, threads, smem, stream, p.mc, mapQ, mapY, p);
      case 2: return launch_cluster(gram_tma_kernel<4, kMaxConsumersWhole2, true>, grid, threads, smem, stream, p.mc, mapQ, mapY, p);
      default: return cudaErrorInvalidValue;
    }
  }
  if (p.rb == 2) {
    switch (variant) {
      case 0: gram_tma_kernel<2, kMaxConsumers, false, 2><<<grid, threads, smem, stream>>>(mapQ, mapY, p); break;
      case 1: gram_tma_kernel<4, kMaxConsumersWhole, false, 2><<<grid, threads, smem, stream>>>(mapQ, mapY, p); break;
      case 2: gram_tma_kernel<4, kMaxConsumersWhole2, false, 2><<<grid, threads, smem, stream>>>(mapQ, mapY, p); break;
      default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
  }
  switch (variant) {
    case 0: gram_tma_kernel<2, kMaxConsumers, false><<<grid, threads, smem, stream>>>(mapQ, mapY, p); break;
    case 1: gram_tma_kernel<4, kMaxConsumersWhole, false><<<grid, threads, smem, stream>>>(mapQ, mapY, p); break;
    case 2: gram_tma_kernel<4, kMaxConsumersWhole2, false><<<grid, threads, smem, stream>>>(mapQ, mapY, p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// Sum the per-chunk partials in chunk order.  Output: packed upper tiles (tile (TI,TJ),
// TI <= TJ, at index TJ(TJ+1)/2 + TI, 8x8 row-major; zeros for TJ >= NTc), plus for the oblique Gram the appended
// ||Q||_F^2 (the oblique partials are upper tiles of Q^T (BQ) too, reading D22).
// Block = 32 consecutive outputs x 8 chunk classes (c mod 8): coalesced 256-B rows, eight
// loads in flight per output, then the eight class sums added in class order -- a fixed order,
// so the result is bitwise reproducible (kReduceThreads threads per block).
__global__ void gram_reduce_kernel(GramReduceParams p) {
  if (SCQR3_GATE_SKIP(p.gate)) return;
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, cls = threadIdx.x >> 5;
  const long long nout = static_cast<long long>(p.NT) * (p.NT + 1) / 2 * 64;
  const long long nall = p.dual ? 2 * nout : nout;  // partial entries to reduce
  const long long e = static_cast<long long>(blockIdx.x) * 32 + lane;
  // tiles of columns past the computed ones (n padded to a TRSM instance) are zero
  const long long ncomp = static_cast<long long>(p.NTc) * (p.NTc + 1) / 2 * 64;
  double s = 0.0;
  if (e < nall && (e < nout ? e : e - nout) < ncomp) {
    const size_t stride = static_cast<size_t>(p.tiles_per_partial) * 64;
    const double* src = p.partials + e;
    for (int c = cls; c < p.chunks; c += 8) s += src[static_cast<size_t>(c) * stride];
  }
  red[cls][lane] = s;
  __syncthreads();
  if (cls == 0 && e < nall) {
    double t = red[0][lane];
    for (int k = 1; k < 8; ++k) t += red[k][lane];
    p.tiles[e < nout ? e : e + 1] = t;  // (dual: the plain Gram follows the ||Q||_F^2 slot)
  }
  if (blockIdx.x == 0 && p.colsq_partials) {
    // ||Q||_F^2 from the Y kernel's per-block partials: thread i sums partials i, i + 256, ...
    // (eight loads in flight), then a fixed-order tree -- deterministic, and ~3 us instead of a
    // 4096-long dependent chain on one thread (~160 us, measured)
    __shared__ double cs[256];
    double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
    int c = threadIdx.x;
    for (; c + 768 < p.colsq_count; c += 1024) {
      t0 += p.colsq_partials[c];
      t1 += p.colsq_partials[c + 256];
      t2 += p.colsq_partials[c + 512];
      t3 += p.colsq_partials[c + 768];
    }
    for (; c < p.colsq_count; c += 256) t0 += p.colsq_partials[c];
    cs[threadIdx.x] = (t0 + t1) + (t2 + t3);
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if (threadIdx.x < o) cs[threadIdx.x] += cs[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) p.tiles[nout] = cs[0];
  }
}

// Y = B Q for the tridiagonal B (Alg. 4 line 1): y_i = d_i q_i + e_{i-1} q_{i-1} + e_i q_{i+1}
// (terms in the oracle's order; the halo rows come from the neighbouring ranks), plus per-block
// partial sums of q_ij^2 (||Q||_F^2 for the oblique shift, reading D4).
#ifndef SCQR3_Y_COLS
#define SCQR3_Y_COLS 4  // columns in flight per thread (measured: 4 beats 2, 8, 16; an unpredicated
                        // pointer-bump path for interior row pairs changed nothing: 0.3598 vs 0.3599 ms)
#endif
__global__ void oblique_y_kernel(ObliqueYParams p) {
  __shared__ double red[32];
  if (SCQR3_GATE_SKIP(p.gate)) return;
  double sq = 0.0;
  // two consecutive rows per thread (measured 5 % faster than one row per thread): one 16-byte
  // load and store per column for the pair, the outer neighbours by two 8-byte loads (L1 hits),
  // SCQR3_Y_COLS columns in flight
  for (long long i0 = 2 * (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x); i0 < p.m;
       i0 += 2 * static_cast<long long>(gridDim.x) * blockDim.x) {
    const bool two = i0 + 1 < p.m;
    const double d0 = p.d[i0], d1 = two ? p.d[i0 + 1] : 0.0;
    const double el = i0 > 0 ? p.e[i0 - 1] : p.e_prev, em = p.e[i0], er = two ? p.e[i0 + 1] : 0.0;
    const bool use_l = i0 > 0 || p.has_prev;
    const bool use_r = i0 + 2 < p.m || p.has_next;
    for (int j0 = 0; j0 < p.n; j0 += SCQR3_Y_COLS) {
      double q0[SCQR3_Y_COLS], q1[SCQR3_Y_COLS], ql[SCQR3_Y_COLS], qr[SCQR3_Y_COLS];
#pragma unroll
      for (int jj = 0; jj < SCQR3_Y_COLS; ++jj) {
        const int j = j0 + jj < p.n ? j0 + jj : p.n - 1;
        const double* q = p.Q + j * p.ldq;
        if (two) {
          const double2 v = __ldcs(reinterpret_cast<const double2*>(q + i0));
          q0[jj] = v.x;
          q1[jj] = v.y;
        } else {
          q0[jj] = q[i0];
          q1[jj] = p.has_next ? p.halo_next[j] : 0.0;  // row i0's lower neighbour (i0 = m-1)
        }
        ql[jj] = i0 > 0 ? q[i0 - 1] : (p.has_prev ? p.halo_prev[j] : 0.0);
        qr[jj] = i0 + 2 < p.m ? q[i0 + 2] : (p.has_next && two ? p.halo_next[j] : 0.0);
      }
#pragma unroll
      for (int jj = 0; jj < SCQR3_Y_COLS; ++jj) {
        const int j = j0 + jj;
        if (j >= p.n) continue;
        double y0 = d0 * q0[jj];  // the oracle's term order: d_i q_i + e_{i-1} q_{i-1} + e_i q_{i+1}
        if (use_l) y0 = fma(el, ql[jj], y0);
        if (two || p.has_next) y0 = fma(em, q1[jj], y0);
        sq = fma(q0[jj], q0[jj], sq);
        double* y = p.Y + j * p.ldy;
        if (two) {
          double y1 = d1 * q1[jj];
          y1 = fma(em, q0[jj], y1);
          if (use_r) y1 = fma(er, qr[jj], y1);
          __stcs(reinterpret_cast<double2*>(y + i0), make_double2(y0, y1));
          sq = fma(q1[jj], q1[jj], sq);
        } else {
          y[i0] = y0;
        }
      }
    }
  }
  // deterministic block reduction
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_down_sync(0xffffffffu, sq, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) p.colsq_partials[blockIdx.x] = v;
  }
}

// Y = B Q for a general sparse metric in CSR, plus the
// ||Q||_F^2 partials like oblique_y_kernel.  One thread per (row, 8-column chunk): consecutive
// threads take consecutive rows, so each nonzero's Q reads are coalesced along the column;
// rows outside [0, m) come from the halo buffers (neighbouring ranks' rows).
#ifndef SCQR3_CSR_COLS
#define SCQR3_CSR_COLS 16  // columns per thread (measured on C5L: 16 beats 4, 8, 32, 64)
#endif
__global__ void csr_y_kernel(ObliqueYParams p) {
  __shared__ double red[32];
  if (SCQR3_GATE_SKIP(p.gate)) return;
  constexpr int C = SCQR3_CSR_COLS;
  const int nch = (p.n + C - 1) / C;
  const long long total = p.m * nch;
  double sq = 0.0;
  for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = k % p.m;
    const int c0 = static_cast<int>(k / p.m) * C;
    const int cw = min(C, p.n - c0);
    double acc[C];
#pragma unroll
    for (int j = 0; j < C; ++j) acc[j] = 0.0;
    for (long long z = p.rp[i]; z < p.rp[i + 1]; ++z) {
      const long long col = p.ci[z];
      const double v = p.cv[z];
      const double* src;
      long long ld;
      if (col < 0) {
        src = p.halo_prev + (col + p.halo);
        ld = p.halo;
      } else if (col >= p.m) {
        if (p.ghosts) {  // ghost row of the sparsity-pattern plan (row-major)
          src = p.ghost + (col - p.m) * p.n;
          ld = 1;
        } else {
          src = p.halo_next + (col - p.m);
          ld = p.halo;
        }
      } else {
        src = p.Q + col;
        ld = p.ldq;
      }
      double qv[C];
#pragma unroll
      for (int j = 0; j < C; ++j) qv[j] = j < cw ? src[(c0 + j) * ld] : 0.0;
#pragma unroll
      for (int j = 0; j < C; ++j) acc[j] = fma(v, qv[j], acc[j]);
      if (col == i) {  // the row's own q (SPD: the diagonal is stored) -> ||Q||_F^2 partial
#pragma unroll
        for (int j = 0; j < C; ++j) sq = fma(qv[j], qv[j], sq);
      }
    }
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (j < cw) __stcs(p.Y + (c0 + j) * p.ldy + i, acc[j]);
  }
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_down_sync(0xffffffffu, sq, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) p.colsq_partials[blockIdx.x] = v;
  }
}

// Tile version of csr_y_kernel (round 2c; launched when nnz <= 12 m, see ObliqueYParams::csr_tile): a CTA owns T = 256 consecutive rows
// and ALL their columns.  The tile's row pointers and, when they fit (at most 12 nonzeros per row
// on average), its column indices and values are staged in shared memory once by coalesced loads,
// so the inner loop's only global loads are the Q entries: no rp -> ci -> Q dependent chain and
// no re-read of the CSR arrays per column chunk.  Thread t owns row i0 + t and takes C = 8
// columns at a time with one pointer bump per load (the per-load index arithmetic and column
// predicates of csr_y_kernel were ~16 instructions per load: ncu showed the issue slots half
// busy at 25 % occupancy); 64 registers -> four CTAs per SM.  Measured on C5L (m = 2e6, n = 64,
// 5-point Laplacian): 0.47 ms (4.6 TB/s of the algorithmic 2.18 GB) against 0.71 ms; DRAM reads
// 1.17 GB = 1.07x the algorithmic bytes.  More loads in flight per thread (C = 16, two nonzeros
// per step) and 128- or 512-row tiles measured slower, __ldg the same, __ldcs slower
// (profiles/csr_y_r02e.md); so did a shared-memory window of the tile's own rows per column
// chunk fed by 1-D bulk copies (0.52 ms) and a row-pair version with 16-byte loads (half the load
// requests, 128 registers: 0.74 ms).  The per-row term order is the CSR order (as in csr_y_kernel and the
// oracle), so Y has the same bits; ||Q||_F^2 is the same squares summed in another fixed order.
__device__ __forceinline__ void csr_src(const ObliqueYParams& p, long long col, int c0, const double*& src,
                                        long long& ld) {
  if (col < 0) {  // a band halo row of the previous rank
    src = p.halo_prev + (col + p.halo);
    ld = p.halo;
  } else if (col >= p.m) {
    if (p.ghosts) {  // ghost row of the sparsity-pattern plan (row-major)
      src = p.ghost + (col - p.m) * p.n;
      ld = 1;
    } else {
      src = p.halo_next + (col - p.m);
      ld = p.halo;
    }
  } else {
    src = p.Q + col;
    ld = p.ldq;
  }
  src += c0 * ld;
}

template <int C, bool STAGED>
__device__ __forceinline__ void csr_row(const ObliqueYParams& p, long long i, long long zb, long long ze,
                                        const int* __restrict__ sci, const double* __restrict__ scv,
                                        long long zoff, double& sq) {
  for (int c0 = 0; c0 < p.n; c0 += C) {
    const int cw = min(C, p.n - c0);
    double acc[C];
#pragma unroll
    for (int j = 0; j < C; ++j) acc[j] = 0.0;
    for (long long z = zb; z < ze; ++z) {
      const long long col = STAGED ? sci[z - zoff] : p.ci[z];
      const double v = STAGED ? scv[z - zoff] : p.cv[z];
      const double* src;
      long long ld;
      csr_src(p, col, c0, src, ld);
      double qv[C];
      if (cw == C) {  // a full chunk: no per-column predicates
#pragma unroll
        for (int j = 0; j < C; ++j, src += ld) qv[j] = *src;
      } else {
#pragma unroll
        for (int j = 0; j < C; ++j) qv[j] = j < cw ? src[j * ld] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < C; ++j) acc[j] = fma(v, qv[j], acc[j]);
      if (col == i) {  // the row's own q (SPD: the diagonal is stored) -> ||Q||_F^2 partial
#pragma unroll
        for (int j = 0; j < C; ++j) sq = fma(qv[j], qv[j], sq);
      }
    }
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (j < cw) __stcs(p.Y + (c0 + j) * p.ldy + i, acc[j]);
  }
}

__global__ void __launch_bounds__(kCsrTileRows, 4) csr_y_tile_kernel(ObliqueYParams p) {
  constexpr int T = kCsrTileRows, C = 8, CAP = kCsrTileNnzPerRow * T;
  __shared__ long long s_rp[T + 1];
  __shared__ int s_ci[CAP];
  __shared__ double s_cv[CAP];
  __shared__ double red[32];
  if (SCQR3_GATE_SKIP(p.gate)) return;
  double sq = 0.0;
  const long long ntiles = (p.m + T - 1) / T;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long i0 = tile * T;
    const int rows = static_cast<int>(min(static_cast<long long>(T), p.m - i0));
    __syncthreads();  // the previous tile's readers are done with the staged arrays
    for (int t = threadIdx.x; t <= rows; t += T) s_rp[t] = p.rp[i0 + t];
    __syncthreads();
    const long long z0 = s_rp[0];
    const long long cnt = s_rp[rows] - z0;
    const bool staged = cnt <= CAP;  // else this tile reads ci / cv from global memory
    if (staged) {
      for (int z = threadIdx.x; z < cnt; z += T) {
        s_ci[z] = p.ci[z0 + z];
        s_cv[z] = p.cv[z0 + z];
      }
    }
    __syncthreads();
    if (static_cast<int>(threadIdx.x) < rows) {
      const long long i = i0 + threadIdx.x;
      const long long zb = s_rp[threadIdx.x], ze = s_rp[threadIdx.x + 1];
      if (staged)
        csr_row<C, true>(p, i, zb, ze, s_ci, s_cv, z0, sq);
      else
        csr_row<C, false>(p, i, zb, ze, nullptr, nullptr, 0, sq);
    }
  }
  // deterministic block reduction
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_down_sync(0xffffffffu, sq, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < T / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) p.colsq_partials[blockIdx.x] = v;
  }
}

// Gershgorin bound max_i sum_k |B_ik| >= ||B||_2 for a CSR metric (reading D4).
__global__ void csr_gershgorin_kernel(const long long* rp, const double* cv, long long m, double* partial) {
  __shared__ double red[32];
  double mx = 0.0;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    double r = 0.0;
    for (long long z = rp[i]; z < rp[i + 1]; ++z) r += fabs(cv[z]);
    mx = fmax(mx, r);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
  }
}

// Argument check of a CSR metric on the device: row_ptr non-decreasing from 0, every column
// index inside [-halo, m + halo).  *bad is set to 1 on any violation.
// *bad = 1 if some v[k] is outside [lo, hi) (the ghost plan's send rows)
__global__ void index_check_kernel(const long long* v, long long cnt, long long lo, long long hi, int* bad) {
  for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < cnt;
       k += static_cast<long long>(gridDim.x) * blockDim.x)
    if (v[k] < lo || v[k] >= hi) *bad = 1;
}

__global__ void csr_check_kernel(const long long* rp, const int* ci, long long m, long long halo, int has_prev,
                                 int has_next, int* bad) {
  // halo rows exist only towards neighbouring ranks: none before rank 0, none after the last
  const long long lo = has_prev ? -halo : 0, hi = has_next ? m + halo : m;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long a = rp[i], b = rp[i + 1];
    if ((i == 0 && a != 0) || b < a) {
      *bad = 1;
      continue;
    }
    for (long long z = a; z < b; ++z)
      if (ci[z] < lo || ci[z] >= hi) *bad = 1;
  }
}

// Gershgorin bound max_i d_i + |e_{i-1}| + |e_i| >= ||B||_2 (reading D4); one partial per block.
__global__ void gershgorin_kernel(const double* d, const double* e, long long m, int has_prev, double e_prev,
                                  int has_next, double* partial) {
  __shared__ double red[32];
  double mx = 0.0;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    double r = d[i];
    if (i > 0) r += fabs(e[i - 1]);
    else if (has_prev) r += fabs(e_prev);
    if (i + 1 < m || has_next) r += fabs(e[i]);
    mx = fmax(mx, r);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
  }
}

__global__ void max_reduce_kernel(const double* partial, int count, double* out) {
  // one warp (max is order independent, so the result is still exact and reproducible)
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  double v = 0.0;
  for (int i = threadIdx.x; i < count; i += 32) v = fmax(v, partial[i]);
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  if (threadIdx.x == 0) *out = v;
}

// packed upper tiles -> full symmetric n x n column-major matrix (kernel-level API only)
__global__ void tiles_to_full_kernel(const double* tiles, int n, double* A) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= static_cast<long long>(n) * n) return;
  const int i = static_cast<int>(k % n), j = static_cast<int>(k / n);
  const int a = i <= j ? i : j, b = i <= j ? j : i;  // upper element (a, b)
  const int TI = a >> 3, TJ = b >> 3;
  const size_t tile = static_cast<size_t>(TJ) * (TJ + 1) / 2 + TI;
  // inside a diagonal tile the upper element (a%8, b%8) is taken so A is exactly symmetric
  A[k] = tiles[tile * 64 + 8 * (a & 7) + (b & 7)];
}

// Deterministic cross-rank sum (opts.deterministic): parts holds nparts rank Grams of count
// entries back to back (ncclAllGather); summed in rank order, identical bits on every rank.
__global__ void rank_sum_kernel(const double* parts, int nparts, long long count, double* out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = parts[i];
  for (int r = 1; r < nparts; ++r) s += parts[static_cast<long long>(r) * count + i];
  out[i] = s;
}

}  // namespace scqr3
