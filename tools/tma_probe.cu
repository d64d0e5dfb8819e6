// Read-bandwidth probe for streaming a tall-skinny column-major fp64 matrix (m x 64) the way the
// n = 64 Gram does: TMA boxes of R rows x 64 columns into a per-CTA stage ring (one producer lane,
// consumer warps that only wait and release), against plain coalesced loads.  Answers whether
// the 16-row SWIZZLE_128B boxes (64 separate 128-B segments per box) cap the read rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -Ipaper_1809_11085_b200/csrc \
//        tools/tma_probe.cu -o tools/tma_probe -lcuda && tools/tma_probe
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "scqr3_dev.cuh"

using namespace scqr3;

template <int ROWS>
__global__ void tma_stream(const __grid_constant__ CUtensorMap map, long long m, int stages, int ncons, double* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  const uint32_t sbytes = ROWS * 64 * 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + stages * sbytes);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], ncons);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const long long total = (m + ROWS - 1) / ROWS;
  const long long s0 = total * blockIdx.x / gridDim.x, s1 = total * (blockIdx.x + 1) / gridDim.x;
  const int nst = static_cast<int>(s1 - s0);
  if (warp == 0) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nst; ++i, ++st) {
        if (st == stages) { st = 0; ph ^= 1u; }
        if (i >= stages) mbar_wait(&empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&full[st], sbytes);
        tma_load_2d(base + st * sbytes, &map, static_cast<int>((s0 + i) * ROWS), 0, &full[st]);
      }
    }
    return;
  }
  double acc = 0.0;
  int st = 0;
  uint32_t ph = 0;
  for (int i = 0; i < nst; ++i, ++st) {
    if (st == stages) { st = 0; ph ^= 1u; }
    mbar_wait(&full[st], ph);
    acc += reinterpret_cast<const double*>(base + st * sbytes)[lane + 32 * (warp - 1)];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  if (acc == 12345.678) sink[0] = acc;
}

template <int RB>
__global__ void tma_stream3(const __grid_constant__ CUtensorMap map, long long m, int stages, int ncons, double* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  const uint32_t sbytes = RB * 16 * 64 * 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + stages * sbytes);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], ncons);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const long long total = m / (16 * RB);
  const long long s0 = total * blockIdx.x / gridDim.x, s1 = total * (blockIdx.x + 1) / gridDim.x;
  const int nst = static_cast<int>(s1 - s0);
  if (warp == 0) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nst; ++i, ++st) {
        if (st == stages) { st = 0; ph ^= 1u; }
        if (i >= stages) mbar_wait(&empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&full[st], sbytes);
        const int rb0 = static_cast<int>((s0 + i) * RB);
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::
                "r"(smem_u32(base + st * sbytes)), "l"(&map), "r"(0), "r"(rb0), "r"(0), "r"(smem_u32(&full[st]))
            : "memory");
      }
    }
    return;
  }
  double acc = 0.0;
  int st = 0;
  uint32_t ph = 0;
  for (int i = 0; i < nst; ++i, ++st) {
    if (st == stages) { st = 0; ph ^= 1u; }
    mbar_wait(&full[st], ph);
    acc += reinterpret_cast<const double*>(base + st * sbytes)[lane + 32 * (warp - 1)];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  if (acc == 12345.678) sink[0] = acc;
}

// plain loads: warp w of the grid takes 32-row groups; lane = row, loop over the 64 columns
__global__ void ldg_stream(const double* X, long long m, long long ld, double* sink) {
  const long long groups = (m + 31) / 32;
  double acc = 0.0;
  const int lane = threadIdx.x & 31;
  for (long long gi = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; gi < groups;
       gi += static_cast<long long>(gridDim.x) * blockDim.x / 32) {
    const long long r = gi * 32 + lane;
    if (r < m) {
      double v[16];
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 16) {
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = __ldcs(X + r + (c0 + c) * ld);
#pragma unroll
        for (int c = 0; c < 16; ++c) acc += v[c];
      }
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

int main() {
  const long long m = 10000000, n = 64, ld = m;
  double* X;
  double* sink;
  cudaMalloc(&X, m * n * 8);
  cudaMalloc(&sink, 8);
  cudaMemset(X, 0, m * n * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    return best;
  };
  const double bytes = 8.0 * m * n;
  auto run_tma = [&](auto kern, int rows, CUtensorMapSwizzle swz, int stages, int occ, int ncons, const char* name) {
    CUtensorMap map;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(n)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(rows), 64};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, X, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("%s: encode failed %d\n", name, (int)r);
      return;
    }
    const size_t smem = 1024 + static_cast<size_t>(stages) * rows * 64 * 8 + 16 * stages;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const int grid = 148 * occ;
    const float ms = timeit([&] { kern<<<grid, 32 * (1 + ncons), smem>>>(map, m, stages, ncons, sink); });
    cudaError_t e = cudaGetLastError();
    printf("%-34s rows=%3d stages=%2d ctas/SM=%d: %.3f ms  %.2f TB/s %s\n", name, rows, stages, occ, ms,
           bytes / ms / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  run_tma(tma_stream<16>, 16, CU_TENSOR_MAP_SWIZZLE_128B, 8, 3, 6, "TMA 16x64 swz128 (Gram n=64)");
  run_tma(tma_stream<16>, 16, CU_TENSOR_MAP_SWIZZLE_128B, 8, 1, 6, "TMA 16x64 swz128, 1 CTA/SM");
  run_tma(tma_stream<16>, 16, CU_TENSOR_MAP_SWIZZLE_128B, 16, 2, 6, "TMA 16x64 swz128, 16 stages");
  run_tma(tma_stream<32>, 32, CU_TENSOR_MAP_SWIZZLE_NONE, 8, 2, 6, "TMA 32x64 no swizzle");
  run_tma(tma_stream<64>, 64, CU_TENSOR_MAP_SWIZZLE_NONE, 4, 2, 6, "TMA 64x64 no swizzle");
  run_tma(tma_stream<64>, 64, CU_TENSOR_MAP_SWIZZLE_NONE, 6, 1, 6, "TMA 64x64 no swizzle 1 CTA");
  run_tma(tma_stream<128>, 128, CU_TENSOR_MAP_SWIZZLE_NONE, 3, 1, 6, "TMA 128x64 no swizzle");
  // 3-D view (16 rows, row blocks of 16, columns) with SWIZZLE_128B: a box of RB row blocks
  // fetches RB x 128 contiguous bytes per column while every 128-B line stays swizzled
  auto run_3d = [&](int rb, int stages, int occ, const char* name) {
    CUtensorMap map;
    cuuint64_t dims[3] = {16, static_cast<cuuint64_t>(m / 16), static_cast<cuuint64_t>(n)};
    cuuint64_t strides[2] = {128, static_cast<cuuint64_t>(ld) * 8};
    cuuint32_t box[3] = {16, static_cast<cuuint32_t>(rb), 64};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, X, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("%s: encode failed %d\n", name, (int)r);
      return;
    }
    auto kern = rb == 2 ? tma_stream3<2> : rb == 4 ? tma_stream3<4> : tma_stream3<8>;
    const size_t smem = 1024 + static_cast<size_t>(stages) * rb * 16 * 64 * 8 + 16 * stages;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const float ms = timeit([&] { kern<<<148 * occ, 32 * 7, smem>>>(map, m, stages, 6, sink); });
    cudaError_t e = cudaGetLastError();
    printf("%-34s rows=%3d stages=%2d ctas/SM=%d: %.3f ms  %.2f TB/s %s\n", name, 16 * rb, stages, occ, ms,
           bytes / ms / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  run_3d(2, 8, 2, "TMA 3-D {16,2,64} swz128");
  run_3d(4, 4, 2, "TMA 3-D {16,4,64} swz128");
  run_3d(8, 3, 1, "TMA 3-D {16,8,64} swz128");
  {
    const float ms = timeit([&] { ldg_stream<<<148 * 8, 256>>>(X, m, ld, sink); });
    printf("%-34s: %.3f ms  %.2f TB/s\n", "LDG 32 rows x 16 cols in flight", ms, bytes / ms / 1e9);
  }
  return 0;
}
