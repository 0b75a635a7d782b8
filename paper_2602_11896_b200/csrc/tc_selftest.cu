// tc_selftest.cu — test-only export: one-CTA tcgen05 kind::tf32 GEMM (3xTF32) exercising every
// primitive of tc.cuh (canonical K-major layouts, SMEM descriptors, TMEM alloc, mma, commit,
// mbarrier, bulk copy, tcgen05.ld). D[128][N] = A[128][K] . B[N][K]^T, fp32 in/out.
#include <cuda_runtime.h>

#include "../../include/jtfs.h"
#include "common.cuh"
#include "tc.cuh"

namespace jtfs {

__global__ void __launch_bounds__(128) k_tc_selftest(const float* __restrict__ A, const float* __restrict__ Bimg,
                                                     float* __restrict__ D, int N, int K, int three) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t Kc = (uint32_t)K;
  float* a_hi = reinterpret_cast<float*>(sm);
  float* a_lo = a_hi + 128 * K;
  float* b_hi = a_lo + 128 * K;   // bulk-copied image: [hi | lo], each N*K floats in canonical layout
  float* b_lo = b_hi + N * K;
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    tc::mbar_init(&bar_load, 1);
    tc::mbar_init(&bar_mma, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tmem_base, 256);
  // A: split + canonical layout by threads
  for (int i = tid; i < 128 * K; i += 128) {
    int r = i / K, k = i % K;
    float hi, lo;
    tc::split_tf32(A[i], hi, lo);
    uint32_t o = tc::core_off(r, k, Kc) / 4;
    a_hi[o] = hi;
    a_lo[o] = lo;
  }
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    uint32_t bytes = (uint32_t)(2 * N * K * 4);
    tc::mbar_expect_tx(&bar_load, bytes);
    tc::bulk_g2s(b_hi, Bimg, bytes, &bar_load);
    tc::mbar_wait(&bar_load, 0);
    const uint32_t idesc = tc::idesc_tf32(128, (uint32_t)N);
    const uint32_t sboA = Kc * 32, sboB = Kc * 32;
    for (int s = 0; s < K / 8; ++s) {
      uint64_t ah = tc::sdesc(tc::smem_u32(a_hi) + 256 * s, 128, sboA);
      uint64_t al = tc::sdesc(tc::smem_u32(a_lo) + 256 * s, 128, sboA);
      uint64_t bh = tc::sdesc(tc::smem_u32(b_hi) + 256 * s, 128, sboB);
      uint64_t bl = tc::sdesc(tc::smem_u32(b_lo) + 256 * s, 128, sboB);
      tc::mma_tf32(tbase, ah, bh, idesc, s > 0 ? 1u : 0u);
      if (three) {
        tc::mma_tf32(tbase, ah, bl, idesc, 1u);
        tc::mma_tf32(tbase, al, bh, idesc, 1u);
      }
    }
    tc::mma_commit(&bar_mma);
  }
  __syncwarp();
  tc::mbar_wait(&bar_mma, 0);
  tc::tc_fence_after();
  const int row = warp * 32 + (tid & 31);
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tc::tmem_ld16(tbase + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, v);
#pragma unroll
    for (int j = 0; j < 16; ++j) D[row * N + c + j] = v[j];
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 256);
}

// same GEMM with A staged in TMEM (tcgen05.st) and issued as the TS variant of tcgen05.mma
__global__ void __launch_bounds__(128) k_tc_selftest_ts(const float* __restrict__ A, const float* __restrict__ Bimg,
                                                        float* __restrict__ D, int N, int K, int three) {
  extern __shared__ __align__(1024) uint8_t sm[];
  float* b_hi = reinterpret_cast<float*>(sm);
  float* b_lo = b_hi + N * K;
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    tc::mbar_init(&bar_load, 1);
    tc::mbar_init(&bar_mma, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tmem_base, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = tmem_base;
  const uint32_t ta_hi = tbase + 256, ta_lo = tbase + 256 + (uint32_t)K;
  // each thread = one row of A: write hi/lo to its TMEM lane, 16 columns at a time
  const int row = tid;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  for (int c = 0; c < K; c += 16) {
    float hi[16], lo[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float h = 0.f, l = 0.f;
      if (c + j < K) tc::split_tf32(A[row * K + c + j], h, l);
      hi[j] = h;
      lo[j] = l;
    }
    tc::tmem_st16(ta_hi + lane_off + (uint32_t)c, hi);
    tc::tmem_st16(ta_lo + lane_off + (uint32_t)c, lo);
  }
  tc::tmem_wait_st();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (tid == 0) {
    uint32_t bytes = (uint32_t)(2 * N * K * 4);
    tc::mbar_expect_tx(&bar_load, bytes);
    tc::bulk_g2s(b_hi, Bimg, bytes, &bar_load);
    tc::mbar_wait(&bar_load, 0);
    const uint32_t idesc = tc::idesc_tf32(128, (uint32_t)N);
    const uint32_t sboB = (uint32_t)K * 32;
    for (int s = 0; s < K / 8; ++s) {
      uint64_t bh = tc::sdesc(tc::smem_u32(b_hi) + 256 * s, 128, sboB);
      uint64_t bl = tc::sdesc(tc::smem_u32(b_lo) + 256 * s, 128, sboB);
      tc::mma_tf32_ts(tbase, ta_hi + 8 * s, bh, idesc, s > 0 ? 1u : 0u);
      if (three) {
        tc::mma_tf32_ts(tbase, ta_hi + 8 * s, bl, idesc, 1u);
        tc::mma_tf32_ts(tbase, ta_lo + 8 * s, bh, idesc, 1u);
      }
    }
    tc::mma_commit(&bar_mma);
  }
  __syncwarp();
  tc::mbar_wait(&bar_mma, 0);
  tc::tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tc::tmem_ld16(tbase + lane_off + (uint32_t)c, v);
#pragma unroll
    for (int j = 0; j < 16; ++j) D[row * N + c + j] = v[j];
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

}  // namespace jtfs

extern "C" jtfs_status jtfs_debug_tc_gemm_ts(const float* A, const float* Bimg, float* D, int N, int K, int three,
                                             jtfs_stream_t stream) {
  if (N < 16 || N > 256 || N % 16 || K < 16 || K % 16 || K > 128) return JTFS_ERR_SIZE;
  size_t sm = (size_t)(2 * N * K) * 4;
  cudaFuncSetAttribute(jtfs::k_tc_selftest_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  jtfs::k_tc_selftest_ts<<<1, 128, sm, (cudaStream_t)stream>>>(A, Bimg, D, N, K, three);
  jtfs::count_launch();
  return cudaGetLastError() == cudaSuccess ? JTFS_OK : JTFS_ERR_CUDA;
}

extern "C" jtfs_status jtfs_debug_tc_gemm(const float* A, const float* Bimg, float* D, int N, int K, int three,
                                          jtfs_stream_t stream) {
  if (N < 16 || N > 256 || N % 16 || K < 8 || K % 8) return JTFS_ERR_SIZE;
  size_t sm = (size_t)(2 * 128 * K + 2 * N * K) * 4;
  if (sm > 200 * 1024) return JTFS_ERR_SIZE;
  cudaFuncSetAttribute(jtfs::k_tc_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  jtfs::k_tc_selftest<<<1, 128, sm, (cudaStream_t)stream>>>(A, Bimg, D, N, K, three);
  jtfs::count_launch();
  return cudaGetLastError() == cudaSuccess ? JTFS_OK : JTFS_ERR_CUDA;
}
