// Microbenchmarks for the tcgen05 joint-stage kernels: TMEM ld/st throughput and kind::tf32 MMA rate
// per N (single CTA per SM, clock64 timing). Build: nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2602_11896_b200/csrc/tc.cuh"
using namespace jtfs;

__global__ void __launch_bounds__(128, 1) k_tmem(long long* out, int iters, int mode) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  const uint32_t lq = (uint32_t)(warp * 32) << 16;
  float v[16];
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x + i;
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int c = 0; c < 512; c += 16) {
      if (mode == 0) { tc::tmem_ld16_nowait(tbase + lq + c, v); }
      else { tc::tmem_st16(tbase + lq + c, v); }
    }
    if (mode == 0) { tc::tmem_wait_ld(); acc += v[0] + v[15]; }
    else tc::tmem_wait_st();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) out[1000] = 1;
  tc::tc_fence_before(); __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

// back-to-back kind::tf32 MMAs M=128 x N x K=8 from SMEM (zeros), one elected thread issues
__global__ void __launch_bounds__(128, 1) k_mma(long long* out, int n_mma, int N, int ts) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  float* A = reinterpret_cast<float*>(sm);
  for (int i = threadIdx.x; i < 128 * 64 + 256 * 64; i += 128) A[i] = 0.f;
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  tc::fence_async_smem();
  tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  long long t0 = clock64();
  if (warp == 0) {
    const uint64_t dA = tc::sdesc(tc::smem_u32(A), 128, 64 * 32);
    const uint64_t dB = tc::sdesc(tc::smem_u32(A + 128 * 64), 128, 64 * 32);
    const uint32_t idesc = tc::idesc_tf32(128, (uint32_t)N);
    if (tc::elect_one()) {
      if (ts) {
        for (int i = 0; i < n_mma; ++i) tc::mma_tf32_ts(tbase, tbase + 256 + 8u * (i & 7), dB + 16u * (i & 7), idesc, 1u);
      } else {
        for (int i = 0; i < n_mma; ++i) tc::mma_tf32(tbase, dA + 16u * (i & 7), dB + 16u * (i & 7), idesc, 1u);
      }
      tc::mma_commit(&bar);
    }
    __syncwarp();
    tc::mbar_wait(&bar, 0);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc::tc_fence_before(); __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

// ping-pong: MMA warp issues one 128x64x8 MMA + commit -> epilogue warps (4) wait, tcgen05.ld 32 cols,
// tcgen05.st 64 cols, arrive -> MMA warp waits, repeat. Measures the bwd per-tile protocol latency.
__global__ void __launch_bounds__(160, 1) k_pingpong(long long* out, int iters, int nmma) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ uint64_t b1, b2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* A = reinterpret_cast<float*>(sm);
  for (int i = threadIdx.x; i < 128 * 64 + 256 * 64; i += 160) A[i] = 0.f;
  if (threadIdx.x == 0) { tc::mbar_init(&b1, 1); tc::mbar_init(&b2, 4); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  tc::fence_async_smem();
  tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  long long t0 = clock64();
  if (warp == 4) {
    const uint64_t dA = tc::sdesc(tc::smem_u32(A), 128, 64 * 32);
    const uint64_t dB = tc::sdesc(tc::smem_u32(A + 128 * 64), 128, 64 * 32);
    const uint32_t idesc = tc::idesc_tf32(128, 64);
    for (int it = 0; it < iters; ++it) {
      if (it > 0) tc::mbar_wait(&b2, (it - 1) & 1);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        for (int i = 0; i < nmma; ++i) tc::mma_tf32(tbase, dA + 16u * (i & 7), dB + 16u * (i & 7), idesc, 1u);
        tc::mma_commit(&b1);
      }
      __syncwarp();
    }
    tc::mbar_wait(&b2, (iters - 1) & 1);
  } else {
    const uint32_t lq = (uint32_t)(warp * 32) << 16;
    float v[32];
    for (int it = 0; it < iters; ++it) {
      tc::mbar_wait(&b1, it & 1);
      tc::tc_fence_after();
      tc::tmem_ld16_nowait(tbase + lq, v);
      tc::tmem_ld16_nowait(tbase + lq + 16, v + 16);
      tc::tmem_wait_ld();
      for (int i = 0; i < 32; ++i) v[i] = v[i] * 0.5f;
      tc::tmem_st16(tbase + lq + 128, v);
      tc::tmem_st16(tbase + lq + 144, v + 16);
      tc::tmem_st16(tbase + lq + 192, v);
      tc::tmem_st16(tbase + lq + 208, v + 16);
      tc::tmem_wait_st();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&b2);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 128) out[blockIdx.x] = t1 - t0;
  tc::tc_fence_before(); __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

// contention: warp 4 issues the bwd per-tile MMA mix (15 SS N=64 + 24 TS N=48) `iters` times while
// warps 0-3 (if epi) stream tcgen05.ld 32 cols + tcgen05.st 64 cols per round, unsynchronised.
__global__ void __launch_bounds__(160, 1) k_contend(long long* out, int iters, int epi) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  float* A = reinterpret_cast<float*>(sm);
  for (int i = threadIdx.x; i < 128 * 64 + 256 * 64; i += 160) A[i] = 0.f;
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); done = 0; }
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  tc::fence_async_smem();
  tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  long long t0 = clock64();
  if (warp == 4) {
    const uint64_t dA = tc::sdesc(tc::smem_u32(A), 128, 64 * 32);
    const uint64_t dB = tc::sdesc(tc::smem_u32(A + 128 * 64), 128, 64 * 32);
    const uint32_t id1 = tc::idesc_tf32(128, 64), id2 = tc::idesc_tf32(128, 48);
    if (tc::elect_one()) {
      for (int it = 0; it < iters; ++it) {
        for (int i = 0; i < 15; ++i) tc::mma_tf32(tbase, dA + 16u * (i & 7), dB + 16u * (i & 7), id1, 1u);
        for (int i = 0; i < 24; ++i) tc::mma_tf32_ts(tbase + 256, tbase + 128 + 8u * (i & 7), dB + 16u * (i & 7), id2, 1u);
      }
      tc::mma_commit(&bar);
    }
    __syncwarp();
    tc::mbar_wait(&bar, 0);
    if (threadIdx.x == 128) { out[blockIdx.x] = clock64() - t0; done = 1; }
  } else if (epi) {
    const uint32_t lq = (uint32_t)(warp * 32) << 16;
    float v[32];
    for (int i = 0; i < 32; ++i) v[i] = 1.f;
    int rounds = 0;
    while (!done && rounds < 100000) {
      tc::tmem_ld16_nowait(tbase + lq + 64, v);
      tc::tmem_ld16_nowait(tbase + lq + 80, v + 16);
      tc::tmem_wait_ld();
      tc::tmem_st16(tbase + lq + 192, v);
      tc::tmem_st16(tbase + lq + 208, v + 16);
      tc::tmem_st16(tbase + lq + 224, v);
      tc::tmem_st16(tbase + lq + 240, v + 16);
      tc::tmem_wait_st();
      ++rounds;
    }
    if (threadIdx.x == 0) out[200 + blockIdx.x] = rounds;
  }
  tc::tc_fence_before(); __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

// per-instruction timing of the MMA-issue path: n MMAs (N=128, TS) then commit, then a try_wait on an
// already-completed mbarrier, then the wait for the commit
__global__ void __launch_bounds__(128, 1) k_issue(long long* out, int n) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar, done_bar;
  const int warp = threadIdx.x >> 5;
  float* B = reinterpret_cast<float*>(sm);
  for (int i = threadIdx.x; i < 128 * 64 * 2; i += 128) B[i] = 0.f;
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::mbar_init(&done_bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  tc::fence_async_smem();
  tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  if (threadIdx.x == 0) tc::mbar_arrive(&done_bar);   // completes phase 0
  __syncthreads();
  if (warp == 0) {
    const uint64_t dB = tc::sdesc(tc::smem_u32(B), 128, 64 * 32);
    const uint32_t idesc = tc::idesc_tf32(128, 128);
    long long t0 = 0, t1 = 0, t2 = 0, t3 = 0, t4 = 0;
    if (tc::elect_one()) {
      t0 = clock64();
      for (int i = 0; i < n; ++i) tc::mma_tf32_ts(tbase, tbase + 256 + 8u * (i & 7), dB + 16u * (i & 7), idesc, 1u);
      t1 = clock64();
      tc::mma_commit(&bar);
      t2 = clock64();
    }
    __syncwarp();
    tc::mbar_wait(&done_bar, 0);   // already complete
    t3 = clock64();
    tc::mbar_wait(&bar, 0);
    t4 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; }
  }
  tc::tc_fence_before(); __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

int main() {
  long long* d; cudaMalloc(&d, 2000 * 8);
  long long h[148];
  int iters = 200;
  for (int mode = 0; mode < 2; ++mode) {
    k_tmem<<<148, 128>>>(d, iters, mode);
    cudaDeviceSynchronize();
    k_tmem<<<148, 128>>>(d, iters, mode);
    cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
    double bytes = (double)iters * 512 * 128 * 4;   // whole TMEM per iter
    printf("tmem %s: %.1f cycles/iter, %.1f B/cycle/SM (err %s)\n", mode ? "st" : "ld", (double)h[0] / iters,
           bytes / h[0], cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int Ns[] = {16, 32, 48, 64, 128, 176, 256};
  for (int ts = 0; ts < 2; ++ts)
  for (int N : Ns) {
    if (ts && N > 240) continue;
    int n = 2000;
    k_mma<<<148, 128, 200 * 1024>>>(d, n, N, ts);
    cudaDeviceSynchronize();
    k_mma<<<148, 128, 200 * 1024>>>(d, n, N, ts);
    cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
    printf("mma tf32 %s 128x%dx8: %.1f cycles/mma (model N/2 = %d) (err %s)\n", ts ? "TS" : "SS", N, (double)h[0] / n, N / 2,
           cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(k_pingpong, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int nm : {1, 15}) {
    int it = 2000;
    k_pingpong<<<148, 160, 200 * 1024>>>(d, it, nm);
    cudaDeviceSynchronize();
    k_pingpong<<<148, 160, 200 * 1024>>>(d, it, nm);
    cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
    printf("pingpong (%d MMA N=64 + commit -> ld 32 / st 64 cols -> arrive): %.1f cycles/round (err %s)\n", nm,
           (double)h[0] / it, cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(k_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int n : {1, 4, 8, 16, 30, 60}) {
    k_issue<<<1, 128, 200 * 1024>>>(d, n);
    cudaDeviceSynchronize();
    k_issue<<<1, 128, 200 * 1024>>>(d, n);
    long long hh[4];
    cudaMemcpy(hh, d, 4 * 8, cudaMemcpyDeviceToHost);
    printf("issue %2d TS N=128 MMAs: issue %lld cyc, commit %lld, wait(complete bar) %lld, wait(commit) %lld (%s)\n", n,
           hh[0], hh[1], hh[2], hh[3], cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(k_contend, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int epi = 0; epi < 2; ++epi) {
    int it = 200;
    k_contend<<<148, 160, 200 * 1024>>>(d, it, epi);
    cudaDeviceSynchronize();
    k_contend<<<148, 160, 200 * 1024>>>(d, it, epi);
    long long hh[400];
    cudaMemcpy(hh, d, 400 * 8, cudaMemcpyDeviceToHost);
    printf("contend epi=%d: %.1f cycles per bwd tile MMA mix (ideal 15*48+24*24 = 1296); epi rounds %lld (err %s)\n",
           epi, (double)hh[0] / it, hh[200], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
