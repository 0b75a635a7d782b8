// Bulk-copy (cp.async.bulk, TMA engine) throughput from L2 into SMEM with an mbarrier ring, all SMs
// concurrently: the B-image stream pattern of the joint-stage kernels.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2602_11896_b200/csrc/tc.cuh"
using namespace jtfs;

__global__ void __launch_bounds__(64, 1) k_bulk(const float* src, int64_t src_floats, long long* out, int chunk_bytes,
                                               int NS, int nchunks) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[16], empty[16];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
    tc::fence_mbar_init();
  }
  __syncthreads();
  long long t0 = clock64();
  const int64_t per = chunk_bytes / 4;
  const int64_t nsrc = src_floats / per;
  if (warp == 0) {
    int stage = 0; uint32_t ph = 0;
    for (int i = 0; i < nchunks; ++i) {
      tc::mbar_wait(&empty[stage], ph ^ 1);
      if (tc::elect_one()) {
        tc::mbar_expect_tx(&full[stage], (uint32_t)chunk_bytes);
        const float* s = src + ((blockIdx.x * 7 + i) % nsrc) * per;
        tc::bulk_g2s(sm + (size_t)stage * chunk_bytes, s, (uint32_t)chunk_bytes, &full[stage]);
      }
      __syncwarp();
      if (++stage == NS) { stage = 0; ph ^= 1; }
    }
  } else {
    int stage = 0; uint32_t ph = 0;
    for (int i = 0; i < nchunks; ++i) {
      tc::mbar_wait(&full[stage], ph);
      if (tc::elect_one()) tc::mbar_arrive(&empty[stage]);
      __syncwarp();
      if (++stage == NS) { stage = 0; ph ^= 1; }
    }
    if (threadIdx.x == 32) out[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  const int64_t nf = 40ll << 20 >> 2;   // 40 MB source (L2 resident)
  float* src; cudaMalloc(&src, nf * 4); cudaMemset(src, 0, nf * 4);
  long long* d; cudaMalloc(&d, 148 * 8);
  long long h[148];
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int cb : {4096, 8192, 16384, 32768, 65536})
    for (int ns : {2, 3, 4, 6, 8, 12}) {
      if ((int64_t)cb * ns > 200 * 1024 || ns > 16) continue;
      const int nch = (int)((64ll << 20) / cb / 148 * 4);   // ~256 MB total traffic
      k_bulk<<<148, 64, cb * ns>>>(src, nf, d, cb, ns, nch);
      k_bulk<<<148, 64, cb * ns>>>(src, nf, d, cb, ns, nch);
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("chunk %6d B x %2d stages: %6.1f B/cycle/SM (%.2f TB/s chip at 1.965 GHz) %s\n", cb, ns,
             (double)cb * nch / mx, (double)cb * nch / mx * 148 * 1.965e9 / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
