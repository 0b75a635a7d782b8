// common.cuh — shared device helpers for the libjtfs kernels (product path only).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace jtfs {

// Count of kernel launches issued by the library (reported by bench.py as gpu_launches).
void count_launch(int n = 1);
// Profiling hooks (jtfs_prof_enable): CUDA events around the joint-stage kernels.
void prof_begin(cudaStream_t st, int id);
void prof_end(cudaStream_t st, int id);

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }

__device__ __forceinline__ int64_t pmod64(int64_t a, int64_t m) {
  int64_t r = a % m;
  return r < 0 ? r + m : r;
}

// Batched rows: for signal b and row r, element 0 is at base + b*stride_b + off + r*L.
struct Rows {
  int64_t stride_b, off, count, L;
};

// Path-shard ownership of one jtfs_loss_grad call (include/jtfs.h): bit bi = second-order block bi
// (blocks go to shards by the planner's LPT rule, Plan::block_owner), bit 63 = order 1 (shard 0).
constexpr uint64_t kOwnOrder1 = 1ull << 63;
constexpr uint64_t kOwnAll = ~0ull;
__host__ __device__ __forceinline__ bool owns_block(uint64_t own, int bi) { return (own >> bi) & 1ull; }

}  // namespace jtfs
