// kernels_tc.cu — the joint lambda_1 stage forward on the 5th-generation tensor cores (tcgen05).
//
// For one block n2 and a tile of 128 time columns, every frequential filter f is the exact dense
// matrix M_f[r][n] = h_f[(r 2^k_f - n) mod P] (zero-pad to P, circular convolution along n1,
// decimation by 2^k_f: P:276-295). The complex product W_f^T = Y2^T M_f^T is a real GEMM
//     D[c][2r+po] = sum_{n,pi} A[c][2n+pi] B[2r+po][2n+pi]
// with A[c][2n+pi] = (Re,Im) Y2[n][c] and B = [[Re M, -Im M], [Im M, Re M]] interleaved, so that
// TMEM lane c (a time column) holds Re/Im W of 64 consecutive lambda_1 rows side by side. 3xTF32:
// D = A_hi B_hi + A_hi B_lo + A_lo B_hi, fp32 accumulation in TMEM (north_star: "a genuine dense
// contraction with a 3xTF32 split").
//   warp 0      producer: cp.async.bulk of pre-split B images (planner, canonical K-major layout)
//   warp 1      MMA issuer (one thread): tcgen05.mma kind::tf32, M=128, N=128, K=8
//   warps 4..11 epilogue: tcgen05.ld -> |W| (Eq.2) -> phi_F over rows (Eq.4, R17) in registers
// A (the Y2 tile, hi/lo) stays resident in SMEM for all filters of the block; TMEM is double
// buffered so the epilogue of row tile t overlaps the MMAs of row tile t+1.
#include <cuda_runtime.h>

#include "device.cuh"
#include "tc.cuh"

namespace jtfs {

constexpr int kTcRows = 64;         // lambda_1 rows per row tile (N = 128)
constexpr int kTcN = 2 * kTcRows;   // MMA N
constexpr int kTcKc = 32;           // B chunk (k' elements) per pipeline stage
constexpr int kTcThreads = 384;     // 12 warps

__device__ __forceinline__ int find_tc(const int64_t* __restrict__ tiles, int n, int64_t t) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (__ldg(tiles + mid) <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

struct TcArgs {
  const float2* Y2; int64_t y_sb;
  float* o; int64_t o_sb;
  const JointUnit* units; const BlockInfo* binfo;
  const TcBlock* blocks; const int64_t* tiles; int n_tc_blocks;
  const float* img;                 // B images
  const float* wts;                 // phi_F weights [unit][rho][NT*64]
  const TcUnit* tcu;                // per unit image / weight offsets
  int nfr, shard, n_shards;
};

constexpr int kTcMaxStages = 8;

template <int CT, int KAP>
__global__ void __launch_bounds__(kTcThreads, 1) k_joint_fwd_tc(TcArgs a, int NS) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[kTcMaxStages], empty[kTcMaxStages], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int jb = find_tc(a.tiles, a.n_tc_blocks, blockIdx.x);
  const TcBlock TB = a.blocks[jb];
  const BlockInfo bf = a.binfo[TB.bi];
  const int64_t col0 = (blockIdx.x - a.tiles[jb]) * (int64_t)(128 * CT);
  const int b = blockIdx.y;
  const int K = TB.K, K2 = TB.K2;
  float* a_hi = reinterpret_cast<float*>(sm);              // [CT][128][K2] canonical
  float* a_lo = a_hi + CT * 128 * K2;
  float* bst = a_lo + CT * 128 * K2;                        // NS stages x (2 x 128 x kTcKc)
  float* red = bst + NS * 2 * kTcN * kTcKc;                 // [CT][KAP][128]

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { tc::mbar_init(&tfull[s], 1); tc::mbar_init(&tempty[s], 8); }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(&tmem_base, CT == 1 ? 256 : 512);
  // ---- A: Y2 tile -> tf32 hi/lo, canonical K-major, k' = 2n + (re, im); zero padded
  const float2* ysrc = a.Y2 + b * a.y_sb + bf.y_off;
  for (int idx = tid; idx < CT * 128 * (K2 / 2); idx += kTcThreads) {
    const int c = idx & 127;
    const int rest = idx >> 7;
    const int n = rest % (K2 / 2), m = rest / (K2 / 2);
    const int64_t col = col0 + m * 128 + c;
    float2 v = make_float2(0.f, 0.f);
    if (n < K && col < bf.n_cols) v = ysrc[(int64_t)n * bf.T2 + (bf.c_lo + col) % bf.T2];
    float h0, l0, h1, l1;
    tc::split_tf32(v.x, h0, l0);
    tc::split_tf32(v.y, h1, l1);
    const uint32_t o = (uint32_t)(m * 128 * K2) + tc::core_off((uint32_t)c, (uint32_t)(2 * n), (uint32_t)K2) / 4;
    *reinterpret_cast<float2*>(a_hi + o) = make_float2(h0, h1);
    *reinterpret_cast<float2*>(a_lo + o) = make_float2(l0, l1);
  }
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = tmem_base;
  const int nchunks = (K2 + kTcKc - 1) / kTcKc;

  if (warp == 0) {
    // ===================== producer: B chunks via the bulk-copy engine (whole warp, one lane issues)
    int stage = 0;
    uint32_t ph = 0;
    for (int f = 0; f < a.nfr; ++f) {
      const int u = TB.bi * a.nfr + f;
      if (u % a.n_shards != a.shard) continue;
      const TcUnit tu = a.tcu[u];
      const float* src = a.img + tu.img_off;
      for (int t = 0; t < tu.NT; ++t) {
        for (int ch = 0; ch < nchunks; ++ch) {
          const int kc = min(kTcKc, K2 - ch * kTcKc);
          const uint32_t bytes = (uint32_t)(2 * kTcN * kc * 4);
          tc::mbar_wait(&empty[stage], ph ^ 1);
          if (tc::elect_one()) {
            tc::mbar_expect_tx(&full[stage], bytes);
            tc::bulk_g2s(bst + stage * 2 * kTcN * kTcKc, src, bytes, &full[stage]);
          }
          __syncwarp();
          src += 2 * kTcN * kc;
          if (++stage == NS) { stage = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (warp-uniform loop, one elected lane issues)
    const uint32_t idesc = tc::idesc_tf32(128, kTcN);
    const uint32_t sboA = (uint32_t)K2 * 32u;
    // descriptors differ only in the start-address field: add (byte offset >> 4) to the low word
    const uint64_t dA_hi = tc::sdesc(tc::smem_u32(a_hi), 128, sboA);
    const uint64_t dA_lo = tc::sdesc(tc::smem_u32(a_lo), 128, sboA);
    const uint32_t aStepM = (uint32_t)(128 * K2 * 4) >> 4;
    const uint32_t bst_s = tc::smem_u32(bst);
    int stage = 0, buf = 0;
    uint32_t ph = 0, bph = 0;
    for (int f = 0; f < a.nfr; ++f) {
      const int u = TB.bi * a.nfr + f;
      if (u % a.n_shards != a.shard) continue;
      const TcUnit tu = a.tcu[u];
      for (int t = 0; t < tu.NT; ++t) {
        tc::mbar_wait(&tempty[buf], bph ^ 1);
        tc::tc_fence_after();
        const uint32_t dbase = tbase + (uint32_t)(buf * CT * kTcN);
        for (int ch = 0; ch < nchunks; ++ch) {
          const int kc = min(kTcKc, K2 - ch * kTcKc);
          tc::mbar_wait(&full[stage], ph);
          tc::tc_fence_after();
          const uint32_t bh = bst_s + (uint32_t)(stage * 2 * kTcN * kTcKc * 4);
          const uint64_t dB_hi = tc::sdesc(bh, 128, (uint32_t)kc * 32u);
          const uint64_t dB_lo = tc::sdesc(bh + (uint32_t)(kTcN * kc * 4), 128, (uint32_t)kc * 32u);
          if (tc::elect_one()) {
            for (int ks = 0; ks < kc / 8; ++ks) {
              const uint32_t kg = (uint32_t)(ch * (kTcKc / 8) + ks);
#pragma unroll
              for (int m = 0; m < CT; ++m) {
                const uint32_t d = dbase + (uint32_t)(m * kTcN);
                const uint64_t ao = (uint64_t)(m * aStepM + 16u * kg);
                tc::mma_tf32(d, dA_hi + ao, dB_hi + 16u * ks, idesc, (ch > 0 || ks > 0) ? 1u : 0u);
                tc::mma_tf32(d, dA_hi + ao, dB_lo + 16u * ks, idesc, 1u);
                tc::mma_tf32(d, dA_lo + ao, dB_hi + 16u * ks, idesc, 1u);
              }
            }
            tc::mma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == NS) { stage = 0; ph ^= 1; }
        }
        if (tc::elect_one()) tc::mma_commit(&tfull[buf]);
        __syncwarp();
        if (++buf == 2) { buf = 0; bph ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: |W| and phi_F over rows, per time column (TMEM lane)
    const int e = warp - 4;
    const int q = e & 3, h = e >> 2;        // lane quadrant, column half (32 complex rows)
    const int c = q * 32 + lane;            // time column within the tile
    int buf = 0;
    uint32_t bph = 0;
    for (int f = 0; f < a.nfr; ++f) {
      const int u = TB.bi * a.nfr + f;
      if (u % a.n_shards != a.shard) continue;
      const JointUnit U = a.units[u];
      const TcUnit tu = a.tcu[u];
      const int ro = U.rows_out;
      const float* wt = a.wts + tu.wt_off;
      const int ldw = tu.NT * kTcRows;
      float oacc[CT][KAP];
#pragma unroll
      for (int m = 0; m < CT; ++m)
#pragma unroll
        for (int r = 0; r < KAP; ++r) oacc[m][r] = 0.f;
      for (int t = 0; t < tu.NT; ++t) {
        // lane l holds the phi_F weights of row (t*64 + h*32 + l); broadcast by shuffles below
        float wl[KAP];
#pragma unroll
        for (int r = 0; r < KAP; ++r) wl[r] = (r < ro) ? __ldg(wt + r * ldw + t * kTcRows + h * 32 + lane) : 0.f;
        tc::mbar_wait(&tfull[buf], bph);
        tc::tc_fence_after();
#pragma unroll
        for (int m = 0; m < CT; ++m) {
          float v[64];
          const uint32_t ta = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * CT * kTcN + m * kTcN + h * 64);
          tc::tmem_ld16_nowait(ta, v);
          tc::tmem_ld16_nowait(ta + 16, v + 16);
          tc::tmem_ld16_nowait(ta + 32, v + 32);
          tc::tmem_ld16_nowait(ta + 48, v + 48);
          tc::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float mod = tc::sqrt_approx(fmaf(v[2 * i], v[2 * i], v[2 * i + 1] * v[2 * i + 1]));
#pragma unroll
            for (int r = 0; r < KAP; ++r) oacc[m][r] = fmaf(__shfl_sync(0xffffffffu, wl[r], i), mod, oacc[m][r]);
          }
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tempty[buf]);
        if (++buf == 2) { buf = 0; bph ^= 1; }
      }
      // combine the two row halves in a fixed order, write o[rho][col]
      if (h == 1) {
#pragma unroll
        for (int m = 0; m < CT; ++m)
#pragma unroll
          for (int r = 0; r < KAP; ++r) red[(m * KAP + r) * 128 + c] = oacc[m][r];
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (h == 0) {
#pragma unroll
        for (int m = 0; m < CT; ++m) {
          const int64_t colg = col0 + m * 128 + c;
          if (colg < bf.n_cols) {
            float* dst = a.o + b * a.o_sb + U.o_off + colg;
#pragma unroll
            for (int r = 0; r < KAP; ++r)
              if (r < ro) dst[(int64_t)r * bf.n_cols] = oacc[m][r] + red[(m * KAP + r) * 128 + c];
          }
        }
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tbase, CT == 1 ? 256 : 512);
}

static size_t tc_smem(int CT, int KAP, int NS, int K2) {
  return (size_t)(2 * CT * 128 * K2 + NS * 2 * kTcN * kTcKc + CT * KAP * 128) * 4 + 1024;
}

template <int CT, int KAP>
static void launch_tc(const TcArgs& a, int K2max, int64_t ntiles, int B, cudaStream_t st) {
  // as many 32 KB B stages as fit next to the resident A tile (<= 8)
  int NS = kTcMaxStages;
  while (NS > 2 && tc_smem(CT, KAP, NS, K2max) > 225 * 1024) --NS;
  size_t sm = tc_smem(CT, KAP, NS, K2max);
  cudaFuncSetAttribute(k_joint_fwd_tc<CT, KAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  dim3 g((unsigned)ntiles, (unsigned)B);
  k_joint_fwd_tc<CT, KAP><<<g, kTcThreads, sm, st>>>(a, NS);
  count_launch();
}

void launch_joint_fwd_tc(const Plan& p, const DeviceTables& d, const float2* Y2, int64_t y_sb, float* o,
                         int64_t o_sb, int shard, int n_shards, int B, cudaStream_t st) {
  for (int cls = 0; cls < kTcClasses; ++cls) {
    const TcClass& C = d.tc[cls];
    if (C.n_blocks == 0) continue;
    TcArgs a{Y2, y_sb, o, o_sb, d.units, d.binfo, C.blocks, C.tiles, C.n_blocks, d.tc_img, d.tc_wts, d.tc_units,
             (int)p.L_fr.size(), shard, n_shards};
    // class = (CT, KAP): 0:(2,2) 1:(2,4) 2:(2,8) 3:(1,2) 4:(1,4) 5:(1,8)
    switch (cls) {
      case 0: launch_tc<2, 2>(a, C.K2max, C.ntiles, B, st); break;
      case 1: launch_tc<2, 4>(a, C.K2max, C.ntiles, B, st); break;
      case 2: launch_tc<2, 8>(a, C.K2max, C.ntiles, B, st); break;
      case 3: launch_tc<1, 2>(a, C.K2max, C.ntiles, B, st); break;
      case 4: launch_tc<1, 4>(a, C.K2max, C.ntiles, B, st); break;
      case 5: launch_tc<1, 8>(a, C.K2max, C.ntiles, B, st); break;
    }
  }
}

}  // namespace jtfs
