// kernels_tc.cu — the joint lambda_1 stage (SURVEY §8(a) A5 forward, A7 backward) on the
// 5th-generation tensor cores (tcgen05, kind::tf32, accumulators in TMEM).
//
// For one block n2 and a tile of 128 time columns, every frequential filter f is the exact dense
// matrix M_f[r][n] = h_f[(r 2^k_f - n) mod P] (zero-pad to P, circular convolution along n1,
// decimation by 2^k_f: P:276-295). The complex product W_f^T = Y2^T M_f^T is a real GEMM
//     D[c][2r+po] = sum_{n,pi} A[c][2n+pi] B[2r+po][2n+pi]
// with A[c][2n+pi] = (Re,Im) Y2[n][c] and B = [[Re M, -Im M], [Im M, Re M]] interleaved, so that
// TMEM lane c (a time column) holds Re/Im W of 64 consecutive lambda_1 rows side by side. 3xTF32:
// D = A_hi B_hi + A_hi B_lo + A_lo B_hi, fp32 accumulation in TMEM (north_star: "a genuine dense
// contraction with a 3xTF32 split"). B is the same for every column tile and signal: the planner
// pre-splits it into tf32 hi/lo images in the canonical K-major layout, streamed by the bulk-copy
// engine (cp.async.bulk) through an mbarrier ring; A (the Y2 tile) stays resident in SMEM.
//
// Forward (k_joint_fwd_tc):  warp 0 producer, warp 1 MMA issuer (elected lane), warps 4..11
//   epilogue: tcgen05.ld -> |W| (Eq.2) -> phi_F over rows (Eq.4, R17) in registers -> o.
//   TMEM double buffered: the epilogue of row tile t overlaps the MMAs of row tile t+1.
// Backward (k_joint_bwd_tc), per 32-row tile g of every filter:
//   GEMM1  D1 = W recomputed (forward B images, N = 64)
//   epi    g_W = (W/|W|) Phi_F^T g_o (R22 dead zone) -> tf32 hi/lo -> TMEM (tcgen05.st) = A2
//   GEMM2  D2[c][2n+po] += sum_kk A2[c][kk] B2[2n+po][kk] (A from TMEM), B2 = conj(M_f) images,
//          i.e. g_Y2^T += g_W^T conj(M_f), accumulated in TMEM over all filters and row tiles.
//   The MMA warp issues GEMM1(g+1) before GEMM2(g), so the tensor core works while the epilogue
//   turns D1(g) into A2(g).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "device.cuh"
#include "tc.cuh"

namespace jtfs {

constexpr int kTcRows = 64;         // lambda_1 rows per forward row tile (N = 128)
constexpr int kTcN = 2 * kTcRows;   // forward MMA N
constexpr int kTcThreads = 384;     // 12 warps
constexpr int kTcMaxStages = 8;
constexpr int kTcMaxStages2 = 16;   // backward ring 2 (B2 chunks)
constexpr int kBwRows = 32;         // rows per backward tile (GEMM1 N = 64, GEMM2 K = 64)
#ifndef JTFS_BW_EPIW
#define JTFS_BW_EPIW 16
#endif
constexpr int kBwEpiWarps = JTFS_BW_EPIW;   // backward epilogue warps: 4 TMEM lane quadrants x 4 (or 2) row groups
constexpr int kBwRpw = kBwRows / (kBwEpiWarps / 4);            // rows per epilogue warp (8)
constexpr int kBwThreads = 128 + 32 * kBwEpiWarps;             // + producers / MMA issuers (warps 0-3)
constexpr int kBwN1 = 2 * kBwRows;

__device__ __forceinline__ int find_tc(const int64_t* __restrict__ tiles, int n, int64_t t) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (__ldg(tiles + mid) <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// A tile: Y2[n0 + n][col0 + c] -> tf32 hi/lo, canonical K-major [128][K2], k' = 2n + (re, im)
__device__ __forceinline__ void build_a(float* a_hi, float* a_lo, const float2* __restrict__ ysrc,
                                        const BlockInfo& bf, int64_t col0, int K, int K2, int tid, int nthr,
                                        int n0 = 0) {
  for (int idx = tid; idx < 128 * (K2 / 2); idx += nthr) {
    const int c = idx & 127;
    const int n = idx >> 7;
    const int64_t col = col0 + c;
    float2 v = make_float2(0.f, 0.f);
    if (n0 + n < K && col < bf.n_cols) v = ysrc[(int64_t)(n0 + n) * bf.T2 + (bf.c_lo + col) % bf.T2];
    float h0, l0, h1, l1;
    tc::split_tf32(v.x, h0, l0);
    tc::split_tf32(v.y, h1, l1);
    const uint32_t o = tc::core_off((uint32_t)c, (uint32_t)(2 * n), (uint32_t)K2) / 4;
    if (a_hi) *reinterpret_cast<float2*>(a_hi + o) = make_float2(h0, h1);
    *reinterpret_cast<float2*>(a_lo + o) = make_float2(l0, l1);
  }
}

struct TcArgs {
  const float2* Y2; int64_t y_sb;
  float* o; int64_t o_sb;
  const JointUnit* units; const BlockInfo* binfo;
  const TcBlock* blocks; const int64_t* tiles; int n_tc_blocks;
  const float* img;                 // forward B images
  const float* wts;                 // phi_F weights [unit][rho][NT*64]
  const TcUnit* tcu;                // per unit image / weight offsets
  int nfr;
  uint64_t own;
  float* wbuf; int64_t wb_sb;       // split-K blocks: per-signal W buffer
  int part, pmode;                  // K part of this launch; kPm* bits
  int ng;                           // filter groups: CTA x handles column tile x % ntiles, filters f = x / ntiles mod ng
  long long* trace;                 // JTFS_TC_TRACE builds: per-tile event clocks of CTA (0, 0)
  int fexpt;                        // timing experiments only (JTFS_TC_FEXPT: 1 no W loads, 2 no W stores,
                                    // 4 no B-image copies after the first two tiles, 8 no modulus / phi_F)
  const float* thr;                 // per-signal modulus dead zone (R22), for the kept phase store
};
// K-part modes: load / store the fp32 W partials, finish (modulus, phi_F), and keep the phase of the final W
// for the backward (kPmPhase, "phase store": the backward needs only W/|W| and the dead-zone decision)
constexpr int kPmLoad = 1, kPmStore = 2, kPmFinish = 4, kPmPhase = 8;
constexpr float kPhaseScale = 32767.f;   // phase store: 2 x int16 fixed point per cell (|error| <= 1.6e-5)
static const int g_tc_fexpt = [] {
  const char* e = std::getenv("JTFS_TC_FEXPT");
  return e ? std::atoi(e) : 0;
}();
#ifdef JTFS_TC_TRACE
#define TC_TRACE(ev, g)                                                                  \
  do {                                                                                   \
    if (a.trace && blockIdx.x == 0 && blockIdx.y == 0 && (g) < 512) a.trace[(ev) * 512 + (g)] = clock64(); \
  } while (0)
#else
#define TC_TRACE(ev, g) do {} while (0)
#endif

// =====================================================================================
// forward
// =====================================================================================
template <int CT, int KAP>
__global__ void __launch_bounds__(kTcThreads, 1) k_joint_fwd_tc(TcArgs a, int NS, int STG) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[kTcMaxStages], empty[kTcMaxStages], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  // logical warp roles: 0 producer, 1 MMA issuer, 4.. epilogue. The epilogue occupies the LOW physical
  // warps so the producer and the MMA issuer get the higher warp ids, which the scheduler favours
  // (highest-id-first arbitration): otherwise the busy epilogue warps starve the issuing warp.
  const int tid = threadIdx.x, lane = tid & 31, pw = tid >> 5;
  const int warp = pw >= 8 ? pw - 8 : pw + 4;
  const int jb = 0;                                         // one block per launch
  const int ntl = (int)(a.tiles[1] - a.tiles[0]);
  const int ct = (int)blockIdx.x % ntl, grp = (int)blockIdx.x / ntl;
  const TcBlock TB = a.blocks[jb];
  const BlockInfo bf = a.binfo[TB.bi];
  const int64_t col0 = (int64_t)ct * (128 * CT);
  const int b = blockIdx.y;
  const int K = TB.K, kcw = TB.kcw;
  const int kp_lo = TB.ks ? a.part * TB.kpw : 0;            // k' range of this launch (split-K blocks)
  const int K2 = TB.ks ? min(TB.kpw, TB.K2 - kp_lo) : TB.K2;
  const int pmode = TB.ks ? a.pmode : kPmFinish;
  // A (the Y2 tile, tf32 hi/lo) placement: both halves in TMEM (tsa, TS-form MMAs), both in SMEM (SS form),
  // or hybrid (hyb, CT = 1): A_hi in TMEM and A_lo in SMEM -- a whole K up to 384 in one part, so split-K
  // blocks need no fp32 W partials round trip through HBM
  const bool hyb = TB.hyb != 0;
  const bool tsa = !hyb && tc_fwd_tsa(CT, K2);            // A in TMEM (TS-form MMAs)
  const int nbuf = hyb ? (256 + K2 <= 512 ? 2 : 1) : tc_fwd_nbuf(CT, K2);   // TMEM accumulator buffers
  float* a_hi = reinterpret_cast<float*>(sm);              // [CT][128][K2] canonical (SS form)
  float* a_lo = hyb ? a_hi : a_hi + CT * 128 * K2;         // hybrid: only A_lo in SMEM
  float* bst = tsa ? a_hi : a_lo + CT * 128 * K2;           // NS stages x STG floats
  float* red = bst + NS * STG;                              // [CT][KAP][128]
  float* swt = red + CT * KAP * 128;                        // KAP <= 8: [8 epilogue warps][32 rows][KAP] phi_F weights

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { tc::mbar_init(&tfull[s], 1); tc::mbar_init(&tempty[s], 8); }
    tc::fence_mbar_init();
  }
  const int tcols = (CT == 1 && !tsa && !hyb) ? 256 : 512;
  if (warp == 1) tc::tmem_alloc(&tmem_base, tcols);
  const float2* ysrc = a.Y2 + b * a.y_sb + bf.y_off;
  if (!tsa && !hyb)
    for (int m = 0; m < CT; ++m)
      build_a(a_hi + m * 128 * K2, a_lo + m * 128 * K2, ysrc, bf, col0 + m * 128, K, K2, tid, kTcThreads, kp_lo / 2);
  if (hyb) build_a(nullptr, a_lo, ysrc, bf, col0, K, K2, tid, kTcThreads, kp_lo / 2);
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = tmem_base;
  // TS form: A hi at TMEM columns [256, 256 + K2), lo at [256 + K2, 256 + 2 K2)
  const uint32_t taa_hi = tbase + 128 * (uint32_t)nbuf, taa_lo = taa_hi + (uint32_t)K2;
  if (tsa || hyb) {
    if (warp >= 4 && warp < 8) {
      const uint32_t lq = (uint32_t)((warp & 3) * 32) << 16;
      const int64_t col = col0 + (warp & 3) * 32 + lane;
      const float2* ycol = ysrc + (bf.c_lo + (col < bf.n_cols ? col : 0)) % bf.T2;
      const int n0 = kp_lo / 2;
      for (int k0 = 0; k0 < K2; k0 += 16) {
        float hi[16], lo[16];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int n = n0 + k0 / 2 + j;
          float2 v = make_float2(0.f, 0.f);
          if (n < K && k0 / 2 + j < K2 / 2 && col < bf.n_cols) v = ycol[(int64_t)n * bf.T2];
          tc::split_tf32(v.x, hi[2 * j], lo[2 * j]);
          tc::split_tf32(v.y, hi[2 * j + 1], lo[2 * j + 1]);
        }
        if (K2 - k0 >= 16) {
          tc::tmem_st16(taa_hi + lq + (uint32_t)k0, hi);
          if (!hyb) tc::tmem_st16(taa_lo + lq + (uint32_t)k0, lo);
        } else {
          tc::tmem_st8(taa_hi + lq + (uint32_t)k0, hi);
          if (!hyb) tc::tmem_st8(taa_lo + lq + (uint32_t)k0, lo);
        }
      }
      tc::tmem_wait_st();
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
  }
  const int nchunks = (K2 + kcw - 1) / kcw;
  // Two MMA issuers (see below) when there are two accumulator buffers: tiles alternate between them and
  // so do the B stages, split into two rings of NS / 2 stages (one ring per issuer: a stage is then only
  // ever waited on by one thread, which keeps the parity waits unambiguous). A ring needs >= 2 stages
  // when a tile spans several chunks (load of chunk c + 1 under the MMAs of chunk c).
  const int nis = (nbuf == 2 && NS >= 2 && (nchunks == 1 || NS >= 4)) ? 2 : 1;
  const int NSr = NS / nis;

  if (warp == 0) {
    // ===================== producer: B chunks via the bulk-copy engine (one elected lane issues)
    int stage_r[2] = {0, 0}, gt = 0;
    uint32_t ph_r[2] = {0, 0};
    for (int f = 0; f < a.nfr; ++f) {
      const int u = TB.bi * a.nfr + f;
      if (!owns_block(a.own, TB.bi) || f % a.ng != grp) continue;
      const TcUnit tu = a.tcu[u];
      for (int t = 0; t < tu.NT; ++t) {
        // row tile t of the unit's image: chunks of the full K2, starting at this launch's k' range
        const float* src = a.img + tu.img_off + (int64_t)t * (2 * kTcN * TB.K2) + 2 * kTcN * kp_lo;
        const int r = gt % nis;
        int& stage = stage_r[r];
        uint32_t& ph = ph_r[r];
        for (int ch = 0; ch < nchunks; ++ch) {
          const int kc = min(kcw, K2 - ch * kcw);
          const uint32_t bytes = (uint32_t)(2 * kTcN * kc * 4);
          const int sg = r * NSr + stage;
          tc::mbar_wait(&empty[sg], ph ^ 1);
          if ((a.fexpt & 4) && gt > 1) {   // timing experiment: B images of the first tiles only
            if (tc::elect_one()) tc::mbar_arrive(&full[sg]);
          } else if (tc::elect_one()) {
            tc::mbar_expect_tx(&full[sg], bytes);
            tc::bulk_g2s(bst + sg * STG, src, bytes, &full[sg]);
          }
          __syncwarp();
          src += 2 * kTcN * kc;
          if (++stage == NSr) { stage = 0; ph ^= 1; }
        }
        ++gt;
      }
    }
  } else if (warp == 1 || (warp == 3 && nis == 2)) {
    // ===================== MMA issuers (warp-uniform loops, one elected lane issues). The tensor pipe's
    // issue queue holds only ~3 MMAs (~200 cycles of N=128 work) while a commit plus a barrier wait costs
    // ~200 cycles even when the phase has completed (tools/ubench/tmem_mma.cu k_issue), so one issuer
    // drains the pipe at every chunk and tile boundary. With two accumulator buffers, warp 1 issues the
    // even tiles (buffer 0, stage ring 0) and warp 3 the odd ones (buffer 1, ring 1): one's waits overlap
    // the other's MMAs.
    const int q = warp == 3 ? 1 : 0;
    // a unit's last row tile with <= 32 rows runs N = 64 MMAs (rows 32..63 are padding)
    const uint32_t idesc_full = tc::idesc_tf32(128, kTcN), idesc_half = tc::idesc_tf32(128, kTcN / 2);
    const uint32_t sboA = (uint32_t)K2 * 32u;
    // descriptors differ only in the start-address field: add (byte offset >> 4) to the low word
    const uint64_t dA_hi = tc::sdesc(tc::smem_u32(a_hi), 128, sboA);
    const uint64_t dA_lo = tc::sdesc(tc::smem_u32(a_lo), 128, sboA);
    const uint32_t aStepM = (uint32_t)(128 * K2 * 4) >> 4;
    const uint32_t bst_s = tc::smem_u32(bst);
    int stage = 0, gt = 0;
    int buf = q;
    uint32_t ph = 0, bph = 0;
    for (int f = 0; f < a.nfr; ++f) {
      const int u = TB.bi * a.nfr + f;
      if (!owns_block(a.own, TB.bi) || f % a.ng != grp) continue;
      const TcUnit tu = a.tcu[u];
      for (int t = 0; t < tu.NT; ++t) {
        if (gt % nis != q) {   // the other issuer's tile (other ring)
          ++gt;
          continue;
        }
        tc::mbar_wait(&tempty[buf], bph ^ 1);
        tc::tc_fence_after();
        if (lane == 0) TC_TRACE(0, gt);
        const uint32_t dbase = tbase + (uint32_t)(buf * CT * kTcN);
        const uint32_t idesc = (t == tu.NT - 1 && a.units[u].n_rows - t * kTcRows <= kTcRows / 2) ? idesc_half
                                                                                                  : idesc_full;
        for (int ch = 0; ch < nchunks; ++ch) {
          const int kc = min(kcw, K2 - ch * kcw);
          tc::mbar_wait(&full[q * NSr + stage], ph);
          tc::tc_fence_after();
          if (lane == 0 && ch == 0) TC_TRACE(1, gt);
          const uint32_t bh = bst_s + (uint32_t)((q * NSr + stage) * STG * 4);
          const uint64_t dB_hi = tc::sdesc(bh, 128, (uint32_t)kc * 32u);
          const uint64_t dB_lo = tc::sdesc(bh + (uint32_t)(kTcN * kc * 4), 128, (uint32_t)kc * 32u);
          if (tc::elect_one()) {
            for (int ks = 0; ks < kc / 8; ++ks) {
              const uint32_t kg = (uint32_t)(ch * (kcw / 8) + ks);
              if (tsa) {
                tc::mma_tf32_ts(dbase, taa_hi + 8u * kg, dB_hi + 16u * ks, idesc, (ch > 0 || ks > 0) ? 1u : 0u);
                tc::mma_tf32_ts(dbase, taa_hi + 8u * kg, dB_lo + 16u * ks, idesc, 1u);
                tc::mma_tf32_ts(dbase, taa_lo + 8u * kg, dB_hi + 16u * ks, idesc, 1u);
              } else if (hyb) {   // A_hi from TMEM (TS form), A_lo from SMEM (SS form)
                tc::mma_tf32_ts(dbase, taa_hi + 8u * kg, dB_hi + 16u * ks, idesc, (ch > 0 || ks > 0) ? 1u : 0u);
                tc::mma_tf32_ts(dbase, taa_hi + 8u * kg, dB_lo + 16u * ks, idesc, 1u);
                tc::mma_tf32(dbase, dA_lo + 16u * kg, dB_hi + 16u * ks, idesc, 1u);
              } else {
#pragma unroll
                for (int m = 0; m < CT; ++m) {
                  const uint32_t d = dbase + (uint32_t)(m * kTcN);
                  const uint64_t ao = (uint64_t)(m * aStepM + 16u * kg);
                  tc::mma_tf32(d, dA_hi + ao, dB_hi + 16u * ks, idesc, (ch > 0 || ks > 0) ? 1u : 0u);
                  tc::mma_tf32(d, dA_hi + ao, dB_lo + 16u * ks, idesc, 1u);
                  tc::mma_tf32(d, dA_lo + ao, dB_hi + 16u * ks, idesc, 1u);
                }
              }
            }
            tc::mma_commit(&empty[q * NSr + stage]);
          }
          __syncwarp();
          if (++stage == NSr) { stage = 0; ph ^= 1; }
        }
        if (tc::elect_one()) tc::mma_commit(&tfull[buf]);
        __syncwarp();
        if (lane == 0) TC_TRACE(2, gt);
        ++gt;
        if (nis == 2) bph ^= 1;                          // own buffer q, every own tile
        else if (++buf == nbuf) { buf = 0; bph ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: |W| and phi_F over rows, per time column (TMEM lane)
    const int e = warp - 4;
    const int q = e & 3, h = e >> 2;        // lane quadrant, column half (32 complex rows)
    const int c = q * 32 + lane;            // time column within the tile
    int buf = 0, ge = 0;
    uint32_t bph = 0;
    for (int f = 0; f < a.nfr; ++f) {
      const int u = TB.bi * a.nfr + f;
      if (!owns_block(a.own, TB.bi) || f % a.ng != grp) continue;
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
        // lane l stages the phi_F weights of row (t*64 + h*32 + l) in the warp's SMEM slab [row][KAP]; the math
        // below reads a row's weights as broadcast vector loads (one LDS per 2-4 outputs instead of one SHFL
        // per output). The previous tile's reads are done: same warp, program order, then __syncwarp.
        float wl[KAP];   // KAP >= 16: kept in registers and broadcast by shuffles (the slab would cost stages)
#pragma unroll
        for (int r = 0; r < KAP; ++r) wl[r] = (r < ro) ? __ldg(wt + r * ldw + t * kTcRows + h * 32 + lane) : 0.f;
        if constexpr (KAP <= 8) {
          __syncwarp();
          float* my = swt + (e * 32 + lane) * KAP;
          if constexpr (KAP >= 4) {
#pragma unroll
            for (int r = 0; r < KAP; r += 4)
              *reinterpret_cast<float4*>(my + r) = make_float4(wl[r], wl[r + 1], wl[r + 2], wl[r + 3]);
          } else {
            *reinterpret_cast<float2*>(my) = make_float2(wl[0], wl[1]);
          }
          __syncwarp();
        }
        tc::mbar_wait(&tfull[buf], bph);
        tc::tc_fence_after();
        if (warp == 4 && lane == 0) TC_TRACE(5, ge);
        // rows h*32 .. of a half tile (see the issuer) are padding and their TMEM columns were not written
        const bool skip = h == 1 && t == tu.NT - 1 && U.n_rows - t * kTcRows <= kTcRows / 2;
#pragma unroll
        for (int m = 0; m < CT; ++m) {
          float v[64];
          const uint32_t ta = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * CT * kTcN + m * kTcN + h * 64);
          if (skip) {
            if (m == CT - 1) {
              tc::tc_fence_before();
              __syncwarp();
              if (lane == 0) tc::mbar_arrive(&tempty[buf]);
            }
            continue;
          }
          tc::tmem_ld16_nowait(ta, v);
          tc::tmem_ld16_nowait(ta + 16, v + 16);
          tc::tmem_ld16_nowait(ta + 32, v + 32);
          tc::tmem_ld16_nowait(ta + 48, v + 48);
          tc::tmem_wait_ld();
          if (m == CT - 1) {
            // the accumulator buffer is free once its last column block sits in registers: release it
            // before the math so the next tile's MMAs overlap it (essential with one buffer, K2 > 128)
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[buf]);
          }
          if (pmode != kPmFinish) {
            // split-K: W of (tile t, column c, rows h*32 ..) accumulated across the K parts. Layout per
            // (column tile, 64-row tile): [float4 group g = (2 row + re/im) / 4][column c] -- a warp's 32
            // columns of one group are 512 contiguous bytes (coalesced loads and stores)
            float4* wp = reinterpret_cast<float4*>(a.wbuf + b * a.wb_sb + TB.wp_off) +
                         ((int64_t)ct * TB.wp_tiles + tu.wp_tile0 + t) * (128 * 32) + (h * 16) * 128 + c;
            if ((pmode & kPmLoad) && !(a.fexpt & 1)) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float4 w = wp[i * 128];
                v[4 * i] += w.x; v[4 * i + 1] += w.y; v[4 * i + 2] += w.z; v[4 * i + 3] += w.w;
              }
            }
            if ((pmode & kPmStore) && !(pmode & kPmPhase) && !(a.fexpt & 2)) {
#pragma unroll
              for (int i = 0; i < 16; ++i)
                wp[i * 128] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            }
            if ((pmode & kPmPhase) && !(a.fexpt & 2)) {
              // phase store: per cell (c, s) = round(32767 W/|W|) as two int16 (0 in the R22 dead zone, decided
              // here on the final fp32 W exactly as the backward's recompute path decides it); per (column
              // tile, 64-row tile) [16-byte group][column c], 4 rows per group, so a warp's 32 columns of one
              // group are 512 contiguous bytes; half the bytes of the fp32 W
              const float th2 = fmaxf(a.thr[b] * a.thr[b], 1.17549435e-38f);
              // half h's groups start at h * wph / 256: with fp32 partials in the tile (wph = 4096) that is the
              // start of the half's own partial region, which only this thread (column c) has read -- the
              // store never overwrites a partial another thread still has to load
              uint4* pq = reinterpret_cast<uint4*>(a.wbuf + b * a.wb_sb + TB.wp_off) +
                          ((int64_t)ct * TB.wp_tiles + tu.wp_tile0 + t) * TB.wph + (h * (TB.wph >> 8)) * 128 + c;
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                uint32_t wd[4];
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                  const float re = v[8 * i + 2 * q4], im = v[8 * i + 2 * q4 + 1];
                  const float m2 = fmaf(re, re, im * im);
                  int cs = 0, sn = 0;
                  if (m2 > th2) {
                    const float sc = kPhaseScale * rsqrtf(m2);
                    cs = __float2int_rn(fminf(fmaxf(re * sc, -kPhaseScale), kPhaseScale));
                    sn = __float2int_rn(fminf(fmaxf(im * sc, -kPhaseScale), kPhaseScale));
                  }
                  wd[q4] = (uint32_t)(uint16_t)(int16_t)cs | ((uint32_t)(uint16_t)(int16_t)sn << 16);
                }
                pq[i * 128] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
              }
            }
            if (!(pmode & kPmFinish)) continue;
          }
          if (a.fexpt & 8) {   // timing experiment: no modulus / phi_F math
#pragma unroll
            for (int r = 0; r < KAP; ++r) oacc[m][r] += v[r];
            continue;
          }
          const float* sw = swt + e * 32 * KAP;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float mod = tc::sqrt_approx(fmaf(v[2 * i], v[2 * i], v[2 * i + 1] * v[2 * i + 1]));
#pragma unroll
            for (int r = 0; r < KAP; r += 2) {   // outputs r, r + 1 as one packed FMA (FFMA2, bit-identical)
              float2 w2;
              if constexpr (KAP > 8) {
                w2 = make_float2(__shfl_sync(0xffffffffu, wl[r], i), __shfl_sync(0xffffffffu, wl[r + 1], i));
              } else if constexpr (KAP >= 4) {
                const float4 w4 = *reinterpret_cast<const float4*>(sw + i * KAP + (r & ~3));   // broadcast
                w2 = (r & 2) ? make_float2(w4.z, w4.w) : make_float2(w4.x, w4.y);
              } else {
                w2 = *reinterpret_cast<const float2*>(sw + i * KAP);
              }
              const float2 o2 = tc::fma2(w2, make_float2(mod, mod), make_float2(oacc[m][r], oacc[m][r + 1]));
              oacc[m][r] = o2.x;
              oacc[m][r + 1] = o2.y;
            }
          }
        }
        if (warp == 4 && lane == 0) TC_TRACE(6, ge);
        ++ge;
        if (++buf == nbuf) { buf = 0; bph ^= 1; }
      }
      if (!(pmode & kPmFinish)) continue;
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
  if (warp == 1) tc::tmem_dealloc(tbase, tcols);
}

static size_t tc_fwd_smem(int CT, int KAP, int NS, int K2, int STG, bool hyb = false) {
  const size_t a = hyb ? (size_t)128 * K2 : (tc_fwd_tsa(CT, K2) ? 0 : (size_t)2 * CT * 128 * K2);
  return (a + NS * STG + CT * KAP * 128 + (KAP <= 8 ? 8 * 32 * KAP : 0)) * 4 + 1024;
}

// forward B ring stages that fit (the planner rejects chunk widths that leave fewer than 3; 2 in hybrid mode)
int tc_fwd_stages(int CT, int KAP, int K2, int kcw, bool hyb) {
  const int STG = 2 * kTcN * kcw;
  int NS = kTcMaxStages;
  while (NS > 0 && tc_fwd_smem(CT, KAP, NS, K2, STG, hyb) > 224 * 1024) --NS;
  return NS;
}

#ifdef JTFS_TC_TRACE
static const int g_trace_fwd_k = [] {
  const char* e = std::getenv("JTFS_TRACE_K");
  return e ? std::atoi(e) : 34;
}();
#endif

// filter groups of a launch: fixed per block by the planner (about two waves of 148 SMs per signal),
// independent of the batch so that micro-batching leaves every summation order, hence the bits, unchanged
static int tc_groups(const TcClass& C, int B) {
  (void)B;
  return C.ngmax;
}

template <int CT, int KAP>
static void launch_tc(const TcArgs& a, const TcClass& C, int B, cudaStream_t st) {
  const int STG = 2 * kTcN * C.kcw;
  const int NS = tc_fwd_stages(CT, KAP, C.K2max, C.kcw, C.hyb != 0);
  const size_t sm = tc_fwd_smem(CT, KAP, NS, C.K2max, STG, C.hyb != 0);
  cudaFuncSetAttribute(k_joint_fwd_tc<CT, KAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  dim3 g((unsigned)(C.ntiles * a.ng), (unsigned)B);
  k_joint_fwd_tc<CT, KAP><<<g, kTcThreads, sm, st>>>(a, NS, STG);
  count_launch();
}

void launch_joint_fwd_tc(const Plan& p, const DeviceTables& d, const float2* Y2, int64_t y_sb, float* o,
                         int64_t o_sb, float* wbuf, int64_t wb_sb, bool keep_w, const float* thr, uint64_t own, int B,
                         const cudaStream_t* ss, int ns) {
  int li = 0;
  for (const TcClass& C : d.tc) {
    const cudaStream_t st = ss[li++ % ns];
    if (C.n_blocks == 0 || !owns_block(own, C.bi)) continue;   // path shards: own blocks only
    const int nparts = C.ks ? C.nparts : 1;
    for (int part = 0; part < nparts; ++part) {   // split-K parts run in order on one stream
      int pmode = kPmFinish;
      if (C.ks) {
        pmode = (part > 0 ? kPmLoad : 0) | (part < nparts - 1 ? kPmStore : 0) |
                (part == nparts - 1 ? kPmFinish | (keep_w ? kPmPhase : 0) : 0);
      }
      TcArgs a{Y2, y_sb, o, o_sb, d.units, d.binfo, C.blocks, C.tiles, C.n_blocks, d.tc_img, d.tc_wts, d.tc_units,
               (int)p.L_fr.size(), own, wbuf, wb_sb, part, pmode, tc_groups(C, B), nullptr, g_tc_fexpt, thr};
#ifdef JTFS_TC_TRACE
      static long long* ftrace = nullptr;
      if (!ftrace) cudaMalloc(&ftrace, 16 * 512 * 8);
      if (C.Kmax == g_trace_fwd_k && part == 0) { cudaMemsetAsync(ftrace, 0, 16 * 512 * 8, st); a.trace = ftrace; }
#endif
      // class = 8 * ct_kind + kap_kind (CT = 2 for ct_kind 0)
      switch (C.cls) {
        case 0: launch_tc<2, 2>(a, C, B, st); break;
        case 1: launch_tc<2, 4>(a, C, B, st); break;
        case 2: launch_tc<2, 8>(a, C, B, st); break;
        case 8: launch_tc<1, 2>(a, C, B, st); break;
        case 9: launch_tc<1, 4>(a, C, B, st); break;
        case 10: launch_tc<1, 8>(a, C, B, st); break;
        case 11: launch_tc<1, 16>(a, C, B, st); break;
        case 12: launch_tc<1, 32>(a, C, B, st); break;
      }
#ifdef JTFS_TC_TRACE
      if (a.trace) {
        static long long h[16 * 512];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, a.trace, sizeof(h), cudaMemcpyDeviceToHost);
        if (FILE* fo = fopen("gpurun_out/tc_trace_fwd.bin", "wb")) { fwrite(h, 1, sizeof(h), fo); fclose(fo); }
      }
#endif
    }
  }
}

// =====================================================================================
// backward
// =====================================================================================
struct TcBwArgs {
  const float2* Y2; int64_t y_sb;
  const float* go; int64_t go_sb;
  float2* gY; int64_t gy_sb;
  const JointUnit* units; const BlockInfo* binfo;
  const TcBlock* blocks; const int64_t* tiles; int n_tc_blocks;
  const float* img;                 // forward B images (64-row tiles, kcw-wide chunks)
  const float* img2;                // backward B2 images [unit][tile32][chunk][hi|lo][N2 x kb2]
  const float* img1b;               // backward GEMM1 images [unit][tile32][chunk][hi|lo][64 x kc]
  const float* wts;
  const TcUnit* tcu;
  int nfr;
  uint64_t own;
  const float* thr;
  int expt;                         // timing experiments only (JTFS_TC_EXPT); 0 in production
  const float* wbuf; int64_t wb_sb; // split-K blocks: W left by the forward (GEMM1 skipped)
  int ng;                           // filter groups (see TcArgs); ng > 1: D2 partials to gp, reduced after
  float2* gp; int64_t gp_sb;
  long long* trace;                 // JTFS_TC_TRACE builds: per-tile event clocks of CTA (0, 0)
  int bmode;                        // tc_bwd_mode preference (tc_bwd_mode_pref)
};


template <int KAP>
__global__ void __launch_bounds__(kBwThreads, 1) k_joint_bwd_tc(TcBwArgs a, int NS1, int STG1, int NS2, int STG2) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full1[kTcMaxStages], empty1[kTcMaxStages], full2[kTcMaxStages2], empty2[kTcMaxStages2];
  // tile barriers in one struct: the epilogue addresses them from one base register (see eb below)
  __shared__ struct { uint64_t tfull[2], tempty[2], a2full[2], a2empty[2], d2full; } tb_;
  uint64_t* const tfull = tb_.tfull; uint64_t* const tempty = tb_.tempty;
  uint64_t* const a2full = tb_.a2full; uint64_t* const a2empty = tb_.a2empty;
  uint64_t& d2full = tb_.d2full;
  __shared__ uint32_t tmem_base;
  // logical warp roles: 0/2 producers, 1/3 MMA issuers, 4.. epilogue (epilogue on the low physical warps so
  // the producers and issuers get the higher, favoured warp ids; see the forward kernel)
  const int tid = threadIdx.x, lane = tid & 31, pw = tid >> 5;
  const int warp = pw >= kBwEpiWarps ? pw - kBwEpiWarps : pw + 4;
  const int jb = 0;                                     // one block per launch
  const int ntl = (int)(a.tiles[1] - a.tiles[0]);
  const int ct = (int)blockIdx.x % ntl, grp = (int)blockIdx.x / ntl;
  const TcBlock TB = a.blocks[jb];
  const BlockInfo bf = a.binfo[TB.bi];
  const int64_t col0 = (int64_t)ct * 128;
  const int b = blockIdx.y;
  const int K = TB.K, K2 = TB.K2, kcw = TB.kcw, kB2c = TB.kb2;
  const int N2 = ((2 * K + 15) / 16) * 16;
  const bool ksm = TB.ks != 0;                         // split-K block: W from the forward, no GEMM1
  int nab, ta;                                         // A2 buffers; Y2 tile in TMEM (GEMM1 TS form)
  if (ksm) { nab = N2 <= 256 ? 2 : 1; ta = 0; }
  else tc_bwd_mode(K, K2, &nab, &ta, a.bmode);
  float* a_hi = reinterpret_cast<float*>(sm);          // [128][K2] (SMEM mode only)
  float* a_lo = a_hi + 128 * K2;
  float* bst1 = (ta || ksm) ? a_hi : a_lo + 128 * K2;   // ring 1 (GEMM1 B images): NS1 x STG1 floats
  float* bst2 = bst1 + NS1 * STG1;                      // ring 2 (GEMM2 B2 images): NS2 x STG2 floats

  if (tid == 0) {
    for (int s = 0; s < NS1; ++s) { tc::mbar_init(&full1[s], 1); tc::mbar_init(&empty1[s], 1); }
    for (int s = 0; s < NS2; ++s) { tc::mbar_init(&full2[s], 1); tc::mbar_init(&empty2[s], 1); }
    for (int s = 0; s < 2; ++s) { tc::mbar_init(&tfull[s], 1); tc::mbar_init(&tempty[s], kBwEpiWarps); }
    for (int s = 0; s < 2; ++s) { tc::mbar_init(&a2full[s], kBwEpiWarps); tc::mbar_init(&a2empty[s], 1); }
    tc::mbar_init(&d2full, 1);
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(&tmem_base, 512);
  if (!ta && !ksm) build_a(a_hi, a_lo, a.Y2 + b * a.y_sb + bf.y_off, bf, col0, K, K2, tid, kBwThreads);
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  // TMEM columns: D1 buffers [0,64) [64,128); A2 buffer j: hi [128+128j, +64), lo [192+128j, +64);
  // D2 [128+128 nab, +N2); TMEM mode: A hi [D2 end, +K2), A lo [+K2, +K2)
  const uint32_t tbase = tmem_base;
  const uint32_t ta2 = tbase + (ksm ? 0u : 128u);       // split-K: no D1
  const uint32_t d2 = ta2 + 128 * (uint32_t)nab;
  const uint32_t taa_hi = d2 + (uint32_t)N2, taa_lo = taa_hi + (uint32_t)K2;
  if (ta && warp >= 4 && warp < 8) {
    // Y2 tile -> tf32 hi/lo rows of TMEM (lane = time column, column = k' = 2n + re/im)
    const uint32_t lq = (uint32_t)((warp & 3) * 32) << 16;
    const int64_t col = col0 + (warp & 3) * 32 + lane;
    const float2* ysrc = a.Y2 + b * a.y_sb + bf.y_off + (bf.c_lo + (col < bf.n_cols ? col : 0)) % bf.T2;
    for (int k0 = 0; k0 < K2; k0 += 16) {
      float hi[16], lo[16];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int n = k0 / 2 + j;
        float2 v = make_float2(0.f, 0.f);
        if (n < K && col < bf.n_cols) v = ysrc[(int64_t)n * bf.T2];
        tc::split_tf32(v.x, hi[2 * j], lo[2 * j]);
        tc::split_tf32(v.y, hi[2 * j + 1], lo[2 * j + 1]);
      }
      if (K2 - k0 >= 16) {
        tc::tmem_st16(taa_hi + lq + (uint32_t)k0, hi);
        tc::tmem_st16(taa_lo + lq + (uint32_t)k0, lo);
      } else {
        tc::tmem_st8(taa_hi + lq + (uint32_t)k0, hi);
        tc::tmem_st8(taa_lo + lq + (uint32_t)k0, lo);
      }
    }
    tc::tmem_wait_st();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const int nchunks = (K2 + kcw - 1) / kcw;

  if (warp == 0 || warp == 2) {
    // ===================== producers: warp 0 streams the GEMM1 B images (ring 1), warp 2 the GEMM2
    // B2 images (ring 2); separate rings let B2 run ahead while GEMM2 waits for the epilogue
    const bool p1 = warp == 0;
    int stage = 0;
    uint32_t ph = 0;
    for (int f = 0; f < (p1 && ksm ? 0 : a.nfr); ++f) {   // no GEMM1 (ring 1) in split-K mode
      const int u = TB.bi * a.nfr + f;
      if (!owns_block(a.own, TB.bi) || f % a.ng != grp) continue;
      const TcUnit tu = a.tcu[u];
      const int NT32 = (int)((a.units[u].n_rows + kBwRows - 1) / kBwRows);
      for (int t32 = 0; t32 < NT32; ++t32) {
        if (p1) {
          // 32-row tile t32 of the backward GEMM1 images, every chunk [hi 64 x kc | lo 64 x kc]: one bulk
          // copy per chunk (each copy costs the SM's copy engine ~400 cycles whatever its size)
          const float* src = a.img1b + tu.img1b_off + (int64_t)t32 * (2 * kBwN1 * K2);
          for (int ch = 0; ch < nchunks; ++ch) {
            const int kc = min(kcw, K2 - ch * kcw);
            const uint32_t bytes = (uint32_t)(2 * kBwN1 * kc * 4);
            tc::mbar_wait(&empty1[stage], ph ^ 1);
            if ((a.expt & 2) && t32 > 0) {
              if (tc::elect_one()) tc::mbar_arrive(&full1[stage]);
            } else if (tc::elect_one()) {
              tc::mbar_expect_tx(&full1[stage], bytes);
              tc::bulk_g2s(bst1 + stage * STG1, src, bytes, &full1[stage]);
            }
            __syncwarp();
            src += 2 * kBwN1 * kc;
            if (++stage == NS1) { stage = 0; ph ^= 1; }
          }
        } else {
          const float* src = a.img2 + tu.img2_off + (int64_t)t32 * (2 * N2 * 64);
          for (int ch = 0; ch < 64 / kB2c; ++ch) {
            const uint32_t bytes = (uint32_t)(2 * N2 * kB2c * 4);
            tc::mbar_wait(&empty2[stage], ph ^ 1);
            if ((a.expt & 2) && t32 > 0) {
              if (tc::elect_one()) tc::mbar_arrive(&full2[stage]);
            } else if (tc::elect_one()) {
              tc::mbar_expect_tx(&full2[stage], bytes);
              tc::bulk_g2s(bst2 + stage * STG2, src, bytes, &full2[stage]);
            }
            __syncwarp();
            src += 2 * N2 * kB2c;
            if (++stage == NS2) { stage = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1 || warp == 3) {
    // ===================== MMA issuers: warp 1 GEMM1 (recompute W), warp 3 GEMM2 (g_Y2^T accumulation).
    // Two issuing threads keep the tensor pipe fed: GEMM1 of later tiles queues while GEMM2 waits for
    // the epilogue's A2 or its B2 chunk (tcgen05.commit tracks each thread's own MMAs).
    const uint32_t idesc1 = tc::idesc_tf32(128, kBwN1);
    // GEMM2 N = N2 (<= 384): UMMA N <= 256, so wider D2 is covered by two MMAs over row halves of B2
    const int N2a = N2 > 256 ? ((N2 / 2 + 15) / 16) * 16 : N2;
    const uint32_t idesc2 = tc::idesc_tf32(128, (uint32_t)N2a);
    const uint32_t idesc2b = tc::idesc_tf32(128, (uint32_t)(N2 - N2a > 0 ? N2 - N2a : 16));
    const uint32_t sboA = (uint32_t)K2 * 32u;
    const uint64_t dA_hi = tc::sdesc(tc::smem_u32(a_hi), 128, sboA);
    const uint64_t dA_lo = tc::sdesc(tc::smem_u32(a_lo), 128, sboA);
    const uint32_t bst1_s = tc::smem_u32(bst1), bst2_s = tc::smem_u32(bst2);
    int stage1 = 0, stage2 = 0, buf = 0;
    uint32_t ph1 = 0, ph2 = 0, bph = 0;
    int g2 = 0;   // GEMM2 count
    int g1 = 0;   // GEMM1 count
    auto gemm1 = [&]() {
      if (lane == 0) TC_TRACE(0, g1);
      tc::mbar_wait(&tempty[buf], bph ^ 1);
      if (lane == 0) TC_TRACE(13, g1);
      const uint32_t d = tbase + (uint32_t)(buf * kBwN1);
      for (int ch = 0; ch < nchunks; ++ch) {
        const int kc = min(kcw, K2 - ch * kcw);
        tc::mbar_wait(&full1[stage1], ph1);
        tc::tc_fence_after();
        if (lane == 0 && ch == 0) TC_TRACE(14, g1);
        const uint32_t off = bst1_s + (uint32_t)(stage1 * STG1 * 4);
        const uint64_t dbh = tc::sdesc(off, 128, (uint32_t)kc * 32u);
        const uint64_t dbl = tc::sdesc(off + (uint32_t)(kBwN1 * kc * 4), 128, (uint32_t)kc * 32u);
        if (tc::elect_one()) {
          for (int ks = 0; ks < kc / 8; ++ks) {
            const uint32_t kg = (uint32_t)(ch * (kcw / 8) + ks);
            if (ta) {
              tc::mma_tf32_ts(d, taa_hi + 8u * kg, dbh + 16u * ks, idesc1, (ch > 0 || ks > 0) ? 1u : 0u);
              tc::mma_tf32_ts(d, taa_hi + 8u * kg, dbl + 16u * ks, idesc1, 1u);
              tc::mma_tf32_ts(d, taa_lo + 8u * kg, dbh + 16u * ks, idesc1, 1u);
            } else {
              tc::mma_tf32(d, dA_hi + 16u * kg, dbh + 16u * ks, idesc1, (ch > 0 || ks > 0) ? 1u : 0u);
              tc::mma_tf32(d, dA_hi + 16u * kg, dbl + 16u * ks, idesc1, 1u);
              tc::mma_tf32(d, dA_lo + 16u * kg, dbh + 16u * ks, idesc1, 1u);
            }
          }
          tc::mma_commit(&empty1[stage1]);
          if (ch == nchunks - 1) tc::mma_commit(&tfull[buf]);
        }
        __syncwarp();
        if (++stage1 == NS1) { stage1 = 0; ph1 ^= 1; }
      }
      if (++buf == 2) { buf = 0; bph ^= 1; }
      if (lane == 0) TC_TRACE(1, g1);
      ++g1;
    };
    auto gemm2 = [&]() {
      if (lane == 0) TC_TRACE(2, g2);
      const int ab = nab == 2 ? (g2 & 1) : 0;
      const uint32_t aph = (uint32_t)((nab == 2 ? (g2 >> 1) : g2) & 1);
      const uint32_t ta2_hi = ta2 + 128u * ab, ta2_lo = ta2_hi + 64u;
      tc::mbar_wait(&a2full[ab], aph);
      tc::tc_fence_after();
      if (lane == 0) TC_TRACE(3, g2);
      for (int ch = 0; ch < 64 / kB2c; ++ch) {
        tc::mbar_wait(&full2[stage2], ph2);
        tc::tc_fence_after();
        if (lane == 0 && ch == 0) TC_TRACE(9, g2);
        if (lane == 0 && ch == 64 / kB2c - 1) TC_TRACE(11, g2);
        const uint32_t bh = bst2_s + (uint32_t)(stage2 * STG2 * 4);
        const uint64_t dbh = tc::sdesc(bh, 128, (uint32_t)kB2c * 32u);
        const uint64_t dbl = tc::sdesc(bh + (uint32_t)(N2 * kB2c * 4), 128, (uint32_t)kB2c * 32u);
        if (tc::elect_one()) {
          for (int ks = 0; ks < ((a.expt & 4) ? 0 : kB2c / 8); ++ks) {
            const uint32_t kg = (uint32_t)(ch * (kB2c / 8) + ks);
            tc::mma_tf32_ts(d2, ta2_hi + 8u * kg, dbh + 16u * ks, idesc2, (g2 > 0 || kg > 0) ? 1u : 0u);
            tc::mma_tf32_ts(d2, ta2_hi + 8u * kg, dbl + 16u * ks, idesc2, 1u);
            tc::mma_tf32_ts(d2, ta2_lo + 8u * kg, dbh + 16u * ks, idesc2, 1u);
            if (N2a < N2) {   // rows N2a .. N2-1 of B2 start (N2a / 8) core-matrix groups further
              const uint64_t o2 = (uint64_t)((N2a / 8) * kB2c * 32) >> 4;
              const uint32_t d2b = d2 + (uint32_t)N2a;
              tc::mma_tf32_ts(d2b, ta2_hi + 8u * kg, dbh + o2 + 16u * ks, idesc2b, (g2 > 0 || kg > 0) ? 1u : 0u);
              tc::mma_tf32_ts(d2b, ta2_hi + 8u * kg, dbl + o2 + 16u * ks, idesc2b, 1u);
              tc::mma_tf32_ts(d2b, ta2_lo + 8u * kg, dbh + o2 + 16u * ks, idesc2b, 1u);
            }
          }
          tc::mma_commit(&empty2[stage2]);
          if (ch == 64 / kB2c - 1) tc::mma_commit(&a2empty[ab]);
        }
        __syncwarp();
        if (lane == 0 && ch == 0) TC_TRACE(10, g2);
        if (lane == 0 && ch == 64 / kB2c - 1) TC_TRACE(12, g2);
        if (++stage2 == NS2) { stage2 = 0; ph2 ^= 1; }
      }
      if (lane == 0) TC_TRACE(4, g2);
      ++g2;
    };
    int G = 0;
    for (int f = 0; f < a.nfr; ++f) {
      const int u = TB.bi * a.nfr + f;
      if (!owns_block(a.own, TB.bi) || f % a.ng != grp) continue;
      G += (int)((a.units[u].n_rows + kBwRows - 1) / kBwRows);
    }
    if (warp == 1) {
      if (!ksm)
        for (int g = 0; g < G; ++g) gemm1();
    } else {
      for (int g = 0; g < G; ++g) gemm2();
      if (tc::elect_one()) tc::mma_commit(&d2full);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ===================== epilogue: warp (q, h) owns TMEM lane quadrant q and rows h*8 .. h*8+7 of a tile
    const int e = warp - 4;
    const int q = e & 3, h = e >> 2;
    const int c = q * 32 + lane;
    const int64_t colg = col0 + c;
    const float th2 = fmaxf(a.thr[b] * a.thr[b], 1.17549435e-38f);   // R22 dead zone (and |w|^2 > FLT_MIN)
    const uint32_t lq = (uint32_t)(q * 32) << 16;
    // this warp's TMEM lane quadrant + column offset of its rows, opaque (not re-derived from SR_TID per tile)
    uint32_t lqh = lq + (uint32_t)(h * 2 * kBwRpw);
    asm volatile("" : "+r"(lqh));
    int buf = 0;
    uint32_t bph = 0;
    int g = 0;
    // shared-window address of tb_ kept opaque in one register: tfull +0, tempty +16, a2full +32, a2empty +48
    // (the compiler otherwise re-derives each barrier's address from SR_CgaCtaId at every use: ~5
    // instructions and an S2R latency per barrier operation, four operations per tile and warp)
    uint32_t eb = tc::smem_u32(&tb_);
    asm volatile("" : "+r"(eb));
    // g_o (and, split-K, the W phase) of the next tile / unit are loaded one tile ahead
    auto next_unit = [&](int f) {
      while (f < a.nfr && (!owns_block(a.own, TB.bi) || f % a.ng != grp)) ++f;
      return f;
    };
    // phi_F weights of this warp's 8 rows of tile t (row block of output r at + r * ldw): read as two
    // warp-uniform float4 loads per r (broadcast) and folded into g_W's row factors before the tile's W is
    // waited for. (A register-less "prefetch" load of the next tile's lines is dropped by ptxas as dead code,
    // and staging them in SMEM by cp.async a tile ahead measured slower: the extra instructions cost more than
    // the L2 latency they hide.)
    auto wrow = [&](int u, int t) { return a.wts + a.tcu[u].wt_off + t * kBwRows + h * kBwRpw; };
    auto load_go = [&](int u, float* gor) {
      const JointUnit U = a.units[u];
#pragma unroll
      for (int r = 0; r < KAP; ++r)
        gor[r] = (r < U.rows_out && colg < bf.n_cols) ? a.go[b * a.go_sb + U.o_off + (int64_t)r * bf.n_cols + colg]
                                                       : 0.f;
    };
    // split-K mode: the phase of W (tile, column, this warp's 8 rows) from the forward's phase store, one
    // tile ahead; layout per (column tile, 64-row tile): [16-byte group][column], 2 x int16 per cell, row r in
    // group (r / 32) * wph / 256 + (r % 32) / 4
    const uint4* wcol = ksm ? reinterpret_cast<const uint4*>(a.wbuf + b * a.wb_sb + TB.wp_off) +
                                  (int64_t)ct * TB.wp_tiles * TB.wph + (h * (kBwRpw / 4)) * 128 + c
                            : nullptr;
    auto load_wv = [&](int u, int t32, uint4* wv) {
      const uint4* q4 = wcol + (int64_t)(a.tcu[u].wp_tile0 + (t32 >> 1)) * TB.wph + ((t32 & 1) * (TB.wph >> 8)) * 128;
#pragma unroll
      for (int i = 0; i < kBwRpw / 4; ++i) wv[i] = q4[i * 128];
    };
    int f = next_unit(0);
    float gor_n[KAP];
    uint4 wv_n[kBwRpw / 4];
    if (f < a.nfr) {
      load_go(TB.bi * a.nfr + f, gor_n);
      if (ksm) load_wv(TB.bi * a.nfr + f, 0, wv_n);
    }
    for (; f < a.nfr;) {
      const int u = TB.bi * a.nfr + f;
      const JointUnit U = a.units[u];
      float gor[KAP];
#pragma unroll
      for (int r = 0; r < KAP; ++r) gor[r] = gor_n[r];
      const int NT32 = (int)((U.n_rows + kBwRows - 1) / kBwRows);
      const int fn = next_unit(f + 1);
      const int ldw = a.tcu[u].NT * kTcRows;
      const float* wbase = wrow(u, 0);   // per unit: no dependent offset load per tile
      for (int t = 0; t < NT32; ++t, ++g) {
        // gv[i] = (Phi_F^T g_o)[row i] for this column (Eq. 4 adjoint)
        float gv[kBwRpw];
        {
          const float* wr = wbase + t * kBwRows;
#pragma unroll
          for (int i = 0; i < kBwRpw; ++i) gv[i] = 0.f;
#pragma unroll
          for (int r = 0; r < KAP; ++r) {
            if (r < U.rows_out) {
#pragma unroll
              for (int j = 0; j < kBwRpw / 4; ++j) {
                const float4 w0 = __ldg(reinterpret_cast<const float4*>(wr + (int64_t)r * ldw) + j);
                gv[4 * j] = fmaf(w0.x, gor[r], gv[4 * j]); gv[4 * j + 1] = fmaf(w0.y, gor[r], gv[4 * j + 1]);
                gv[4 * j + 2] = fmaf(w0.z, gor[r], gv[4 * j + 2]); gv[4 * j + 3] = fmaf(w0.w, gor[r], gv[4 * j + 3]);
              }
            }
          }
        }
        float v[2 * kBwRpw];
        if (ksm) {   // decode the phase store: (re, im) = W/|W| (0 in the dead zone)
          constexpr float kInv = 1.f / kPhaseScale;
#pragma unroll
          for (int i = 0; i < kBwRpw / 4; ++i) {
            const uint32_t wd[4] = {wv_n[i].x, wv_n[i].y, wv_n[i].z, wv_n[i].w};
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              v[8 * i + 2 * q4] = (float)(int16_t)(wd[q4] & 0xffffu) * kInv;
              v[8 * i + 2 * q4 + 1] = (float)(int16_t)(wd[q4] >> 16) * kInv;
            }
          }
        }
        if (t + 1 < NT32) {
          if (ksm) load_wv(u, t + 1, wv_n);
        } else if (fn < a.nfr) {
          load_go(TB.bi * a.nfr + fn, gor_n);
          if (ksm) load_wv(TB.bi * a.nfr + fn, 0, wv_n);
        }
        if (!ksm) {
          tc::mbar_wait_a(eb + 8u * buf, bph);
          tc::tc_fence_after();
          if (warp == 4 && lane == 0) TC_TRACE(5, g);
          const uint32_t ta = tbase + lqh + (uint32_t)(buf * kBwN1);
#pragma unroll
          for (int j = 0; j < kBwRpw / 8; ++j) tc::tmem_ld16_nowait(ta + 16u * j, v + 16 * j);
          tc::tmem_wait_ld();
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive_a(eb + 16u + 8u * buf);
          if (++buf == 2) { buf = 0; bph ^= 1; }
        }
        float ghi[2 * kBwRpw], glo[2 * kBwRpw];
        if (a.expt & 1) {
#pragma unroll
          for (int i = 0; i < 2 * kBwRpw; ++i) ghi[i] = glo[i] = v[i] * 0.f;
        } else
        {
        // g_W = (W/|W|) Phi_F^T g_o (Eq.4 adjoint, modulus adjoint with the R22 dead zone); the split-K test sits
        // outside the unrolled row loop (one uniform branch per tile instead of one per row)
        if (!ksm) {                                      // split-K: (re, im) is already the phase (or 0)
#pragma unroll
          for (int i = 0; i < kBwRpw; ++i) {
            const float m2 = fmaf(v[2 * i], v[2 * i], v[2 * i + 1] * v[2 * i + 1]);
            gv[i] = m2 > th2 ? gv[i] * tc::rsqrt_approx(m2) : 0.f;
          }
        }
#pragma unroll
        for (int i = 0; i < kBwRpw; ++i) {
          const float re = v[2 * i], im = v[2 * i + 1];
          const float s = gv[i];
          // (re, im) s and the lo halves as packed pairs (FMUL2 / FADD2); hi rounded on the integer pipe
          const float2 g2 = tc::mul2(make_float2(re, im), make_float2(s, s));
          const float2 h2 = make_float2(tc::tf32_rna(g2.x), tc::tf32_rna(g2.y));
          const float2 l2 = tc::sub2(g2, h2);
          ghi[2 * i] = h2.x; ghi[2 * i + 1] = h2.y;
          glo[2 * i] = l2.x; glo[2 * i + 1] = l2.y;
        }
        }
        // A2 buffer ab (TMEM) is free once the GEMM2 that last read it completed
        if (warp == 4 && lane == 0) TC_TRACE(6, g);
        const int ab = nab == 2 ? (g & 1) : 0;
        const uint32_t ta2_hi = ta2 + 128u * ab, ta2_lo = ta2_hi + 64u;
        tc::mbar_wait_a(eb + 48u + 8u * ab, (uint32_t)(((nab == 2 ? (g >> 1) : g) & 1) ^ 1));
        tc::tc_fence_after();
        if (warp == 4 && lane == 0) TC_TRACE(7, g);
#pragma unroll
        for (int j = 0; j < kBwRpw / 8; ++j) {
          tc::tmem_st16(ta2_hi + lqh + (uint32_t)(16 * j), ghi + 16 * j);
          tc::tmem_st16(ta2_lo + lqh + (uint32_t)(16 * j), glo + 16 * j);
        }
        tc::tmem_wait_st();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_a(eb + 32u + 8u * ab);
        if (warp == 4 && lane == 0) TC_TRACE(8, g);
      }
      f = fn;
    }
    // final: D2 (g_Y2^T for this column tile) -> g_Y2[n][col]
    if (g > 0) {
      tc::mbar_wait(&d2full, 0);
      tc::tc_fence_after();
    }
    if (h == 0) {
      // ng == 1: g_Y2[n][col]; ng > 1: this group's partial gp[grp][n][col] (reduced by k_gy_reduce)
      const int64_t dstride = a.ng > 1 ? bf.n_cols : bf.T2;
      float2* dst = a.ng > 1 ? a.gp + b * a.gp_sb + TB.gp_off + (int64_t)grp * K * bf.n_cols + (colg < bf.n_cols ? colg : 0)
                             : a.gY + b * a.gy_sb + bf.y_off + (bf.c_lo + (colg < bf.n_cols ? colg : 0)) % bf.T2;
      for (int c0 = 0; c0 < N2; c0 += 16) {
        float v[16];
        if (g > 0) {
          tc::tmem_ld16(d2 + lq + (uint32_t)c0, v);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        if (colg < bf.n_cols) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int n = c0 / 2 + i;
            if (n < K) dst[(int64_t)n * dstride] = make_float2(v[2 * i], v[2 * i + 1]);
          }
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tbase, 512);
}

// backward B rings (floats per stage, stage counts); the planner picks kb2 with the same rule
void tc_bwd_rings(int K, int K2, int kcw, int kb2, int* NS1, int* STG1, int* NS2, int* STG2) {
  const int N2 = ((2 * K + 15) / 16) * 16;
  *STG1 = 2 * kBwN1 * kcw;
  *STG2 = 2 * N2 * kb2;
  if (K2 == 0) {   // split-K block: no GEMM1 (W comes from the forward), ring 2 only
    *NS1 = 0;
    *NS2 = (int)std::min<long>(kTcMaxStages2, (224L * 1024 - 1024) / (*STG2 * 4));
    return;
  }
  int nab, ta;
  tc_bwd_mode(K, K2, &nab, &ta, tc_bwd_mode_pref());
  const long avail = 224L * 1024 - 1024 - (ta ? 0L : (long)2 * 128 * K2 * 4);
  // ring 2 holds up to three tiles of B2 chunks (GEMM2 runs a tile behind GEMM1 and a B2 tile takes
  // ~2 us to land from L2), ring 1 the rest
  int n2 = std::min(kTcMaxStages2, std::max(3, 192 / kb2));
  while (n2 > 2 && avail - (long)n2 * *STG2 * 4 < 2L * *STG1 * 4) --n2;
  *NS2 = n2;
  *NS1 = (int)std::min<long>(kTcMaxStages, (avail - (long)n2 * *STG2 * 4) / (*STG1 * 4));
}

int tc_bwd_mode_pref() {
  static const int m = [] {
    const char* e = std::getenv("JTFS_BWD_MODE");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}

static const int g_tc_expt = [] {
  const char* e = std::getenv("JTFS_TC_EXPT");
  return e ? std::atoi(e) : 0;
}();

template <int KAP>
static void launch_tc_bwd(const TcBwArgs& a, const TcClass& C, int B, cudaStream_t st) {
  int NS1, NS2, STG1, STG2;
  tc_bwd_rings(C.Kmax, C.ks ? 0 : C.K2max, C.kcw, C.kb2, &NS1, &STG1, &NS2, &STG2);
  int nab, ta;
  tc_bwd_mode(C.Kmax, C.K2max, &nab, &ta, tc_bwd_mode_pref());
  if (C.ks) ta = 1;   // no A tile in SMEM
  const size_t sm = (size_t)((ta ? 0 : 2 * 128 * C.K2max) + NS1 * STG1 + NS2 * STG2) * 4 + 1024;
  cudaFuncSetAttribute(k_joint_bwd_tc<KAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  dim3 g((unsigned)(C.ntiles * a.ng), (unsigned)B);
  k_joint_bwd_tc<KAP><<<g, kBwThreads, sm, st>>>(a, NS1, STG1, NS2, STG2);
  count_launch();
}

// g_Y2[n][col] = sum over filter groups of the partials (fixed order: deterministic)
__global__ void k_gy_reduce(const float2* __restrict__ gp, int64_t gp_sb, int64_t gp_off, float2* __restrict__ gY,
                            int64_t gy_sb, BlockInfo bf, int K, int ng) {
  const int b = blockIdx.y;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (int64_t)K * bf.n_cols) return;
  const int64_t n = q / bf.n_cols, col = q % bf.n_cols;
  const float2* src = gp + b * gp_sb + gp_off + q;
  float2 acc = src[0];
  for (int g = 1; g < ng; ++g) {
    const float2 v = src[(int64_t)g * K * bf.n_cols];
    acc.x += v.x;
    acc.y += v.y;
  }
  gY[b * gy_sb + bf.y_off + n * bf.T2 + (bf.c_lo + col) % bf.T2] = acc;
}

void launch_joint_bwd_tc(const Plan& p, const DeviceTables& d, const float2* Y2, int64_t y_sb, const float* go,
                         int64_t go_sb, float2* gY, int64_t gy_sb, const float* wbuf, int64_t wb_sb,
                         float2* gp, int64_t gp_sb, const float* thr, uint64_t own, int B,
                         const cudaStream_t* ss, int ns) {
  int li = 0;
  for (const TcClass& C : d.tcb) {
    const cudaStream_t st = ss[li++ % ns];
    if (C.n_blocks == 0 || !owns_block(own, C.bi)) continue;   // path shards: own blocks only
    TcBwArgs a{Y2, y_sb, go, go_sb, gY, gy_sb, d.units, d.binfo, C.blocks, C.tiles, C.n_blocks, d.tc_img,
               d.tc_img2, d.tc_img1b, d.tc_wts, d.tc_units, (int)p.L_fr.size(), own, thr, g_tc_expt, wbuf, wb_sb,
               tc_groups(C, B), gp, gp_sb, nullptr, tc_bwd_mode_pref()};
#ifdef JTFS_TC_TRACE
    static long long* trace = nullptr;
    if (!trace) cudaMalloc(&trace, 16 * 512 * 8);
    if (C.Kmax == g_trace_fwd_k) { cudaMemsetAsync(trace, 0, 16 * 512 * 8, st); a.trace = trace; }
#endif
    switch (C.cls) {  // class = kap_kind (KAP = 2 << kap_kind)
      case 0: launch_tc_bwd<2>(a, C, B, st); break;
      case 1: launch_tc_bwd<4>(a, C, B, st); break;
      case 2: launch_tc_bwd<8>(a, C, B, st); break;
      case 3: launch_tc_bwd<16>(a, C, B, st); break;
      case 4: launch_tc_bwd<32>(a, C, B, st); break;
    }
    if (a.ng > 1) {
      const BlockInfo& bf = p.binfo[C.bi];
      dim3 gr((unsigned)((C.Kmax * bf.n_cols + 255) / 256), (unsigned)B);
      k_gy_reduce<<<gr, 256, 0, st>>>(gp, gp_sb, C.gp_off, gY, gy_sb, bf, C.Kmax, a.ng);
      count_launch();
    }
#ifdef JTFS_TC_TRACE
    if (a.trace) {
      static long long h[16 * 512];
      cudaStreamSynchronize(st);
      cudaMemcpy(h, a.trace, sizeof(h), cudaMemcpyDeviceToHost);
      if (FILE* fo = fopen("gpurun_out/tc_trace.bin", "wb")) { fwrite(h, 1, sizeof(h), fo); fclose(fo); }
    }
#endif
  }
}

}  // namespace jtfs
