// kernels_frfft.cu — the joint lambda_1 stage by the paper's own route, an FFT
// along n1 per time column (`frequency_scattering`), for the blocks whose K = n1_max is
// too large for the resident-tile tensor-core kernels (kernels_tc.cu). FP32 CUDA-core arithmetic.
//
// One CTA = (block n2, C time columns, signal). For each column y = Y2[0:K][c] zero-padded to P rows
// (P:276-277):
//   forward   Y^ = FFT_P(y)
//             per filter f of L_fr (both spins and phi_F, R12):
//               W^_f[m] = (1/2^kf) sum_b Y^[m + b L_f] psi^_f[m + b L_f]   (cdgmm + subsample_fourier,
//                                                                         fold-mean)
//               w_f = IFFT_{L_f}(W^_f)
//               u = |w_f| (Eq.2) on the needed rows; o[rho][c] = sum_r g_kf[(rho 2^d - r) mod L_f] u[r]
//               (phi_F over log-frequency with stride F, Eq.4, R17)
//   backward  recompute w_f; g_u[r] = sum_rho g_kf[(rho 2^d - r) mod L_f] g_o[rho][c] (phi_F adjoint);
//             g_w = (w/|w|) g_u (modulus adjoint, R22 dead zone); G^[m] += psi^_f[m] DFT_{L_f}(g_w)[m mod L_f]
//             (adjoint of the fold = periodic extension; psi^ real => self-adjoint, R21);
//             g_y = IFFT_P(G^) restricted to n < K.
// The forward FFT of y and the accumulator G^ are shared by all 2N_fr+1 filters of the block, so each
// column is transformed once per filter bank instead of once per filter.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdlib>

#include "device.cuh"
#include "fft_dev.cuh"

namespace jtfs {

constexpr int kFfThreads = 256;

struct FfArgs {
  const float2* Y2; int64_t y_sb;
  float* o; int64_t o_sb;             // forward: o (output); backward: g_o (input)
  float2* gY; int64_t gy_sb;          // backward output g_Y2
  const JointUnit* units; const BlockInfo* binfo;
  const int32_t* blist; const int64_t* tiles; int nb;
  const float* spec;                  // [nfr][P] level-0 responses of L_fr
  const float* wts; const int64_t* wt_off;  // per unit [rows_out][n_rows]
  const float2* tw;
  const float* thr;
  int nfr, P, lgP;
  uint64_t own;
};

__device__ __forceinline__ int ff_find(const int64_t* __restrict__ tiles, int n, int64_t t) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (__ldg(tiles + mid) <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// SMEM twiddle table W_P^e, e < P, from the global 4096-entry table (P <= 4096)
__device__ __forceinline__ void ff_twiddles(float2* tws, const float2* __restrict__ tw, int lgP) {
  for (int e = threadIdx.x; e < (1 << lgP); e += kFfThreads) tws[e] = __ldg(tw + (e << (12 - lgP)));
}

// Y^[c][.] = FFT_P of the zero-padded column c of the block (C columns from col0)
template <int C>
__device__ __forceinline__ void ff_load_fft(CfSmem Yh, const float2* tws, const FfArgs& a, const BlockInfo& bf,
                                            int K, int64_t col0, int b) {
  const int P = a.P;
  const float2* ysrc = a.Y2 + b * a.y_sb + bf.y_off;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int64_t col = col0 + c;
    const bool ok = col < bf.n_cols;
    const int64_t cc = (bf.c_lo + (ok ? col : 0)) & (bf.T2 - 1);
    for (int n = threadIdx.x; n < P; n += kFfThreads) {
      float2 v = make_float2(0.f, 0.f);
      if (n < K && ok) v = ysrc[(int64_t)n * bf.T2 + cc];
      Yh(c, n, v);
    }
  }
  __syncthreads();
  col_fft<kFfThreads>(C, a.lgP, false, tws, a.lgP, Yh, Yh, Yh);
}

// W[c][m] = (1/P) sum_{b < 2^kf} Y^[c][m + b L_f] psi^_f[m + b L_f], m < L_f (cdgmm + fold-mean; the
// 1/2^kf and the 1/L_f of the unscaled inverse DFT that follows give 1/P). One spectrum load serves
// the C columns.
template <int C>
__device__ __forceinline__ void ff_fold(CfSmem W, CfSmem Yh, const float* __restrict__ spec, int P, int kf) {
  const int Lf = P >> kf, nrep = 1 << kf;
  const float sc = 1.f / (float)P;
  for (int m = threadIdx.x; m < Lf; m += kFfThreads) {
    float2 acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = make_float2(0.f, 0.f);
    for (int q = 0; q < nrep; ++q) {
      const int mm = m + q * Lf;
      const float h = __ldg(spec + mm);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const float2 v = Yh(c, mm);
        acc[c].x = fmaf(h, v.x, acc[c].x);
        acc[c].y = fmaf(h, v.y, acc[c].y);
      }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) W(c, m, make_float2(acc[c].x * sc, acc[c].y * sc));
  }
  __syncthreads();
}

// storer of the forward's inverse transform: modulus of the needed rows (Eq.2), Md[c][i], r = r_lo + i
struct StMod {
  float* Md;
  int P, rlo, nr, Lmask;
  __device__ __forceinline__ void operator()(int c, int r, float2 w) const {
    const int i = (r - rlo) & Lmask;
    if (i < nr) Md[c * P + i] = sqrtf(fmaf(w.x, w.x, w.y * w.y));
  }
};

// storer of the final inverse transform: g_Y2[n][col] = G[n] / P for n < K
struct StOut {
  float2* gdst;
  int64_t col0, c_lo, T2m, n_cols;
  int K;
  float sc;
  __device__ __forceinline__ void operator()(int c, int n, float2 v) const {
    const int64_t cg = col0 + c;
    if (n < K && cg < n_cols) gdst[(int64_t)n * (T2m + 1) + ((c_lo + cg) & T2m)] = make_float2(v.x * sc, v.y * sc);
  }
};

template <int C, int MINB>
__global__ void __launch_bounds__(kFfThreads, MINB) k_joint_fwd_fft(FfArgs a) {
  extern __shared__ __align__(16) float2 ffsm[];
  const int li = ff_find(a.tiles, a.nb, blockIdx.x);
  const int bi = a.blist[li];
  const BlockInfo bf = a.binfo[bi];
  const int64_t col0 = (int64_t)(blockIdx.x - a.tiles[li]) * C;
  const int b = blockIdx.y;
  const int P = a.P;
  const int K = a.units[bi * a.nfr].n1_max;
  const CfSmem Yh{ffsm, P};                          // [C][P]
  const CfSmem Wk{ffsm + C * P, P};                  // [C][P]; its first C*P floats double as Md
  float2* tws = ffsm + 2 * C * P;                    // [P]
  float* Md = reinterpret_cast<float*>(Wk.s);
  ff_twiddles(tws, a.tw, a.lgP);
  ff_load_fft<C>(Yh, tws, a, bf, K, col0, b);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int f = 0; f < a.nfr; ++f) {
    const int u = bi * a.nfr + f;
    if (!owns_block(a.own, bi)) continue;
    const JointUnit U = a.units[u];
    const int Lf = (int)U.Lf, nr = (int)U.n_rows, ro = U.rows_out;
    ff_fold<C>(Wk, Yh, a.spec + (int64_t)f * P, P, U.kf);
    const StMod st{Md, P, (int)U.r_lo, nr, Lf - 1};
    col_fft<kFfThreads>(C, a.lgP - U.kf, true, tws, a.lgP, Wk, st, Wk);
    // phi_F over rows (Eq.4): o[rho][c] = sum_i wts[rho][i] Md[c][i]. Warp w takes rho pairs w, w + 8, ...;
    // lanes stride the rows; butterfly shuffle reduction in a fixed order (deterministic).
    const float* wt = a.wts + a.wt_off[u];
    for (int pp = warp; 2 * pp < ro; pp += kFfThreads / 32) {
      const int r0 = 2 * pp, r1 = 2 * pp + 1;
      const bool two = r1 < ro;
      const float* w0p = wt + (int64_t)r0 * nr;
      const float* w1p = wt + (int64_t)(two ? r1 : r0) * nr;
      float a0[C], a1[C];
#pragma unroll
      for (int c = 0; c < C; ++c) a0[c] = a1[c] = 0.f;
      for (int i = lane; i < nr; i += 32) {
        const float w0 = __ldg(w0p + i), w1 = __ldg(w1p + i);
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const float m = Md[c * P + i];
          a0[c] = fmaf(w0, m, a0[c]);
          a1[c] = fmaf(w1, m, a1[c]);
        }
      }
#pragma unroll
      for (int sh = 16; sh > 0; sh >>= 1)
#pragma unroll
        for (int c = 0; c < C; ++c) {
          a0[c] += __shfl_xor_sync(0xffffffffu, a0[c], sh);
          a1[c] += __shfl_xor_sync(0xffffffffu, a1[c], sh);
        }
      if (lane < 2 * C) {
        const int c = lane & (C - 1);
        const int rho = lane < C ? r0 : r1;
        float v = 0.f;
#pragma unroll
        for (int cc = 0; cc < C; ++cc) if (cc == c) v = lane < C ? a0[cc] : a1[cc];
        const int64_t cg = col0 + c;
        if (rho < ro && cg < bf.n_cols) a.o[b * a.o_sb + U.o_off + (int64_t)rho * bf.n_cols + cg] = v;
      }
    }
    __syncthreads();   // Md (= Wk) is overwritten by the next filter's transform
  }
}

template <int C, int MINB>
__global__ void __launch_bounds__(kFfThreads, MINB) k_joint_bwd_fft(FfArgs a) {
  static_assert(C == 4, "g_o rows are packed as float4");
  extern __shared__ __align__(16) float2 ffsm[];
  __shared__ float4 gos[kFfMaxRo];
  const int li = ff_find(a.tiles, a.nb, blockIdx.x);
  const int bi = a.blist[li];
  const BlockInfo bf = a.binfo[bi];
  const int64_t col0 = (int64_t)(blockIdx.x - a.tiles[li]) * C;
  const int b = blockIdx.y;
  const int P = a.P;
  const int K = a.units[bi * a.nfr].n1_max;
  const CfSmem Yh{ffsm, P};
  const CfSmem Wk{ffsm + C * P, P};
  const CfSmem G{ffsm + 2 * C * P, P};    // accumulated spectrum of g_y
  float2* tws = ffsm + 3 * C * P;         // [P]
  const int tid = threadIdx.x;
  for (int idx = tid; idx < C * P; idx += kFfThreads) G.s[idx] = make_float2(0.f, 0.f);
  ff_twiddles(tws, a.tw, a.lgP);
  ff_load_fft<C>(Yh, tws, a, bf, K, col0, b);
  const float th2 = a.thr[b] * a.thr[b];
  for (int f = 0; f < a.nfr; ++f) {
    const int u = bi * a.nfr + f;
    if (!owns_block(a.own, bi)) continue;
    const JointUnit U = a.units[u];
    const int Lf = (int)U.Lf, nr = (int)U.n_rows, rlo = (int)U.r_lo, ro = U.rows_out;
    // g_o of this unit for the CTA's columns, packed per rho
    for (int rho = tid; rho < ro; rho += kFfThreads) {
      float g[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const int64_t cg = col0 + c;
        g[c] = (cg < bf.n_cols) ? a.o[b * a.o_sb + U.o_off + (int64_t)rho * bf.n_cols + cg] : 0.f;
      }
      gos[rho] = make_float4(g[0], g[1], g[2], g[3]);
    }
    const float* sp = a.spec + (int64_t)f * P;
    ff_fold<C>(Wk, Yh, sp, P, U.kf);                                      // (its barrier orders gos)
    col_fft<kFfThreads>(C, a.lgP - U.kf, true, tws, a.lgP, Wk, Wk, Wk);   // w
    // g_w = (w/|w|) * sum_rho wts[rho][i] g_o[rho][c] on the needed rows, 0 elsewhere
    const float* wt = a.wts + a.wt_off[u];
    for (int r = tid; r < Lf; r += kFfThreads) {
      const int i = (r - rlo) & (Lf - 1);
      float gu[C] = {0.f, 0.f, 0.f, 0.f};
      if (i < nr) {
        for (int rho = 0; rho < ro; ++rho) {
          const float wv = __ldg(wt + (int64_t)rho * nr + i);
          const float4 g = gos[rho];
          gu[0] = fmaf(wv, g.x, gu[0]); gu[1] = fmaf(wv, g.y, gu[1]);
          gu[2] = fmaf(wv, g.z, gu[2]); gu[3] = fmaf(wv, g.w, gu[3]);
        }
      }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const float2 w = Wk(c, r);
        const float m2 = fmaf(w.x, w.x, w.y * w.y);
        const float s = (i < nr && m2 > FLT_MIN && m2 > th2) ? gu[c] * rsqrtf(m2) : 0.f;
        Wk(c, r, make_float2(w.x * s, w.y * s));
      }
    }
    __syncthreads();
    col_fft<kFfThreads>(C, a.lgP - U.kf, false, tws, a.lgP, Wk, Wk, Wk);   // DFT_{L_f}(g_w)
    // G^[c][m] += psi^_f[m] DFT(g_w)[m mod L_f] (adjoint of the fold = periodic extension; psi^ real, R21)
    for (int m = tid; m < P; m += kFfThreads) {
      const float h = __ldg(sp + m);
      const int mw = m & (Lf - 1);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const float2 v = Wk(c, mw), g = G(c, m);
        G(c, m, make_float2(fmaf(h, v.x, g.x), fmaf(h, v.y, g.y)));
      }
    }
    __syncthreads();
  }
  const StOut out{a.gY + b * a.gy_sb + bf.y_off, col0, bf.c_lo, bf.T2 - 1, bf.n_cols, K, 1.f / (float)P};
  col_fft<kFfThreads>(C, a.lgP, true, tws, a.lgP, G, out, G);
}

constexpr int kFfC = 4;   // columns per CTA (C x P <= 16 x 256 points per SMEM FFT call)

static int ilog2i(int64_t v) {
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return l;
}

static size_t ff_smem(int P, bool bwd) {
  return (size_t)(bwd ? 3 : 2) * kFfC * P * 8 + (size_t)P * 8;   // column buffers + twiddles [P]
}

void launch_joint_fft(const Plan& p, const DeviceTables& d, bool bwd, const float2* Y2, int64_t y_sb, float* o,
                      int64_t o_sb, float2* gY, int64_t gy_sb, const float* thr, uint64_t own, int B,
                      cudaStream_t st) {
  const FfList& L = bwd ? d.ffb : d.ffw;
  if (L.nb == 0 || L.ntiles == 0) return;
  FfArgs a{Y2, y_sb, o, o_sb, gY, gy_sb, d.units, d.binfo, L.blist, L.tiles, L.nb, d.fr_spec, d.u_wts,
           d.u_wt_off, d.tw, thr, (int)p.L_fr.size(), (int)p.P, ilog2i(p.P), own};
  const size_t sm = ff_smem((int)p.P, bwd);
  dim3 g((unsigned)L.ntiles, (unsigned)B);
  // forward: 80-register variant with 3 CTAs per SM (measured faster than 128 registers at 2 per SM);
  // JTFS_FF_MINB=2 selects the latter (A/B)
  static const int minb = [] {
    const char* e = std::getenv("JTFS_FF_MINB");
    return e ? std::atoi(e) : 3;
  }();
  if (bwd) {
    cudaFuncSetAttribute(k_joint_bwd_fft<kFfC, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_joint_bwd_fft<kFfC, 2><<<g, kFfThreads, sm, st>>>(a);
  } else if (minb == 3) {
    cudaFuncSetAttribute(k_joint_fwd_fft<kFfC, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_joint_fwd_fft<kFfC, 3><<<g, kFfThreads, sm, st>>>(a);
  } else {
    cudaFuncSetAttribute(k_joint_fwd_fft<kFfC, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_joint_fwd_fft<kFfC, 2><<<g, kFfThreads, sm, st>>>(a);
  }
  count_launch();
}

int64_t joint_fft_tiles(int64_t n_cols) { return (n_cols + kFfC - 1) / kFfC; }

}  // namespace jtfs
