// kernels_fr.cu — frequential (lambda_1-axis) stages and the time averaging of the JTFS path.
//
//  * order-1 frequential scattering of S1 (spinned=False, P:264-305 with P:341) and its adjoint
//  * k_joint_fwd / k_joint_bwd: the dominant joint stage. Per block n2 and
//    per time column t the spinned frequential filter f is the exact dense matrix
//    M_f[r][n] = h_f[(r 2^k_f - n) mod P] (zero-pad to P, circular convolution, decimation), so
//      W_f = M_f Y2,  U = |W_f| (Eq.2),  o = Phi_F U (Eq.4 over log-frequency, R17)
//    and the backward is g_W = (W/|W|) Phi_F^T g_o, g_Y2 += M_f^H g_W (R21, R22).
//    FP32 CUDA-core register-tiled contraction over K = n1_max, fused with the modulus and phi_F.
//  * phi_T along time at level s2 with decimation to stride T (Eq.4) and its adjoint; loss (R19).
#include <cuda_runtime.h>

#include <cfloat>

#include "device.cuh"

namespace jtfs {

__device__ __forceinline__ int find_idx(const int64_t* __restrict__ tiles, int n, int64_t t) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (__ldg(tiles + mid) <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// j-range of a symmetric truncated kernel of half width H on a circle of length L
__device__ __forceinline__ void sym_range(int64_t H, int64_t L, int64_t* jlo, int64_t* jhi) {
  if (2 * H + 1 > L) { *jlo = -(L / 2) + 1; *jhi = L / 2; } else { *jlo = -H; *jhi = H; }
}

__device__ __forceinline__ int64_t cdist(int64_t a, int64_t L) {  // circular |a| on L
  a %= L;
  if (a < 0) a += L;
  return a > L - a ? L - a : a;
}

// =====================================================================================
// Order 1 (S1 frequential scattering, non-spinned)
// W1[f][i][t] = sum_{n < N1} h_f[(r_i 2^k_f - n) mod P] S1t[n][t],  r_i = (r_lo_f + i) mod L_f
// =====================================================================================
__global__ void k_o1_W(const float* __restrict__ S1t, int64_t S1t_sb, float2* __restrict__ W1, int64_t W1_sb,
                       const float2* __restrict__ hfr, const int64_t* __restrict__ rlo,
                       const int64_t* __restrict__ nrows, const int32_t* __restrict__ kf_of,
                       const int32_t* __restrict__ hH, int N1, int P, int64_t Ft) {
  const int f = blockIdx.y, b = blockIdx.z;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = q / Ft, t = q % Ft;
  if (i >= nrows[f]) return;
  const int kf = kf_of[f];
  const int64_t Lf = P >> kf;
  const int64_t r = (rlo[f] + i) & (Lf - 1);
  const int hb = (int)((r << kf) & (P - 1));
  const float* x = S1t + b * S1t_sb + t;
  const float2* h = hfr + (int64_t)f * P;
  float2 acc = make_float2(0.f, 0.f);
  // h_f[(hb - n) mod P] vanishes unless n is within the support half-width H of hb (circularly)
  const int H = hH[f];
  const int span = 2 * H + 1 >= P ? P : 2 * H + 1;
  for (int q = 0; q < span; ++q) {
    const int n = (hb - H + q) & (P - 1);
    if (n >= N1) continue;
    const float v = x[(int64_t)n * Ft];
    const float2 hv = __ldg(h + ((hb - n) & (P - 1)));
    acc.x = fmaf(hv.x, v, acc.x);
    acc.y = fmaf(hv.y, v, acc.y);
  }
  W1[b * W1_sb + ((int64_t)f * P + i) * Ft + t] = acc;
}

// V2[f][i][t'] = sum_j tT[|j|] |W1[f][i][(m0 + t' + j) mod Ft]|   (phi_T at level log2T, no decimation)
__global__ void k_o1_time(const float2* __restrict__ W1, int64_t W1_sb, float* __restrict__ V2, int64_t V2_sb,
                          const int64_t* __restrict__ nrows, const float* __restrict__ tT, int64_t H, int P,
                          int64_t Ft, int64_t frames, int64_t m0) {
  const int f = blockIdx.y + 1, b = blockIdx.z;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = q / frames, tp = q % frames;
  if (i >= nrows[f]) return;
  const float2* w = W1 + b * W1_sb + ((int64_t)f * P + i) * Ft;
  int64_t jlo, jhi;
  sym_range(H, Ft, &jlo, &jhi);
  double acc = 0;
  for (int64_t j = jlo; j <= jhi; ++j) {
    int64_t tau = (m0 + tp + j) % Ft;
    if (tau < 0) tau += Ft;
    float2 v = w[tau];
    acc += (double)__ldg(tT + (j < 0 ? -j : j)) * (double)sqrtf(v.x * v.x + v.y * v.y);
  }
  V2[b * V2_sb + ((int64_t)f * P + i) * frames + tp] = (float)acc;
}

// order-1 outputs (paths 1 .. nfr1): f = 0: Re W1 (Eq.3); f > 0: phi_F rows of V2, stride F.
__global__ void __launch_bounds__(256) k_o1_out(const float2* __restrict__ W1, int64_t W1_sb, const float* __restrict__ V2,
                         int64_t V2_sb, float* __restrict__ S, int64_t S_sb, const int64_t* __restrict__ rlo,
                         const int64_t* __restrict__ nrows, const int32_t* __restrict__ kf_of,
                         const float* __restrict__ phiF_k, const int64_t* __restrict__ phiF_off, int log2F, int P,
                         int64_t Ft, int64_t frames, int64_t m0, int rows1) {
  // 64 outputs per CTA, 4 threads each (part = threadIdx.x / 64 takes rows i = part mod 4); partials
  // combined in part order (deterministic)
  __shared__ double part_acc[4][64];
  const int f = blockIdx.y, b = blockIdx.z;
  const int o = threadIdx.x & 63, part = threadIdx.x >> 6;
  const int64_t q = (int64_t)blockIdx.x * 64 + o;
  const int64_t rho = q / frames, tp = q % frames;
  const bool valid = rho < rows1;
  double acc = 0;
  if (valid && f > 0) {
    const int kf = kf_of[f], d = log2F - kf;
    const int64_t Lf = P >> kf;
    const float* g = phiF_k + phiF_off[kf];
    const float* v = V2 + b * V2_sb + (int64_t)f * P * frames + tp;
    const int nr = (int)nrows[f], r0 = (int)rlo[f], Lm = (int)Lf - 1;   // L_f: power of two
    for (int i = part; i < nr; i += 4) {
      const int r = (r0 + i) & Lm;
      const int e = (((int)rho << d) - r) & Lm;
      acc += (double)__ldg(g + e) * (double)v[(int64_t)i * frames];
    }
  }
  part_acc[part][o] = acc;
  __syncthreads();
  if (part != 0 || !valid) return;
  float out;
  if (f == 0) {
    out = W1[b * W1_sb + rho * Ft + m0 + tp].x;
  } else {
    out = (float)(((part_acc[0][o] + part_acc[1][o]) + part_acc[2][o]) + part_acc[3][o]);
  }
  S[b * S_sb + frames + ((int64_t)f * rows1 + rho) * frames + tp] = out;
}

// ---- order-1 adjoints
// gV2[f][i][t'] = sum_rho g_k[(rho 2^d - r_i) mod L_f] r[path 1+f][rho][t']   (f >= 1)
__global__ void k_o1_bwd_rows(const float* __restrict__ rres, int64_t r_sb, float* __restrict__ V2, int64_t V2_sb,
                              const int64_t* __restrict__ rlo, const int64_t* __restrict__ nrows,
                              const int32_t* __restrict__ kf_of, const float* __restrict__ phiF_k,
                              const int64_t* __restrict__ phiF_off, int log2F, int P, int64_t frames, int rows1) {
  const int f = blockIdx.y + 1, b = blockIdx.z;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = q / frames, tp = q % frames;
  if (i >= nrows[f]) return;
  const int kf = kf_of[f], d = log2F - kf;
  const int64_t Lf = P >> kf;
  const int64_t r = (rlo[f] + i) & (Lf - 1);
  const float* g = phiF_k + phiF_off[kf];
  const float* rr = rres + b * r_sb + frames + (int64_t)f * rows1 * frames + tp;
  double acc = 0;
  for (int rho = 0; rho < rows1; ++rho) {
    const int64_t e = (((int64_t)rho << d) - r) & (Lf - 1);
    acc += (double)__ldg(g + e) * (double)rr[(int64_t)rho * frames];
  }
  V2[b * V2_sb + ((int64_t)f * P + i) * frames + tp] = (float)acc;
}

// gW1[f][i][tau] = phase(W1) * sum_{t'} tT[dist(m0+t'-tau)] gV2[f][i][t']   (f >= 1), in place;
// f = 0: gW1[0][rho][tau] = r[path 1][rho][tau - m0] (kept frames), real.
__global__ void k_o1_bwd_time(const float* __restrict__ rres, int64_t r_sb, float2* __restrict__ W1,
                              int64_t W1_sb, const float* __restrict__ V2, int64_t V2_sb,
                              const int64_t* __restrict__ nrows, const float* __restrict__ tT, int64_t H, int P,
                              int64_t Ft, int64_t frames, int64_t m0, const float* __restrict__ thr) {
  const int f = blockIdx.y, b = blockIdx.z;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = q / Ft, tau = q % Ft;
  if (i >= nrows[f]) return;
  float2* w = W1 + b * W1_sb + ((int64_t)f * P + i) * Ft + tau;
  if (f == 0) {
    int64_t tp = tau - m0;
    float g = (tp >= 0 && tp < frames) ? rres[b * r_sb + frames + i * frames + tp] : 0.f;
    *w = make_float2(g, 0.f);
    return;
  }
  const float* gv2 = V2 + b * V2_sb + ((int64_t)f * P + i) * frames;
  double acc = 0;
  // a = (m0 + tp - tau) mod Ft advanced by one per frame (one 64-bit modulo per output)
  const int Fti = (int)Ft;
  int ad = (int)(((m0 - tau) % Ft + Ft) % Ft);
  for (int64_t tp = 0; tp < frames; ++tp) {
    const int dd = ad > Fti - ad ? Fti - ad : ad;
    if (dd <= H) acc += (double)__ldg(tT + dd) * (double)gv2[tp];
    if (++ad == Fti) ad = 0;
  }
  float2 v = *w;
  float m2 = v.x * v.x + v.y * v.y;
  const float th = thr[b];
  float s = (m2 > FLT_MIN && m2 > th * th) ? (float)acc * rsqrtf(m2) : 0.f;
  *w = make_float2(v.x * s, v.y * s);
}

// gS1t[n][tau] = sum_f sum_i Re(conj(h_f[(r_i 2^k_f - n) mod P]) gW1[f][i][tau])
constexpr int kO1Parts = 4;   // threads per output of the order-1 reductions (few outputs: latency bound)
__global__ void __launch_bounds__(256) k_o1_bwd_S1t(const float2* __restrict__ W1, int64_t W1_sb, float* __restrict__ gS1t,
                             int64_t gS_sb, const float2* __restrict__ hfr, const int64_t* __restrict__ rlo,
                             const int64_t* __restrict__ nrows, const int32_t* __restrict__ kf_of,
                             const int32_t* __restrict__ hH, int nfr1, int N1, int P, int64_t Ft) {
  // 64 outputs per CTA, kO1Parts threads each (part = threadIdx.x / 64 takes filters f = part mod
  // kO1Parts); partial sums combined in part order (deterministic)
  __shared__ double part_acc[kO1Parts][64];
  const int b = blockIdx.y;
  const int o = threadIdx.x & 63, part = threadIdx.x >> 6;
  const int64_t q = (int64_t)blockIdx.x * 64 + o;
  const int64_t n = q / Ft, tau = q % Ft;
  double acc = 0;
  if (n < N1) {
    for (int f = part; f < nfr1; f += kO1Parts) {
      const int kf = kf_of[f];
      const int64_t Lf = P >> kf;
      const float2* h = hfr + (int64_t)f * P;
      const float2* g = W1 + b * W1_sb + (int64_t)f * P * Ft + tau;
      float accf = 0.f;
      // rows r with |r 2^kf - n| <= H (circular on P): r in [ceil((n-H)/2^kf), floor((n+H)/2^kf)] mod L_f
      const int H = hH[f];
      const int nr = (int)nrows[f], r0 = (int)rlo[f], Lm = (int)Lf - 1;
      int rs, cnt;
      if (2 * H + 1 >= P) { rs = 0; cnt = (int)Lf; }
      else {
        const int s = 1 << kf;
        const int a = (int)n - H, bnd = (int)n + H;
        rs = a >= 0 ? (a + s - 1) >> kf : -((-a) >> kf);
        const int rhi = bnd >> kf;                          // bnd >= 0
        cnt = min(rhi - rs + 1, (int)Lf);
      }
      for (int qq = 0; qq < cnt; ++qq) {
        const int r = (rs + qq) & Lm;
        const int i = (r - r0) & Lm;
        if (i >= nr) continue;
        const int hb = (r << kf) & (P - 1);
        const float2 hv = __ldg(h + ((hb - (int)n) & (P - 1)));
        const float2 gv = g[(int64_t)i * Ft];
        accf = fmaf(hv.x, gv.x, fmaf(hv.y, gv.y, accf));
      }
      acc += accf;
    }
  }
  part_acc[part][o] = acc;
  __syncthreads();
  if (part == 0 && n < N1) {
    double t = part_acc[0][o];
    for (int k = 1; k < kO1Parts; ++k) t += part_acc[k][o];
    gS1t[b * gS_sb + n * Ft + tau] = (float)t;
  }
}

// =====================================================================================
// Joint stage forward (dominant): one CTA = (unit = (block, filter), 64-column tile, signal)
// =====================================================================================
template <int KAP>
__global__ void __launch_bounds__(256) k_joint_fwd(
    const float2* __restrict__ Y2, int64_t y_sb, float* __restrict__ o, int64_t o_sb,
    const JointUnit* __restrict__ units, const int32_t* __restrict__ ulist, const int64_t* __restrict__ tiles,
    int nlist, const BlockInfo* __restrict__ binfo, const float2* __restrict__ hfr, int P,
    const float* __restrict__ phiF_k, const int64_t* __restrict__ phiF_off, uint64_t own) {
  extern __shared__ float4 smem4[];
  const int li = find_idx(tiles, nlist, blockIdx.x);
  if (!owns_block(own, units[ulist[li]].bi)) return;
  const JointUnit U = units[ulist[li]];
  const BlockInfo bf = binfo[U.bi];
  const int64_t ct = blockIdx.x - tiles[li];
  const int b = blockIdx.y;
  const int K = U.n1_max;
  const int Lf = (int)U.Lf;
  float2* Ys = reinterpret_cast<float2*>(smem4);        // [K][64]
  float2* hs = Ys + K * kJC;                            // [P]
  float* gs = reinterpret_cast<float*>(hs + P);         // [Lf]
  float* red = gs + Lf;                                 // [16][KAP][64] final row-group reduction
  const int tid = threadIdx.x;
  const int64_t col0 = ct * kJC;
  const float2* ysrc = Y2 + b * y_sb + bf.y_off;
  for (int idx = tid; idx < K * kJC; idx += 256) {
    int n = idx / kJC, c = idx % kJC;
    int64_t col = col0 + c;
    float2 v = make_float2(0.f, 0.f);
    if (col < bf.n_cols) v = ysrc[(int64_t)n * bf.T2 + (bf.c_lo + col) % bf.T2];
    Ys[idx] = v;
  }
  for (int idx = tid; idx < P; idx += 256) hs[idx] = hfr[(int64_t)U.f * P + idx];
  const float* gsrc = phiF_k + phiF_off[U.kf];
  for (int idx = tid; idx < Lf; idx += 256) gs[idx] = gsrc[idx];
  __syncthreads();

  const int tr = tid >> 4, tc = tid & 15;
  float opart[KAP][4];
#pragma unroll
  for (int q = 0; q < KAP; ++q)
#pragma unroll
    for (int c = 0; c < 4; ++c) opart[q][c] = 0.f;

  for (int64_t r0 = 0; r0 < U.n_rows; r0 += kJR) {
    int hb[4];
    int rr[4];
    bool valid[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int64_t lr = r0 + tr * 4 + i;
      valid[i] = lr < U.n_rows;
      int r = (int)((U.r_lo + lr) % Lf);
      rr[i] = r;
      hb[i] = (r << U.kf) & (P - 1);
    }
    float2 acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[i][c] = make_float2(0.f, 0.f);
    for (int n = 0; n < K; ++n) {
      const float4* yp = reinterpret_cast<const float4*>(Ys + n * kJC + tc * 4);
      float4 ya = yp[0], yb = yp[1];
      float2 y[4] = {make_float2(ya.x, ya.y), make_float2(ya.z, ya.w), make_float2(yb.x, yb.y),
                     make_float2(yb.z, yb.w)};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float2 h = hs[(hb[i] - n) & (P - 1)];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc[i][c].x = fmaf(h.x, y[c].x, fmaf(-h.y, y[c].y, acc[i][c].x));
          acc[i][c].y = fmaf(h.x, y[c].y, fmaf(h.y, y[c].x, acc[i][c].y));
        }
      }
    }
    // modulus (Eq.2) and phi_F over rows (Eq.4): o[rho][c] += g[(rho 2^d - r) mod Lf] |w[r][c]|
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (!valid[i]) continue;
      float v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = sqrtf(acc[i][c].x * acc[i][c].x + acc[i][c].y * acc[i][c].y);
#pragma unroll
      for (int q = 0; q < KAP; ++q) {
        if (q < U.rows_out) {
          float w = gs[((q << U.d) - rr[i]) & (Lf - 1)];
#pragma unroll
          for (int c = 0; c < 4; ++c) opart[q][c] = fmaf(w, v[c], opart[q][c]);
        }
      }
    }
  }
  // reduce the 16 row groups in a fixed order (deterministic)
  __syncthreads();
#pragma unroll
  for (int q = 0; q < KAP; ++q)
#pragma unroll
    for (int c = 0; c < 4; ++c) red[(tr * KAP + q) * kJC + tc * 4 + c] = opart[q][c];
  __syncthreads();
  for (int idx = tid; idx < U.rows_out * kJC; idx += 256) {
    int q = idx / kJC, c = idx % kJC;
    float s = 0.f;
    for (int g = 0; g < 16; ++g) s += red[(g * KAP + q) * kJC + c];
    int64_t col = col0 + c;
    if (col < bf.n_cols) o[b * o_sb + U.o_off + (int64_t)q * bf.n_cols + col] = s;
  }
}

// =====================================================================================
// Joint stage backward: one CTA = (block, 64-column tile, 64-row range of n1, signal)
// =====================================================================================
__global__ void __launch_bounds__(256) k_joint_bwd(
    const float2* __restrict__ Y2, int64_t y_sb, const float* __restrict__ go, int64_t go_sb,
    float2* __restrict__ gY2, int64_t gy_sb, const JointUnit* __restrict__ units, int nfr,
    const int64_t* __restrict__ tiles, int n_blocks, const BlockInfo* __restrict__ binfo,
    const float2* __restrict__ hfr, int P, const float* __restrict__ phiF_k, const int64_t* __restrict__ phiF_off,
    uint64_t own, int maxLf, const float* __restrict__ thr) {
  extern __shared__ float4 smem4[];
  const int bi = find_idx(tiles, n_blocks, blockIdx.x);
  const BlockInfo bf = binfo[bi];
  const JointUnit U0 = units[bi * nfr];
  const int K = U0.n1_max;
  const int64_t ntc = (bf.n_cols + kJC - 1) / kJC;
  const int64_t loc = blockIdx.x - tiles[bi];
  const int64_t ct = loc % ntc;
  const int nr = (int)(loc / ntc);
  const int n0 = nr * kJN;
  const int KB = min(kJN, K - n0);
  const int b = blockIdx.y;
  const int tid = threadIdx.x;
  const int64_t col0 = ct * kJC;

  float2* Ys = reinterpret_cast<float2*>(smem4);      // [K][64]
  float2* hs = Ys + K * kJC;                          // [P]
  float2* Gw = hs + P;                                // [64][64] (also split-reduction scratch)
  float* gs = reinterpret_cast<float*>(Gw + kJR * kJC);  // [maxLf]
  float* Go = gs + maxLf;                             // [32][64]
  int* hbs = reinterpret_cast<int*>(Go + 32 * kJC);   // [64]

  const float2* ysrc = Y2 + b * y_sb + bf.y_off;
  for (int idx = tid; idx < K * kJC; idx += 256) {
    int n = idx / kJC, c = idx % kJC;
    int64_t col = col0 + c;
    float2 v = make_float2(0.f, 0.f);
    if (col < bf.n_cols) v = ysrc[(int64_t)n * bf.T2 + (bf.c_lo + col) % bf.T2];
    Ys[idx] = v;
  }

  // GEMM2 thread mapping: tiles of 4 n x 4 cols, r-split S
  const int NG = (KB + 3) / 4;
  const int T = NG * 16;
  const int S = max(1, 256 / T);
  const bool g2 = tid < T * S;
  const int tile2 = tid % T, split = tid / T;
  const int ng = tile2 / 16, cg = tile2 % 16;
  float2 gacc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) gacc[i][c] = make_float2(0.f, 0.f);

  const int tr = tid >> 4, tc = tid & 15;
  const float th2 = thr[b] * thr[b];
  for (int f = 0; f < nfr; ++f) {
    const int uidx = bi * nfr + f;
    if (!owns_block(own, bi)) continue;
    const JointUnit U = units[uidx];
    const int Lf = (int)U.Lf;
    __syncthreads();  // previous users of hs/gs/Go are done
    for (int idx = tid; idx < P; idx += 256) hs[idx] = hfr[(int64_t)U.f * P + idx];
    const float* gsrc = phiF_k + phiF_off[U.kf];
    for (int idx = tid; idx < Lf; idx += 256) gs[idx] = gsrc[idx];
    for (int idx = tid; idx < U.rows_out * kJC; idx += 256) {
      int q = idx / kJC, c = idx % kJC;
      int64_t col = col0 + c;
      Go[idx] = (col < bf.n_cols) ? go[b * go_sb + U.o_off + (int64_t)q * bf.n_cols + col] : 0.f;
    }
    __syncthreads();
    for (int64_t r0 = 0; r0 < U.n_rows; r0 += kJR) {
      int hb[4], rr[4];
      bool valid[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int64_t lr = r0 + tr * 4 + i;
        valid[i] = lr < U.n_rows;
        int r = (int)((U.r_lo + lr) % Lf);
        rr[i] = r;
        hb[i] = (r << U.kf) & (P - 1);
      }
      if (tc == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) hbs[tr * 4 + i] = hb[i];
      }
      // GEMM1 recompute: w = M_f y
      float2 acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[i][c] = make_float2(0.f, 0.f);
      for (int n = 0; n < K; ++n) {
        const float4* yp = reinterpret_cast<const float4*>(Ys + n * kJC + tc * 4);
        float4 ya = yp[0], yb = yp[1];
        float2 y[4] = {make_float2(ya.x, ya.y), make_float2(ya.z, ya.w), make_float2(yb.x, yb.y),
                       make_float2(yb.z, yb.w)};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float2 h = hs[(hb[i] - n) & (P - 1)];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            acc[i][c].x = fmaf(h.x, y[c].x, fmaf(-h.y, y[c].y, acc[i][c].x));
            acc[i][c].y = fmaf(h.x, y[c].y, fmaf(h.y, y[c].x, acc[i][c].y));
          }
        }
      }
      // g_v = Phi_F^T g_o ; g_w = (w/|w|) g_v  -> Gw
#pragma unroll
      for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float gv = 0.f;
          if (valid[i]) {
            for (int q = 0; q < U.rows_out; ++q)
              gv = fmaf(gs[((q << U.d) - rr[i]) & (Lf - 1)], Go[q * kJC + tc * 4 + c], gv);
          }
          float m2 = acc[i][c].x * acc[i][c].x + acc[i][c].y * acc[i][c].y;
          float s = (valid[i] && m2 > FLT_MIN && m2 > th2) ? gv * rsqrtf(m2) : 0.f;
          Gw[(tr * 4 + i) * kJC + tc * 4 + c] = make_float2(acc[i][c].x * s, acc[i][c].y * s);
        }
      }
      __syncthreads();
      // GEMM2: gY[n][c] += sum_i conj(h[(hb_i - n) mod P]) Gw[i][c]
      if (g2) {
        for (int i = split; i < kJR; i += S) {
          const int hbi = hbs[i];
          const float4* gp = reinterpret_cast<const float4*>(Gw + i * kJC + cg * 4);
          float4 ga = gp[0], gb = gp[1];
          float2 gw[4] = {make_float2(ga.x, ga.y), make_float2(ga.z, ga.w), make_float2(gb.x, gb.y),
                          make_float2(gb.z, gb.w)};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float2 h = hs[(hbi - (n0 + ng * 4 + j)) & (P - 1)];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              gacc[j][c].x = fmaf(h.x, gw[c].x, fmaf(h.y, gw[c].y, gacc[j][c].x));
              gacc[j][c].y = fmaf(h.x, gw[c].y, fmaf(-h.y, gw[c].x, gacc[j][c].y));
            }
          }
        }
      }
      __syncthreads();
    }
  }
  // reduce the r-splits in a fixed order and write g_Y2 (columns of this tile, rows n0..n0+KB)
  __syncthreads();
  float2* red = Gw;  // S*T*16 <= 256*16 complex = 4096 = kJR*kJC
  if (g2) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int c = 0; c < 4; ++c) red[(split * T + tile2) * 16 + j * 4 + c] = gacc[j][c];
  }
  __syncthreads();
  float2* gdst = gY2 + b * gy_sb + bf.y_off;
  for (int idx = tid; idx < T * 16; idx += 256) {
    int t2 = idx / 16, e = idx % 16;
    int j = e / 4, c = e % 4;
    int n = n0 + (t2 / 16) * 4 + j;
    int cc = (t2 % 16) * 4 + c;
    float2 s = make_float2(0.f, 0.f);
    for (int sp = 0; sp < S; ++sp) s = cadd(s, red[(sp * T + t2) * 16 + e]);
    int64_t col = col0 + cc;
    if (n < n0 + KB && col < bf.n_cols) gdst[(int64_t)n * bf.T2 + (bf.c_lo + col) % bf.T2] = s;
  }
}


// =====================================================================================
// Joint stage backward on CUDA cores for the blocks the tensor-core kernel does not take (large
// n1_max, few columns): one CTA = (block, 32-column tile, signal) over ALL K rows of n1, so W is
// recomputed exactly once; g_Y2 accumulates in SMEM (each thread owns fixed entries: deterministic).
// =====================================================================================
constexpr int kB2C = 32;
__global__ void __launch_bounds__(256) k_joint_bwd2(
    const float2* __restrict__ Y2, int64_t y_sb, const float* __restrict__ go, int64_t go_sb,
    float2* __restrict__ gY2, int64_t gy_sb, const JointUnit* __restrict__ units, int nfr,
    const int64_t* __restrict__ tiles, int n_blocks, const BlockInfo* __restrict__ binfo,
    const float2* __restrict__ hfr, int P, const float* __restrict__ phiF_k, const int64_t* __restrict__ phiF_off,
    uint64_t own, int maxLf, const float* __restrict__ thr) {
  extern __shared__ float4 smem4[];
  const int bi = find_idx(tiles, n_blocks, blockIdx.x);
  const BlockInfo bf = binfo[bi];
  const int K = units[bi * nfr].n1_max;
  const int64_t col0 = (int64_t)(blockIdx.x - tiles[bi]) * kB2C;
  const int b = blockIdx.y;
  const int tid = threadIdx.x;
  float2* Ys = reinterpret_cast<float2*>(smem4);     // [K][32]
  float2* Gy = Ys + K * kB2C;                        // [K][32]
  float2* hs = Gy + K * kB2C;                        // [P]
  float2* Gw = hs + P;                               // [64][32]
  float* gs = reinterpret_cast<float*>(Gw + kJR * kB2C);  // [maxLf]
  float* Go = gs + maxLf;                            // [32][32]
  int* hbs = reinterpret_cast<int*>(Go + 32 * kB2C); // [64]
  const float2* ysrc = Y2 + b * y_sb + bf.y_off;
  for (int idx = tid; idx < K * kB2C; idx += 256) {
    const int n = idx / kB2C, c = idx % kB2C;
    const int64_t col = col0 + c;
    Ys[idx] = (col < bf.n_cols) ? ysrc[(int64_t)n * bf.T2 + (bf.c_lo + col) % bf.T2] : make_float2(0.f, 0.f);
    Gy[idx] = make_float2(0.f, 0.f);
  }
  const float th2 = thr[b] * thr[b];
  const int tr = tid >> 4, tc = tid & 15;            // GEMM1: 4 rows x 2 columns per thread
  const int NG = (K + 3) / 4;                        // GEMM2: tiles of 4 n x 2 columns
  const int ntile2 = NG * 16;
  for (int f = 0; f < nfr; ++f) {
    const int uidx = bi * nfr + f;
    if (!owns_block(own, bi)) continue;
    const JointUnit U = units[uidx];
    const int Lf = (int)U.Lf;
    __syncthreads();
    for (int idx = tid; idx < P; idx += 256) hs[idx] = hfr[(int64_t)U.f * P + idx];
    const float* gsrc = phiF_k + phiF_off[U.kf];
    for (int idx = tid; idx < Lf; idx += 256) gs[idx] = gsrc[idx];
    for (int idx = tid; idx < U.rows_out * kB2C; idx += 256) {
      const int q = idx / kB2C, c = idx % kB2C;
      const int64_t col = col0 + c;
      Go[idx] = (col < bf.n_cols) ? go[b * go_sb + U.o_off + (int64_t)q * bf.n_cols + col] : 0.f;
    }
    __syncthreads();
    for (int64_t r0 = 0; r0 < U.n_rows; r0 += kJR) {
      int hb[4], rr[4];
      bool valid[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t lr = r0 + tr * 4 + i;
        valid[i] = lr < U.n_rows;
        const int r = (int)((U.r_lo + lr) % Lf);
        rr[i] = r;
        hb[i] = (r << U.kf) & (P - 1);
      }
      if (tc == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) hbs[tr * 4 + i] = hb[i];
      }
      float2 acc[4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = make_float2(0.f, 0.f);
#pragma unroll 2
      for (int n = 0; n < K; ++n) {
        const float4 yv = *reinterpret_cast<const float4*>(Ys + n * kB2C + tc * 2);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 h = hs[(hb[i] - n) & (P - 1)];
          acc[i][0].x = fmaf(h.x, yv.x, fmaf(-h.y, yv.y, acc[i][0].x));
          acc[i][0].y = fmaf(h.x, yv.y, fmaf(h.y, yv.x, acc[i][0].y));
          acc[i][1].x = fmaf(h.x, yv.z, fmaf(-h.y, yv.w, acc[i][1].x));
          acc[i][1].y = fmaf(h.x, yv.w, fmaf(h.y, yv.z, acc[i][1].y));
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float gv = 0.f;
          if (valid[i])
            for (int q = 0; q < U.rows_out; ++q)
              gv = fmaf(gs[((q << U.d) - rr[i]) & (Lf - 1)], Go[q * kB2C + tc * 2 + c], gv);
          const float m2 = acc[i][c].x * acc[i][c].x + acc[i][c].y * acc[i][c].y;
          const float s = (valid[i] && m2 > FLT_MIN && m2 > th2) ? gv * rsqrtf(m2) : 0.f;
          Gw[(tr * 4 + i) * kB2C + tc * 2 + c] = make_float2(acc[i][c].x * s, acc[i][c].y * s);
        }
      }
      __syncthreads();
      // GEMM2: Gy[n][c] += sum_i conj(h[(hb_i - n) mod P]) Gw[i][c]
      const int nrow = (int)((U.n_rows - r0) < kJR ? (U.n_rows - r0) : kJR);
      for (int t2 = tid; t2 < ntile2; t2 += 256) {
        const int ng = t2 >> 4, cg = t2 & 15;
        float2 a2[4][2];
#pragma unroll
        for (int j = 0; j < 4; ++j) a2[j][0] = a2[j][1] = make_float2(0.f, 0.f);
        for (int i = 0; i < nrow; ++i) {
          const int hbi = hbs[i];
          const float4 gw = *reinterpret_cast<const float4*>(Gw + i * kB2C + cg * 2);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 h = hs[(hbi - (ng * 4 + j)) & (P - 1)];
            a2[j][0].x = fmaf(h.x, gw.x, fmaf(h.y, gw.y, a2[j][0].x));
            a2[j][0].y = fmaf(h.x, gw.y, fmaf(-h.y, gw.x, a2[j][0].y));
            a2[j][1].x = fmaf(h.x, gw.z, fmaf(h.y, gw.w, a2[j][1].x));
            a2[j][1].y = fmaf(h.x, gw.w, fmaf(-h.y, gw.z, a2[j][1].y));
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int n = ng * 4 + j;
          if (n < K) {
            float2* g0 = Gy + n * kB2C + cg * 2;
            g0[0] = cadd(g0[0], a2[j][0]);
            g0[1] = cadd(g0[1], a2[j][1]);
          }
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();
  float2* gdst = gY2 + b * gy_sb + bf.y_off;
  for (int idx = tid; idx < K * kB2C; idx += 256) {
    const int n = idx / kB2C, c = idx % kB2C;
    const int64_t col = col0 + c;
    if (col < bf.n_cols) gdst[(int64_t)n * bf.T2 + (bf.c_lo + col) % bf.T2] = Gy[idx];
  }
}

// =====================================================================================
// phi_T along time (Eq.4, level s2, stride T) -> packed order-2 coefficients; one warp per output
// =====================================================================================
__global__ void k_phiT_fwd(const float* __restrict__ o, int64_t o_sb, float* __restrict__ S, int64_t S_sb,
                           const JointUnit* __restrict__ units, const int64_t* __restrict__ ucoef, int n_units,
                           const BlockInfo* __restrict__ binfo, const float* __restrict__ phiT_half,
                           const int64_t* __restrict__ phiT_off, const int64_t* __restrict__ phiT_H,
                           int64_t o2_start, int64_t n_o2, int64_t frames, int64_t m0, uint64_t own) {
  const int64_t q = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.y;
  if (q >= n_o2) return;
  const int u = find_idx(ucoef, n_units, q);
  if (!owns_block(own, units[u].bi)) return;
  const JointUnit U = units[u];
  const BlockInfo bf = binfo[U.bi];
  const int64_t loc = q - ucoef[u];
  const int64_t rho = loc / frames, tp = loc % frames;
  const int64_t H = phiT_H[bf.s2];
  const float* t = phiT_half + phiT_off[bf.s2];
  const float* src = o + b * o_sb + U.o_off + rho * bf.n_cols;
  double acc = 0;
  if (bf.n_cols < bf.T2) {
    // unwrapped: column index of position m*D + j is (m - m0)*D + H + j (no modulo)
    const int64_t base = (tp)*bf.D + H;
    for (int64_t j = -H + lane; j <= H; j += 32)
      acc += (double)__ldg(t + (j < 0 ? -j : j)) * (double)src[base + j];
  } else {
    int64_t jlo, jhi;
    sym_range(H, bf.T2, &jlo, &jhi);
    const int64_t cm = (m0 + tp) * bf.D;
    for (int64_t j = jlo + lane; j <= jhi; j += 32) {
      int64_t i = (cm + j - bf.c_lo) % bf.T2;
      if (i < 0) i += bf.T2;
      acc += (double)__ldg(t + (j < 0 ? -j : j)) * (double)src[i];
    }
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (lane == 0) S[b * S_sb + o2_start + q] = (float)acc;
}

// g_o[u][rho][i] = sum_{t'} tT_s2[dist(m0+t')*D - c_i] r[path][rho][t']
__global__ void k_phiT_adj(const float* __restrict__ rres, int64_t r_sb, float* __restrict__ go, int64_t go_sb,
                           const JointUnit* __restrict__ units, const int64_t* __restrict__ uo, int n_units,
                           const BlockInfo* __restrict__ binfo, const float* __restrict__ phiT_half,
                           const int64_t* __restrict__ phiT_off, const int64_t* __restrict__ phiT_H,
                           const int64_t* __restrict__ ucoef, int64_t o2_start, int64_t o_size, int64_t frames,
                           int64_t m0, uint64_t own) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (q >= o_size) return;
  const int u = find_idx(uo, n_units, q);
  if (!owns_block(own, units[u].bi)) return;
  const JointUnit U = units[u];
  const BlockInfo bf = binfo[U.bi];
  const int64_t loc = q - U.o_off;
  const int64_t rho = loc / bf.n_cols, i = loc % bf.n_cols;
  const int64_t H = phiT_H[bf.s2];
  const float* t = phiT_half + phiT_off[bf.s2];
  const float* rr = rres + b * r_sb + o2_start + ucoef[u] + rho * frames;
  double acc = 0;
  if (bf.n_cols < bf.T2) {
    // unwrapped coordinates: column i sits at x = m0*D - H + i; frame m at m*D
    const int64_t x = m0 * bf.D - H + i;
    int64_t mlo = x - H <= 0 ? -((H - x) / bf.D) : (x - H + bf.D - 1) / bf.D;
    int64_t mhi = (x + H) >= 0 ? (x + H) / bf.D : -((-(x + H) + bf.D - 1) / bf.D);
    mlo = mlo < m0 ? m0 : mlo;
    mhi = mhi > m0 + frames - 1 ? m0 + frames - 1 : mhi;
    for (int64_t m = mlo; m <= mhi; ++m) {
      const int64_t dd = m * bf.D - x;
      acc += (double)__ldg(t + (dd < 0 ? -dd : dd)) * (double)rr[m - m0];
    }
  } else {
    const int64_t c = (bf.c_lo + i) % bf.T2;
    for (int64_t tp = 0; tp < frames; ++tp) {
      int64_t dd = cdist((m0 + tp) * bf.D - c, bf.T2);
      if (dd <= H) acc += (double)__ldg(t + dd) * (double)rr[tp];
    }
  }
  go[b * go_sb + q] = (float)acc;
}

constexpr int kPhiTCols = 1024;   // adjoint columns per CTA (jtfs_api.cu builds the tile table with this step)
// ---- phi_T over time, row-tiled: one CTA per (unit, rho) row and kPhiTCols-column tile, the tile's (u, rho,
// first column) read from a per-tile table (broadcast loads), float accumulation.
// g_o[u][rho][i] = sum_{t'} tT_s2[dist((m0+t')D - c_i)] r[path][rho][t']  (adjoint of Eq.4's phi_T + stride)
__global__ void __launch_bounds__(256) k_phiT_adj2(
    const float* __restrict__ rres, int64_t r_sb, float* __restrict__ go, int64_t go_sb,
    const JointUnit* __restrict__ units, const BlockInfo* __restrict__ binfo, const float* __restrict__ phiT_half,
    const int64_t* __restrict__ phiT_off, const int64_t* __restrict__ phiT_H, const int64_t* __restrict__ ucoef,
    const int32_t* __restrict__ tinfo, int64_t o2_start, int frames, int64_t m0, uint64_t own) {
  struct { int u, rho; int64_t c0; } R;
  R.u = __ldg(tinfo + 3 * blockIdx.x);
  R.rho = __ldg(tinfo + 3 * blockIdx.x + 1);
  R.c0 = __ldg(tinfo + 3 * blockIdx.x + 2);
  __shared__ float rr[256];
  const int b = blockIdx.y;
  if (!owns_block(own, units[R.u].bi)) return;
  const JointUnit U = units[R.u];
  const BlockInfo bf = binfo[U.bi];
  const float* rsrc = rres + b * r_sb + o2_start + ucoef[R.u] + (int64_t)R.rho * frames;
  for (int t = threadIdx.x; t < frames; t += 256) rr[t] = rsrc[t];
  __syncthreads();
  const int H = (int)phiT_H[bf.s2];
  const float* tT = phiT_half + phiT_off[bf.s2];
  const int D = bf.D;
  float* gdst = go + b * go_sb + U.o_off + (int64_t)R.rho * bf.n_cols;
  const int lgD = __ffs(D) - 1;
  // kPhiTCols columns per CTA, 256 apart per thread (coalesced stores), one table lookup per CTA
  for (int64_t i = R.c0 + threadIdx.x; i < R.c0 + kPhiTCols && i < bf.n_cols; i += 256) {
    float acc = 0.f;
    if (bf.n_cols < bf.T2) {
      // unwrapped coordinates: column i sits at x = m0 D - H + i; frame m at m D; |m D - x| <= H
      // D is a power of two: ceil / floor division by arithmetic shifts (no 64-bit divides per column)
      const int64_t x = m0 * D - H + i;
      const int64_t lo = x - H, hi = x + H;
      int64_t mlo = -((-lo) >> lgD);
      int64_t mhi = hi >> lgD;
      if (mlo < m0) mlo = m0;
      if (mhi > m0 + frames - 1) mhi = m0 + frames - 1;
      int dd = (int)(mlo * D - x);
      for (int64_t m = mlo; m <= mhi; ++m, dd += D) acc = fmaf(__ldg(tT + (dd < 0 ? -dd : dd)), rr[m - m0], acc);
    } else {
      const int64_t c = (bf.c_lo + i) % bf.T2;
      for (int tp = 0; tp < frames; ++tp) {
        const int64_t dd = cdist((m0 + tp) * D - c, bf.T2);
        if (dd <= H) acc = fmaf(__ldg(tT + dd), rr[tp], acc);
      }
    }
    gdst[i] = acc;
  }
}

// S[coef(u, rho, t')] = sum_j tT_s2[|j|] o[u][rho][col(t' D + j)]: one CTA per (unit, rho) row (tile 0 of
// each row only), the half kernel staged in SMEM when it fits, one warp per frame (lanes stride j)
__global__ void __launch_bounds__(256) k_phiT_fwd2(
    const float* __restrict__ o, int64_t o_sb, float* __restrict__ S, int64_t S_sb,
    const JointUnit* __restrict__ units, const int64_t* __restrict__ ucoef, const BlockInfo* __restrict__ binfo,
    const float* __restrict__ phiT_half, const int64_t* __restrict__ phiT_off, const int64_t* __restrict__ phiT_H,
    const int32_t* __restrict__ rows_u, int64_t o2_start, int frames, int64_t m0, uint64_t own) {
  extern __shared__ float tsm[];
  const int u = rows_u[2 * blockIdx.x], rho = rows_u[2 * blockIdx.x + 1];
  if (!owns_block(own, units[u].bi)) return;
  const int b = blockIdx.y;
  const JointUnit U = units[u];
  const BlockInfo bf = binfo[U.bi];
  const int H = (int)phiT_H[bf.s2];
  const float* tg = phiT_half + phiT_off[bf.s2];
  const bool in_sm = H + 1 <= kPhiTSmem;
  if (in_sm)
    for (int j = threadIdx.x; j <= H; j += 256) tsm[j] = tg[j];
  __syncthreads();
  const float* tT = in_sm ? tsm : tg;
  const float* src = o + b * o_sb + U.o_off + (int64_t)rho * bf.n_cols;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* dst = S + b * S_sb + o2_start + ucoef[u] + (int64_t)rho * frames;
  for (int tp = warp; tp < frames; tp += 8) {
    float acc = 0.f;
    if (bf.n_cols < bf.T2) {
      const int64_t base = (int64_t)tp * bf.D + H;       // unwrapped: column of position m D + j
      for (int j = -H + lane; j <= H; j += 32) acc = fmaf(tT[j < 0 ? -j : j], src[base + j], acc);
    } else {
      int64_t jlo, jhi;
      sym_range(H, bf.T2, &jlo, &jhi);
      const int64_t cm = (m0 + tp) * bf.D;
      for (int64_t j = jlo + lane; j <= jhi; j += 32) {
        int64_t i = (cm + j - bf.c_lo) % bf.T2;
        if (i < 0) i += bf.T2;
        acc = fmaf(tT[j < 0 ? -j : j], src[i], acc);
      }
    }
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sh);
    if (lane == 0) dst[tp] = acc;
  }
}

// ---- phi_T adjoint as a banded GEMM (blocks whose needed columns are not the whole circle, i.e.
// unwrapped halo-pruned columns). For one block all rows (unit, rho) share the column grid: column i sits
// at x = m0 D - H + i, frame t' at (m0 + t') D, so Eq.4's phi_T + stride-T decimation is S[row][t'] =
// sum_i Phi[t'][i] o[row][i] with Phi[t'][i] = tT_s2[|t' D + H - i|] (zero beyond H), and its adjoint is
// g_o = R Phi. (The forward keeps the per-row kernel k_phiT_fwd2: one warp per frame reading a contiguous
// window; a banded-GEMM forward measured slower, 18.0 vs 14.3 ms at c4.)
// adjoint: g_o[row][i] = sum_t' Phi[t'][i] r[row][t'] for a 32-row group and a 256-column tile; the tile's
// frame band (<= 32 frames per pass) and r staged in SMEM; 8 rows x 4 columns per thread
__global__ void __launch_bounds__(256) k_phiT_adj3(
    const float* __restrict__ rres, int64_t r_sb, float* __restrict__ go, int64_t go_sb,
    const int32_t* __restrict__ grp, const int32_t* __restrict__ grows, const int32_t* __restrict__ atiles,
    const JointUnit* __restrict__ units, const BlockInfo* __restrict__ binfo, const float* __restrict__ phiT_half,
    const int64_t* __restrict__ phiT_off, const int64_t* __restrict__ phiT_H, const int64_t* __restrict__ ucoef,
    int64_t o2_start, int frames, uint64_t own) {
  __shared__ __align__(16) float sW[32][256];
  __shared__ float sR[32][33];
  const int gi = atiles[2 * blockIdx.x];
  const int64_t c0 = (int64_t)atiles[2 * blockIdx.x + 1] * 256;
  const int32_t* G = grp + 8 * gi;
  const int r0 = G[0], nr = G[1], bi = G[2];
  if (!owns_block(own, bi)) return;
  const int b = blockIdx.y;
  const BlockInfo bf = binfo[bi];
  const int D = bf.D;
  const int64_t H = phiT_H[bf.s2];
  const float* tT = phiT_half + phiT_off[bf.s2];
  const int tid = threadIdx.x, cq = tid & 63, rg = tid >> 6;
  __shared__ int64_t rcoef[32];                             // residual offset of each row (per signal)
  if (tid < 32)
    rcoef[tid] = tid < nr ? o2_start + ucoef[grows[2 * (r0 + tid)]] + (int64_t)grows[2 * (r0 + tid) + 1] * frames : 0;
  __syncthreads();
  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  // frames reaching columns [c0, c0 + 255]: t' D + 2H >= c0 and t' D <= c0 + 255
  const int64_t mlo = (c0 - 2 * H) <= 0 ? 0 : (c0 - 2 * H + D - 1) / D;
  const int64_t mhi = min((int64_t)frames - 1, (c0 + 255) / D);
  for (int64_t m0 = mlo; m0 <= mhi; m0 += 32) {
    const int nm = (int)min((int64_t)32, mhi - m0 + 1);
    for (int idx = tid; idx < 32 * 32; idx += 256) {
      const int r = idx >> 5, m = idx & 31;
      float v = 0.f;
      if (r < nr && m < nm) v = rres[b * r_sb + rcoef[r] + m0 + m];
      sR[r][m] = v;
    }
    for (int idx = tid; idx < 32 * 256; idx += 256) {
      const int m = idx >> 8, k = idx & 255;
      const int64_t dd = (m0 + m) * D + H - (c0 + k);
      const int64_t ad = dd < 0 ? -dd : dd;
      sW[m][k] = (m < nm && ad <= H) ? __ldg(tT + ad) : 0.f;
    }
    __syncthreads();
    for (int m = 0; m < nm; ++m) {
      const float4 w = *reinterpret_cast<const float4*>(&sW[m][4 * cq]);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float rv = sR[rg * 8 + i][m];
        acc[i][0] = fmaf(rv, w.x, acc[i][0]);
        acc[i][1] = fmaf(rv, w.y, acc[i][1]);
        acc[i][2] = fmaf(rv, w.z, acc[i][2]);
        acc[i][3] = fmaf(rv, w.w, acc[i][3]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = rg * 8 + i;
    if (r >= nr) continue;
    const int u = grows[2 * (r0 + r)], rho = grows[2 * (r0 + r) + 1];
    float* dst = go + b * go_sb + units[u].o_off + (int64_t)rho * bf.n_cols;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = c0 + 4 * cq + j;
      if (c < bf.n_cols) dst[c] = acc[i][j];
    }
  }
}

// loss (R19): r = S - St on owned order-1/2 coefficients (0 elsewhere), E_b = 1/2 sum r^2. Two passes
// for a deterministic sum spread over the SMs: kLossParts CTAs per signal write float64 partials (fixed
// coefficient ranges), one warp per signal adds them in a fixed order.
constexpr int kLossParts = 32;
// LossReport: one CTA per (path, signal), float64 partial sums in a fixed tree order (deterministic)
__global__ void __launch_bounds__(256) k_loss_report(const float* __restrict__ S, const float* __restrict__ St,
                                                     int64_t n_coef, const int64_t* __restrict__ path_off,
                                                     float* __restrict__ rep, int n_paths) {
  __shared__ double red[256];
  const int q = blockIdx.x, b = blockIdx.y;
  const int64_t a = path_off[q], e = path_off[q + 1];
  double acc = 0.0;
  for (int64_t i = a + threadIdx.x; i < e; i += 256) {
    const double r = (double)S[b * n_coef + i] - (double)St[b * n_coef + i];
    acc += r * r;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) rep[(int64_t)b * n_paths + q] = (float)(0.5 * red[0]);
}

void launch_loss_report(const Plan& p, const DeviceTables& d, const float* S, const float* St, float* rep, int B,
                        cudaStream_t st) {
  dim3 g((unsigned)p.paths.size(), (unsigned)B);
  k_loss_report<<<g, 256, 0, st>>>(S, St, p.n_coef, d.path_off, rep, (int)p.paths.size());
  count_launch();
}

__global__ void __launch_bounds__(256) k_loss(const float* __restrict__ S, int64_t S_sb, const float* __restrict__ St,
                                              int64_t St_sb, float* __restrict__ r, int64_t r_sb,
                                              double* __restrict__ part_out, const int32_t* __restrict__ coef_path,
                                              const int32_t* __restrict__ path_unit, int64_t n_coef, uint64_t own) {
  const int b = blockIdx.y;
  const int64_t per = (n_coef + kLossParts - 1) / kLossParts;
  const int64_t lo = blockIdx.x * per, hi = lo + per < n_coef ? lo + per : n_coef;
  __shared__ double part[256];
  double acc = 0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += 256) {
    int pu = path_unit[coef_path[i]];
    const bool mine = (pu == -1) ? (own & kOwnOrder1) != 0 : (pu >= 0 && owns_block(own, pu));
    float d = mine ? S[b * S_sb + i] - St[b * St_sb + i] : 0.f;
    r[b * r_sb + i] = d;
    acc += (double)d * (double)d;
  }
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) part[threadIdx.x] += part[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part_out[b * kLossParts + blockIdx.x] = part[0];
}
__global__ void k_loss_final(const double* __restrict__ part, float* __restrict__ loss, int B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double acc = 0;
  for (int k = 0; k < kLossParts; ++k) acc += part[b * kLossParts + k];
  loss[b] = (float)(0.5 * acc);
}

}  // namespace jtfs

namespace jtfs {

// ------------------------------------------------------------------ launchers
void launch_o1_fwd(const Plan& p, const DeviceTables& d, const float* S1t, int64_t S1t_sb, float2* W1,
                   int64_t W1_sb, float* V2, int64_t V2_sb, float* S, int64_t S_sb, int B, cudaStream_t st) {
  const int nfr1 = 1 + (int)p.psi_fr_plus.size();
  const int P = (int)p.P;
  const int64_t m0 = p.pad_left / p.T;
  dim3 g1((unsigned)((p.P * p.Ft + 255) / 256), (unsigned)nfr1, (unsigned)B);
  k_o1_W<<<g1, 256, 0, st>>>(S1t, S1t_sb, W1, W1_sb, d.hfr, d.o1_rlo, d.o1_nrows, d.kf_of, d.hfr_H,
                             (int)p.psi1.size(), P, p.Ft);
  if (nfr1 > 1) {
    dim3 g2((unsigned)((p.P * p.frames + 255) / 256), (unsigned)(nfr1 - 1), (unsigned)B);
    k_o1_time<<<g2, 256, 0, st>>>(W1, W1_sb, V2, V2_sb, d.o1_nrows, d.phiT_half + p.phiT_off[p.log2T],
                                  p.phiT_H[p.log2T], P, p.Ft, p.frames, m0);
  }
  dim3 g3((unsigned)((p.o1_rows_out * p.frames + 63) / 64), (unsigned)nfr1, (unsigned)B);
  k_o1_out<<<g3, 256, 0, st>>>(W1, W1_sb, V2, V2_sb, S, S_sb, d.o1_rlo, d.o1_nrows, d.kf_of, d.phiF_k, d.phiF_off,
                               p.log2F, P, p.Ft, p.frames, m0, p.o1_rows_out);
  count_launch(nfr1 > 1 ? 3 : 2);
}

void launch_o1_bwd(const Plan& p, const DeviceTables& d, const float* r, int64_t r_sb, float2* W1,
                   int64_t W1_sb, float* V2, int64_t V2_sb, const float* S1t, int64_t S1t_sb, float* gS1t,
                   int64_t gS1t_sb, const float* thr, int B, cudaStream_t st) {
  (void)S1t; (void)S1t_sb;
  const int nfr1 = 1 + (int)p.psi_fr_plus.size();
  const int P = (int)p.P;
  const int64_t m0 = p.pad_left / p.T;
  if (nfr1 > 1) {
    dim3 g1((unsigned)((p.P * p.frames + 255) / 256), (unsigned)(nfr1 - 1), (unsigned)B);
    k_o1_bwd_rows<<<g1, 256, 0, st>>>(r, r_sb, V2, V2_sb, d.o1_rlo, d.o1_nrows, d.kf_of, d.phiF_k, d.phiF_off,
                                      p.log2F, P, p.frames, p.o1_rows_out);
    count_launch();
  }
  dim3 g2((unsigned)((p.P * p.Ft + 255) / 256), (unsigned)nfr1, (unsigned)B);
  k_o1_bwd_time<<<g2, 256, 0, st>>>(r, r_sb, W1, W1_sb, V2, V2_sb, d.o1_nrows, d.phiT_half + p.phiT_off[p.log2T],
                                    p.phiT_H[p.log2T], P, p.Ft, p.frames, m0, thr);
  dim3 g3((unsigned)((p.psi1.size() * p.Ft + 63) / 64), (unsigned)B);
  k_o1_bwd_S1t<<<g3, 256, 0, st>>>(W1, W1_sb, gS1t, gS1t_sb, d.hfr, d.o1_rlo, d.o1_nrows, d.kf_of, d.hfr_H,
                                   nfr1, (int)p.psi1.size(), P, p.Ft);
  count_launch(2);
}

static size_t joint_fwd_smem(const Plan& p, const DeviceTables& d, int ci, int kap) {
  return (size_t)d.fwd_kmax[ci] * kJC * 8 + (size_t)p.P * 8 + (size_t)d.maxLf * 4 + (size_t)16 * kap * kJC * 4;
}

template <int KAP>
static void launch_joint_fwd_kap(const Plan& p, const DeviceTables& d, int ci, const float2* Y2, int64_t y_sb,
                                 float* o, int64_t o_sb, uint64_t own, int B, cudaStream_t st) {
  if (d.fwd_n[ci] == 0) return;
  size_t sm = joint_fwd_smem(p, d, ci, KAP);
  cudaFuncSetAttribute(k_joint_fwd<KAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  dim3 g((unsigned)d.fwd_ntiles[ci], (unsigned)B);
  k_joint_fwd<KAP><<<g, 256, sm, st>>>(Y2, y_sb, o, o_sb, d.units, d.fwd_ulist[ci], d.fwd_tiles[ci], d.fwd_n[ci],
                                       d.binfo, d.hfr, (int)p.P, d.phiF_k, d.phiF_off, own);
  count_launch();
}

void launch_joint_fwd(const Plan& p, const DeviceTables& d, const float2* Y2, int64_t y_sb, float* o,
                      int64_t o_sb, uint64_t own, int B, cudaStream_t st) {
  launch_joint_fwd_kap<1>(p, d, 0, Y2, y_sb, o, o_sb, own, B, st);
  launch_joint_fwd_kap<2>(p, d, 1, Y2, y_sb, o, o_sb, own, B, st);
  launch_joint_fwd_kap<4>(p, d, 2, Y2, y_sb, o, o_sb, own, B, st);
  launch_joint_fwd_kap<8>(p, d, 3, Y2, y_sb, o, o_sb, own, B, st);
  launch_joint_fwd_kap<16>(p, d, 4, Y2, y_sb, o, o_sb, own, B, st);
  launch_joint_fwd_kap<32>(p, d, 5, Y2, y_sb, o, o_sb, own, B, st);
}

void launch_phiT_fwd(const Plan& p, const DeviceTables& d, const float* o, int64_t o_sb, float* S,
                     int64_t S_sb, uint64_t own, int B, cudaStream_t st) {
  if (d.n_o2 == 0 || d.phT_nrows == 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_phiT_fwd2, cudaFuncAttributeMaxDynamicSharedMemorySize, kPhiTSmem * 4);
    attr = true;
  }
  dim3 g((unsigned)d.phT_nrows, (unsigned)B);
  k_phiT_fwd2<<<g, 256, kPhiTSmem * 4, st>>>(o, o_sb, S, S_sb, d.units, d.ucoef, d.binfo, d.phiT_half, d.phiT_off,
                                             d.phiT_H, d.phT_rows_u, d.o2_start, (int)p.frames, p.pad_left / p.T,
                                             own);
  count_launch();
}

void launch_loss(const Plan& p, const DeviceTables& d, const float* S, int64_t S_sb, const float* St,
                 int64_t St_sb, float* r, int64_t r_sb, float* loss, double* part, uint64_t own, int B,
                 cudaStream_t st) {
  k_loss<<<dim3(kLossParts, B), 256, 0, st>>>(S, S_sb, St, St_sb, r, r_sb, part, d.coef_path, d.path_owner_unit,
                                              p.n_coef, own);
  k_loss_final<<<(B + 127) / 128, 128, 0, st>>>(part, loss, B);
  count_launch(2);
}

void launch_phiT_adj(const Plan& p, const DeviceTables& d, const float* r, int64_t r_sb, float* go,
                     int64_t go_sb, uint64_t own, int B, cudaStream_t st) {
  if (p.o_size == 0 || d.phT_ntiles == 0) return;
  if (d.ph3_natiles > 0) {
    k_phiT_adj3<<<dim3((unsigned)d.ph3_natiles, (unsigned)B), 256, 0, st>>>(
        r, r_sb, go, go_sb, d.ph3_groups, d.ph3_rows, d.ph3_atiles, d.units, d.binfo, d.phiT_half, d.phiT_off,
        d.phiT_H, d.ucoef, d.o2_start, (int)p.frames, own & d.ph3_mask);
    count_launch();
  }
  const uint64_t rest = own & ~d.ph3_mask & ((d.n_blocks >= 64 ? ~0ull : (1ull << d.n_blocks) - 1));
  if (rest == 0) return;
  dim3 g((unsigned)d.phT_ntiles, (unsigned)B);
  k_phiT_adj2<<<g, 256, 0, st>>>(r, r_sb, go, go_sb, d.units, d.binfo, d.phiT_half, d.phiT_off, d.phiT_H, d.ucoef,
                                 d.phT_tiles, d.o2_start, (int)p.frames,
                                 p.pad_left / p.T, rest);
  count_launch();
}

void launch_joint_bwd(const Plan& p, const DeviceTables& d, const float2* Y2, int64_t y_sb, const float* go,
                      int64_t go_sb, float2* gY2, int64_t gy_sb, const float* thr, uint64_t own, int B,
                      cudaStream_t st) {
  if (d.n_blocks == 0 || d.bwd_ntiles == 0) return;
  const size_t sm = (size_t)2 * d.Kmax_simt_bwd * kB2C * 8 + (size_t)p.P * 8 + (size_t)kJR * kB2C * 8 +
                    (size_t)d.maxLf * 4 + (size_t)32 * kB2C * 4 + 64 * 4;
  cudaFuncSetAttribute(k_joint_bwd2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  dim3 g((unsigned)d.bwd_ntiles, (unsigned)B);
  k_joint_bwd2<<<g, 256, sm, st>>>(Y2, y_sb, go, go_sb, gY2, gy_sb, d.units, (int)p.L_fr.size(), d.bwd_tiles,
                                   d.n_blocks, d.binfo, d.hfr, (int)p.P, d.phiF_k, d.phiF_off, own,
                                   d.maxLf, thr);
  count_launch();
}

}  // namespace jtfs
