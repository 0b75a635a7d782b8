// kernels_time.cu — time-axis stages of the JTFS path on sm_100a: padding, Fourier-domain
// filtering + subsampling (cdgmm + subsample_fourier), modulus, and
// the adjoints of those stages for the gradient; plus the metamer update.
// All HBM-bound; coalesced along the contiguous time / frequency axis.
#include <cuda_runtime.h>

#include <algorithm>

#include "device.cuh"

namespace jtfs {

__device__ __forceinline__ int64_t floor_div(int64_t a, int64_t b) {  // b > 0
  return a >= 0 ? a / b : -((-a + b - 1) / b);
}

__device__ __forceinline__ int find_job(const int64_t* __restrict__ tiles, int n, int64_t t) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (__ldg(tiles + mid) <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// R10 half-sample symmetric extension: xp[i] = x[e(i - pad_left)], e = 2N-periodic even extension.
__global__ void k_reflect_pad(const float* __restrict__ x, int64_t sx, double2* __restrict__ xp, int64_t N,
                              int64_t N_pad, int64_t pad_left) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N_pad) return;
  int b = blockIdx.y;
  int64_t t = (i - pad_left) % (2 * N);
  if (t < 0) t += 2 * N;
  int64_t src = t < N ? t : 2 * N - 1 - t;
  xp[(int64_t)b * N_pad + i] = make_double2((double)__ldg(x + b * sx + src), 0.0);
}

void launch_reflect_pad(const float* x, int64_t sx, double2* xp, const Plan& p, int B, cudaStream_t st) {
  dim3 g((unsigned)((p.N_pad + 255) / 256), (unsigned)B);
  k_reflect_pad<<<g, 256, 0, st>>>(x, sx, xp, p.N, p.N_pad, p.pad_left);
  count_launch();
}

// out[m] = scale * sum_{s in [lo, lo+len), s = m (mod L_out)} h[s-lo] * in[s mod L_in]
// i.e. cdgmm with a support-limited real response, then subsample_fourier (fold-mean).
template <class TI> struct GAcc { using T = float2; using R = float; };
template <> struct GAcc<double2> { using T = double2; using R = double; };
__device__ __forceinline__ void st_c(float2* p, double re, double im) { *p = make_float2((float)re, (float)im); }
__device__ __forceinline__ void st_c(double2* p, double re, double im) { *p = make_double2(re, im); }

template <class TI, class TO, class VT>
__global__ void __launch_bounds__(kGatherThreads) k_gather(const TI* __restrict__ in, int64_t in_sb,
                                                            TO* __restrict__ out, int64_t out_sb,
                                                            const GatherJob* __restrict__ jobs,
                                                            const int64_t* __restrict__ tiles, int njobs,
                                                            const VT* __restrict__ vals, uint64_t own) {
  using R = typename GAcc<TI>::R;
  const int64_t tile = blockIdx.x;
  const int b = blockIdx.y;
  const int j = find_job(tiles, njobs, tile);
  const GatherJob J = jobs[j];
  if (J.blk >= 0 && !owns_block(own, J.blk)) return;   // layer-2 block of another path shard
  const TI* src = in + b * in_sb + J.in_off;
  const int tsz = J.tl ? kGatherTileT : kGatherTile;
  const int64_t m0 = (tile - tiles[j]) * tsz;
  // T-layout jobs (layer-2 rows > 4096 points, whose inverse FFT then runs row-contiguous): the tile's
  // 4096 outputs are staged in SMEM [kk][k1] (m = m0 + k1 + L1 kk; k1 XOR-swizzled by kk, conflict-free
  // both ways) and written as runs of 4096 / L1 consecutive k2 per k1 row of the T-layout
  constexpr bool kCanT = sizeof(TO) == 8;
  __shared__ TO stg[kCanT ? kGatherTileT : 1];
  const int64_t L1t = J.L_out >> 12;
  const int lgL1t = J.tl ? 63 - __clzll(L1t) : 0;   // L1t: power of two (shifts, not 64-bit divides)
  for (int64_t m = m0 + threadIdx.x; m < J.L_out && m < m0 + tsz; m += kGatherThreads) {
    // L_in, L_out: powers of two (grid lengths N_pad >> k)
    int64_t s = J.lo + ((m - J.lo) & (J.L_out - 1));          // smallest s >= lo with s = m mod L_out
    R ax = 0, ay = 0;
    const int64_t msk = J.L_in - 1;
    for (; s < J.lo + J.len; s += J.L_out) {
      const R h = (R)__ldg(vals + J.val_off + (s - J.lo));
      const TI z = src[s & msk];
      R vx = (R)z.x, vy = (R)z.y;
      if (J.par >= 0) {   // pair-packed real rows (plan.h GatherJob::par)
        const TI w = src[(-s) & msk];
        if (J.par == 0) { vx = (R)0.5 * ((R)z.x + (R)w.x); vy = (R)0.5 * ((R)z.y - (R)w.y); }
        else { vx = (R)0.5 * ((R)z.y + (R)w.y); vy = (R)0.5 * ((R)w.x - (R)z.x); }
      }
      ax += h * vx;
      ay += h * vy;
    }
    if (kCanT && J.tl) {
      const int ml = (int)(m - m0), kk = ml >> lgL1t, k1 = ml & ((int)L1t - 1);
      st_c(stg + kk * L1t + (k1 ^ (kk & (L1t - 1))), (double)(ax * (R)J.scale), (double)(ay * (R)J.scale));
    } else {
      st_c(out + b * out_sb + J.out_off + m, (double)(ax * (R)J.scale), (double)(ay * (R)J.scale));
    }
  }
  if (kCanT && J.tl) {
    __syncthreads();
    const int lgW = 12 - lgL1t;                      // W = 4096 / L1t
    TO* dst = out + b * out_sb + J.out_off + (m0 >> lgL1t);
    for (int i = threadIdx.x; i < kGatherTileT; i += kGatherThreads) {
      const int k1 = i >> lgW, kk = i & ((1 << lgW) - 1);
      dst[((int64_t)k1 << 12) + kk] = stg[(kk << lgL1t) + (k1 ^ (kk & ((int)L1t - 1)))];
    }
  }
}

template <class TI, class TO, class VT>
static void gather_t(const TI* in, int64_t in_sb, TO* out, int64_t out_sb, const GatherJob* jobs,
                     const int64_t* tiles, int njobs, int64_t ntiles, const VT* vals, int B, cudaStream_t st,
                     uint64_t own = kOwnAll) {
  if (njobs <= 0 || ntiles <= 0) return;
  dim3 g((unsigned)ntiles, (unsigned)B);
  k_gather<TI, TO, VT><<<g, kGatherThreads, 0, st>>>(in, in_sb, out, out_sb, jobs, tiles, njobs, vals, own);
  count_launch();
}
void launch_gather(const float2* in, int64_t in_sb, float2* out, int64_t out_sb, const GatherJob* jobs,
                   const int64_t* tiles, int njobs, int64_t ntiles, const float* vals, int B, cudaStream_t st,
                   uint64_t own) {
  gather_t(in, in_sb, out, out_sb, jobs, tiles, njobs, ntiles, vals, B, st, own);
}
void launch_gather_dd(const double2* in, int64_t in_sb, double2* out, int64_t out_sb, const GatherJob* jobs,
                      const int64_t* tiles, int njobs, int64_t ntiles, const double* vals, int B, cudaStream_t st) {
  gather_t(in, in_sb, out, out_sb, jobs, tiles, njobs, ntiles, vals, B, st);
}
void launch_gather_df(const double2* in, int64_t in_sb, float2* out, int64_t out_sb, const GatherJob* jobs,
                      const int64_t* tiles, int njobs, int64_t ntiles, const float* vals, int B, cudaStream_t st,
                      uint64_t own) {
  gather_t(in, in_sb, out, out_sb, jobs, tiles, njobs, ntiles, vals, B, st, own);
}

// U1 = |Z1| as float64 rows for the next FFT, which runs in float64: the FFT's rounding is
// relative to the whole row (dominated by the envelope's mean), and the second-layer bands it feeds are far
// below that (reading R22). The rows are real, so two of a level group share one complex FFT
// (pair packing, the R2C trick): packed row p of group g = U1[2p] + i U1[2p + 1] (imaginary 0 for an odd
// last row); the gathers unpack the two spectra (GatherJob::par).
__global__ void k_modulus_pack(const float2* __restrict__ z, int64_t zsb, double2* __restrict__ u, int64_t usb,
                               PackGroups G) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= G.pstart[G.n]) return;
  int g = 0;
  while (g + 1 < G.n && q >= G.pstart[g + 1]) ++g;
  const int64_t loc = q - G.pstart[g];
  const int lgL = G.lgL[g];
  const int64_t p = loc >> lgL, e = loc & ((int64_t(1) << lgL) - 1);
  const float2* zr = z + blockIdx.y * zsb + G.off[g] + ((2 * p) << lgL) + e;
  const float2 va = zr[0];
  const float2 vb = (2 * p + 1 < G.count[g]) ? zr[int64_t(1) << lgL] : make_float2(0.f, 0.f);
  u[blockIdx.y * usb + q] =   // compact packed layout: element q
      make_double2((double)sqrtf(va.x * va.x + va.y * va.y), (double)sqrtf(vb.x * vb.x + vb.y * vb.y));
}

void launch_modulus_pack(const float2* z, int64_t zsb, double2* u, int64_t usb, const PackGroups& G, int B,
                         cudaStream_t st) {
  const int64_t n = G.pstart[G.n];
  dim3 g((unsigned)((n + 255) / 256), (unsigned)B);
  k_modulus_pack<<<g, 256, 0, st>>>(z, zsb, u, usb, G);
  count_launch();
}

// position of natural element n of a row of 2^lgL points in the T-layout of the four-step (fft.cuh):
// n = k1 + L1 k2 sits at k1 4096 + k2 (rows of <= 4096 points are natural)
__device__ __forceinline__ int64_t t_pos(int64_t n, int lgL) {
  if (lgL <= 12) return n;
  const int lgL1 = lgL - 12;
  return ((n & ((int64_t(1) << lgL1) - 1)) << 12) + (n >> lgL1);
}

// debug stage U1: unpack the pair-packed float64 rows -> fp32 [sum L1] in the natural row layout
__global__ void k_unpack_u1(const double2* __restrict__ u, int64_t usb, float* __restrict__ out, int64_t out_sb,
                            PackGroups G, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int g = 0;
  while (g + 1 < G.n && i >= G.off[g + 1]) ++g;
  const int lgL = G.lgL[g];
  const int64_t r = (i - G.off[g]) >> lgL, e = (i - G.off[g]) & ((int64_t(1) << lgL) - 1);
  const double2 v = u[blockIdx.y * usb + G.pstart[g] + ((r >> 1) << lgL) + t_pos(e, lgL)];
  out[blockIdx.y * out_sb + i] = (float)((r & 1) ? v.y : v.x);
}

// debug stage Z1: rows in T-layout -> natural order
__global__ void k_untranspose_rows(const float2* __restrict__ z, int64_t zsb, float2* __restrict__ out,
                                   int64_t out_sb, PackGroups G, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int g = 0;
  while (g + 1 < G.n && i >= G.off[g + 1]) ++g;
  const int lgL = G.lgL[g];
  const int64_t r = (i - G.off[g]) >> lgL, e = (i - G.off[g]) & ((int64_t(1) << lgL) - 1);
  out[blockIdx.y * out_sb + i] = z[blockIdx.y * zsb + G.off[g] + (r << lgL) + t_pos(e, lgL)];
}

void launch_untranspose_rows(const float2* z, int64_t zsb, float2* out, int64_t out_sb, const PackGroups& G,
                             int64_t n, int B, cudaStream_t st) {
  dim3 g((unsigned)((n + 255) / 256), (unsigned)B);
  k_untranspose_rows<<<g, 256, 0, st>>>(z, zsb, out, out_sb, G, n);
  count_launch();
}

void launch_unpack_u1(const double2* u, int64_t usb, float* out, int64_t out_sb, const PackGroups& G, int64_t n,
                      int B, cudaStream_t st) {
  dim3 g((unsigned)((n + 255) / 256), (unsigned)B);
  k_unpack_u1<<<g, 256, 0, st>>>(u, usb, out, out_sb, G, n);
  count_launch();
}

// real parts of float64 complex rows -> fp32 (debug stage U1)
__global__ void k_real_rows_d(const double2* __restrict__ in, int64_t in_sb, float* __restrict__ out, int64_t out_sb,
                              int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[blockIdx.y * out_sb + i] = (float)in[blockIdx.y * in_sb + i].x;
}

void launch_real_rows_d(const double2* in, int64_t in_sb, float* out, int64_t out_sb, int64_t n, int B,
                        cudaStream_t st) {
  dim3 g((unsigned)((n + 255) / 256), (unsigned)B);
  k_real_rows_d<<<g, 256, 0, st>>>(in, in_sb, out, out_sb, n);
  count_launch();
}

__global__ void k_real_rows(const float2* __restrict__ in, int64_t in_sb, int64_t in_off, float* __restrict__ out,
                            int64_t out_sb, int64_t out_off, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[blockIdx.y * out_sb + out_off + i] = in[blockIdx.y * in_sb + in_off + i].x;
}

void launch_real_rows(const float2* in, int64_t in_sb, int64_t in_off, float* out, int64_t out_sb,
                      int64_t out_off, int64_t n, int B, cudaStream_t st) {
  dim3 g((unsigned)((n + 255) / 256), (unsigned)B);
  k_real_rows<<<g, 256, 0, st>>>(in, in_sb, in_off, out, out_sb, out_off, n);
  count_launch();
}

// S0 = phi_T * x_p at stride T, unpadded (R14, R16): path 0 of the packed vector.
__global__ void k_s0_out(const float2* __restrict__ s0c, int64_t s0_sb, float* __restrict__ S, int64_t S_sb,
                         int64_t m0, int64_t frames) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= frames) return;
  S[blockIdx.y * S_sb + t] = s0c[blockIdx.y * s0_sb + m0 + t].x;
}

void launch_s0_out(const float2* s0c, int64_t s0_sb, float* S, int64_t S_sb, const Plan& p, int B,
                   cudaStream_t st) {
  dim3 g((unsigned)((p.frames + 255) / 256), (unsigned)B);
  k_s0_out<<<g, 256, 0, st>>>(s0c, s0_sb, S, S_sb, p.pad_left / p.T, p.frames);
  count_launch();
}

// Adjoint of layer 2 and of the S1 time average, in Fourier (R21: responses are real, so the
// adjoint of "multiply + fold-mean + IFFT" is "FFT + periodic extension + multiply"):
//   g_hat_U1[n1][m] = phiT_k1[m] GS[n1][m mod Ft] + sum_{blocks with n1 < n1_max} psi2_k1[m] GY[n1][m mod T2]
constexpr int kU1AdjTile = 1024;   // elements per CTA (jtfs_api.cu builds u1adj_tiles with this size)
__global__ void __launch_bounds__(256) k_adj_gather_u1(
    const float2* __restrict__ GS, int64_t GS_sb, const float2* __restrict__ GY, int64_t GY_sb,
    float2* __restrict__ out, int64_t out_sb, const int64_t* __restrict__ tiles, int N1,
    const int64_t* __restrict__ l1_off, const int32_t* __restrict__ n1_k1, const Support* __restrict__ phiT_sup,
    const Support* __restrict__ psi2_sup, const BlockInfo* __restrict__ binfo, const int32_t* __restrict__ nmax,
    int n_blocks, int log2T, int64_t N_pad, int64_t Ft, const float* __restrict__ vals, uint64_t own) {
  const int64_t tile = blockIdx.x;
  const int b = blockIdx.y;
  const int n1 = find_job(tiles, N1, tile);
  const int k1 = n1_k1[n1];
  const int64_t L1 = N_pad >> k1;
  // the CTA's filter n1 is fixed: the blocks that reach it, with their psi2 support and Y2 layout, are
  // gathered once into SMEM (the per-element loop then reads broadcast SMEM instead of chains of
  // dependent global loads)
  constexpr int kMaxB = 32;
  __shared__ int64_t s_lo[kMaxB], s_len[kMaxB], s_off[kMaxB], s_y[kMaxB], s_T2[kMaxB];
  __shared__ int s_nb;
  if (threadIdx.x == 0) {
    int nb = 0;
    for (int bi = 0; bi < n_blocks && nb < kMaxB; ++bi) {
      if (n1 >= nmax[bi] || !owns_block(own, bi)) continue;   // path shards: own blocks only
      const Support sp = psi2_sup[bi * (log2T + 1) + k1];
      const BlockInfo bf = binfo[bi];
      s_lo[nb] = sp.lo; s_len[nb] = sp.len; s_off[nb] = sp.off;
      s_y[nb] = bf.y_off + (int64_t)n1 * bf.T2; s_T2[nb] = bf.T2;
      ++nb;
    }
    s_nb = nb;
  }
  __syncthreads();
  const Support spT = phiT_sup[k1];
  const int nb = s_nb;
  // kU1AdjTile elements per CTA, 256 apart per thread (coalesced), one setup per CTA. Blocks whose rows
  // are longer than 4096 points hold their spectra in the four-step's T-layout (bin k1 + L1b k2 at
  // k1 4096 + k2, fft.cuh): the CTA's 1024 consecutive bins are staged in SMEM by runs of 1024 / L1b
  // consecutive k2 per k1 row ([kk][k1], k1 XOR-swizzled by kk), double-buffered (one barrier per block).
  // Summation order per element: phi_T term, then blocks ascending (as in the natural-layout loop).
  constexpr int kR = kU1AdjTile / 256;
  __shared__ float2 stg[2][kU1AdjTile];
  // within-row indices fit 32 bits (rows <= 2^22 points); powers of two divide by shifts
  const int L1m = (int)L1 - 1;
  const int mt0 = (int)((tile - tiles[n1]) * kU1AdjTile);
  const float2* gsrow = GS + b * GS_sb + (int64_t)n1 * Ft;
  const int Ftm = (int)Ft - 1;
  float2 acc[kR];
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int m = mt0 + threadIdx.x + 256 * r;
    acc[r] = make_float2(0.f, 0.f);
    const int t = (m - (int)spT.lo) & L1m;
    if (m <= L1m && t < (int)spT.len) {
      float h = __ldg(vals + spT.off + t);
      float2 v = gsrow[m & Ftm];
      acc[r] = make_float2(h * v.x, h * v.y);
    }
  }
  int sb = 0;
  for (int i = 0; i < nb; ++i) {
    const int T2 = (int)s_T2[i], lo = (int)s_lo[i], len = (int)s_len[i];
    const int d0 = (mt0 - lo) & L1m;
    if (len <= 0 || (d0 >= len && d0 + kU1AdjTile <= L1m + 1)) continue;   // CTA-uniform: no overlap
    const float2* gy = GY + b * GY_sb + s_y[i];
    const float* hv = vals + s_off[i];
    if (T2 > 4096) {
      const int lgL1b = __ffs(T2) - 1 - 12, L1b = 1 << lgL1b;      // L1b = T2 / 4096
      const int lgWb = 10 - lgL1b;                                  // Wb = 1024 / L1b
      const int mm0 = mt0 & (T2 - 1);
      const float2* src = gy + (mm0 >> lgL1b);
      for (int e = threadIdx.x; e < kU1AdjTile; e += 256) {
        const int kq = e >> lgWb, kk = e & ((1 << lgWb) - 1);
        stg[sb][(kk << lgL1b) + (kq ^ (kk & (L1b - 1)))] = src[((int64_t)kq << 12) + kk];
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        const int m = mt0 + threadIdx.x + 256 * r;
        const int t = (m - lo) & L1m;
        if (m <= L1m && t < len) {
          const int ml = threadIdx.x + 256 * r, kk = ml >> lgL1b, kq = ml & (L1b - 1);
          const float h = __ldg(hv + t);
          const float2 v = stg[sb][(kk << lgL1b) + (kq ^ (kk & (L1b - 1)))];
          acc[r].x = fmaf(h, v.x, acc[r].x);
          acc[r].y = fmaf(h, v.y, acc[r].y);
        }
      }
      sb ^= 1;
    } else {
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        const int m = mt0 + threadIdx.x + 256 * r;
        const int t = (m - lo) & L1m;
        if (m <= L1m && t < len) {
          const float h = __ldg(hv + t);
          const float2 v = gy[m & (T2 - 1)];
          acc[r].x = fmaf(h, v.x, acc[r].x);
          acc[r].y = fmaf(h, v.y, acc[r].y);
        }
      }
    }
  }
  float2* orow = out + b * out_sb + l1_off[n1];
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int m = mt0 + threadIdx.x + 256 * r;
    if (m <= L1m) orow[m] = acc[r];
  }
}

void launch_adj_gather_u1(const Plan& p, const DeviceTables& d, const float2* GS, int64_t GS_sb,
                          const float2* GY, int64_t GY_sb, float2* out, int64_t out_sb, int B,
                          cudaStream_t st, uint64_t own) {
  dim3 g((unsigned)d.u1adj_ntiles, (unsigned)B);
  k_adj_gather_u1<<<g, 256, 0, st>>>(GS, GS_sb, GY, GY_sb, out, out_sb, d.u1adj_tiles, (int)p.psi1.size(),
                                     d.l1_off, d.n1_k1, d.phiT_sup, d.psi2_sup, d.binfo, d.blk_nmax,
                                     d.n_blocks, p.log2T, p.N_pad, p.Ft, d.spec_vals, own);
  count_launch();
}

// Modulus adjoint (R22): g_Z1 = (Z1/|Z1|) * Re(g_U1), 0 where |Z1| < thr (in float64: Z1 is the
// complex64 copy of the float64 first layer, and cells down to the dead zone keep their phase).
__global__ void k_phase_mul(const float2* __restrict__ z, const float2* __restrict__ gu, int64_t gsb,
                            float2* __restrict__ out, int64_t n, int64_t sb, const float* __restrict__ thr) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t o = blockIdx.y * sb + i;
  const float2 v = z[o];
  const double m2 = (double)v.x * v.x + (double)v.y * v.y;
  const double g = gu[blockIdx.y * gsb + i].x;
  const double t = thr[blockIdx.y];
  const double s = (m2 > 0.0 && m2 >= t * t) ? g / sqrt(m2) : 0.0;
  out[o] = make_float2((float)(v.x * s), (float)(v.y * s));
}

void launch_phase_mul(const float2* z, const float2* gu, int64_t gsb, float2* out, int64_t n_per_b, int64_t sb,
                      const float* thr, int B, cudaStream_t st) {
  dim3 g((unsigned)((n_per_b + 255) / 256), (unsigned)B);
  k_phase_mul<<<g, 256, 0, st>>>(z, gu, gsb, out, n_per_b, sb, thr);
  count_launch();
}

// R22 dead-zone radius of the modulus adjoint: thr[b] = eps * RMS(y_b), eps = 1e-12;
// float64 partial sums combined in a fixed tree order (deterministic)
__global__ void __launch_bounds__(256) k_mod_threshold(const float* __restrict__ y, int64_t N, float eps,
                                                       float* __restrict__ thr) {
  __shared__ double red[256];
  const float* src = y + (int64_t)blockIdx.x * N;
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < N; i += 256) m += (double)src[i] * (double)src[i];
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) thr[blockIdx.x] = (float)((double)eps * sqrt(red[0] / (double)N));
}

void launch_mod_threshold(const float* y, int64_t N, float eps, float* thr, int B, cudaStream_t st) {
  k_mod_threshold<<<B, 256, 0, st>>>(y, N, eps, thr);
  count_launch();
}

// Adjoint of layer 1 in Fourier: g_hat_x[m] = sum_n1 psi1[m] GZ[n1][m mod L1], n1 over the
// precomputed list of filters whose support meets the 256-bin tile (fixed order: deterministic).
__global__ void __launch_bounds__(256) k_adj_gather_x(const float2* __restrict__ GZ, int64_t GZ_sb,
                                                      float2* __restrict__ out, int64_t out_sb,
                                                      const int32_t* __restrict__ tstart,
                                                      const int32_t* __restrict__ list,
                                                      const Support* __restrict__ psi1_sup,
                                                      const int64_t* __restrict__ l1_off,
                                                      const int32_t* __restrict__ n1_k1, int64_t N_pad,
                                                      const float* __restrict__ vals) {
  const int64_t tile = blockIdx.x;
  const int b = blockIdx.y;
  const int64_t m = tile * 256 + threadIdx.x;
  if (m >= N_pad) return;
  float2 acc = make_float2(0.f, 0.f);
  for (int q = tstart[tile]; q < tstart[tile + 1]; ++q) {
    const int n1 = list[q];
    const Support sp = psi1_sup[n1];
    int64_t t = m - sp.lo;
    t %= N_pad; if (t < 0) t += N_pad;
    if (t < sp.len) {
      float h = __ldg(vals + sp.off + t);
      const int64_t L1 = N_pad >> n1_k1[n1];
      float2 v = GZ[b * GZ_sb + l1_off[n1] + (m & (L1 - 1))];
      acc.x = fmaf(h, v.x, acc.x);
      acc.y = fmaf(h, v.y, acc.y);
    }
  }
  out[b * out_sb + m] = acc;
}

void launch_adj_gather_x(const Plan& p, const DeviceTables& d, const float2* GZ, int64_t GZ_sb, float2* out,
                         int64_t out_sb, int B, cudaStream_t st) {
  dim3 g((unsigned)(p.N_pad / 256), (unsigned)B);
  k_adj_gather_x<<<g, 256, 0, st>>>(GZ, GZ_sb, out, out_sb, d.gx_tile_start, d.gx_list, d.psi1_sup, d.l1_off,
                                    d.n1_k1, p.N_pad, d.spec_vals);
  count_launch();
}

// real rows -> complex rows (imaginary 0), for the FFT of a real gradient
__global__ void k_real_to_complex(const float* __restrict__ in, int64_t in_sb, float2* __restrict__ out,
                                  int64_t out_sb, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[blockIdx.y * out_sb + i] = make_float2(in[blockIdx.y * in_sb + i], 0.f);
}

void launch_real_to_complex(const float* in, int64_t in_sb, float2* out, int64_t out_sb, int64_t n, int B,
                            cudaStream_t st) {
  dim3 g((unsigned)((n + 255) / 256), (unsigned)B);
  k_real_to_complex<<<g, 256, 0, st>>>(in, in_sb, out, out_sb, n);
  count_launch();
}

// Adjoint of the reflect padding (R10): g[i] = sum over padded positions p with src(p) = i of Re(gxp[p]).
__global__ void k_reflect_adj(const float2* __restrict__ gxp, int64_t sxp, float* __restrict__ g, int64_t sg,
                              int64_t N, int64_t N_pad, int64_t pad_left) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int b = blockIdx.y;
  const float2* src = gxp + b * sxp;
  const int64_t P2 = 2 * N;
  float acc = 0.f;
  for (int w = 0; w < 2; ++w) {
    int64_t base = (w == 0) ? i : (P2 - 1 - i);
    // p = pad_left + base + P2*k in [0, N_pad)
    int64_t kmin = floor_div(-pad_left - base + P2 - 1, P2);
    int64_t kmax = floor_div(N_pad - 1 - pad_left - base, P2);
    for (int64_t k = kmin; k <= kmax; ++k) acc += src[pad_left + base + P2 * k].x;
  }
  g[b * sg + i] = acc;
}

void launch_reflect_adj(const float2* gxp, int64_t sxp, float* g, int64_t sg, const Plan& p, int B,
                        cudaStream_t st) {
  dim3 gr((unsigned)((p.N + 255) / 256), (unsigned)B);
  k_reflect_adj<<<gr, 256, 0, st>>>(gxp, sxp, g, sg, p.N, p.N_pad, p.pad_left);
  count_launch();
}

// ---- colored-noise initialisation ("a colored Gaussian noise y0 whose power spectral density
// matches S1 x"; reading R25): per-band gains g[n1] = a[n1] / sqrt(pi/4 nu[n1]) where a is the
// per-row RMS (over frames) of the order-1 beta = 0 path of S_target interpolated at rho = n1 / F.
__global__ void __launch_bounds__(256) k_cn_gains(const float* __restrict__ St, int64_t St_sb, float* __restrict__ g,
                                                  int64_t g_sb, const double* __restrict__ nu, int64_t off,
                                                  int rows, int64_t frames, int N1, int F) {
  __shared__ double r[1024];
  __shared__ int any;
  const int b = blockIdx.x;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  for (int rho = threadIdx.x; rho < rows; rho += blockDim.x) {
    const float* s = St + b * St_sb + off + (int64_t)rho * frames;
    double acc = 0.0;
    for (int64_t t = 0; t < frames; ++t) acc += (double)s[t] * (double)s[t];
    r[rho] = sqrt(acc / (double)frames);
    if (r[rho] > 0.0) any = 1;
  }
  __syncthreads();
  for (int n1 = threadIdx.x; n1 < N1; n1 += blockDim.x) {
    const double pos = (double)n1 / (double)F;     // np.interp semantics: clamp beyond the last row
    int i0 = (int)floor(pos);
    double a;
    if (i0 >= rows - 1) a = r[rows - 1];
    else a = r[i0] + (pos - (double)i0) * (r[i0 + 1] - r[i0]);
    g[b * g_sb + n1] = (float)(a / sqrt(0.78539816339744831 * nu[n1]));
  }
  if (threadIdx.x == 0) g[b * g_sb + N1] = any ? 0.f : 1.f;   // 1 = all-zero profile: white fallback
}

void launch_cn_gains(const Plan& p, const DeviceTables& d, const float* St, int64_t St_sb, float* g, int64_t g_sb,
                     int B, cudaStream_t st) {
  const int rows = (int)((p.psi1.size() + p.F - 1) / p.F);
  k_cn_gains<<<B, 256, 0, st>>>(St, St_sb, g, g_sb, d.cn_nu, p.frames, rows, p.frames, (int)p.psi1.size(),
                                (int)p.F);
  count_launch();
}

// X[m] *= G[m], G[m] = sum_n1 g[n1] |psi1_hat(m')|^2 / den[m'], m' = min(m, N_pad - m) (even: y0 real);
// the filters meeting bin m' come from the per-256-bin CSR list of the layer-1 adjoint gather
__global__ void __launch_bounds__(256) k_cn_shape(float2* __restrict__ X, int64_t X_sb, const float* __restrict__ g,
                                                  int64_t g_sb, const int32_t* __restrict__ tstart,
                                                  const int32_t* __restrict__ list, const Support* __restrict__ sup,
                                                  const float* __restrict__ vals, const float* __restrict__ den,
                                                  int64_t N_pad, int64_t tile) {
  const int b = blockIdx.y;
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= N_pad) return;
  const int64_t mm = m <= N_pad / 2 ? m : N_pad - m;
  const int64_t tl = mm / tile;
  float acc = 0.f;
  for (int q = tstart[tl]; q < tstart[tl + 1]; ++q) {
    const int n1 = list[q];
    const Support sp = sup[n1];
    int64_t t = (mm - sp.lo) % N_pad;
    if (t < 0) t += N_pad;
    if (t < sp.len) {
      const float h = __ldg(vals + sp.off + t);
      acc = fmaf(g[b * g_sb + n1] * h, h, acc);
    }
  }
  const float G = acc / den[mm];
  float2* x = X + b * X_sb + m;
  *x = make_float2(x->x * G, x->y * G);
}

void launch_cn_shape(const Plan& p, const DeviceTables& d, float2* X, int64_t X_sb, const float* g, int64_t g_sb,
                     int B, cudaStream_t st) {
  dim3 gr((unsigned)((p.N_pad + 255) / 256), (unsigned)B);
  k_cn_shape<<<gr, 256, 0, st>>>(X, X_sb, g, g_sb, d.gx_tile_start, d.gx_list, d.psi1_sup, d.spec_vals, d.cn_den,
                                 p.N_pad, p.gx_tile);
  count_launch();
}

// y0[i] = Re X[pad_left + i] (the IFFT output), or 1e-4 white[pad_left + i] for an all-zero profile
__global__ void k_cn_crop(const float2* __restrict__ X, int64_t X_sb, const float* __restrict__ white,
                          const float* __restrict__ g, int64_t g_sb, float* __restrict__ y0, int64_t N,
                          int64_t N_pad, int64_t pad_left, int N1) {
  const int b = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const bool fb = g[b * g_sb + N1] != 0.f;
  y0[b * N + i] = fb ? 1e-4f * white[b * N_pad + pad_left + i] : X[b * X_sb + pad_left + i].x;
}

void launch_cn_crop(const Plan& p, const float2* X, int64_t X_sb, const float* white, const float* g, int64_t g_sb,
                    float* y0, int B, cudaStream_t st) {
  dim3 gr((unsigned)((p.N + 255) / 256), (unsigned)B);
  k_cn_crop<<<gr, 256, 0, st>>>(X, X_sb, white, g, g_sb, y0, p.N, p.N_pad, p.pad_left, (int)p.psi1.size());
  count_launch();
}

// non-finite check (JTFS_ERR_NUMERIC): flag = 1 if any x[i] is NaN or +-inf
__global__ void k_check_finite(const float* __restrict__ x, int64_t n, int32_t* __restrict__ flag) {
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

void launch_check_finite(const float* x, int64_t n, int32_t* flag, cudaStream_t st) {
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 8);
  k_check_finite<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, st>>>(x, n, flag);
  count_launch();
}

// ---- metamer update (R23-R24): per-signal bold-driver decision, then momentum step.
__global__ void k_metamer_decide(float* mu, float* loss_prev, const float* loss, int32_t* accepted,
                                 const int32_t* active, int B, float grow, float shrink) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (active && !active[b]) {   // frozen (early stop / rejection cap): state kept
    accepted[b] = 0;
    return;
  }
  float E = loss[b];
  if (E <= loss_prev[b]) {
    accepted[b] = 1;
    loss_prev[b] = E;
    mu[b] = mu[b] * grow;
  } else {
    accepted[b] = 0;
    mu[b] = mu[b] * shrink;
  }
}

__global__ void k_metamer_apply(float* __restrict__ y, float* __restrict__ u, float* __restrict__ y_prev,
                                float* __restrict__ g_prev, const float* __restrict__ mu,
                                const int32_t* __restrict__ accepted, const int32_t* __restrict__ active,
                                const float* __restrict__ g, int64_t sg, int64_t N, float momentum) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int b = blockIdx.y;
  const int64_t o = (int64_t)b * N + i;
  if (active && !active[b]) {   // frozen at the best iterate
    y[o] = y_prev[o];
    u[o] = 0.f;
    return;
  }
  float gg, yy, uu;
  if (accepted[b]) {
    yy = y[o];
    gg = g[(int64_t)b * sg + i];
    y_prev[o] = yy;
    g_prev[o] = gg;
    uu = u[o];
  } else {
    yy = y_prev[o];
    gg = g_prev[o];
    uu = 0.f;
  }
  uu = momentum * uu - mu[b] * gg;
  u[o] = uu;
  y[o] = yy + uu;
}

void launch_metamer(float* y, float* u, float* y_prev, float* g_prev, float* mu, float* loss_prev,
                    const float* loss, int32_t* accepted, const int32_t* active, const float* g, int64_t sg,
                    int64_t N, int B, float momentum, float grow, float shrink, cudaStream_t st) {
  k_metamer_decide<<<(B + 127) / 128, 128, 0, st>>>(mu, loss_prev, loss, accepted, active, B, grow, shrink);
  dim3 gr((unsigned)((N + 255) / 256), (unsigned)B);
  k_metamer_apply<<<gr, 256, 0, st>>>(y, u, y_prev, g_prev, mu, accepted, active, g, sg, N, momentum);
  count_launch(2);
}

}  // namespace jtfs
