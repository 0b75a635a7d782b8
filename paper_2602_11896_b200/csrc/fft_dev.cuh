// fft_dev.cuh — device building blocks of the hand-written FFT (fft.cu) shared with the FFT route of
// the joint lambda_1 stage (kernels_frfft.cu): complex helpers, radix-4/2 Stockham passes in SMEM.
#pragma once
#include <cuda_runtime.h>

#ifndef JTFS_CF_INLINE
#define JTFS_CF_INLINE __noinline__
#endif

namespace jtfs {

constexpr int kTw = 4096;  // twiddle table length

template <class C> struct Cx;
template <> struct Cx<float2> {
  using R = float;
  __device__ static float2 mk(float a, float b) { return make_float2(a, b); }
};
template <> struct Cx<double2> {
  using R = double;
  __device__ static double2 mk(double a, double b) { return make_double2(a, b); }
};

template <class C> __device__ __forceinline__ C t_add(C a, C b) { return Cx<C>::mk(a.x + b.x, a.y + b.y); }
template <class C> __device__ __forceinline__ C t_sub(C a, C b) { return Cx<C>::mk(a.x - b.x, a.y - b.y); }
template <class C> __device__ __forceinline__ C t_mul(C a, C b) {
  return Cx<C>::mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
template <class TO, class C> __device__ __forceinline__ TO t_cvt(C v);
template <> __device__ __forceinline__ float2 t_cvt<float2, float2>(float2 v) { return v; }
template <> __device__ __forceinline__ double2 t_cvt<double2, double2>(double2 v) { return v; }
template <> __device__ __forceinline__ float2 t_cvt<float2, double2>(double2 v) {
  return make_float2((float)v.x, (float)v.y);
}
template <> __device__ __forceinline__ double2 t_cvt<double2, float2>(float2 v) {
  return make_double2(v.x, v.y);
}

template <class C>
__device__ __forceinline__ void dft4(C& a0, C& a1, C& a2, C& a3, bool inv) {
  C t0 = t_add(a0, a2), t1 = t_sub(a0, a2), t2 = t_add(a1, a3), t3 = t_sub(a1, a3);
  a0 = t_add(t0, t2);
  a2 = t_sub(t0, t2);
  C mt3 = inv ? Cx<C>::mk(-t3.y, t3.x) : Cx<C>::mk(t3.y, -t3.x);  // (+/-i) * t3
  a1 = t_add(t1, mt3);
  a3 = t_sub(t1, mt3);
}

template <class C>
__device__ __forceinline__ C twid(const C* __restrict__ tw, int e, bool inv) {
  C w = tw[e];
  return inv ? Cx<C>::mk(w.x, -w.y) : w;
}

// One Stockham pass of radix R over M sequences of length n in SMEM (element i of sequence c at
// s[i*es + c*ss]). `ileave` = sequences interleaved (ss == 1): consecutive threads -> sequences.
template <class C, int R, int THREADS>
__device__ __forceinline__ void stockham_pass(C* s, int n, int M, int es, int ss, bool ileave, int Ns, bool inv,
                                              const C* __restrict__ tw) {
  constexpr int MAXB = (R == 4) ? 4 : 8;
  const int nbr = n / R;
  const int nb = nbr * M;
  C v[MAXB][R];
  int dst[MAXB];
#pragma unroll
  for (int i = 0; i < MAXB; ++i) {
    int q = threadIdx.x + i * THREADS;
    dst[i] = -1;
    if (q < nb) {
      int c, j;
      if (ileave) { c = q % M; j = q / M; } else { c = q / nbr; j = q % nbr; }
      int k = j % Ns;
      int tstep = kTw / (Ns * R);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        C a = s[(j + r * nbr) * es + c * ss];
        if (r > 0 && k > 0) a = t_mul(a, twid(tw, r * k * tstep, inv));
        v[i][r] = a;
      }
      if (R == 4) {
        dft4(v[i][0], v[i][1], v[i][2], v[i][3], inv);
      } else {
        C a = v[i][0], b = v[i][1];
        v[i][0] = t_add(a, b);
        v[i][1] = t_sub(a, b);
      }
      dst[i] = ((j / Ns) * Ns * R + k) * es + c * ss;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < MAXB; ++i) {
    if (dst[i] >= 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) s[dst[i] + r * Ns * es] = v[i][r];
    }
  }
  __syncthreads();
}

template <class C, int THREADS>
__device__ void smem_fft(C* s, int n, int M, int es, int ss, bool ileave, bool inv, const C* __restrict__ tw) {
  int Ns = 1;
  while (Ns * 4 <= n) {
    stockham_pass<C, 4, THREADS>(s, n, M, es, ss, ileave, Ns, inv, tw);
    Ns *= 4;
  }
  if (Ns < n) stockham_pass<C, 2, THREADS>(s, n, M, es, ss, ileave, Ns, inv, tw);
}


// =====================================================================================
// Batched short FFTs of several sequences in SMEM, radix-16 Stockham (two radix-4 levels in registers,
// W16 twiddles as constants) plus one radix-8/4/2 pass; complex type Cp = float2 or double2.
// Sequence layouts:
//   SeqCol<Cp>:   element e of sequence c at s[c * cs + sidx(e)], sidx(e) = e ^ ((e >> 4) & 15): the XOR
//                 swizzle keeps the radix-16 scatter and the gathers conflict-free without padding;
//                 threads walk the elements of one sequence (c slowest).
//   SeqInter<Cp>: element e of sequence c at s[e * nseq + c] (sequences interleaved, c fastest): for
//                 column transforms loaded straight from row-major global memory.
// The first pass reads through a loader ld(c, e) and the last writes through a storer st(c, e, v), so
// producers (cdgmm + fold, twiddles) and consumers (modulus, spectrum accumulation, scaling,
// transposition) fuse into the transform. Capacity: nseq * L <= NPT * NT (NPT points per thread).
// =====================================================================================
__device__ __forceinline__ int sidx(int e) { return e ^ ((e >> 4) & 15); }

template <class Cp>
__device__ __forceinline__ Cp cmul_t(Cp a, Cp b) {
  return Cx<Cp>::mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmul_f(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmul_f(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// X[k] for k = k1 + 4 k2 ends in slot 4 k1 + k2 (read back with dft16_slot)
template <class Cp>
__device__ __forceinline__ void dft16(Cp (&a)[16], bool inv) {
  using R = typename Cx<Cp>::R;
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4(a[n2], a[4 + n2], a[8 + n2], a[12 + n2], inv);
  const R c1 = (R)0.92387953251128675613, s1 = (R)0.38268343236508977173, r2 = (R)0.70710678118654752440;
  const R sg = inv ? (R)1 : (R)-1;
  // slot 4 k1 + n2 *= W16^(n2 k1)
  const Cp w1 = Cx<Cp>::mk(c1, sg * s1), w2 = Cx<Cp>::mk(r2, sg * r2), w3 = Cx<Cp>::mk(s1, sg * c1);
  const Cp w4 = Cx<Cp>::mk(0, sg), w6 = Cx<Cp>::mk(-r2, sg * r2), w9 = Cx<Cp>::mk(-c1, -sg * s1);
  a[5] = cmul_f(a[5], w1);  a[6] = cmul_f(a[6], w2);   a[7] = cmul_f(a[7], w3);
  a[9] = cmul_f(a[9], w2);  a[10] = cmul_f(a[10], w4); a[11] = cmul_f(a[11], w6);
  a[13] = cmul_f(a[13], w3); a[14] = cmul_f(a[14], w6); a[15] = cmul_f(a[15], w9);
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft4(a[4 * k1], a[4 * k1 + 1], a[4 * k1 + 2], a[4 * k1 + 3], inv);
}
__host__ __device__ constexpr int dft16_slot(int r) { return 4 * (r & 3) + (r >> 2); }

template <class Cp>
__device__ __forceinline__ void dft8(Cp (&a)[8], bool inv) {
  using R = typename Cx<Cp>::R;
  // n = 2 n1 + n2 (n1 < 4, n2 < 2), k = k1 + 4 k2: DFT4 over n1, twiddle W8^(n2 k1), DFT2 over n2
  dft4(a[0], a[2], a[4], a[6], inv);
  dft4(a[1], a[3], a[5], a[7], inv);
  const R r2 = (R)0.70710678118654752440, sg = inv ? (R)1 : (R)-1;
  // slot 2 k1 + n2 holds (k1, n2)
  a[3] = cmul_f(a[3], Cx<Cp>::mk(r2, sg * r2));
  a[5] = Cx<Cp>::mk(-sg * a[5].y, sg * a[5].x);                 // * W8^2 = (0, sg)
  a[7] = cmul_f(a[7], Cx<Cp>::mk(-r2, sg * r2));
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    const Cp x = a[2 * k1], y = a[2 * k1 + 1];
    a[2 * k1] = t_add(x, y);
    a[2 * k1 + 1] = t_sub(x, y);
  }
}
__host__ __device__ constexpr int dft8_slot(int r) { return 2 * (r & 3) + (r >> 2); }

template <class Cp>
struct SeqCol {
  Cp* s;
  int cs;
  static constexpr bool kCFast = false;
  __device__ __forceinline__ Cp operator()(int c, int e) const { return s[c * cs + sidx(e)]; }
  __device__ __forceinline__ void operator()(int c, int e, Cp v) const { s[c * cs + sidx(e)] = v; }
};
template <class Cp>
struct SeqInter {
  Cp* s;
  int nseq;
  static constexpr bool kCFast = true;
  __device__ __forceinline__ Cp operator()(int c, int e) const { return s[e * nseq + c]; }
  __device__ __forceinline__ void operator()(int c, int e, Cp v) const { s[e * nseq + c] = v; }
};
using CfSmem = SeqCol<float2>;

// One Stockham pass of radix R (16, 8, 4, 2) over nseq = 2^lgC sequences of length L = 2^lgL (sub-transform
// size Ns = 2^lgNs before the pass). tws = SMEM table W_{2^lgT}^e = exp(-2 pi i e / 2^lgT), e < 2^lgT,
// 2^lgT >= L; lgT = -1: the per-pass table of length L (fft.cuh fft_pass_tables). All loads happen before the barrier and all stores after it (in place when ld and st address
// the same buffer). CFAST: consecutive threads take consecutive sequences.
template <class Cp, int R, int NT, int NPT, bool CFAST, class LD, class ST>
__device__ JTFS_CF_INLINE void cf_pass(int lgC, int lgL, int lgNs, bool inv, const Cp* tws, int lgT, LD ld, ST st) {
  using RT = typename Cx<Cp>::R;
  constexpr int lgR = R == 16 ? 4 : (R == 8 ? 3 : (R == 4 ? 2 : 1));
  constexpr int NB = NPT / R > 0 ? NPT / R : 1;                      // butterflies per thread
  const int lgnbr = lgL - lgR;
  const int nb = 1 << (lgC + lgnbr);
  const int Ns = 1 << lgNs;
  const int tsh = lgT - lgNs - lgR;                                 // 2^lgT / (Ns R) = 2^tsh
  const RT sg = inv ? (RT)-1 : (RT)1;
  Cp v[NB][R];
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const int q = threadIdx.x + i * NT;
    if (q < nb) {
      const int c = CFAST ? (q & ((1 << lgC) - 1)) : (q >> lgnbr);
      const int j = CFAST ? (q >> lgC) : (q & ((1 << lgnbr) - 1));
      const int k = j & (Ns - 1);
#pragma unroll
      for (int r = 0; r < R; ++r) v[i][r] = ld(c, j + (r << lgnbr));
      if (k > 0) {
#pragma unroll
        for (int r = 1; r < R; ++r) {
          Cp w = lgT < 0 ? tws[(Ns - 1) + (r - 1) * Ns + k] : tws[(r * k) << tsh];
          w.y *= sg;
          v[i][r] = cmul_f(v[i][r], w);
        }
      }
      if constexpr (R == 16) {
        dft16(v[i], inv);
      } else if constexpr (R == 8) {
        dft8(v[i], inv);
      } else if constexpr (R == 4) {
        dft4(v[i][0], v[i][1], v[i][2], v[i][3], inv);
      } else {
        const Cp x = v[i][0], y = v[i][1];
        v[i][0] = t_add(x, y);
        v[i][1] = t_sub(x, y);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const int q = threadIdx.x + i * NT;
    if (q < nb) {
      const int c = CFAST ? (q & ((1 << lgC) - 1)) : (q >> lgnbr);
      const int j = CFAST ? (q >> lgC) : (q & ((1 << lgnbr) - 1));
      const int base = ((j >> lgNs) << (lgNs + lgR)) + (j & (Ns - 1));
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int slot = R == 16 ? dft16_slot(r) : (R == 8 ? dft8_slot(r) : r);
        st(c, base + (r << lgNs), v[i][slot]);
      }
    }
  }
  __syncthreads();
}

// Batched FFT (forward e^-, or unscaled inverse e^+) of 2^lgC sequences of length 2^lgL: the first pass
// reads through ld, the last writes through st, intermediate passes run in place in `buf`.
template <class Cp, int NT, int NPT, class LD, class ST, class BUF>
__device__ __forceinline__ void seq_fft(int lgC, int lgL, bool inv, const Cp* tws, int lgT, LD ld, ST st, BUF buf) {
  constexpr bool CF = BUF::kCFast;
  const int n16 = lgL / 4, rem = lgL - 4 * n16;
  const int npass = n16 + (rem ? 1 : 0);
  int lgNs = 0;
  for (int p = 0; p < n16; ++p, lgNs += 4) {
    const bool first = p == 0, last = p == npass - 1;
    if (first && last) cf_pass<Cp, 16, NT, NPT, CF>(lgC, lgL, lgNs, inv, tws, lgT, ld, st);
    else if (first) cf_pass<Cp, 16, NT, NPT, CF>(lgC, lgL, lgNs, inv, tws, lgT, ld, buf);
    else if (last) cf_pass<Cp, 16, NT, NPT, CF>(lgC, lgL, lgNs, inv, tws, lgT, buf, st);
    else cf_pass<Cp, 16, NT, NPT, CF>(lgC, lgL, lgNs, inv, tws, lgT, buf, buf);
  }
  if (rem) {
    const bool first = n16 == 0;
    if (rem == 3) {
      if (first) cf_pass<Cp, 8, NT, NPT, CF>(lgC, lgL, lgNs, inv, tws, lgT, ld, st);
      else cf_pass<Cp, 8, NT, NPT, CF>(lgC, lgL, lgNs, inv, tws, lgT, buf, st);
    } else if (rem == 2) {
      if (first) cf_pass<Cp, 4, NT, NPT, CF>(lgC, lgL, lgNs, inv, tws, lgT, ld, st);
      else cf_pass<Cp, 4, NT, NPT, CF>(lgC, lgL, lgNs, inv, tws, lgT, buf, st);
    } else {
      if (first) cf_pass<Cp, 2, NT, NPT, CF>(lgC, lgL, lgNs, inv, tws, lgT, ld, st);
      else cf_pass<Cp, 2, NT, NPT, CF>(lgC, lgL, lgNs, inv, tws, lgT, buf, st);
    }
  }
}

// float2 column FFTs of the FFT route (kernels_frfft.cu): C columns (C a power of two), NT threads, 16
// points per thread
template <int NT, class LD, class ST>
__device__ __forceinline__ void col_fft(int C, int lgL, bool inv, const float2* tws, int lgT, LD ld, ST st,
                                        CfSmem buf) {
  const int lgC = C == 1 ? 0 : (C == 2 ? 1 : (C == 4 ? 2 : 3));
  seq_fft<float2, NT, 16>(lgC, lgL, inv, tws, lgT, ld, st, buf);
}

}  // namespace jtfs
