// fft.cu — batched power-of-two complex FFTs for sm_100a, hand written (no cuFFT).
//
// Radix-16 Stockham passes in SMEM (fft_dev.cuh: two radix-4 levels in registers, one radix-8/4/2
// pass for the remainder) with the loads of the first pass and the stores of the last pass going
// straight to global memory. Lengths <= 4096 run in one kernel (k_fft_small, 4096 / L rows per CTA);
// longer lengths L = L1 * 4096 use the four-step scheme:
//   A) L1-point column transforms in place, times the twiddle W_L^{n2 k1} (k_fft_colA; sequences
//      interleaved in SMEM so the strided columns load and store coalesced)
//   B) 4096-point row transforms written transposed to the output (k_fft_rowB)
// Used for rfft/ifft/cfft of the listings P:203, P:209, P:211, P:235, P:282, P:285 and their
// adjoints. Forward = exp(-2 pi i k n / L); inverse = exp(+...) / L (numpy convention).
// Templated on the compute type (float2 or double2) and on the input/output element types: the
// first layer (signal -> X_hat -> Z1) runs in float64 so that the phase Z1/|Z1| used by the
// modulus adjoint stays accurate in near-silent bands ("precision").
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "fft.cuh"
#include "fft_dev.cuh"
#include "plan.h"

namespace jtfs {

template <class C> struct FftTw;
template <> struct FftTw<float2> {
  static const float2* base(const FftTables& t) { return t.twp; }
  static const float2* tw2(const FftTables& t, int lg) { return t.tw2_f[lg]; }
};
template <> struct FftTw<double2> {
  static const double2* base(const FftTables& t) { return t.twpd; }
  static const double2* tw2(const FftTables& t, int lg) { return t.tw2_d[lg]; }
};

// SMEM copy of the per-pass twiddle table of length L = 2^lgL (fft_pass_tables; cf_pass with lgT = -1)
template <class C, int NT>
__device__ __forceinline__ void load_twiddles(C* tws, const C* __restrict__ tw, int lgL) {
  for (int e = threadIdx.x; e < (1 << lgL); e += NT) tws[e] = tw[(1 << lgL) + e];
}

// ---------------------------------------------------------------- L <= 4096: 4096 / L rows per CTA
template <class TI, class C>
struct LdRows {  // first pass reads global rows (converted to the compute type), zero past the last row
  const TI* src;
  int lgL, rows;
  __device__ __forceinline__ C operator()(int c, int e) const {
    return c < rows ? t_cvt<C>(src[((int64_t)c << lgL) + e]) : Cx<C>::mk(0, 0);
  }
};
template <class TO, class C>
struct StRows {  // last pass writes global rows, scaled
  TO* dst;
  int lgL, rows;
  typename Cx<C>::R sc;
  __device__ __forceinline__ void operator()(int c, int e, C v) const {
    if (c < rows) dst[((int64_t)c << lgL) + e] = t_cvt<TO>(Cx<C>::mk(v.x * sc, v.y * sc));
  }
};

template <class TI, class TO, class C>
__global__ void __launch_bounds__(256, sizeof(C) == 8 ? 2 : 1) k_fft_small(const TI* __restrict__ in, TO* __restrict__ out, Rows ri, Rows ro,
                                                   int lgL, int lgM, int inv, double scale,
                                                   const C* __restrict__ tw) {
  extern __shared__ __align__(16) uint8_t smraw[];
  C* s = reinterpret_cast<C*>(smraw);          // [M][L] (swizzled sequences)
  C* tws = s + (1 << (lgL + lgM));             // [L]
  const int b = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x << lgM;
  const int rows = (int)((ri.count - r0) < (1 << lgM) ? (ri.count - r0) : (1 << lgM));
  load_twiddles<C, 256>(tws, tw, lgL);
  __syncthreads();
  const LdRows<TI, C> ld{in + b * ri.stride_b + ri.off + (r0 << lgL), lgL, rows};
  const StRows<TO, C> st{out + b * ro.stride_b + ro.off + (r0 << lgL), lgL, rows, (typename Cx<C>::R)scale};
  const SeqCol<C> buf{s, 1 << lgL};
  seq_fft<C, 256, 16>(lgM, lgL, inv != 0, tws, -1, ld, st, buf);
}

// Several row groups of (possibly different) lengths <= 4096 in one launch: CTA x belongs to the group
// whose CTA range holds it (the job list travels in the kernel parameters).
struct FftJob {
  int64_t off, count;   // first row element (same offset in and out), rows
  int lgL, cta0;        // log2 length, first CTA
};
constexpr int kMaxFftJobs = 24;
struct FftJobs {
  FftJob j[kMaxFftJobs];
  int n;
};
template <class TI, class TO, class C>
__global__ void __launch_bounds__(256, sizeof(C) == 8 ? 2 : 1) k_fft_small_multi(const TI* __restrict__ in, TO* __restrict__ out,
                                                         int64_t in_sb, int64_t out_sb, FftJobs J, int inv,
                                                         const C* __restrict__ tw) {
  extern __shared__ __align__(16) uint8_t smraw[];
  int jx = 0;
  while (jx + 1 < J.n && (int)blockIdx.x >= J.j[jx + 1].cta0) ++jx;
  const int64_t off = J.j[jx].off, count = J.j[jx].count;
  const int lgL = J.j[jx].lgL, lgM = 12 - lgL;
  C* s = reinterpret_cast<C*>(smraw);          // [M][L] (swizzled sequences), M L = 4096
  C* tws = s + 4096;                           // [L]
  const int b = blockIdx.y;
  const int64_t r0 = (int64_t)((int)blockIdx.x - J.j[jx].cta0) << lgM;
  const int rows = (int)((count - r0) < (1 << lgM) ? (count - r0) : (1 << lgM));
  load_twiddles<C, 256>(tws, tw, lgL);
  __syncthreads();
  const typename Cx<C>::R sc = inv ? (typename Cx<C>::R)1 / (typename Cx<C>::R)(1 << lgL) : (typename Cx<C>::R)1;
  const LdRows<TI, C> ld{in + b * in_sb + off + (r0 << lgL), lgL, rows};
  const StRows<TO, C> st{out + b * out_sb + off + (r0 << lgL), lgL, rows, sc};
  const SeqCol<C> buf{s, 1 << lgL};
  seq_fft<C, 256, 16>(lgM, lgL, inv != 0, tws, -1, ld, st, buf);
}

// ---------------------------------------------------------------- four-step A: columns
// x viewed as [L1][L2] (n = n1 L2 + n2). For the CTA's CW columns n2: y[k1][n2] = sum_n1 x[n1][n2]
// W_L1^{n1 k1}, times W_L^{n2 k1}, written back in place. W_L^{n2 k1} = tw2[k1 4096 + n2] (fft_fourstep_table:
// consecutive columns read consecutive words).
template <class C>
struct LdCols {
  const C* base;   // row n1 at base + n1 * L2
  int L2;
  __device__ __forceinline__ C operator()(int c, int n1) const { return base[(int64_t)n1 * L2 + c]; }
};
template <class C>
struct StColsTw {
  C* base;
  int L2, c0, inv;
  const C* tw2;
  __device__ __forceinline__ void operator()(int c, int k1, C v) const {
    C w = tw2[((int64_t)k1 << 12) + c0 + c];
    if (inv) w.y = -w.y;
    base[(int64_t)k1 * L2 + c] = cmul_f(v, w);
  }
};

template <class C>
__global__ void __launch_bounds__(256, sizeof(C) == 8 ? 3 : 2) k_fft_colA(C* __restrict__ data, Rows ri, int lgL1, int L2, int lgCW, int inv,
                                                  const C* __restrict__ tw, const C* __restrict__ tw2) {
  extern __shared__ __align__(16) uint8_t smraw[];
  C* s = reinterpret_cast<C*>(smraw);                  // [L1][CW] interleaved
  C* tws = s + (1 << (lgL1 + lgCW));                   // [L1]
  const int64_t r = blockIdx.y;
  const int b = blockIdx.z;
  const int64_t L = (int64_t)L2 << lgL1;
  const int c0 = blockIdx.x << lgCW;
  C* base = data + b * ri.stride_b + ri.off + r * L + c0;
  load_twiddles<C, 256>(tws, tw, lgL1);
  __syncthreads();
  const LdCols<C> ld{base, L2};
  const StColsTw<C> st{base, L2, c0, inv, tw2};
  const SeqInter<C> buf{s, 1 << lgCW};
  seq_fft<C, 256, 16>(lgCW, lgL1, inv != 0, tws, -1, ld, st, buf);
}

// ---------------------------------------------------------------- four-step B: rows, transposed out
// For rows k1 in [k1_0, k1_0 + M): X[k1 + L1 k2] = sum_n2 y[k1][n2] W_L2^{n2 k2}.
template <class C, class TO, int NPT, int NT>
__global__ void __launch_bounds__(NT) k_fft_rowB(const C* __restrict__ in, TO* __restrict__ out, Rows ri, Rows ro,
                                                  int L1, int lgM, int inv, double scale, const C* __restrict__ tw) {
  extern __shared__ __align__(16) uint8_t smraw[];
  constexpr int lgL2 = 12, L2 = 4096;
  C* s = reinterpret_cast<C*>(smraw);                 // [M][L2] swizzled
  C* tws = s + (L2 << lgM);                           // [L2]
  const int64_t r = blockIdx.y;
  const int b = blockIdx.z;
  const int64_t L = (int64_t)L1 * L2;
  const int M = 1 << lgM;
  const int k10 = blockIdx.x * M;
  const C* src = in + b * ri.stride_b + ri.off + r * L + (int64_t)k10 * L2;
  TO* dst = out + b * ro.stride_b + ro.off + r * L;
  load_twiddles<C, NT>(tws, tw, lgL2);
  __syncthreads();
  const LdRows<C, C> ld{src, lgL2, M};
  const SeqCol<C> buf{s, L2};
  seq_fft<C, NT, NPT>(lgM, lgL2, inv != 0, tws, -1, ld, buf, buf);
  const typename Cx<C>::R sc = (typename Cx<C>::R)scale;
  for (int i = threadIdx.x; i < (L2 << lgM); i += NT) {
    const int m = i & (M - 1), k2 = i >> lgM;
    const C v = buf(m, k2);
    dst[(int64_t)k2 * L1 + k10 + m] = t_cvt<TO>(Cx<C>::mk(v.x * sc, v.y * sc));
  }
}

// ---------------------------------------------------------------- "T-layout" passes (no transposition)
template <class C, class TO>
struct StRowT {  // row m of the CTA at dst + m * 4096, element n2; T -> natural twiddle W_L^{(k10 + m) n2} if tw2
  TO* dst;
  int k10, inv;
  typename Cx<C>::R sc;
  const C* tw2;
  __device__ __forceinline__ void operator()(int m, int n2, C v) const {
    if (tw2) {
      C w = tw2[((int64_t)(k10 + m) << 12) + n2];
      if (inv) w.y = -w.y;
      v = cmul_f(v, w);
    }
    dst[((int64_t)m << 12) + n2] = t_cvt<TO>(Cx<C>::mk(v.x * sc, v.y * sc));
  }
};
// A four-step transform whose rows are stored in place keeps every global access row-contiguous: the
// natural -> T pair (k_fft_colA, then k_fft_rowT without twiddle) leaves X[k1 + L1 k2] at position
// k1 L2 + k2, and the T -> natural pair (k_fft_rowT with the twiddle W_L^{k1 n2} on its store, then
// k_fft_colT) takes a row-major T-layout input back to natural order. Chains whose consumers are
// elementwise (Z1 -> |Z1| -> U1 FFT; g_U1 -> phase -> g_Z1 FFT) run in T-layout in between.
// Occupancy (row passes are HBM bound; a CTA's load, compute and store phases only overlap with other
// CTAs'): one row x 256 threads per CTA with the twiddle table read through L1 (TWG): float32 32 KB,
// 4 CTAs per SM at 64 registers; float64 64 KB, 2 CTAs per SM at 128 registers (measured on the B200 against
// 4 rows x 1024 threads and 2 rows x 512 threads with SMEM twiddles: c4 652.7 -> 638 ms/step).
template <class C, class TO, int NPT, int NT, bool TWG, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_fft_rowT(const C* __restrict__ in, TO* __restrict__ out, Rows ri, Rows ro,
                                                  int lgL1, int lgM, int inv, double scale, const C* __restrict__ tw,
                                                  const C* __restrict__ tw2) {
  extern __shared__ __align__(16) uint8_t smraw[];
  constexpr int lgL2 = 12, L2 = 4096;
  C* s = reinterpret_cast<C*>(smraw);                 // [M][L2] swizzled
  const int64_t r = blockIdx.y;
  const int b = blockIdx.z;
  const int64_t L = (int64_t)L2 << lgL1;
  const int M = 1 << lgM;
  const int k10 = blockIdx.x * M;
  const C* src = in + b * ri.stride_b + ri.off + r * L + (int64_t)k10 * L2;
  TO* dst = out + b * ro.stride_b + ro.off + r * L + (int64_t)k10 * L2;
  const C* tws = tw + L2;                             // per-pass table of length 4096 (global, via L1)
  if constexpr (!TWG) {
    C* t = s + (L2 << lgM);                           // [L2]
    load_twiddles<C, NT>(t, tw, lgL2);
    __syncthreads();
    tws = t;
  }
  const LdRows<C, C> ld{src, lgL2, M};
  const SeqCol<C> buf{s, L2};
  // the last radix-16 pass stores straight to global memory (consecutive threads hold consecutive n2 of a
  // row: coalesced), with the T -> natural twiddle and the scale applied on the way; in place is safe (every
  // load of the CTA's rows happens in the first pass)
  const StRowT<C, TO> st{dst, k10, inv, (typename Cx<C>::R)scale, tw2};
  seq_fft<C, NT, NPT>(lgM, lgL2, inv != 0, tws, -1, ld, st, buf);
}

template <class C, class TO>
struct StCols {
  TO* base;
  int L2;
  typename Cx<C>::R sc;
  __device__ __forceinline__ void operator()(int c, int n1, C v) const {
    base[(int64_t)n1 * L2 + c] = t_cvt<TO>(Cx<C>::mk(v.x * sc, v.y * sc));
  }
};

// column pass of the T -> natural pair: L1-point transforms of columns, no twiddle, out of place
template <class C, class TO>
__global__ void __launch_bounds__(256, sizeof(C) == 8 ? 3 : 2) k_fft_colT(const C* __restrict__ in, TO* __restrict__ out,
                                                                         Rows ri, Rows ro, int lgL1, int L2, int lgCW,
                                                                         int inv, double scale,
                                                                         const C* __restrict__ tw) {
  extern __shared__ __align__(16) uint8_t smraw[];
  C* s = reinterpret_cast<C*>(smraw);                  // [L1][CW] interleaved
  C* tws = s + (1 << (lgL1 + lgCW));                   // [L1]
  const int64_t r = blockIdx.y;
  const int b = blockIdx.z;
  const int64_t L = (int64_t)L2 << lgL1;
  const int c0 = blockIdx.x << lgCW;
  load_twiddles<C, 256>(tws, tw, lgL1);
  __syncthreads();
  const LdCols<C> ld{in + b * ri.stride_b + ri.off + r * L + c0, L2};
  const StCols<C, TO> st{out + b * ro.stride_b + ro.off + r * L + c0, L2, (typename Cx<C>::R)scale};
  const SeqInter<C> buf{s, 1 << lgCW};
  seq_fft<C, 256, 16>(lgCW, lgL1, inv != 0, tws, -1, ld, st, buf);
}

// ---------------------------------------------------------------- host side
template <class T>
static std::vector<T> twiddles() {
  std::vector<T> t(kTw);
  for (int e = 0; e < kTw; ++e) {
    double a = -2.0 * 3.14159265358979323846 * (double)e / (double)kTw;
    t[e].x = (decltype(t[e].x))std::cos(a);
    t[e].y = (decltype(t[e].y))std::sin(a);
  }
  return t;
}
std::vector<float2> fft_twiddle_table() { return twiddles<float2>(); }

template <class T>
static std::vector<T> pass_tables() {
  std::vector<T> t(2 * kTw);
  for (int lg = 1; lg <= 12; ++lg) {
    T* tab = t.data() + (1 << lg);
    const int n16 = lg / 4, rem = lg - 4 * n16;
    int Ns = 1;
    for (int p = 0; p < n16 + (rem ? 1 : 0); ++p) {
      const int R = p < n16 ? 16 : (1 << rem);
      for (int r = 1; r < R; ++r)
        for (int k = 0; k < Ns; ++k) {
          const double a = -2.0 * 3.14159265358979323846 * (double)(r * k) / (double)(Ns * R);
          tab[(Ns - 1) + (r - 1) * Ns + k].x = (decltype(tab[0].x))std::cos(a);
          tab[(Ns - 1) + (r - 1) * Ns + k].y = (decltype(tab[0].x))std::sin(a);
        }
      Ns *= R;
    }
  }
  return t;
}
std::vector<float2> fft_pass_tables() { return pass_tables<float2>(); }
std::vector<double2> fft_pass_tables_d() { return pass_tables<double2>(); }
std::vector<double2> fft_twiddle_table_d() { return twiddles<double2>(); }

// four-step twiddles for L = 2^lgL > 4096: tw2[k1 4096 + n2] = W_L^{k1 n2}, k1 < L / 4096, n2 < 4096 (float64
// evaluation of the reduced exponent; one table of L entries per length)
template <class T>
static void fourstep_table(int lgL, std::vector<T>* t) {
  const int64_t L = int64_t(1) << lgL, L1 = L >> 12;
  t->resize((size_t)L);
  for (int64_t k1 = 0; k1 < L1; ++k1)
    for (int64_t n2 = 0; n2 < 4096; ++n2) {
      const double a = -2.0 * 3.14159265358979323846 * (double)((k1 * n2) & (L - 1)) / (double)L;
      (*t)[(size_t)((k1 << 12) + n2)].x = (decltype((*t)[0].x))std::cos(a);
      (*t)[(size_t)((k1 << 12) + n2)].y = (decltype((*t)[0].x))std::sin(a);
    }
}
void fft_fourstep_table_f(int lgL, std::vector<float2>* t) { fourstep_table(lgL, t); }
void fft_fourstep_table_d(int lgL, std::vector<double2>* t) { fourstep_table(lgL, t); }

static int ilog2_exact(int64_t v) {
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return l;
}

template <class TI, class TO, class C>
static cudaError_t fft_launch_t(const TI* in, TO* out, Rows ri, Rows ro, int B, bool inverse, const FftTables& T,
                                cudaStream_t st, int layout = kLayoutNatural) {
  // row passes: float32 4 rows per CTA, 1024 threads x 16 points (transposed stores in full 32-byte
  // sectors); float64 2 rows, 512 threads (SMEM); 256 threads x 32 points measured slower
  constexpr int kRowLgM = sizeof(C) == 8 ? 2 : 1;
  constexpr int kRowNT = sizeof(C) == 8 ? 1024 : 512;
  constexpr int kRowNPT = (4096 << kRowLgM) / kRowNT;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fft_rowB<C, TO, kRowNPT, kRowNT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(((4096 << kRowLgM) + 4096) * sizeof(C)));
    cudaFuncSetAttribute(k_fft_colA<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(8192 * sizeof(C)));
    cudaFuncSetAttribute(k_fft_small<TI, TO, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(8192 * sizeof(C)));
    attr = true;
  }
  const int64_t L = ri.L;
  const int lgL = ilog2_exact(L);
  const double scale = inverse ? 1.0 / (double)L : 1.0;
  if (ri.count <= 0 || B <= 0) return cudaSuccess;
  const C* tw = FftTw<C>::base(T);
  if (L <= 4096) {
    const int lgM = 12 - lgL;
    dim3 grid((unsigned)((ri.count + (1 << lgM) - 1) >> lgM), (unsigned)B);
    k_fft_small<TI, TO, C><<<grid, 256, (size_t)(4096 + L) * sizeof(C), st>>>(in, out, ri, ro, lgL, lgM,
                                                                           inverse ? 1 : 0, scale, tw);
    count_launch();
    return cudaGetLastError();
  }
  // four-step; step A runs in place on `in` (it is clobbered; requires TI == C), step B writes `out`
  static_assert(sizeof(TI) == sizeof(C), "four-step input must already be in the compute type");
  const int L2 = 4096, lgL1 = lgL - 12, L1 = 1 << lgL1;
  const int lgCW = std::min(12, 12 - lgL1);                   // CW * L1 = 4096 points per CTA
  if (layout != kLayoutNatural) {
    static bool attrT = false;
    if (!attrT) {
      cudaFuncSetAttribute(k_fft_rowT<C, TO, 16, 256, true, (sizeof(C) == 8 ? 4 : 2)>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(4096 * sizeof(C)));
      cudaFuncSetAttribute(k_fft_rowT<C, C, 16, 256, true, (sizeof(C) == 8 ? 4 : 2)>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(4096 * sizeof(C)));
      cudaFuncSetAttribute(k_fft_colT<C, TO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(8192 * sizeof(C)));
      attrT = true;
    }
    constexpr int kTLgM = 0, kTNT = 256, kTMinB = sizeof(C) == 8 ? 4 : 2;
    constexpr bool kTwg = true;
    const int lgM = std::min(kTLgM, lgL1);
    const size_t smT = (size_t)((4096 << lgM) + (kTwg ? 0 : 4096)) * sizeof(C);
    C* io = reinterpret_cast<C*>(const_cast<TI*>(in));
    if (layout == kLayoutToT) {   // natural -> T: columns (twiddled, in place), then rows stored in place
      dim3 ga((unsigned)(L2 >> lgCW), (unsigned)ri.count, (unsigned)B);
      k_fft_colA<C><<<ga, 256, (size_t)(4096 + L1) * sizeof(C), st>>>(io, ri, lgL1, L2, lgCW, inverse ? 1 : 0, tw,
                                                                      FftTw<C>::tw2(T, lgL));
      dim3 gb((unsigned)(L1 >> lgM), (unsigned)ri.count, (unsigned)B);
      k_fft_rowT<C, TO, 16, kTNT, kTwg, kTMinB><<<gb, kTNT, smT, st>>>(io, out, ri, ro, lgL1, lgM, inverse ? 1 : 0, scale,
                                                                 tw, nullptr);
    } else {                      // T -> natural: rows (twiddled on store, in place), then columns out of place
      dim3 gb((unsigned)(L1 >> lgM), (unsigned)ri.count, (unsigned)B);
      k_fft_rowT<C, C, 16, kTNT, kTwg, kTMinB><<<gb, kTNT, smT, st>>>(io, io, ri, ri, lgL1, lgM, inverse ? 1 : 0, 1.0, tw,
                                                               FftTw<C>::tw2(T, lgL));
      dim3 ga((unsigned)(L2 >> lgCW), (unsigned)ri.count, (unsigned)B);
      k_fft_colT<C, TO><<<ga, 256, (size_t)(4096 + L1) * sizeof(C), st>>>(io, out, ri, ro, lgL1, L2, lgCW,
                                                                          inverse ? 1 : 0, scale, tw);
    }
    count_launch(2);
    return cudaGetLastError();
  }
  {
    dim3 grid((unsigned)(L2 >> lgCW), (unsigned)ri.count, (unsigned)B);
    k_fft_colA<C><<<grid, 256, (size_t)(4096 + L1) * sizeof(C), st>>>(
        reinterpret_cast<C*>(const_cast<TI*>(in)), ri, lgL1, L2, lgCW, inverse ? 1 : 0, tw, FftTw<C>::tw2(T, lgL));
  }
  {
    const int lgM = std::min(kRowLgM, lgL1);
    dim3 grid((unsigned)(L1 >> lgM), (unsigned)ri.count, (unsigned)B);
    k_fft_rowB<C, TO, kRowNPT, kRowNT><<<grid, kRowNT, (size_t)((4096 << lgM) + 4096) * sizeof(C), st>>>(
        reinterpret_cast<const C*>(in), out, ri, ro, L1, lgM, inverse ? 1 : 0, scale, tw);
  }
  count_launch(2);
  return cudaGetLastError();
}

// Row groups sharing the batch strides: groups of length <= 4096 go into grouped launches (up to
// kMaxFftJobs per launch), longer ones through fft_launch_t (four-step).
template <class TI, class TO, class C>
static cudaError_t fft_groups_t(const TI* in, TO* out, int64_t in_sb, int64_t out_sb, const FftGroup* g, int ng,
                                int B, bool inverse, const FftTables& T, cudaStream_t st, int layout = kLayoutNatural) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fft_small_multi<TI, TO, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(8192 * sizeof(C)));
    attr = true;
  }
  FftJobs J{};
  int ctas = 0;
  auto flush = [&]() -> cudaError_t {
    if (J.n == 0) return cudaSuccess;
    int maxL = 0;
    for (int i = 0; i < J.n; ++i) maxL = std::max(maxL, 1 << J.j[i].lgL);
    k_fft_small_multi<TI, TO, C><<<dim3((unsigned)ctas, (unsigned)B), 256, (size_t)(4096 + maxL) * sizeof(C), st>>>(
        in, out, in_sb, out_sb, J, inverse ? 1 : 0, FftTw<C>::base(T));
    count_launch();
    J.n = 0;
    ctas = 0;
    return cudaGetLastError();
  };
  cudaError_t e;
  for (int i = 0; i < ng; ++i) {
    if (g[i].count <= 0 || B <= 0) continue;
    if (g[i].L > 4096) {
      Rows ri{in_sb, g[i].off, g[i].count, g[i].L}, ro{out_sb, g[i].off, g[i].count, g[i].L};
      if ((e = fft_launch_t<TI, TO, C>(in, out, ri, ro, B, inverse, T, st, layout))) return e;
      continue;
    }
    const int lgL = ilog2_exact(g[i].L), lgM = 12 - lgL;
    const int n = (int)((g[i].count + (1 << lgM) - 1) >> lgM);
    if (J.n == kMaxFftJobs && (e = flush())) return e;
    J.j[J.n++] = FftJob{g[i].off, g[i].count, lgL, ctas};
    ctas += n;
  }
  return flush();
}
cudaError_t fft_groups(const float2* in, float2* out, int64_t in_sb, int64_t out_sb, const FftGroup* g, int ng,
                       int B, bool inverse, const FftTables& T, cudaStream_t st, int layout) {
  return fft_groups_t<float2, float2, float2>(in, out, in_sb, out_sb, g, ng, B, inverse, T, st, layout);
}
cudaError_t fft_groups_df(const double2* in, float2* out, int64_t in_sb, int64_t out_sb, const FftGroup* g, int ng,
                          int B, bool inverse, const FftTables& T, cudaStream_t st, int layout) {
  return fft_groups_t<double2, float2, double2>(in, out, in_sb, out_sb, g, ng, B, inverse, T, st, layout);
}
cudaError_t fft_groups_dd(const double2* in, double2* out, int64_t in_sb, int64_t out_sb, const FftGroup* g, int ng,
                          int B, bool inverse, const FftTables& T, cudaStream_t st, int layout) {
  return fft_groups_t<double2, double2, double2>(in, out, in_sb, out_sb, g, ng, B, inverse, T, st, layout);
}

cudaError_t fft_launch(const float2* in, float2* out, Rows ri, Rows ro, int B, bool inverse, const FftTables& T,
                       cudaStream_t st) {
  return fft_launch_t<float2, float2, float2>(in, out, ri, ro, B, inverse, T, st);
}
cudaError_t fft_launch_dd(const double2* in, double2* out, Rows ri, Rows ro, int B, bool inverse,
                          const FftTables& T, cudaStream_t st) {
  return fft_launch_t<double2, double2, double2>(in, out, ri, ro, B, inverse, T, st);
}
cudaError_t fft_launch_df(const double2* in, float2* out, Rows ri, Rows ro, int B, bool inverse,
                          const FftTables& T, cudaStream_t st) {
  return fft_launch_t<double2, float2, double2>(in, out, ri, ro, B, inverse, T, st);
}

}  // namespace jtfs
