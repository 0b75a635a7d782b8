// fft.cu — batched power-of-two complex FFTs for sm_100a, hand written (no cuFFT).
//
// Shared-memory Stockham autosort with radix-4 passes (+ one radix-2 pass for odd log2 n); each
// butterfly is staged in registers so the pass runs in place in SMEM. Lengths <= 4096 run in one
// kernel (several short rows per CTA); longer lengths L = L1 * 4096 use the four-step scheme:
//   A) L1-point column transforms in place + twiddle W_L^{n2 k1}   (k_fft_colA)
//   B) 4096-point row transforms written transposed to the output  (k_fft_rowB)
// Used for rfft/ifft/cfft of the listings P:203, P:209, P:211, P:235, P:282, P:285 and their
// adjoints. Forward = exp(-2 pi i k n / L); inverse = exp(+...) / L (numpy convention).
// Templated on the compute type (float2 or double2) and on the input/output element types: the
// first layer (signal -> X_hat -> Z1) runs in float64 so that the phase Z1/|Z1| used by the
// modulus adjoint stays accurate in near-silent bands ("precision").
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "fft.cuh"
#include "fft_dev.cuh"

namespace jtfs {

// ---------------------------------------------------------------- n <= 4096, M rows per CTA
template <class TI, class TO, class C>
__global__ void __launch_bounds__(256) k_fft_small(const TI* __restrict__ in, TO* __restrict__ out, Rows ri, Rows ro,
                                                   int n, int M, int inv, double scale, const C* __restrict__ tw) {
  extern __shared__ __align__(16) uint8_t smraw[];
  C* s = reinterpret_cast<C*>(smraw);
  const int b = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * M;
  const int rows = (int)((ri.count - r0) < M ? (ri.count - r0) : M);
  const TI* src = in + b * ri.stride_b + ri.off + r0 * n;
  TO* dstp = out + b * ro.stride_b + ro.off + r0 * n;
  const int tot = rows * n;
  for (int i = threadIdx.x; i < M * n; i += 256) s[i] = (i < tot) ? t_cvt<C>(src[i]) : Cx<C>::mk(0, 0);
  __syncthreads();
  smem_fft<C, 256>(s, n, M, 1, n, false, inv != 0, tw);
  const typename Cx<C>::R sc = (typename Cx<C>::R)scale;
  for (int i = threadIdx.x; i < tot; i += 256) dstp[i] = t_cvt<TO>(Cx<C>::mk(s[i].x * sc, s[i].y * sc));
}

// ---------------------------------------------------------------- four-step A: columns
// x viewed as [L1][L2] (n = n1*L2 + n2). For the CTA's CW columns n2: y[k1][n2] =
// sum_n1 x[n1][n2] W_L1^{n1 k1}, times W_L^{n2 k1}; written back in place.
__device__ __forceinline__ void sincospi_t(float a, float* s, float* c) { sincospif(a, s, c); }
__device__ __forceinline__ void sincospi_t(double a, double* s, double* c) { sincospi(a, s, c); }

template <class C>
__global__ void __launch_bounds__(512) k_fft_colA(C* __restrict__ data, Rows ri, int L1, int L2, int CW, int inv,
                                                  const C* __restrict__ tw) {
  extern __shared__ __align__(16) uint8_t smraw[];
  C* s = reinterpret_cast<C*>(smraw);
  using R = typename Cx<C>::R;
  const int64_t r = blockIdx.y;
  const int b = blockIdx.z;
  const int64_t L = (int64_t)L1 * L2;
  C* base = data + b * ri.stride_b + ri.off + r * L;
  const int c0 = blockIdx.x * CW;
  for (int i = threadIdx.x; i < L1 * CW; i += 512) {
    int n1 = i / CW, c = i % CW;
    s[i] = base[(int64_t)n1 * L2 + c0 + c];
  }
  __syncthreads();
  smem_fft<C, 512>(s, L1, CW, CW, 1, true, inv != 0, tw);
  const R sgn = inv ? (R)2 : (R)-2;
  for (int i = threadIdx.x; i < L1 * CW; i += 512) {
    int k1 = i / CW, c = i % CW;
    int64_t e = ((int64_t)(c0 + c) * k1) % L;  // exact; 2e/L exact in fp32 (L <= 2^22)
    R sn, cs;
    sincospi_t(sgn * (R)e / (R)L, &sn, &cs);
    base[(int64_t)k1 * L2 + c0 + c] = t_mul(s[i], Cx<C>::mk(cs, sn));
  }
}

// ---------------------------------------------------------------- four-step B: rows, transposed out
// For rows k1 in [k1_0, k1_0 + M): X[k1 + L1 k2] = sum_n2 y[k1][n2] W_L2^{n2 k2}.
template <class C, class TO>
__global__ void __launch_bounds__(1024) k_fft_rowB(const C* __restrict__ in, TO* __restrict__ out, Rows ri, Rows ro,
                                                   int L1, int L2, int M, int inv, double scale,
                                                   const C* __restrict__ tw) {
  extern __shared__ __align__(16) uint8_t smraw[];
  C* s = reinterpret_cast<C*>(smraw);
  const int64_t r = blockIdx.y;
  const int b = blockIdx.z;
  const int64_t L = (int64_t)L1 * L2;
  const int k10 = blockIdx.x * M;
  const C* src = in + b * ri.stride_b + ri.off + r * L + (int64_t)k10 * L2;
  TO* dst = out + b * ro.stride_b + ro.off + r * L;
  for (int i = threadIdx.x; i < M * L2; i += 1024) s[i] = src[i];
  __syncthreads();
  smem_fft<C, 1024>(s, L2, M, 1, L2, false, inv != 0, tw);
  const typename Cx<C>::R sc = (typename Cx<C>::R)scale;
  for (int i = threadIdx.x; i < M * L2; i += 1024) {
    int m = i % M, k2 = i / M;
    C v = s[m * L2 + k2];
    dst[(int64_t)k2 * L1 + k10 + m] = t_cvt<TO>(Cx<C>::mk(v.x * sc, v.y * sc));
  }
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
std::vector<double2> fft_twiddle_table_d() { return twiddles<double2>(); }

template <class TI, class TO, class C>
static cudaError_t fft_launch_t(const TI* in, TO* out, Rows ri, Rows ro, int B, bool inverse, const C* tw,
                                cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fft_rowB<C, TO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (sizeof(C) == 8 ? 4 : 2) * 4096 * (int)sizeof(C));
    cudaFuncSetAttribute(k_fft_colA<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * (int)sizeof(C));
    cudaFuncSetAttribute(k_fft_small<TI, TO, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * (int)sizeof(C));
    attr = true;
  }
  const int64_t L = ri.L;
  const double scale = inverse ? 1.0 / (double)L : 1.0;
  if (ri.count <= 0 || B <= 0) return cudaSuccess;
  if (L <= 4096) {
    int M = (int)(L >= 1024 ? 1 : 1024 / L);
    dim3 grid((unsigned)((ri.count + M - 1) / M), (unsigned)B);
    k_fft_small<TI, TO, C><<<grid, 256, (size_t)M * L * sizeof(C), st>>>(in, out, ri, ro, (int)L, M,
                                                                         inverse ? 1 : 0, scale, tw);
    count_launch();
    return cudaGetLastError();
  }
  // four-step; step A runs in place on `in` (it is clobbered; requires TI == C), step B writes `out`
  static_assert(sizeof(TI) == sizeof(C), "four-step input must already be in the compute type");
  const int L2 = 4096, L1 = (int)(L / 4096);
  // columns per CTA: ~8192 elements per CTA, at least 16 columns (>= 128-byte rows)
  const int CW = std::max(16, std::min(L2, 8192 / L1));
  {
    dim3 grid((unsigned)(L2 / CW), (unsigned)ri.count, (unsigned)B);
    k_fft_colA<C><<<grid, 512, (size_t)L1 * CW * sizeof(C), st>>>(reinterpret_cast<C*>(const_cast<TI*>(in)), ri,
                                                                     L1, L2, CW, inverse ? 1 : 0, tw);
  }
  {
    const int Mmax = sizeof(C) == 8 ? 4 : 2;   // rows per CTA: 128 KB of SMEM
    const int M = L1 >= Mmax ? Mmax : L1;
    dim3 grid((unsigned)(L1 / M), (unsigned)ri.count, (unsigned)B);
    k_fft_rowB<C, TO><<<grid, 1024, (size_t)M * L2 * sizeof(C), st>>>(reinterpret_cast<const C*>(in), out, ri, ro,
                                                                        L1, L2, M, inverse ? 1 : 0, scale, tw);
  }
  count_launch(2);
  return cudaGetLastError();
}

cudaError_t fft_launch(const float2* in, float2* out, Rows ri, Rows ro, int B, bool inverse, const float2* tw,
                       cudaStream_t st) {
  return fft_launch_t<float2, float2, float2>(in, out, ri, ro, B, inverse, tw, st);
}
cudaError_t fft_launch_dd(const double2* in, double2* out, Rows ri, Rows ro, int B, bool inverse,
                          const double2* tw, cudaStream_t st) {
  return fft_launch_t<double2, double2, double2>(in, out, ri, ro, B, inverse, tw, st);
}
cudaError_t fft_launch_df(const double2* in, float2* out, Rows ri, Rows ro, int B, bool inverse,
                          const double2* tw, cudaStream_t st) {
  return fft_launch_t<double2, float2, double2>(in, out, ri, ro, B, inverse, tw, st);
}

}  // namespace jtfs
