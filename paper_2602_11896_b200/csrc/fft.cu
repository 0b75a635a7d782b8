// fft.cu — batched power-of-two complex FFTs for sm_100a, hand written (no cuFFT).
//
// Shared-memory Stockham autosort with radix-4 passes (+ one radix-2 pass for odd log2 n); each
// butterfly is staged in registers so the pass runs in place in SMEM. Lengths <= 4096 run in one
// kernel (several short rows per CTA); longer lengths L = L1 * 4096 use the four-step scheme:
//   A) L1-point column transforms in place + twiddle W_L^{n2 k1}   (k_fft_colA)
//   B) 4096-point row transforms written transposed to the output  (k_fft_rowB)
// Used for rfft/ifft/cfft of the listings P:203, P:209, P:211, P:235, P:282, P:285 and their
// adjoints. Forward = exp(-2 pi i k n / L); inverse = exp(+...) / L (numpy convention).
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "common.cuh"
#include "fft.cuh"

namespace jtfs {

static constexpr int kTw = 4096;  // twiddle table length

__device__ __forceinline__ void dft4(float2& a0, float2& a1, float2& a2, float2& a3, bool inv) {
  float2 t0 = cadd(a0, a2), t1 = csub(a0, a2), t2 = cadd(a1, a3), t3 = csub(a1, a3);
  a0 = cadd(t0, t2);
  a2 = csub(t0, t2);
  float2 mt3 = inv ? make_float2(-t3.y, t3.x) : make_float2(t3.y, -t3.x);  // (+/-i) * t3
  a1 = cadd(t1, mt3);
  a3 = csub(t1, mt3);
}

__device__ __forceinline__ float2 twid(const float2* __restrict__ tw, int e, bool inv) {
  float2 w = __ldg(tw + e);
  return inv ? make_float2(w.x, -w.y) : w;
}

// One Stockham pass of radix R over M sequences of length n in SMEM (element i of sequence c at
// s[i*es + c*ss]). `ileave` = sequences interleaved (ss == 1): consecutive threads -> sequences.
template <int R, int THREADS>
__device__ __forceinline__ void stockham_pass(float2* s, int n, int M, int es, int ss, bool ileave,
                                              int Ns, bool inv, const float2* __restrict__ tw) {
  constexpr int MAXB = (R == 4) ? 4 : 8;
  const int nbr = n / R;
  const int nb = nbr * M;
  float2 v[MAXB][R];
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
        float2 a = s[(j + r * nbr) * es + c * ss];
        if (r > 0 && k > 0) a = cmul(a, twid(tw, r * k * tstep, inv));
        v[i][r] = a;
      }
      if (R == 4) {
        dft4(v[i][0], v[i][1], v[i][2], v[i][3], inv);
      } else {
        float2 a = v[i][0], b = v[i][1];
        v[i][0] = cadd(a, b);
        v[i][1] = csub(a, b);
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

template <int THREADS>
__device__ void smem_fft(float2* s, int n, int M, int es, int ss, bool ileave, bool inv,
                         const float2* __restrict__ tw) {
  int Ns = 1;
  while (Ns * 4 <= n) {
    stockham_pass<4, THREADS>(s, n, M, es, ss, ileave, Ns, inv, tw);
    Ns *= 4;
  }
  if (Ns < n) stockham_pass<2, THREADS>(s, n, M, es, ss, ileave, Ns, inv, tw);
}

// ---------------------------------------------------------------- n <= 4096, M rows per CTA
__global__ void __launch_bounds__(256) k_fft_small(const float2* __restrict__ in, float2* __restrict__ out,
                                                   Rows ri, Rows ro, int n, int M, int inv, float scale,
                                                   const float2* __restrict__ tw) {
  extern __shared__ float2 s[];
  const int b = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * M;
  const int rows = (int)((ri.count - r0) < M ? (ri.count - r0) : M);
  const float2* src = in + b * ri.stride_b + ri.off + r0 * n;
  float2* dstp = out + b * ro.stride_b + ro.off + r0 * n;
  const int tot = rows * n;
  for (int i = threadIdx.x; i < M * n; i += 256) s[i] = (i < tot) ? src[i] : make_float2(0.f, 0.f);
  __syncthreads();
  smem_fft<256>(s, n, M, 1, n, false, inv != 0, tw);
  for (int i = threadIdx.x; i < tot; i += 256) dstp[i] = cscale(s[i], scale);
}

// ---------------------------------------------------------------- four-step A: columns
// x viewed as [L1][L2] (n = n1*L2 + n2). For the CTA's CW columns n2: y[k1][n2] =
// sum_n1 x[n1][n2] W_L1^{n1 k1}, times W_L^{n2 k1}; written back in place.
__global__ void __launch_bounds__(512) k_fft_colA(float2* __restrict__ data, Rows ri, int L1, int L2, int CW,
                                                  int inv, const float2* __restrict__ tw) {
  extern __shared__ float2 s[];
  const int64_t r = blockIdx.y;
  const int b = blockIdx.z;
  const int64_t L = (int64_t)L1 * L2;
  float2* base = data + b * ri.stride_b + ri.off + r * L;
  const int c0 = blockIdx.x * CW;
  for (int i = threadIdx.x; i < L1 * CW; i += 512) {
    int n1 = i / CW, c = i % CW;
    s[i] = base[(int64_t)n1 * L2 + c0 + c];
  }
  __syncthreads();
  smem_fft<512>(s, L1, CW, CW, 1, true, inv != 0, tw);
  const float sgn = inv ? 2.0f : -2.0f;
  for (int i = threadIdx.x; i < L1 * CW; i += 512) {
    int k1 = i / CW, c = i % CW;
    int64_t e = ((int64_t)(c0 + c) * k1) % L;   // exact; 2e/L exact in fp32 (L <= 2^22)
    float sn, cs;
    sincospif(sgn * (float)e / (float)L, &sn, &cs);
    base[(int64_t)k1 * L2 + c0 + c] = cmul(s[i], make_float2(cs, sn));
  }
}

// ---------------------------------------------------------------- four-step B: rows, transposed out
// For rows k1 in [k1_0, k1_0 + M): X[k1 + L1 k2] = sum_n2 y[k1][n2] W_L2^{n2 k2}.
__global__ void __launch_bounds__(1024) k_fft_rowB(const float2* __restrict__ in, float2* __restrict__ out,
                                                   Rows ri, Rows ro, int L1, int L2, int M, int inv, float scale,
                                                   const float2* __restrict__ tw) {
  extern __shared__ float2 s[];
  const int64_t r = blockIdx.y;
  const int b = blockIdx.z;
  const int64_t L = (int64_t)L1 * L2;
  const int k10 = blockIdx.x * M;
  const float2* src = in + b * ri.stride_b + ri.off + r * L + (int64_t)k10 * L2;
  float2* dst = out + b * ro.stride_b + ro.off + r * L;
  for (int i = threadIdx.x; i < M * L2; i += 1024) s[i] = src[i];
  __syncthreads();
  smem_fft<1024>(s, L2, M, 1, L2, false, inv != 0, tw);
  for (int i = threadIdx.x; i < M * L2; i += 1024) {
    int m = i % M, k2 = i / M;
    dst[(int64_t)k2 * L1 + k10 + m] = cscale(s[m * L2 + k2], scale);
  }
}

// ---------------------------------------------------------------- host side
static bool g_attr_done = false;

void fft_init_attributes() {
  if (g_attr_done) return;
  cudaFuncSetAttribute(k_fft_rowB, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 4096 * 8);
  cudaFuncSetAttribute(k_fft_colA, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8);
  g_attr_done = true;
}

std::vector<float2> fft_twiddle_table() {
  std::vector<float2> t(kTw);
  for (int e = 0; e < kTw; ++e) {
    double a = -2.0 * 3.14159265358979323846 * (double)e / (double)kTw;
    t[e] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  return t;
}

cudaError_t fft_launch(const float2* in, float2* out, Rows ri, Rows ro, int B, bool inverse,
                       const float2* tw, cudaStream_t st) {
  fft_init_attributes();
  const int64_t L = ri.L;
  const float scale = inverse ? (float)(1.0 / (double)L) : 1.0f;
  if (ri.count <= 0 || B <= 0) return cudaSuccess;
  if (L <= 4096) {
    int M = (int)(L >= 1024 ? 1 : 1024 / L);
    dim3 grid((unsigned)((ri.count + M - 1) / M), (unsigned)B);
    k_fft_small<<<grid, 256, (size_t)M * L * sizeof(float2), st>>>(in, out, ri, ro, (int)L, M,
                                                                     inverse ? 1 : 0, scale, tw);
    count_launch();
    return cudaGetLastError();
  }
  // four-step; step A runs in place on `in` (it is clobbered), step B writes `out`
  const int L2 = 4096, L1 = (int)(L / 4096);
  const int CW = L1 >= 1024 ? 8 : 16;
  {
    dim3 grid((unsigned)(L2 / CW), (unsigned)ri.count, (unsigned)B);
    k_fft_colA<<<grid, 512, (size_t)L1 * CW * sizeof(float2), st>>>(const_cast<float2*>(in), ri, L1, L2, CW,
                                                                    inverse ? 1 : 0, tw);
  }
  {
    const int M = L1 >= 4 ? 4 : L1;
    dim3 grid((unsigned)(L1 / M), (unsigned)ri.count, (unsigned)B);
    k_fft_rowB<<<grid, 1024, (size_t)M * L2 * sizeof(float2), st>>>(in, out, ri, ro, L1, L2, M,
                                                                     inverse ? 1 : 0, scale, tw);
  }
  count_launch(2);
  return cudaGetLastError();
}

}  // namespace jtfs
