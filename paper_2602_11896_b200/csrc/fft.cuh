// fft.cuh — host entry points of the hand-written batched FFT (fft.cu).
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"

namespace jtfs {
// Out-of-place batched C2C FFT of B x ri.count rows of length ri.L (power of two, 2..2^22).
// For L > 4096 the input rows are clobbered (four-step scheme runs its first step in place).
// `tw` = device twiddle table (fft_twiddle_table / _d). Inverse includes the 1/L factor.
cudaError_t fft_launch(const float2* in, float2* out, Rows ri, Rows ro, int B, bool inverse,
                       const float2* tw, cudaStream_t st);
// float64 compute: double -> double, double -> float (output rounded to complex64)
cudaError_t fft_launch_dd(const double2* in, double2* out, Rows ri, Rows ro, int B, bool inverse,
                          const double2* tw, cudaStream_t st);
cudaError_t fft_launch_df(const double2* in, float2* out, Rows ri, Rows ro, int B, bool inverse,
                          const double2* tw, cudaStream_t st);
std::vector<float2> fft_twiddle_table();
std::vector<double2> fft_twiddle_table_d();
}  // namespace jtfs
