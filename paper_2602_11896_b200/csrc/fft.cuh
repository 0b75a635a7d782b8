// fft.cuh — host entry points of the hand-written batched FFT (fft.cu).
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"

namespace jtfs {
// Device twiddle tables: the 4096-entry W_4096^e tables (float, double) and, per length L = 2^lg > 4096, the
// four-step table tw2[k1 4096 + n2] = W_L^{k1 n2} (k1 < L / 4096): the column pass (consecutive columns n2)
// and the T -> natural row pass (consecutive n2) read it coalesced.
struct FftTables {
  const float2* tw = nullptr;
  const double2* twd = nullptr;
  const float2* twp = nullptr;     // per-pass tables (fft_pass_tables), lengths 2 .. 4096
  const double2* twpd = nullptr;
  const float2* tw2_f[23] = {};
  const double2* tw2_d[23] = {};
};
// Out-of-place batched C2C FFT of B x ri.count rows of length ri.L (power of two, 2..2^22).
// For L > 4096 the input rows are clobbered (four-step scheme runs its first step in place).
// Inverse includes the 1/L factor.
cudaError_t fft_launch(const float2* in, float2* out, Rows ri, Rows ro, int B, bool inverse, const FftTables& T,
                       cudaStream_t st);
// float64 compute: double -> double, double -> float (output rounded to complex64)
cudaError_t fft_launch_dd(const double2* in, double2* out, Rows ri, Rows ro, int B, bool inverse,
                          const FftTables& T, cudaStream_t st);
cudaError_t fft_launch_df(const double2* in, float2* out, Rows ri, Rows ro, int B, bool inverse,
                          const FftTables& T, cudaStream_t st);
// Storage order of rows longer than 4096 points (four-step transforms): natural, or the "T-layout" in
// which element k1 + L1 k2 (L1 = L / 4096) sits at k1 4096 + k2 -- the order the row pass leaves when it
// stores in place, used between elementwise stages (fft.cu). Rows of <= 4096 points are always natural.
constexpr int kLayoutNatural = 0, kLayoutToT = 1, kLayoutFromT = 2;
// Row groups {off, count, L} (offsets shared by in and out, per-signal strides in_sb / out_sb): groups of
// length <= 4096 run in grouped launches, longer ones as four-step transforms.
struct FftGroup;
cudaError_t fft_groups(const float2* in, float2* out, int64_t in_sb, int64_t out_sb, const FftGroup* g, int ng,
                       int B, bool inverse, const FftTables& T, cudaStream_t st, int layout = kLayoutNatural);
cudaError_t fft_groups_dd(const double2* in, double2* out, int64_t in_sb, int64_t out_sb, const FftGroup* g, int ng,
                          int B, bool inverse, const FftTables& T, cudaStream_t st, int layout = kLayoutNatural);
cudaError_t fft_groups_df(const double2* in, float2* out, int64_t in_sb, int64_t out_sb, const FftGroup* g, int ng,
                          int B, bool inverse, const FftTables& T, cudaStream_t st, int layout = kLayoutNatural);
std::vector<float2> fft_twiddle_table();
// Per-pass twiddles for the in-SMEM transforms of length L = 2^lg <= 4096, table of L at [L, 2L): pass p of
// seq_fft (radix R_p, sub-transform size Ns_p) holds W_{Ns_p R_p}^{r k} at (Ns_p - 1) + (r - 1) Ns_p + k,
// r < R_p, k < Ns_p (sum over passes of (R_p - 1) Ns_p = L - 1 entries), so lanes with consecutive k read
// consecutive words (the strided W_4096 table puts lanes of one pass in the same bank).
std::vector<float2> fft_pass_tables();
std::vector<double2> fft_pass_tables_d();
std::vector<double2> fft_twiddle_table_d();
void fft_fourstep_table_f(int lgL, std::vector<float2>* t);
void fft_fourstep_table_d(int lgL, std::vector<double2>* t);
}  // namespace jtfs
