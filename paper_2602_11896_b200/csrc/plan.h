// plan.h — host-side JTFS plan (float64) and the device tables derived from it.
// The planner is independent of oracle/ (no shared code): it re-derives every rule from PAPER.md
// and the readings of DESIGN.md §2.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/jtfs.h"

namespace jtfs {

struct Filter {
  double xi = 0, sigma = 0, kappa = 0;
  int j = 0, spin = 1;
  bool phi = false;  // Gaussian low-pass (phi_T / phi_F) instead of Morlet (Eq.1)
};

struct Block {
  int n2, n1_max, s2, j2;
};

// Support-limited spectrum of a filter on an L-point grid: values for bins lo .. lo+len-1 (taken
// modulo L), stored at vals[off .. off+len).
struct Support {
  int64_t lo, len, off, L;
};

// One gather-fold job: out[m] = scale * sum_{s in [lo, lo+len), s = m mod L_out} in[s mod L_in] *
// h[s - lo], for m in [0, L_out).  (cdgmm + subsample_fourier)
struct GatherJob {
  int64_t in_off, L_in, lo, len, val_off, out_off, L_out;
  float scale;
  int32_t blk;   // second-order block of a layer-2 job (path shards skip unowned blocks), -1 otherwise
  int32_t par;   // -1: plain complex row; 0 / 1: the row is the real / imaginary half of a pair-packed row
                 // whose FFT carries two real rows (Z = U_a + i U_b): U_a^[s] = (Z[s] + conj Z[-s]) / 2,
                 // U_b^[s] = (Z[s] - conj Z[-s]) / 2i
  int32_t tl;    // 1: the output row (L_out > 4096 points) is written in the four-step's T-layout (fft.cuh):
                 // element m = k1 + L1 k2 at k1 4096 + k2, so that its inverse FFT runs row-contiguous
};

// Batched FFT group: `count` rows of length L starting at `off` (per signal).
struct FftGroup {
  int64_t off, count, L;
};

// Per (block, frequential filter) unit of the joint lambda_1 stage.
struct JointUnit {
  int32_t bi, f, kf, d;          // block, filter (L_fr index), k_f, log2F - k_f
  int32_t n1_max, rows_out;      // K and kept rows (ceil(n1_max/F))
  int64_t Lf, r_lo, n_rows;      // row grid length P>>kf, needed row range (circular)
  int64_t o_off;                 // offset of this unit's o[rows_out][n_cols] in the o buffer
  int32_t path;                  // path index
  int32_t pad;
};

struct BlockInfo {
  int64_t y_off;                 // offset (complex elements) of the block in Y2 (per signal)
  int64_t T2, c_lo, n_cols;      // columns, needed column range (circular on T2)
  int32_t s2, D;                 // level, decimation 2^(log2T - s2)
};

// Tensor-core (tcgen05) joint-stage tables (kernels_tc.cu)
struct TcUnit {
  int64_t img_off, wt_off;   // offsets (floats) of the unit's B images / phi_F weights
  int64_t img2_off;          // offset of the backward B2 images (32-row tiles)
  int64_t img1b_off;         // offset of the backward GEMM1 images (32-row tiles, [hi 64 x kc | lo 64 x kc])
  int32_t NT;                // row tiles of 64 (0 = unit not on the tensor-core path)
  int32_t wp_tile0;          // split-K blocks: index of the unit's first 64-row tile in the block's W buffer
};
struct TcBlock {
  int32_t bi, K, K2, cls;    // block, n1_max, padded 2K, launch class
  int32_t kcw, kb2;          // B-image chunk widths: forward/GEMM1 (k' elements), backward B2 (kk elements)
  int32_t ks, nparts;        // split-K block (A tile too large for SMEM): number of K parts
  int32_t kpw, wp_tiles;     // part width (k' elements, multiple of kcw); 64-row tiles per column tile
  int64_t wp_off;            // offset (floats, per signal) of the block's W buffer
  int32_t ngmax;             // filter groups a launch may split into (few column tiles -> more CTAs)
  int32_t wph;               // 16-byte words per 64-row tile of the kept phase store (2048; 4096 when the
                             // tile also carries fp32 K-part partials): see kernels_tc.cu "phase store"
  int64_t gp_off;            // backward: offset (complex, per signal) of the block's g_Y2 partials
  int32_t hyb;               // forward "hybrid" one-part split-K: A_hi in TMEM (TS form), A_lo in SMEM (SS form),
                             // for K2 too large for both halves in TMEM (kernels_tc.cu)
  int32_t pad3;
};
// forward class = 8 * ct_kind + kap_kind (ct_kind 0: 2 column tiles, 1: one; KAP = 2 << kap_kind,
// rows_out <= 2, 4, 8, 16, 32); backward class = kap_kind
// Split-K blocks (K too large for a resident A tile, SURVEY §8(a) A5 large n1_max): the forward runs
// in nparts launches over k' ranges of width kpw, accumulating the complex W of every cell in a
// per-signal buffer (first part stores, middle parts add, the last adds and finishes: modulus, phi_F)
// and leaving the full W there; the backward reads W instead of recomputing GEMM1.
// backward TMEM plan (kernels_tc.cu): A2 double-buffered (nab = 2) when D2 leaves room; the Y2 tile A in
// TMEM (ta = 1, GEMM1 in the TS form) when D1 + A2 + D2 + A_hi + A_lo fit in 512 columns.
inline
#ifdef __CUDACC__
__host__ __device__
#endif
void tc_bwd_mode(int K, int K2, int* nab, int* ta, int pref = 0) {
  const int N2 = ((2 * K + 15) / 16) * 16;
  // pref 1 (JTFS_BWD_MODE=1, tuning): double-buffered A2 with the Y2 tile in SMEM (GEMM1 SS form) wherever
  // the TS form would leave a single A2 buffer
  if (pref == 1 && N2 <= 128 && 384 + N2 + 2 * K2 > 512 && 384 + N2 <= 512) { *nab = 2; *ta = 0; return; }
  if (N2 <= 128 && 384 + N2 + 2 * K2 <= 512) { *nab = 2; *ta = 1; }
  else if (256 + N2 + 2 * K2 <= 512) { *nab = 1; *ta = 1; }
  else { *nab = N2 <= 128 ? 2 : 1; *ta = 0; }
}
int tc_bwd_mode_pref();   // host: JTFS_BWD_MODE (default 0)
// backward B ring sizing shared by the planner (chooses kb2) and the launcher (kernels_tc.cu)
void tc_bwd_rings(int K, int K2, int kcw, int kb2, int* NS1, int* STG1, int* NS2, int* STG2);
int tc_fwd_stages(int CT, int KAP, int K2, int kcw, bool hyb = false);
// forward TMEM plan: the Y2 tile (hi + lo, 2 K2 columns) goes to TMEM and the MMAs take the TS form when
// it fits beside the double-buffered accumulators (CT = 1: 2 x 128 columns); the SS form reads A and B
// from SMEM at 8 KB per N = 128 MMA, which saturates SMEM bandwidth together with the B stream
inline
#ifdef __CUDACC__
__host__ __device__
#endif
bool tc_fwd_tsa(int CT, int K2) { return CT == 1 && 128 + 2 * K2 <= 512; }
// accumulator buffers of the forward: 2 (epilogue of tile t overlaps the MMAs of tile t + 1) unless the TS
// form only fits beside a single one (K2 > 128)
inline
#ifdef __CUDACC__
__host__ __device__
#endif
int tc_fwd_nbuf(int CT, int K2) { return (tc_fwd_tsa(CT, K2) && 256 + 2 * K2 > 512) ? 1 : 2; }

struct DeviceTables;  // device pointers (jtfs_api.cu)

struct Plan {
  // ---- hyper-parameters
  int64_t N = 0, T = 0, F = 0;
  int J = 0, Q = 0, J_fr = 0, Q_fr = 0, log2T = 0, log2F = 0;
  int Q2 = 1;                                   // second-layer quality factor (R7)
  // ---- filterbanks
  std::vector<Filter> psi1, psi2, psi_fr_plus, L_fr;
  Filter phiT, phiF;
  // ---- sizes
  int64_t N_pad = 0, pad_left = 0, P = 0, frames = 0, Ft = 0, n_coef = 0;
  std::vector<Block> blocks;
  std::vector<jtfs_path_t> paths;
  // ---- derived GPU layout (per signal, in elements)
  std::vector<int64_t> L1, L1_off;     // per n1: length N_pad>>k1 and offset in sum L1
  int64_t sumL1 = 0, sumY2 = 0, o_size = 0, o1_W_size = 0;
  std::vector<BlockInfo> binfo;
  std::vector<JointUnit> units;        // order-2 (block, filter) units in path order
  std::vector<FftGroup> l1_groups, y2_groups;
  std::vector<FftGroup> l1_pgroups;             // pair-packed U1 rows: ceil(count / 2) rows per level (R2C pairs),
                                                // compact offsets (complex128 elements)
  int64_t u1p_size = 0;                         // complex128 elements of the packed U1 / U1_hat rows
  std::vector<GatherJob> l1_jobs, s1_jobs, l2_jobs;
  GatherJob s0_job{};
  // order-1 unit rows (per f in xi >= 0 prefix)
  std::vector<int64_t> o1_rlo, o1_nrows;
  int32_t o1_rows_out = 0;
  // kernels
  std::vector<float> spec_vals;                 // all support-limited spectra
  std::vector<Support> psi1_sup;                // [N1] on N_pad
  std::vector<double> spec_vals_d;              // float64 psi1 spectra of the forward first layer
  std::vector<Support> psi1_sup_d;              // [N1] on N_pad, offsets into spec_vals_d (l1_jobs)
  // colored-noise initialisation (reading R25): nu[n1] = (1/N_pad) sum_m |psi1_hat[m]|^2,
  // den[m] = sum_n1 |psi1_hat(m/N_pad)|^2 + delta for m in [0, N_pad/2]
  std::vector<double> cn_nu;
  std::vector<float> cn_den;
  std::vector<Support> psi2_sup;                // [n_blocks][log2T+1] on N_pad>>k (len 0 unused)
  std::vector<Support> phiT_sup;                // [log2T+1] on N_pad>>k
  std::vector<float> hfr;                       // [n_fr_all][P][2] row kernels (complex)
  std::vector<double> hfr_d;                    // same in float64 (for the tensor-core images)
  std::vector<int32_t> hfr_H;                   // [n_fr_all] support half-width of h_f (1e-9 relative)
  std::vector<TcUnit> tc_units;                 // [n_units]
  std::vector<TcBlock> tc_blocks;               // tensor-core eligible blocks
  std::vector<char> blk_tc;                     // [n_blocks] 1 = forward on the tensor-core path
  std::vector<char> blk_tcb;                    // [n_blocks] 1 = backward on the tensor-core path
  std::vector<double> block_cost;               // [n_blocks] path-shard LPT cost (planner.cpp)
  // phi_T banded-GEMM adjoint (kernels_fr.cu k_phiT_adj3) over the halo-pruned blocks
  std::vector<int32_t> ph3_groups, ph3_rows, ph3_atiles;
  uint64_t ph3_mask = 0;
  double order1_cost = 0.0;
  std::vector<char> blk_ks;                     // [n_blocks] 1 = split-K tensor-core block
  std::vector<TcBlock> tcb_blocks;              // backward-eligible blocks (cls = KAP class)
  int64_t ks_w_floats = 0;                      // per-signal W buffer of the split-K blocks
  int64_t gp_complex = 0;                       // per-signal g_Y2 partials of the filter-group split
  std::vector<float> tc_img, tc_wts, tc_img2, tc_img1b;
  // FFT route of the joint stage (kernels_frfft.cu)
  std::vector<float> fr_spec;                   // [n_fr_all][P] level-0 responses of L_fr on the P grid
  std::vector<float> u_wts;                     // per unit [rows_out][n_rows] phi_F weights
  std::vector<int64_t> u_wt_off;                // [n_units] offsets into u_wts
  std::vector<float> phiF_k;                    // concat over k of P>>k real kernels
  std::vector<int64_t> phiF_off;                // [log2F+1]
  std::vector<float> phiT_half;                 // concat over s of half kernels t_s[0..H_s]
  std::vector<int64_t> phiT_off, phiT_H;        // [log2T+1]
  std::vector<int64_t> phiT_L;                  // [log2T+1] grid length N_pad>>s
  // adjoint gather of d/dx spectrum: tiles of N_pad with the list of n1 touching each
  int64_t gx_tile = 256;
  std::vector<int32_t> gx_tile_start, gx_list;  // CSR over tiles
  // reflect-pad adjoint needs nothing extra.
  DeviceTables* dev = nullptr;
  int dev_id = -1;
  ~Plan();
};

// planner.cpp
int make_plan(int64_t N, int J, int Q, int J_fr, int Q_fr, int64_t T, int64_t F, Plan* p, std::string* err,
              int Q2 = 1);
double response_at(const Filter& f, double omega);   // periodised level-0 response
void level_response(const Filter& f, int64_t L0, int k, std::vector<double>* out);

}  // namespace jtfs
