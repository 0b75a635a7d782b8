// device.cuh — device copies of the plan tables and the kernel launchers (kernels_*.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.cuh"
#include "fft.cuh"
#include "plan.h"

namespace jtfs {

struct TcClass {
  TcBlock* blocks = nullptr;
  int64_t* tiles = nullptr;
  int n_blocks = 0;
  int64_t ntiles = 0;
  int K2max = 0, Kmax = 0, kcw = 32, kb2 = 8;
  int cls = 0;                     // kernel variant (TcBlock::cls)
  int ks = 0, nparts = 1;          // split-K block: K parts of the forward
  int hyb = 0;                     // forward hybrid one-part mode (TcBlock::hyb)
  int ngmax = 1;                   // filter groups the launch may use (TcBlock::ngmax)
  int64_t n_cols = 0;              // columns of the block
  int bi = 0;                      // block index
  int64_t gp_off = 0;              // backward g_Y2 partials offset (TcBlock::gp_off)
};

struct FfList {                    // blocks on the FFT route of the joint stage + column-tile prefix
  int32_t* blist = nullptr;
  int64_t* tiles = nullptr;
  int nb = 0;
  int64_t ntiles = 0;
};

struct DeviceTables {
  float* spec_vals = nullptr;
  double* spec_vals_d = nullptr;   // float64 psi1 spectra (l1_jobs)
  double* cn_nu = nullptr;          // colored-noise tables (R25)
  float* cn_den = nullptr;
  GatherJob* l1_jobs = nullptr;     int64_t* l1_tiles = nullptr;   int n_l1 = 0;   int64_t l1_ntiles = 0;
  GatherJob* s1_jobs = nullptr;     int64_t* s1_tiles = nullptr;   int n_s1 = 0;   int64_t s1_ntiles = 0;
  GatherJob* l2_jobs = nullptr;     int64_t* l2_tiles = nullptr;   int n_l2 = 0;   int64_t l2_ntiles = 0;
  GatherJob* s0_job = nullptr;      int64_t* s0_tiles = nullptr;   int64_t s0_ntiles = 0;
  Support* psi1_sup = nullptr;
  Support* psi2_sup = nullptr;      // [n_blocks][log2T+1]
  Support* phiT_sup = nullptr;      // [log2T+1]
  float2* hfr = nullptr;            // [n_fr][P]
  float* phiF_k = nullptr;          int64_t* phiF_off = nullptr;
  float* phiT_half = nullptr;       int64_t* phiT_off = nullptr;   int64_t* phiT_H = nullptr;
  JointUnit* units = nullptr;       int n_units = 0;
  BlockInfo* binfo = nullptr;       int n_blocks = 0;
  // forward unit lists per rows_out class KAP in {1,2,4,8,16,32}: unit indices + tile prefix
  int32_t* fwd_ulist[6] = {};       int64_t* fwd_tiles[6] = {};    int fwd_n[6] = {};  int64_t fwd_ntiles[6] = {};
  int fwd_kmax[6] = {};
  int32_t* kf_of = nullptr;         // [n_fr] k_f per frequential filter
  int32_t* hfr_H = nullptr;         // [n_fr] support half-width of h_f
  // phi_T kernels: (unit, rho) rows in unit order and the prefix of their 256-column tiles
  int32_t* phT_rows_u = nullptr;    int32_t* phT_tiles = nullptr;   /* per adjoint tile: u, rho, c0 */  int phT_nrows = 0;  int64_t phT_ntiles = 0;
  int32_t* blk_nmax = nullptr;      // [n_blocks]
  // phi_T banded-GEMM adjoint (k_phiT_adj3) for the halo-pruned blocks: 32-row groups {first row, rows,
  // block, -, ...}, their (unit, rho) rows, tiles (group, 256-column tile), the mask of the blocks covered
  int32_t* ph3_groups = nullptr;    int32_t* ph3_rows = nullptr;   int32_t* ph3_atiles = nullptr;
  int ph3_ngroups = 0;  int64_t ph3_natiles = 0;  uint64_t ph3_mask = 0;
  int64_t* ucoef = nullptr;         // [n_units] coefficient offset of the unit's path - o2_start
  int64_t* uo = nullptr;            // [n_units] o_off
  int64_t o2_start = 0, n_o2 = 0;
  int maxLf = 0, max_rows_out = 0;
  int64_t* bwd_tiles = nullptr;     int64_t bwd_ntiles = 0;        // prefix over blocks of (col tiles x n ranges)
  int32_t* coef_path = nullptr;     // [n_coef]
  int64_t* path_off = nullptr;      // [n_paths + 1] coefficient offsets (LossReport)
  int32_t* path_owner_unit = nullptr;  // [n_paths]: -2 order 0, -1 order 1, else unit index
  int64_t* l1_off = nullptr;        int32_t* n1_k1 = nullptr;      // per n1 offsets, k1
  int64_t* u1adj_tiles = nullptr;   int64_t u1adj_ntiles = 0;      // prefix over n1 of L1 tiles
  int32_t* gx_tile_start = nullptr; int32_t* gx_list = nullptr;
  int64_t* o1_rlo = nullptr;        int64_t* o1_nrows = nullptr;
  float2* tw = nullptr;
  double2* twd = nullptr;
  FftTables fftt;                   // views of tw/twd + four-step tables (owned: fs_bufs)
  std::vector<void*> fs_bufs;
  int Kmax = 0, Kmax_simt_bwd = 0;
  // tensor-core joint stage
  float* tc_img = nullptr;
  float* tc_wts = nullptr;
  TcUnit* tc_units = nullptr;
  std::vector<TcClass> tc;         // one launch per tensor-core block (forward)
  float* tc_img2 = nullptr;
  float* tc_img1b = nullptr;
  std::vector<TcClass> tcb;        // one launch per tensor-core block (backward)
  // FFT route (kernels_frfft.cu)
  float* fr_spec = nullptr;
  float* u_wts = nullptr;
  int64_t* u_wt_off = nullptr;
  FfList ffw, ffb;
};

constexpr int kGatherThreads = 256;                 // threads per CTA of the gather kernels
constexpr int kGatherTile = 4 * kGatherThreads;     // outputs per CTA (4 per thread, 256 apart)
constexpr int kGatherTileT = 4096;                  // outputs per CTA of a T-layout job (staged in SMEM)
constexpr int kPhiTSmem = 12288;   // phi_T half kernel staged in SMEM up to this many taps
constexpr int kJC = 64;            // joint stage: columns per CTA
constexpr int kJR = 64;            // joint stage: rows per chunk
constexpr int kJN = 64;            // joint backward: n1 rows per CTA

// ---- kernels_time.cu
void launch_reflect_pad(const float* x, int64_t sx, double2* xp, const Plan& p, int B, cudaStream_t st);
void launch_gather(const float2* in, int64_t in_sb, float2* out, int64_t out_sb, const GatherJob* jobs,
                   const int64_t* tiles, int njobs, int64_t ntiles, const float* vals, int B, cudaStream_t st,
                   uint64_t own = kOwnAll);
void launch_gather_dd(const double2* in, int64_t in_sb, double2* out, int64_t out_sb, const GatherJob* jobs,
                      const int64_t* tiles, int njobs, int64_t ntiles, const double* vals, int B, cudaStream_t st);
void launch_gather_df(const double2* in, int64_t in_sb, float2* out, int64_t out_sb, const GatherJob* jobs,
                      const int64_t* tiles, int njobs, int64_t ntiles, const float* vals, int B, cudaStream_t st,
                      uint64_t own = kOwnAll);
// level groups of the layer-1 rows for the pair-packed U1 FFT (<= kMaxPackGroups distinct lengths)
constexpr int kMaxPackGroups = 24;
struct PackGroups {
  int64_t off[kMaxPackGroups];          // first row element of the group (natural layout)
  int64_t pstart[kMaxPackGroups + 1];   // packed (compact) offset of each group = Plan::l1_pgroups[g].off
  int count[kMaxPackGroups];            // rows of the group
  int lgL[kMaxPackGroups];              // log2 row length
  int n;
};
PackGroups pack_groups(const Plan& p);
void launch_modulus_pack(const float2* z, int64_t zsb, double2* u, int64_t usb, const PackGroups& G, int B,
                         cudaStream_t st);
void launch_unpack_u1(const double2* u, int64_t usb, float* out, int64_t out_sb, const PackGroups& G, int64_t n,
                      int B, cudaStream_t st);
void launch_untranspose_rows(const float2* z, int64_t zsb, float2* out, int64_t out_sb, const PackGroups& G,
                             int64_t n, int B, cudaStream_t st);
void launch_real_rows_d(const double2* in, int64_t in_sb, float* out, int64_t out_sb, int64_t n, int B,
                        cudaStream_t st);
void launch_real_rows(const float2* in, int64_t in_sb, int64_t in_off, float* out, int64_t out_sb,
                      int64_t out_off, int64_t n, int B, cudaStream_t st);
void launch_s0_out(const float2* s0c, int64_t s0_sb, float* S, int64_t S_sb, const Plan& p, int B,
                   cudaStream_t st);
void launch_adj_gather_u1(const Plan& p, const DeviceTables& d, const float2* GS, int64_t GS_sb,
                          const float2* GY, int64_t GY_sb, float2* out, int64_t out_sb, int B,
                          cudaStream_t st, uint64_t own = kOwnAll);
void launch_phase_mul(const float2* z, const float2* gu, int64_t gsb, float2* out, int64_t n_per_b, int64_t sb,
                      const float* thr, int B, cudaStream_t st);
// reading R22: the modulus adjoint uses phase 0 where |z| < kEpsMod * RMS(y_b)
constexpr float kEpsMod = 1e-12f;
void launch_mod_threshold(const float* y, int64_t N, float eps, float* thr, int B, cudaStream_t st);
void launch_adj_gather_x(const Plan& p, const DeviceTables& d, const float2* GZ, int64_t GZ_sb, float2* out,
                         int64_t out_sb, int B, cudaStream_t st);
void launch_real_to_complex(const float* in, int64_t in_sb, float2* out, int64_t out_sb, int64_t n, int B,
                            cudaStream_t st);
void launch_reflect_adj(const float2* gxp, int64_t sxp, float* g, int64_t sg, const Plan& p, int B,
                        cudaStream_t st);
// colored-noise initialisation (R25): per-band gains from the order-1 beta = 0 path of S_target
// (g [B][N1 + 1], last entry = fallback flag), spectral shaping of X = FFT(white), crop of the IFFT
void launch_cn_gains(const Plan& p, const DeviceTables& d, const float* St, int64_t St_sb, float* g, int64_t g_sb,
                     int B, cudaStream_t st);
void launch_cn_shape(const Plan& p, const DeviceTables& d, float2* X, int64_t X_sb, const float* g, int64_t g_sb,
                     int B, cudaStream_t st);
void launch_cn_crop(const Plan& p, const float2* X, int64_t X_sb, const float* white, const float* g, int64_t g_sb,
                    float* y0, int B, cudaStream_t st);
void launch_check_finite(const float* x, int64_t n, int32_t* flag, cudaStream_t st);
void launch_metamer(float* y, float* u, float* y_prev, float* g_prev, float* mu, float* loss_prev,
                    const float* loss, int32_t* accepted, const int32_t* active, const float* g, int64_t sg,
                    int64_t N, int B, float momentum, float grow, float shrink, cudaStream_t st);

// ---- kernels_fr.cu
void launch_o1_fwd(const Plan& p, const DeviceTables& d, const float* S1t, int64_t S1t_sb, float2* W1,
                   int64_t W1_sb, float* V2, int64_t V2_sb, float* S, int64_t S_sb, int B, cudaStream_t st);
void launch_o1_bwd(const Plan& p, const DeviceTables& d, const float* r, int64_t r_sb, float2* W1,
                   int64_t W1_sb, float* V2, int64_t V2_sb, const float* S1t, int64_t S1t_sb, float* gS1t,
                   int64_t gS1t_sb, const float* thr, int B, cudaStream_t st);
void launch_joint_fwd(const Plan& p, const DeviceTables& d, const float2* Y2, int64_t y_sb, float* o,
                      int64_t o_sb, uint64_t own, int B, cudaStream_t st);
void launch_phiT_fwd(const Plan& p, const DeviceTables& d, const float* o, int64_t o_sb, float* S,
                     int64_t S_sb, uint64_t own, int B, cudaStream_t st);
// per-path LossReport: rep[b][q] = 1/2 sum over path q's coefficients of (S - St)^2
void launch_loss_report(const Plan& p, const DeviceTables& d, const float* S, const float* St, float* rep, int B,
                        cudaStream_t st);
void launch_loss(const Plan& p, const DeviceTables& d, const float* S, int64_t S_sb, const float* St,
                 int64_t St_sb, float* r, int64_t r_sb, float* loss, double* part, uint64_t own, int B,
                 cudaStream_t st);
void launch_phiT_adj(const Plan& p, const DeviceTables& d, const float* r, int64_t r_sb, float* go,
                     int64_t go_sb, uint64_t own, int B, cudaStream_t st);
// the per-block launches go round-robin over the ns streams ss (forked from and joined to the caller's)
// split-K blocks accumulate W in wbuf (per-signal stride wb_sb) and leave it there when keep_w (backward)
void launch_joint_fwd_tc(const Plan& p, const DeviceTables& d, const float2* Y2, int64_t y_sb, float* o,
                         int64_t o_sb, float* wbuf, int64_t wb_sb, bool keep_w, const float* thr, uint64_t own,
                         int B, const cudaStream_t* ss, int ns);
void launch_joint_bwd_tc(const Plan& p, const DeviceTables& d, const float2* Y2, int64_t y_sb, const float* go,
                         int64_t go_sb, float2* gY, int64_t gy_sb, const float* wbuf, int64_t wb_sb,
                         float2* gp, int64_t gp_sb, const float* thr, uint64_t own, int B,
                         const cudaStream_t* ss, int ns);
void launch_joint_bwd(const Plan& p, const DeviceTables& d, const float2* Y2, int64_t y_sb, const float* go,
                      int64_t go_sb, float2* gY2, int64_t gy_sb, const float* thr, uint64_t own, int B,
                      cudaStream_t st);

// ---- kernels_frfft.cu
void launch_joint_fft(const Plan& p, const DeviceTables& d, bool bwd, const float2* Y2, int64_t y_sb, float* o,
                      int64_t o_sb, float2* gY, int64_t gy_sb, const float* thr, uint64_t own, int B,
                      cudaStream_t st);
int64_t joint_fft_tiles(int64_t n_cols);
constexpr int kFfMaxP = 1024;      // FFT route: C x P <= 4096 points per CTA
constexpr int kFfMaxRo = 64;       // FFT route backward: rows_out <= 64

}  // namespace jtfs
