// planner.cpp — JTFS plan in float64 (host). Cites PAPER.md lines (P:n) and DESIGN.md readings.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "plan.h"

namespace jtfs {

static const double kSigma0 = 0.1;
static const double kPi = 3.14159265358979323846;

// Generator of PAPER.md:167-191 evaluated verbatim in float64 (R1: r = r_psi = sqrt(0.5); R2).
static std::vector<std::pair<double, double>> anden_generator(int J, int Q) {
  std::vector<std::pair<double, double>> out;
  const double r_psi = std::sqrt(0.5);
  double xi = std::max(1. / (1. + std::pow(2., 3. / Q)), 0.35);
  double factor = 1. / std::pow(2., 1. / Q);
  double sigma = (1 - factor) / (1 + factor) * xi / std::sqrt(2 * std::log(1. / r_psi));
  double sigma_min = kSigma0 / std::pow(2., J);
  if (sigma <= sigma_min) {
    xi = sigma;
  } else {
    out.emplace_back(xi, sigma);
    while (sigma > (sigma_min * std::pow(2., 1. / Q))) {   // constant-Q region
      xi /= std::pow(2., 1. / Q);
      sigma /= std::pow(2., 1. / Q);
      out.emplace_back(xi, sigma);
    }
  }
  double elbow_xi = xi;                                      // constant-bandwidth region
  for (int q = 0; q < Q - 1; ++q) {
    xi -= 1. / Q * elbow_xi;
    out.emplace_back(xi, sigma_min);
  }
  return out;
}

// R3: j = max(0, floor(-log2(min(|xi| + 5 sigma, 1/2))) - 1)
static int dyadic_scale(double xi, double sigma) {
  double v = std::min(std::fabs(xi) + 5 * sigma, 0.5);
  int j = (int)std::floor(-std::log2(v)) - 1;
  return j < 0 ? 0 : j;
}

// sum_{q in Z} exp(-(nu + q - c)^2 / (2 s^2)), all terms that do not underflow (|.| < 40 s).
static double gauss_periodised(double nu, double c, double s) {
  double lo = std::floor(c - nu - 40 * s), hi = std::ceil(c - nu + 40 * s);
  double acc = 0;
  for (double q = lo; q <= hi; q += 1.0) {
    double t = nu + q - c;
    acc += std::exp(-t * t / (2 * s * s));
  }
  return acc;
}

static double kappa_of(double xi, double sigma) {  // R4
  return gauss_periodised(0.0, xi, sigma) / gauss_periodised(0.0, 0.0, sigma);
}

// Level-k response at nu (cycles per level-k sample). The fold-sum of the level-0 periodised
// response onto L0/2^k bins (R9) equals the periodised Morlet with xi*2^k, sigma*2^k (same kappa).
static double response_level_nu(const Filter& f, int k, double nu) {
  double sc = std::ldexp(1.0, k);
  double s = f.sigma * sc;
  if (f.phi) return gauss_periodised(nu, 0.0, s);
  return 2.0 * (gauss_periodised(nu, f.xi * sc, s) - f.kappa * gauss_periodised(nu, 0.0, s));
}

double response_at(const Filter& f, double omega) { return response_level_nu(f, 0, omega); }

void level_response(const Filter& f, int64_t L0, int k, std::vector<double>* out) {
  int64_t L = L0 >> k;
  out->resize(L);
  for (int64_t m = 0; m < L; ++m) (*out)[m] = response_level_nu(f, k, (double)m / (double)L);
}

// Support (bins where |response| may exceed `cut`, relative to the Gaussian peak) of the level-k response
// on an L-bin grid; the values are appended to *vals (float or double).
template <class V>
static Support support_of(const Filter& f, int k, int64_t L, std::vector<V>* vals, double cut = 1e-10) {
  double sc = std::ldexp(1.0, k);
  double s = f.sigma * sc, c = f.xi * sc;
  double a, b;
  if (f.phi) {
    double w = std::sqrt(2 * std::log(1.0 / cut));
    a = -w * s; b = w * s;
  } else {
    double w = std::sqrt(2 * std::log(2.0 / cut));
    a = c - w * s; b = c + w * s;
    if (2.0 / cut * f.kappa > 1.0) {
      double w2 = std::sqrt(2 * std::log(2.0 / cut * f.kappa));
      a = std::min(a, -w2 * s); b = std::max(b, w2 * s);
    }
  }
  int64_t lo = (int64_t)std::floor(a * L), hi = (int64_t)std::ceil(b * L);
  int64_t len = hi - lo + 1;
  if (len >= L) { lo = 0; len = L; }
  Support sp{lo, len, (int64_t)vals->size(), L};
  for (int64_t t = 0; t < len; ++t)
    vals->push_back((V)response_level_nu(f, k, (double)(lo + t) / (double)L));
  return sp;
}

// Closed-form (Poisson-summed) time-domain kernel of a level-k response on the L0 grid:
// h_k[n] = 2^k sum_r H(2^k n + r L0), H_psi(t) = 2 s sqrt(2 pi) e^{-2 pi^2 s^2 t^2}(e^{2 pi i xi t}
// - kappa), H_phi(t) = s sqrt(2 pi) e^{-2 pi^2 s^2 t^2}.
static void time_kernel(const Filter& f, int64_t L0, int k, int64_t n, double* re, double* im) {
  double s = f.sigma;
  double sc = std::ldexp(1.0, k);
  double reach = 1.40 / s + 2.0;
  int64_t rmax = (int64_t)std::ceil(reach / (double)L0) + 1;
  double ar = 0, ai = 0;
  for (int64_t r = -rmax; r <= rmax; ++r) {
    double t = sc * (double)n + (double)r * (double)L0;
    double e = s * std::sqrt(2 * kPi) * std::exp(-2 * kPi * kPi * s * s * t * t);
    if (e == 0.0) continue;
    if (f.phi) {
      ar += e;
    } else {
      ar += 2 * e * (std::cos(2 * kPi * f.xi * t) - f.kappa);
      ai += 2 * e * std::sin(2 * kPi * f.xi * t);
    }
  }
  *re = sc * ar;
  *im = sc * ai;
}

static int64_t next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p *= 2;
  return p;
}
static int ilog2(int64_t n) {
  int l = 0;
  while ((int64_t(1) << (l + 1)) <= n) ++l;
  return l;
}
static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
static int64_t pmod(int64_t a, int64_t m) { return ((a % m) + m) % m; }

// tf32 rounding identical to cvt.rna.tf32.f32 (nearest, ties away from zero, 13 bits dropped)
static float tf32_rna_host(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) != 0x7F800000u) u = (u + 0x1000u) & 0xFFFFE000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}
static uint32_t core_off_host(uint32_t r, uint32_t k, uint32_t Kc) {
  return (r >> 3) * (Kc * 32u) + (k >> 2) * 128u + (r & 7u) * 16u + (k & 3u) * 4u;
}

// Tensor-core images (kernels_tc.cu): for every unit of an eligible block (K <= 60, rows_out <= 8)
// and every row tile of 64 rows, B = [[Re M, -Im M], [Im M, Re M]] (interleaved) split into tf32
// hi/lo, in K-chunks of 32 in the canonical K-major layout; plus the phi_F weights per row.
static void build_tc_tables(Plan* p) {
  const int nfr = (int)p->L_fr.size();
  p->tc_units.assign(p->units.size(), TcUnit{0, 0, 0, 0, 0, 0});
  p->blk_tc.assign(p->blocks.size(), 0);
  p->blk_tcb.assign(p->blocks.size(), 0);
  p->blk_ks.assign(p->blocks.size(), 0);
  p->ks_w_floats = 0;
  p->gp_complex = 0;
  for (size_t bi = 0; bi < p->blocks.size(); ++bi) {
    const int K = p->blocks[bi].n1_max;
    const int K2 = ((2 * K + 7) / 8) * 8;
    const int N2 = ((2 * K + 15) / 16) * 16;
    int ro_max = 0;
    for (int f = 0; f < nfr; ++f) ro_max = std::max(ro_max, p->units[bi * nfr + f].rows_out);
    if (ro_max > 32 || N2 > 384) continue;                  // FFT route (kernels_frfft.cu)
    int kap = 0;
    while ((2 << kap) < ro_max) ++kap;
    // resident A tile (128 x K2 x 8 B) when it fits with >= 3 B stages, else split-K parts
    int ks = 0, nparts = 1, kpw = K2, kcw = 16;
    const int CT = (K2 <= 64 && kap <= 2) ? 2 : 1;
    // resident Y2 tile when it fits the TMEM (TS form) or two column tiles share the B stream (K2 <= 64);
    // else the tile in SMEM (SS form) while it fits (K2 <= 168); larger K goes split-K: the forward's parts
    // stay in the TS form and the backward reads the forward's W instead of recomputing GEMM1. (Measured
    // at c2: converting the K2 = 136 / 168 blocks to split-K in two parts costs more in W traffic, 24 B per
    // cell, than it saves; in one part, 16 B per cell, it is a gain: see above.)
    // "Split-K in one part" for 130 <= K2 <= 192 (A tile in TMEM, one accumulator buffer): the forward
    // stores W (8 B per modulus cell) and the backward reads it instead of recomputing GEMM1, which frees
    // its SMEM from the 128 x K2 A tile for wide B2 chunks (with the A tile resident the rings fell to
    // 8-16-wide B2 chunks: many ~400-cycle bulk copies per 32-row tile). Measured: c2 21.31 -> 20.88 ms,
    // c4 660.0 -> 649.4 ms per step. Applied while the block's W buffer stays <= 2 GB per signal (c5's
    // blocks would cut its micro-batch from 17 to 6 signals). JTFS_KS1_MIN / JTFS_KS1_MAXW: tuning.
    static const int ks1_min = [] {
      const char* e = std::getenv("JTFS_KS1_MIN");
      return e ? std::atoi(e) : 130;
    }();
    static const double ks1_maxw = [] {
      const char* e = std::getenv("JTFS_KS1_MAXW");
      return e ? std::atof(e) : 2e9;
    }();
    double w_bytes = 0;
    {
      int wpt = 0;
      for (int f = 0; f < nfr; ++f) wpt += (int)((p->units[bi * nfr + f].n_rows + 63) / 64);
      w_bytes = (double)((p->binfo[bi].n_cols + 127) / 128) * wpt * 128 * 64 * 4;   // phase store, 4 B per cell
    }
    if (K2 >= ks1_min && CT == 1 && tc_fwd_tsa(1, K2) && kap <= 4 && w_bytes <= ks1_maxw) {
      ks = 1;
      kcw = 16;
      for (int w : {64, 32, 16}) {
        if (w > K2) continue;
        if (tc_fwd_stages(1, 2 << kap, K2, w) >= 3) { kcw = w; break; }
      }
      nparts = 1;
      kpw = (K2 + kcw - 1) / kcw * kcw;
    } else if (kap <= 2 && (CT == 2 || tc_fwd_tsa(1, K2) || K2 <= 168)) {
      // widest B chunk (fewest hand-offs per tile; one chunk per tile when small) leaving >= 3 stages
      // (each bulk copy costs the copy engine ~400 cycles whatever its size: one copy per tile if possible)
      // Preferred: a width that also allows the forward's two MMA issuers (two accumulator buffers and two
      // stage rings, each >= 2 stages when a tile spans several chunks; kernels_tc.cu) -- measured at c2:
      // the second issuer hides the per-chunk barrier waits and outweighs the extra copies.
      kcw = 0;
      for (int pass = 0; pass < 2 && !kcw; ++pass)
        for (int w : {K2, 64, 32}) {
          if (w > 128 || w > K2) continue;
          const int ns = tc_fwd_stages(CT, 2 << kap, K2, w), nch = (K2 + w - 1) / w;
          const bool two = tc_fwd_nbuf(CT, K2) == 2 && (nch == 1 ? ns >= 2 : ns >= 4);
          if (ns >= 3 && (pass == 1 || two)) { kcw = w; break; }
        }
      if (!kcw) kcw = 16;
    } else {
      ks = 1;
      // fewest balanced K parts whose A tile fits TMEM (TS-form MMAs), each part m whole chunks with the
      // fewest chunks (m) that leave >= 3 stages
      int best_np = 0, best_w = 16;
      for (int np = 2; np <= 8 && !best_np; ++np) {
        const int kp0 = ((K2 + np - 1) / np + 7) / 8 * 8;
        for (int m = 1; m <= 4; ++m) {
          const int w = ((kp0 + m - 1) / m + 7) / 8 * 8;
          const int ns = tc_fwd_stages(1, 2 << kap, m * w, w);
          if (tc_fwd_tsa(1, m * w) && tc_fwd_nbuf(1, m * w) == 2 && ns >= 3 &&
              (np - 1) * m * w < K2) {
            best_np = np;
            best_w = w;
            break;
          }
        }
      }
      if (!best_np) { best_np = (K2 + 127) / 128; best_w = 16; }
      nparts = best_np;
      kcw = best_w;
      kpw = ((K2 + nparts - 1) / nparts + kcw - 1) / kcw * kcw;
    }
    // Hybrid one-part forward instead of K parts (kernels_tc.cu): A_hi in TMEM beside one or two
    // accumulators (128 + K2 <= 512), A_lo in SMEM, so the forward keeps only the phase store (4 B per cell)
    // instead of fp32 W partials (24-40 B per cell over 2-3 parts). B chunks of >= 24 k' keep the copy
    // engine (~400 cycles per bulk copy) below the MMA time (24 cycles per k' of a 64-row tile); widest chunk
    // with >= 3 stages, else >= 2. JTFS_HYB=0: off (A/B timing).
    static const bool hyb_on = [] {
      const char* e = std::getenv("JTFS_HYB");
      return !(e && std::atoi(e) == 0);
    }();
    int hyb = 0;
    if (hyb_on && ks && nparts > 1 && CT == 1 && 128 + K2 <= 512 && w_bytes <= ks1_maxw) {
      int wbest = 0;
      for (int need = 3; need >= 2 && !wbest; --need)
        for (int w = 64; w >= 24; w -= 8)
          if (w <= K2 && tc_fwd_stages(1, 2 << kap, K2, w, true) >= need) { wbest = w; break; }
      if (wbest) {
        hyb = 1;
        nparts = 1;
        kcw = wbest;
        kpw = K2;
      }
    }
    p->blk_tc[bi] = 1;
    p->blk_ks[bi] = (char)ks;
    // backward chunk widths: GEMM1 images (kcwb, own layout) and B2 images (kb2), chosen for the fewest bulk
    // copies per 32-row tile (each costs the copy engine ~400 cycles) with ring 1 >= 2 stages and ring 2
    // holding >= 2 tiles; split-K blocks have no GEMM1
    int kb2 = 8, kcwb = kcw, best = 1 << 30, best_depth = 0;
    for (int wb : {K2, 64, 32, 16}) {
      if (wb > 128 || wb > K2 || wb % 8) continue;
      for (int w : {64, 32, 16, 8}) {
        int ns1, s1, ns2, s2;
        tc_bwd_rings(K, ks ? 0 : K2, wb, w, &ns1, &s1, &ns2, &s2);
        const bool ok = ks ? ns2 >= 2 : (ns1 >= 2 && ns2 >= 2);
        if (!ok) continue;
        // copies per tile, plus a penalty when ring 2 holds less than two tiles of lookahead
        const int cost = (ks ? 0 : (K2 + wb - 1) / wb) + 64 / w + (ns2 * w < 128 ? 2 : 0);
        if (cost < best || (cost == best && ns2 * w > best_depth)) { best = cost; best_depth = ns2 * w; kb2 = w; kcwb = wb; }
      }
      if (ks) break;
    }
    int wp_tiles = 0;
    for (int f = 0; f < nfr; ++f) wp_tiles += (int)((p->units[bi * nfr + f].n_rows + 63) / 64);
    const int64_t n_ct = (p->binfo[bi].n_cols + 127) / 128;
    const int64_t wp_off = ks ? p->ks_w_floats : 0;
    // per 64-row tile: fp32 complex W partials (64 KB) for multi-part blocks; one-part blocks only ever hold
    // the kept phase (2 x int16 per cell, 32 KB)
    const int wph = nparts > 1 ? 4096 : 2048;
    if (ks) p->ks_w_floats += n_ct * wp_tiles * 128 * (nparts > 1 ? 128 : 64);
    // launches with few column tiles split the filters over CTA groups: about two waves of 148 SMs for a
    // batch of kRefBatch signals. Fixed per plan (not per call), so every summation order and hence every
    // bit of a signal's result is independent of the batch / micro-batch it is computed in.
    constexpr int64_t kRefBatch = 8;
    const int64_t n_tiles = (p->binfo[bi].n_cols + 128 * CT - 1) / (128 * CT);
    const int ngmax =
        (int)std::min<int64_t>(nfr, std::max<int64_t>(1, (296 + n_tiles * kRefBatch - 1) / (n_tiles * kRefBatch)));
    p->tc_blocks.push_back({(int32_t)bi, K, K2, 8 * (CT == 2 ? 0 : 1) + kap, kcw, kb2, ks, nparts, kpw, wp_tiles,
                            wp_off, ngmax, wph, 0, hyb, 0});
    int ns1, s1, ns2, s2;
    tc_bwd_rings(K, ks ? 0 : K2, kcwb, kb2, &ns1, &s1, &ns2, &s2);
    const bool bwd = best < (1 << 30) && (ks ? ns2 >= 2 : (N2 <= 256 && ns1 >= 2 && ns2 >= 2));
    if (std::getenv("JTFS_PLAN_DUMP")) {   // tuning aid: one line per tensor-core block
      int64_t rows = 0, prow = 0, prow32 = 0;
      for (int f = 0; f < nfr; ++f) {
        rows += p->units[bi * nfr + f].n_rows;
        prow += (p->units[bi * nfr + f].n_rows + 63) / 64 * 64;
        prow32 += (p->units[bi * nfr + f].n_rows + 31) / 32 * 32;
      }
      const int kw = ks ? kpw : K2;
      std::fprintf(stderr,
                   "tc block %zu: K=%d K2=%d CT=%d KAP=%d ks=%d hyb=%d parts=%d kpw=%d kcw=%d fwdNS=%d nch=%d | bwd=%d kcwb=%d "
                   "kb2=%d ns1=%d ns2=%d | cols=%lld rows=%lld pad64=%lld pad32=%lld units=%d ng=%d\n",
                   (size_t)bi, K, K2, CT, 2 << kap, ks, hyb, nparts, kpw, kcw, tc_fwd_stages(CT, 2 << kap, kw, kcw, hyb != 0),
                   (kw + kcw - 1) / kcw, (int)bwd, kcwb, kb2, ns1, ns2, (long long)p->binfo[bi].n_cols,
                   (long long)rows, (long long)prow, (long long)prow32, nfr, ngmax);
    }
    if (bwd) {
      p->blk_tcb[bi] = 1;
      const int ngb =
          (int)std::min<int64_t>(nfr, std::max<int64_t>(1, (296 + n_ct * kRefBatch - 1) / (n_ct * kRefBatch)));
      p->tcb_blocks.push_back({(int32_t)bi, K, K2, kap, kcwb, kb2, ks, nparts, kpw, wp_tiles, wp_off, ngb, wph,
                               ngb > 1 ? p->gp_complex : 0});
      if (ngb > 1) p->gp_complex += (int64_t)ngb * K * p->binfo[bi].n_cols;
    }
    int tile0 = 0;
    for (int f = 0; f < nfr; ++f) {
      const int u = (int)bi * nfr + f;
      const JointUnit& U = p->units[u];
      TcUnit tu{};
      tu.NT = (int32_t)((U.n_rows + 63) / 64);
      tu.wp_tile0 = tile0;
      tile0 += tu.NT;
      tu.img_off = (int64_t)p->tc_img.size();
      tu.wt_off = (int64_t)p->tc_wts.size();
      const double* h = p->hfr_d.data() + (size_t)U.f * p->P * 2;
      auto Mval = [&](int64_t lr, int n, double* mr, double* mi) {
        const int64_t r = (U.r_lo + lr) % U.Lf;
        const int64_t e = (((r << U.kf) - n) % p->P + p->P) % p->P;
        *mr = h[2 * e];
        *mi = h[2 * e + 1];
      };
      auto put = [&](std::vector<float>& img, size_t hi_base, size_t lo_base, uint32_t o, double v) {
        const float xf = (float)v;
        const float hi = tf32_rna_host(xf);
        img[hi_base + o] = hi;
        img[lo_base + o] = tf32_rna_host(xf - hi);
      };
      // forward images: per 64-row tile, per kcw-wide chunk: [hi 128 x kc | lo 128 x kc]
      for (int t = 0; t < tu.NT; ++t) {
        for (int ch = 0; ch * kcw < K2; ++ch) {
          const int kc = std::min(kcw, K2 - ch * kcw);
          const size_t base = p->tc_img.size();
          p->tc_img.resize(base + 2 * 128 * kc, 0.f);
          for (int nn = 0; nn < 128; ++nn) {
            const int i = nn / 2, po = nn % 2;
            const int64_t lr = (int64_t)t * 64 + i;
            if (lr >= U.n_rows) continue;
            for (int kl = 0; kl < kc; ++kl) {
              const int kk = ch * kcw + kl, n = kk / 2, pi = kk % 2;
              if (n >= K) continue;
              double mr, mi;
              Mval(lr, n, &mr, &mi);
              // Re W = Re M Re Y - Im M Im Y ; Im W = Im M Re Y + Re M Im Y
              const double v = (po == 0) ? ((pi == 0) ? mr : -mi) : ((pi == 0) ? mi : mr);
              put(p->tc_img, base, base + 128 * kc, core_off_host((uint32_t)nn, (uint32_t)kl, (uint32_t)kc) / 4, v);
            }
          }
        }
      }
      // backward GEMM1 images: per 32-row tile, per kcw-wide chunk: [hi 64 x kc | lo 64 x kc] (the forward
      // image rows of that half tile, contiguous so one bulk copy moves a chunk)
      if (bwd && !ks) {
        tu.img1b_off = (int64_t)p->tc_img1b.size();
        const int NT32 = (int)((U.n_rows + 31) / 32);
        for (int t = 0; t < NT32; ++t) {
          for (int ch = 0; ch * kcwb < K2; ++ch) {
            const int kc = std::min(kcwb, K2 - ch * kcwb);
            const size_t base = p->tc_img1b.size();
            p->tc_img1b.resize(base + 2 * 64 * kc, 0.f);
            for (int nn = 0; nn < 64; ++nn) {
              const int i = nn / 2, po = nn % 2;
              const int64_t lr = (int64_t)t * 32 + i;
              if (lr >= U.n_rows) continue;
              for (int kl = 0; kl < kc; ++kl) {
                const int kk = ch * kcwb + kl, n = kk / 2, pi = kk % 2;
                if (n >= K) continue;
                double mr, mi;
                Mval(lr, n, &mr, &mi);
                const double v = (po == 0) ? ((pi == 0) ? mr : -mi) : ((pi == 0) ? mi : mr);
                put(p->tc_img1b, base, base + 64 * kc, core_off_host((uint32_t)nn, (uint32_t)kl, (uint32_t)kc) / 4, v);
              }
            }
          }
        }
      }
      // backward B2 images: per 32-row tile, per kb2-wide kk chunk: [hi N2 x kb2 | lo N2 x kb2]
      // B2[2n][2i] = Re M, B2[2n][2i+1] = Im M, B2[2n+1][2i] = -Im M, B2[2n+1][2i+1] = Re M
      if (bwd) {
        tu.img2_off = (int64_t)p->tc_img2.size();
        const int NT32 = (int)((U.n_rows + 31) / 32);
        for (int t = 0; t < NT32; ++t) {
          for (int ch = 0; ch < 64 / kb2; ++ch) {
            const size_t base = p->tc_img2.size();
            p->tc_img2.resize(base + 2 * (size_t)N2 * kb2, 0.f);
            for (int nn = 0; nn < N2; ++nn) {
              const int n = nn / 2, po = nn % 2;
              if (n >= K) continue;
              for (int kl = 0; kl < kb2; ++kl) {
                const int kk = ch * kb2 + kl, i = kk / 2, pi = kk % 2;
                const int64_t lr = (int64_t)t * 32 + i;
                if (lr >= U.n_rows) continue;
                double mr, mi;
                Mval(lr, n, &mr, &mi);
                // Re g_Y = Re M Re g_W + Im M Im g_W ; Im g_Y = -Im M Re g_W + Re M Im g_W
                const double v = (po == 0) ? ((pi == 0) ? mr : mi) : ((pi == 0) ? -mi : mr);
                put(p->tc_img2, base, base + (size_t)N2 * kb2,
                    core_off_host((uint32_t)nn, (uint32_t)kl, (uint32_t)kb2) / 4, v);
              }
            }
          }
        }
      }
      // phi_F weights g_kf[(rho 2^d - r) mod L_f] per (rho, local row), 0 beyond n_rows
      const float* g = p->phiF_k.data() + p->phiF_off[U.kf];
      for (int rho = 0; rho < U.rows_out; ++rho)
        for (int64_t lr = 0; lr < (int64_t)tu.NT * 64; ++lr) {
          float w = 0.f;
          if (lr < U.n_rows) {
            const int64_t r = (U.r_lo + lr) % U.Lf;
            w = g[((((int64_t)rho << U.d) - r) % U.Lf + U.Lf) % U.Lf];
          }
          p->tc_wts.push_back(w);
        }
      p->tc_units[u] = tu;
    }
  }
}

int make_plan(int64_t N, int J, int Q, int J_fr, int Q_fr, int64_t T, int64_t F, Plan* p,
              std::string* err, int Q2) {
  auto ispow2 = [](int64_t v) { return v >= 1 && (v & (v - 1)) == 0; };
  if (J < 1 || Q < 1 || J_fr < 1 || Q_fr < 1) { *err = "J, Q, J_fr, Q_fr must be >= 1"; return 1; }
  if (!ispow2(T)) { *err = "T must be a power of two"; return 1; }
  if (!ispow2(F)) { *err = "F must be a power of two"; return 1; }
  int log2T = ilog2(T), log2F = ilog2(F);
  if (!(1 <= log2T && log2T <= J)) { *err = "need 1 <= log2(T) <= J"; return 1; }
  if (!(0 <= log2F && log2F <= J_fr)) { *err = "need 0 <= log2(F) <= J_fr"; return 1; }
  if (N < T || N % T != 0) { *err = "N must be a positive multiple of T"; return 1; }
  if (J > 24 || J_fr > 16 || Q > 64 || Q_fr > 16) { *err = "J <= 24, J_fr <= 16, Q <= 64, Q_fr <= 16"; return 1; }
  if (Q2 < 1 || Q2 > 16) { *err = "need 1 <= Q2 <= 16"; return 1; }

  p->N = N; p->J = J; p->Q = Q; p->J_fr = J_fr; p->Q_fr = Q_fr; p->T = T; p->F = F;
  p->log2T = log2T; p->log2F = log2F;
  auto mk = [](double xi, double s) {
    Filter f; f.xi = xi; f.sigma = s; f.j = dyadic_scale(xi, s); f.kappa = kappa_of(xi, s);
    return f;
  };
  for (auto& q : anden_generator(J, Q)) p->psi1.push_back(mk(q.first, q.second));
  // second-layer temporal filterbank: Q^{tm,2} (R7: Q2 = 1 by default)
  for (auto& q : anden_generator(J, Q2)) p->psi2.push_back(mk(q.first, q.second));
  p->Q2 = Q2;
  for (auto& q : anden_generator(J_fr, Q_fr)) p->psi_fr_plus.push_back(mk(q.first, q.second));
  p->phiT.phi = true; p->phiT.sigma = kSigma0 / (double)T; p->phiT.j = log2T; p->phiT.spin = 0;
  p->phiF.phi = true; p->phiF.sigma = kSigma0 / (double)F; p->phiF.j = log2F; p->phiF.spin = 0;
  p->L_fr.push_back(p->phiF);                                                     // R12
  for (auto f : p->psi_fr_plus) { f.spin = 1; p->L_fr.push_back(f); }
  for (auto f : p->psi_fr_plus) { f.xi = -f.xi; f.spin = -1; p->L_fr.push_back(f); }
  const int N1 = (int)p->psi1.size();
  if (N1 < 1) { *err = "empty first-layer filterbank"; return 1; }

  // R10
  p->N_pad = next_pow2(N + 2 * (int64_t)std::ceil(4.0 * (double)std::max<int64_t>(int64_t(1) << J, T) /
                                                  (0.2 * kPi)));
  if (p->N_pad > (int64_t(1) << 22)) { *err = "N_pad exceeds 2^22"; return 1; }
  p->pad_left = T * ((p->N_pad - N) / (2 * T));
  // R11
  double sfr = p->phiF.sigma;
  for (auto& f : p->psi_fr_plus) sfr = std::min(sfr, f.sigma);
  p->P = next_pow2(N1 + 2 * (int64_t)std::ceil(4.0 / (2 * kPi * sfr)));
  p->frames = N / T;
  p->Ft = p->N_pad / T;
  for (int i = 0; i + 1 < N1; ++i)
    if (p->psi1[i].j > p->psi1[i + 1].j) { *err = "internal: j1 not nondecreasing"; return 1; }
  // kept rows per path: up to 32 on the tensor-core / CUDA-core joint kernels; up to 64 on the FFT route of
  // the joint stage (kernels_frfft.cu, P <= 1024), which route_of picks for blocks beyond 32 rows
  if (ceil_div(N1, F) > 64 || (ceil_div(N1, F) > 32 && p->P > 1024)) {
    *err = "ceil(N1/F) must be <= 32, or <= 64 with P <= 1024 (GPU kernel limit)";
    return 1;
  }
  for (int n2 = 0; n2 < (int)p->psi2.size(); ++n2) {
    int j2 = p->psi2[n2].j, n1_max = 0;
    for (auto& f : p->psi1) n1_max += (j2 > f.j);
    if (n1_max > 0) p->blocks.push_back({n2, n1_max, std::min(j2, log2T), j2});
  }

  // ---- path table (R15, R16)
  int64_t off = 0;
  auto add = [&](int order, int n2, int nfr, int spin, int j2, int jfr, int rows) {
    jtfs_path_t q;
    q.order = order; q.n2 = n2; q.n_fr = nfr; q.spin = spin; q.j2 = j2; q.j_fr = jfr;
    q.rows = rows; q.frames = (int32_t)p->frames; q.offset = off;
    p->paths.push_back(q);
    off += (int64_t)rows * p->frames;
  };
  add(0, -1, -1, 0, -1, -1, 1);
  const int nfr1 = 1 + (int)p->psi_fr_plus.size();
  int rows1 = (int)ceil_div(N1, F);
  for (int f = 0; f < nfr1; ++f) add(1, -1, f, p->L_fr[f].spin, -1, p->L_fr[f].j, rows1);
  for (auto& b : p->blocks)
    for (int f = 0; f < (int)p->L_fr.size(); ++f)
      add(2, b.n2, f, p->L_fr[f].spin, b.j2, p->L_fr[f].j, (int)ceil_div(b.n1_max, F));
  p->n_coef = off;

  // ---- layer-1 layout
  p->L1.resize(N1); p->L1_off.resize(N1);
  int64_t s = 0;
  for (int n1 = 0; n1 < N1; ++n1) {
    int k1 = std::min(p->psi1[n1].j, log2T);
    p->L1[n1] = p->N_pad >> k1; p->L1_off[n1] = s; s += p->L1[n1];
  }
  p->sumL1 = s;
  for (int n1 = 0; n1 < N1;) {
    int n = n1;
    while (n < N1 && p->L1[n] == p->L1[n1]) ++n;
    p->l1_groups.push_back({p->L1_off[n1], n - n1, p->L1[n1]});
    // pair-packed U1 rows, compact: group after group, ceil(count / 2) rows of L (complex128 elements)
    p->l1_pgroups.push_back({p->u1p_size, (n - n1 + 1) / 2, p->L1[n1]});
    p->u1p_size += (int64_t)((n - n1 + 1) / 2) * p->L1[n1];
    if (p->l1_groups.size() > 24) { *err = "more than 24 first-layer levels"; return 1; }   // PackGroups
    n1 = n;
  }

  // ---- spectra (support-limited; threshold 1e-10 absolute, DESIGN R26)
  std::vector<float>& V = p->spec_vals;
  for (int n1 = 0; n1 < N1; ++n1) p->psi1_sup.push_back(support_of(p->psi1[n1], 0, p->N_pad, &V));
  // the forward first layer (float64) uses float64 psi1 spectra cut at 1e-17 of the peak: its
  // rounding floor must sit below the R22 dead zone (1e-12 RMS) so that the phase Z1/|Z1| of every
  // cell outside the dead zone is computed, not noise (R22)
  for (int n1 = 0; n1 < N1; ++n1)
    p->psi1_sup_d.push_back(support_of(p->psi1[n1], 0, p->N_pad, &p->spec_vals_d, 1e-17));
  for (int k = 0; k <= log2T; ++k) p->phiT_sup.push_back(support_of(p->phiT, k, p->N_pad >> k, &V));
  p->psi2_sup.assign(p->blocks.size() * (log2T + 1), Support{0, 0, 0, 0});
  for (size_t bi = 0; bi < p->blocks.size(); ++bi) {
    auto& b = p->blocks[bi];
    for (int k = 0; k <= std::min(b.j2 - 1, log2T); ++k)
      p->psi2_sup[bi * (log2T + 1) + k] = support_of(p->psi2[b.n2], k, p->N_pad >> k, &V);
  }

  // colored-noise initialisation tables (reading R25): band energies and the partition denominator
  {
    const int64_t half = p->N_pad / 2;
    std::vector<double> den(half + 1, 0.0);
    p->cn_nu.assign(N1, 0.0);
    for (int n1 = 0; n1 < N1; ++n1) {
      double nu = 0.0;
      for (int64_t m = 0; m < p->N_pad; ++m) {
        const double h = response_level_nu(p->psi1[n1], 0, (double)m / (double)p->N_pad);
        nu += h * h;
        if (m <= half) den[m] += h * h;
      }
      p->cn_nu[n1] = nu / (double)p->N_pad;
    }
    double mx = 0.0;
    for (double v : den) mx = std::max(mx, v);
    p->cn_den.resize(half + 1);
    for (int64_t m = 0; m <= half; ++m) p->cn_den[m] = (float)(den[m] + 1e-3 * mx);
  }
  // gather jobs: layer 1, S0, S1 time part, layer 2
  for (int n1 = 0; n1 < N1; ++n1) {
    auto& sp = p->psi1_sup_d[n1];
    int k1 = std::min(p->psi1[n1].j, log2T);
    p->l1_jobs.push_back({0, p->N_pad, sp.lo, sp.len, sp.off, p->L1_off[n1], p->L1[n1],
                          (float)std::ldexp(1.0, -k1), -1, -1, 0});
  }
  {
    auto& sp = p->phiT_sup[0];
    p->s0_job = {0, p->N_pad, sp.lo, sp.len, sp.off, 0, p->Ft, (float)std::ldexp(1.0, -log2T), -1, -1, 0};
  }
  // U1_hat rows are pair-packed (l1_pgroups): row n1 of a level group lives in packed row (n1 - first) / 2
  // of the group, parity (n1 - first) & 1
  std::vector<int64_t> u1_in(N1);
  std::vector<int32_t> u1_par(N1);
  for (size_t gi = 0; gi < p->l1_groups.size(); ++gi) {
    const FftGroup& g = p->l1_groups[gi];
    for (int64_t r = 0; r < g.count; ++r) {
      int n1 = -1;
      for (int q = 0; q < N1; ++q) if (p->L1_off[q] == g.off + r * g.L) n1 = q;
      u1_in[n1] = p->l1_pgroups[gi].off + (r / 2) * g.L;   // complex128 elements of the packed spectra
      u1_par[n1] = (int32_t)(r & 1);
    }
  }
  for (int n1 = 0; n1 < N1; ++n1) {
    int k1 = std::min(p->psi1[n1].j, log2T);
    auto& sp = p->phiT_sup[k1];
    p->s1_jobs.push_back({u1_in[n1], p->L1[n1], sp.lo, sp.len, sp.off, (int64_t)n1 * p->Ft, p->Ft,
                          (float)std::ldexp(1.0, -(log2T - k1)), -1, u1_par[n1], 0});
  }
  int64_t yoff = 0;
  for (size_t bi = 0; bi < p->blocks.size(); ++bi) {
    auto& b = p->blocks[bi];
    BlockInfo bf{};
    bf.y_off = yoff; bf.T2 = p->N_pad >> b.s2; bf.s2 = b.s2; bf.D = 1 << (log2T - b.s2);
    for (int n1 = 0; n1 < b.n1_max; ++n1) {
      int k1 = std::min(p->psi1[n1].j, log2T);
      auto& sp = p->psi2_sup[bi * (log2T + 1) + k1];
      p->l2_jobs.push_back({u1_in[n1], p->L1[n1], sp.lo, sp.len, sp.off, yoff + n1 * bf.T2, bf.T2,
                            (float)std::ldexp(1.0, -(b.s2 - k1)), (int32_t)bi, u1_par[n1],
                            bf.T2 > 4096 ? 1 : 0});
    }
    p->y2_groups.push_back({yoff, b.n1_max, bf.T2});
    yoff += (int64_t)b.n1_max * bf.T2;
    p->binfo.push_back(bf);
  }
  p->sumY2 = yoff;
  // k_adj_gather_u1 stages the per-block supports of one filter in SMEM (kMaxB = 32); J <= 24 keeps the
  // block count at most 25
  if (p->binfo.size() > 32) { *err = "more than 32 second-order blocks"; return 1; }

  // ---- frequential row kernels h_f on the P grid (closed form, complex) for all of L_fr
  const int nfr = (int)p->L_fr.size();
  p->hfr.resize((size_t)nfr * p->P * 2);
  for (int f = 0; f < nfr; ++f)
    for (int64_t n = 0; n < p->P; ++n) {
      double re, im;
      time_kernel(p->L_fr[f], p->P, 0, n, &re, &im);
      p->hfr[((size_t)f * p->P + n) * 2] = (float)re;
      p->hfr[((size_t)f * p->P + n) * 2 + 1] = (float)im;
      p->hfr_d.push_back(re);
      p->hfr_d.push_back(im);
    }
  // support half-widths of h_f on the circle (|h| >= 1e-9 max|h|, R26): row loops skip the rest
  for (int f = 0; f < nfr; ++f) {
    const double* h = p->hfr_d.data() + (size_t)f * p->P * 2;
    double mx = 0;
    for (int64_t n = 0; n < p->P; ++n) mx = std::max(mx, std::hypot(h[2 * n], h[2 * n + 1]));
    int64_t H = 0;
    for (int64_t n = 0; n <= p->P / 2; ++n) {
      const int64_t m = (p->P - n) % p->P;
      if (std::hypot(h[2 * n], h[2 * n + 1]) >= 1e-9 * mx || std::hypot(h[2 * m], h[2 * m + 1]) >= 1e-9 * mx) H = n;
    }
    p->hfr_H.push_back((int32_t)H);
  }
  // phi_F kernels at levels k = 0..log2F on P>>k grids; truncation half-widths (1e-9 rel)
  std::vector<int64_t> HF(log2F + 1);
  for (int k = 0; k <= log2F; ++k) {
    int64_t L = p->P >> k;
    p->phiF_off.push_back((int64_t)p->phiF_k.size());
    double mx = 0;
    std::vector<double> g(L);
    for (int64_t n = 0; n < L; ++n) {
      double re, im;
      time_kernel(p->phiF, p->P, k, n, &re, &im);
      g[n] = re; mx = std::max(mx, std::fabs(re));
    }
    int64_t H = 0;
    for (int64_t n = 0; n <= L / 2; ++n)
      if (std::fabs(g[n]) >= 1e-9 * mx) H = n;
    HF[k] = H;
    for (int64_t n = 0; n < L; ++n) p->phiF_k.push_back((float)g[n]);
  }
  // phi_T half kernels at levels s = 0..log2T (grid N_pad>>s), truncated at 1e-9 relative
  for (int sl = 0; sl <= log2T; ++sl) {
    int64_t L = p->N_pad >> sl;
    std::vector<double> t;
    double mx = 0;
    for (int64_t n = 0; n <= L / 2; ++n) {
      double re, im;
      time_kernel(p->phiT, p->N_pad, sl, n, &re, &im);
      t.push_back(re); mx = std::max(mx, std::fabs(re));
    }
    int64_t H = 0;
    for (int64_t n = 0; n <= L / 2; ++n)
      if (std::fabs(t[n]) >= 1e-9 * mx) H = n;
    p->phiT_off.push_back((int64_t)p->phiT_half.size());
    p->phiT_H.push_back(H);
    p->phiT_L.push_back(L);
    for (int64_t n = 0; n <= H; ++n) p->phiT_half.push_back((float)t[n]);
  }
  // needed columns per block (exact halo pruning, R26): kept frames at m*D, reach H_s
  int64_t m0 = p->pad_left / T;
  for (auto& bf : p->binfo) {
    int64_t H = p->phiT_H[bf.s2];
    int64_t a = m0 * bf.D - H, b = (m0 + p->frames - 1) * bf.D + H;
    if (b - a + 1 >= bf.T2) { bf.c_lo = 0; bf.n_cols = bf.T2; }
    else { bf.c_lo = pmod(a, bf.T2); bf.n_cols = b - a + 1; }
  }
  // order-2 units in path order; needed rows per unit
  int64_t ooff = 0;
  int path = 1 + nfr1;
  for (size_t bi = 0; bi < p->blocks.size(); ++bi) {
    auto& b = p->blocks[bi];
    for (int f = 0; f < nfr; ++f, ++path) {
      JointUnit u{};
      u.bi = (int)bi; u.f = f; u.kf = std::min(p->L_fr[f].j, log2F); u.d = log2F - u.kf;
      u.n1_max = b.n1_max; u.rows_out = (int)ceil_div(b.n1_max, F);
      u.Lf = p->P >> u.kf;
      int64_t H = HF[u.kf];
      int64_t a = -H, c = (int64_t)(u.rows_out - 1) * (int64_t(1) << u.d) + H;
      if (c - a + 1 >= u.Lf) { u.r_lo = 0; u.n_rows = u.Lf; }
      else { u.r_lo = pmod(a, u.Lf); u.n_rows = c - a + 1; }
      u.o_off = ooff; u.path = path;
      ooff += (int64_t)u.rows_out * p->binfo[bi].n_cols;
      p->units.push_back(u);
    }
  }
  p->o_size = ooff;
  // phi_T adjoint as banded GEMMs over the halo-pruned (unwrapped) blocks: 32-row groups of (unit, rho)
  // rows, 256-column tiles (kernels_fr.cu k_phiT_adj3)
  {
    const int nfr_all = (int)p->L_fr.size();
    for (size_t bi = 0; bi < p->blocks.size(); ++bi) {
      const BlockInfo& bf = p->binfo[bi];
      if (bf.n_cols >= bf.T2) continue;               // whole circle: per-row kernels (k_phiT_fwd2/adj2)
      p->ph3_mask |= 1ull << bi;
      std::vector<int32_t> rows;
      for (int f = 0; f < nfr_all; ++f) {
        const int u = (int)bi * nfr_all + f;
        for (int rho = 0; rho < p->units[u].rows_out; ++rho) { rows.push_back(u); rows.push_back(rho); }
      }
      const int nrows = (int)(rows.size() / 2);
      for (int r0 = 0; r0 < nrows; r0 += 32) {
        const int gi = (int)(p->ph3_groups.size() / 8);
        const int first = (int)(p->ph3_rows.size() / 2);
        for (int r = r0; r < std::min(nrows, r0 + 32); ++r) {
          p->ph3_rows.push_back(rows[2 * r]);
          p->ph3_rows.push_back(rows[2 * r + 1]);
        }
        p->ph3_groups.insert(p->ph3_groups.end(), {first, std::min(32, nrows - r0), (int32_t)bi, 0, 0, 0, 0, 0});
        for (int64_t t = 0; t < (bf.n_cols + 255) / 256; ++t) {
          p->ph3_atiles.push_back(gi);
          p->ph3_atiles.push_back((int32_t)t);
        }
      }
    }
  }
  // path-shard cost model (LPT, jtfs_api.cu block_owner): per block, the joint stage's contraction flops
  // (8 K forward + 16 K backward per modulus cell) plus its time-axis FFTs (5 L log2 L forward and
  // backward per Y2 row); order 1 (shard 0) as its row sums over the needed frames
  p->block_cost.assign(p->blocks.size(), 0.0);
  for (auto& u : p->units)
    p->block_cost[u.bi] += 24.0 * u.n1_max * (double)u.n_rows * (double)p->binfo[u.bi].n_cols;
  for (size_t bi = 0; bi < p->blocks.size(); ++bi) {
    const double T2 = (double)p->binfo[bi].T2;
    p->block_cost[bi] += 10.0 * p->blocks[bi].n1_max * T2 * std::log2(T2);
  }
  p->order1_cost = 8.0 * N1 * (double)p->Ft * (double)nfr1 * 64.0;
  // order-1 needed rows
  p->o1_rows_out = rows1;
  for (int f = 0; f < nfr1; ++f) {
    int kf = std::min(p->L_fr[f].j, log2F), d = log2F - kf;
    int64_t Lf = p->P >> kf, H = HF[kf];
    int64_t a = -H, c = (int64_t)(rows1 - 1) * (int64_t(1) << d) + H;
    if (f == 0) { a = 0; c = rows1 - 1; }   // phi_F path keeps rows directly (no modulus)
    if (c - a + 1 >= Lf) { p->o1_rlo.push_back(0); p->o1_nrows.push_back(Lf); }
    else { p->o1_rlo.push_back(pmod(a, Lf)); p->o1_nrows.push_back(c - a + 1); }
  }
  build_tc_tables(p);
  // FFT route (kernels_frfft.cu): level-0 responses of every frequential filter on the P grid
  // (R4 periodised Morlet / Gaussian, the same response whose inverse DFT is h_f) and per-unit phi_F
  // weights g_kf[(rho 2^d - r) mod L_f] over the unit's needed rows
  {
    std::vector<double> resp;
    for (int f = 0; f < nfr; ++f) {
      level_response(p->L_fr[f], p->P, 0, &resp);
      for (int64_t m = 0; m < p->P; ++m) p->fr_spec.push_back((float)resp[m]);
    }
    for (auto& U : p->units) {
      p->u_wt_off.push_back((int64_t)p->u_wts.size());
      const float* g = p->phiF_k.data() + p->phiF_off[U.kf];
      for (int rho = 0; rho < U.rows_out; ++rho)
        for (int64_t i = 0; i < U.n_rows; ++i) {
          const int64_t r = (U.r_lo + i) % U.Lf;
          p->u_wts.push_back(g[((((int64_t)rho << U.d) - r) % U.Lf + U.Lf) % U.Lf]);
        }
    }
  }
  // adjoint d/dx spectrum gather: CSR of n1 touching each tile of N_pad bins
  int64_t ntile = ceil_div(p->N_pad, p->gx_tile);
  p->gx_tile_start.push_back(0);
  for (int64_t t = 0; t < ntile; ++t) {
    int64_t a = t * p->gx_tile, b = a + p->gx_tile;   // [a, b)
    for (int n1 = 0; n1 < N1; ++n1) {
      auto& sp = p->psi1_sup[n1];
      bool hit = false;
      if (sp.len >= p->N_pad) hit = true;
      else {
        int64_t lo = pmod(sp.lo, p->N_pad);
        // interval [lo, lo+len) modulo N_pad intersects [a, b)?
        for (int w = -1; w <= 1 && !hit; ++w) {
          int64_t l = lo + w * p->N_pad, h = l + sp.len;
          if (l < b && h > a) hit = true;
        }
      }
      if (hit) p->gx_list.push_back(n1);
    }
    p->gx_tile_start.push_back((int32_t)p->gx_list.size());
  }
  return 0;
}

}  // namespace jtfs
