// jtfs_api.cu — C ABI of libjtfs.so (include/jtfs.h): plan handles, device-table upload, workspace
// layout, and the stream-ordered orchestration of the forward, loss + gradient
// and metamer step.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "device.cuh"
#include "fft.cuh"

namespace jtfs {
// JTFS_TC=0 in the environment keeps the joint-stage forward on the FP32 CUDA-core kernel (A/B
// comparison in tests and profiling); both are GPU kernels of this library.
static const bool g_use_tc = [] {
  const char* e = std::getenv("JTFS_TC");
  return !(e && e[0] == '0');
}();
// Route of the joint stage per block: tensor cores (K small enough for a resident A tile), else the
// FFT route along n1 (kernels_frfft.cu). JTFS_FFT_KMIN=k also sends TC-eligible blocks with K >= k to
// the FFT route; JTFS_SIMT=1 uses the dense CUDA-core kernels instead of the FFT route (A/B tests).
static const int g_fft_kmin = [] {
  const char* e = std::getenv("JTFS_FFT_KMIN");
  return e ? std::atoi(e) : 1 << 30;
}();
static const bool g_force_simt = [] {
  const char* e = std::getenv("JTFS_SIMT");
  return e && e[0] == '1';
}();
enum Route { kRouteTc = 0, kRouteFft = 1, kRouteSimt = 2 };
// JTFS_LANES=2 runs loss_grad's micro-batches on two concurrent lanes. Measured slower at c2 (28.3 vs
// 27.2 ms/step: halving the micro-batch costs the tensor-core launches more than the overlap gains), so
// one lane is the default.
static const int g_lanes = [] {
  const char* e = std::getenv("JTFS_LANES");
  return e ? std::atoi(e) : 1;
}();
static int route_of(const Plan& p, size_t bi, bool bwd) {
  const bool tc_ok = g_use_tc && (bwd ? p.blk_tcb[bi] : p.blk_tc[bi]) && p.blocks[bi].n1_max < g_fft_kmin;
  if (tc_ok) return kRouteTc;
  const int ro = (int)((p.blocks[bi].n1_max + p.F - 1) / p.F);
  if (!g_force_simt && p.P <= kFfMaxP && ro <= kFfMaxRo) return kRouteFft;
  return kRouteSimt;
}
static std::atomic<int64_t> g_launches{0};

// Fan-out of the joint stage: the tensor-core blocks and the FFT-route blocks are independent (disjoint
// outputs), so they run on side streams forked from and joined back to the caller's stream; the tail
// of one launch overlaps the next. Streams/events are per host thread and device.
constexpr int kFanStreams = 3;
struct Fanout {
  cudaStream_t s[kFanStreams] = {};
  cudaEvent_t fork = nullptr, join[kFanStreams] = {};
};
constexpr int kMaxLanes = 2;
static Fanout* fanout_get(int lane) {
  static thread_local std::vector<Fanout*> per_dev;
  int dev = 0;
  cudaGetDevice(&dev);
  const int slot = dev * (kMaxLanes + 1) + lane;   // slots 0..kMaxLanes-1: per-lane fan-out sets; kMaxLanes: the lane streams
  if ((int)per_dev.size() <= slot) per_dev.resize(slot + 1, nullptr);
  if (!per_dev[slot]) {
    Fanout* f = new Fanout();
    for (int i = 0; i < kFanStreams; ++i) {
      cudaStreamCreateWithFlags(&f->s[i], cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&f->join[i], cudaEventDisableTiming);
    }
    cudaEventCreateWithFlags(&f->fork, cudaEventDisableTiming);
    per_dev[slot] = f;
  }
  return per_dev[slot];
}
static void fan_fork(Fanout* f, cudaStream_t st) {
  cudaEventRecord(f->fork, st);
  for (int i = 0; i < kFanStreams; ++i) cudaStreamWaitEvent(f->s[i], f->fork, 0);
}
static void fan_join(Fanout* f, cudaStream_t st) {
  for (int i = 0; i < kFanStreams; ++i) {
    cudaEventRecord(f->join[i], f->s[i]);
    cudaStreamWaitEvent(st, f->join[i], 0);
  }
}
void count_launch(int n) { g_launches += n; }

// ---- profiling hooks: events around the dominant kernels, on their launch stream
static std::atomic<int> g_prof{0};
static std::mutex g_prof_mu;
struct ProfRec { int id; cudaEvent_t a, b; };
static std::vector<ProfRec> g_prof_recs;
static thread_local cudaEvent_t t_open[8] = {};
void prof_begin(cudaStream_t st, int id) {
  if (!g_prof.load()) return;
  cudaEventCreate(&t_open[id]);
  cudaEventRecord(t_open[id], st);
}
void prof_end(cudaStream_t st, int id) {
  if (!g_prof.load() || !t_open[id]) return;
  cudaEvent_t b;
  cudaEventCreate(&b);
  cudaEventRecord(b, st);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_recs.push_back({id, t_open[id], b});
  t_open[id] = nullptr;
}
}  // namespace jtfs

using namespace jtfs;

struct jtfs_plan_s {
  Plan p;
  std::mutex mu;
};

static thread_local std::string t_err;
static jtfs_status fail(jtfs_status s, const std::string& m) {
  t_err = m;
  return s;
}
#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) return fail(JTFS_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ------------------------------------------------------------------------------ device tables
template <class T>
static cudaError_t up(const std::vector<T>& v, T** dst) {
  *dst = nullptr;
  if (v.empty()) return cudaSuccess;
  cudaError_t e = cudaMalloc(dst, v.size() * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

static std::vector<int64_t> prefix(const std::vector<int64_t>& counts) {
  std::vector<int64_t> t(counts.size() + 1, 0);
  for (size_t i = 0; i < counts.size(); ++i) t[i + 1] = t[i] + counts[i];
  return t;
}

static void free_tables(DeviceTables* d) {
  if (!d) return;
  void* ptrs[] = {d->spec_vals, d->spec_vals_d, d->cn_nu, d->cn_den, d->l1_jobs, d->l1_tiles, d->s1_jobs, d->s1_tiles, d->l2_jobs, d->l2_tiles,
                  d->s0_job, d->s0_tiles, d->psi1_sup, d->psi2_sup, d->phiT_sup, d->hfr, d->phiF_k,
                  d->phiF_off, d->phiT_half, d->phiT_off, d->phiT_H, d->units, d->binfo, d->kf_of,
                  d->blk_nmax, d->ucoef, d->uo, d->bwd_tiles, d->coef_path, d->path_off, d->path_owner_unit, d->l1_off,
                  d->n1_k1, d->u1adj_tiles, d->gx_tile_start, d->gx_list, d->o1_rlo, d->o1_nrows, d->tw, d->twd,
                  d->fr_spec, d->u_wts, d->u_wt_off, d->hfr_H, d->phT_rows_u, d->phT_tiles, d->ph3_groups, d->ph3_rows, d->ph3_atiles, d->ffw.blist, d->ffw.tiles, d->ffb.blist, d->ffb.tiles};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  for (int c = 0; c < 6; ++c) {
    if (d->fwd_ulist[c]) cudaFree(d->fwd_ulist[c]);
    if (d->fwd_tiles[c]) cudaFree(d->fwd_tiles[c]);
  }
  for (void* q : d->fs_bufs)
    if (q) cudaFree(q);
  for (auto& c : d->tc) {
    if (c.blocks) cudaFree(c.blocks);
    if (c.tiles) cudaFree(c.tiles);
  }
  if (d->tc_img) cudaFree(d->tc_img);
  if (d->tc_img2) cudaFree(d->tc_img2);
  if (d->tc_img1b) cudaFree(d->tc_img1b);
  for (auto& c : d->tcb) {
    if (c.blocks) cudaFree(c.blocks);
    if (c.tiles) cudaFree(c.tiles);
  }
  if (d->tc_wts) cudaFree(d->tc_wts);
  if (d->tc_units) cudaFree(d->tc_units);
  delete d;
}

jtfs::Plan::~Plan() { free_tables(dev); }

static cudaError_t upload(Plan& p) {
  DeviceTables* d = new DeviceTables();
  cudaError_t e;
#define UP(v, f) \
  if ((e = up(v, &d->f)) != cudaSuccess) { free_tables(d); return e; }
  UP(p.spec_vals, spec_vals);
  UP(p.spec_vals_d, spec_vals_d);
  UP(p.cn_nu, cn_nu);
  UP(p.cn_den, cn_den);
  auto job_tiles = [](const std::vector<GatherJob>& jobs) {
    std::vector<int64_t> c;
    for (auto& j : jobs) {
      const int64_t tile = j.tl ? kGatherTileT : kGatherTile;
      c.push_back((j.L_out + tile - 1) / tile);
    }
    return prefix(c);
  };
  std::vector<int64_t> t;
  UP(p.l1_jobs, l1_jobs); t = job_tiles(p.l1_jobs); UP(t, l1_tiles);
  d->n_l1 = (int)p.l1_jobs.size(); d->l1_ntiles = t.back();
  UP(p.s1_jobs, s1_jobs); t = job_tiles(p.s1_jobs); UP(t, s1_tiles);
  d->n_s1 = (int)p.s1_jobs.size(); d->s1_ntiles = t.back();
  UP(p.l2_jobs, l2_jobs); t = job_tiles(p.l2_jobs); UP(t, l2_tiles);
  d->n_l2 = (int)p.l2_jobs.size(); d->l2_ntiles = t.back();
  std::vector<GatherJob> s0{p.s0_job};
  UP(s0, s0_job); t = job_tiles(s0); UP(t, s0_tiles); d->s0_ntiles = t.back();
  UP(p.psi1_sup, psi1_sup);
  UP(p.psi2_sup, psi2_sup);
  UP(p.phiT_sup, phiT_sup);
  {
    std::vector<float2> h(p.hfr.size() / 2);
    for (size_t i = 0; i < h.size(); ++i) h[i] = make_float2(p.hfr[2 * i], p.hfr[2 * i + 1]);
    UP(h, hfr);
  }
  UP(p.phiF_k, phiF_k); UP(p.phiF_off, phiF_off);
  UP(p.phiT_half, phiT_half); UP(p.phiT_off, phiT_off); UP(p.phiT_H, phiT_H);
  UP(p.units, units); d->n_units = (int)p.units.size();
  UP(p.binfo, binfo); d->n_blocks = (int)p.binfo.size();
  // forward unit lists per KAP class
  const int kaps[6] = {1, 2, 4, 8, 16, 32};
  for (int c = 0; c < 6; ++c) {
    std::vector<int32_t> ul;
    std::vector<int64_t> cnt;
    for (size_t u = 0; u < p.units.size(); ++u) {
      int ro = p.units[u].rows_out;
      if (route_of(p, p.units[u].bi, false) != kRouteSimt) continue;   // tensor-core or FFT route
      int cls = 0;
      while (kaps[cls] < ro) ++cls;
      if (cls != c) continue;
      ul.push_back((int32_t)u);
      cnt.push_back((p.binfo[p.units[u].bi].n_cols + kJC - 1) / kJC);
      d->fwd_kmax[c] = std::max(d->fwd_kmax[c], p.units[u].n1_max);
    }
    d->fwd_n[c] = (int)ul.size();
    if (!ul.empty()) {
      t = prefix(cnt);
      UP(ul, fwd_ulist[c]);
      UP(t, fwd_tiles[c]);
      d->fwd_ntiles[c] = t.back();
    }
  }
  // tensor-core classes (forward and backward)
  UP(p.tc_img, tc_img); UP(p.tc_wts, tc_wts); UP(p.tc_units, tc_units); UP(p.tc_img2, tc_img2); UP(p.tc_img1b, tc_img1b);
  // one launch per tensor-core block: each sizes its pipeline for its own K
  auto build_classes = [&](const std::vector<TcBlock>& src, std::vector<TcClass>* out, bool fwd) -> cudaError_t {
    for (auto& tb : src) {
      if (route_of(p, tb.bi, !fwd) != kRouteTc) continue;
      TcClass c;
      const int CT = (fwd && tb.cls < 3) ? 2 : 1;
      std::vector<TcBlock> bl{tb};
      std::vector<int64_t> tt{0, (p.binfo[tb.bi].n_cols + 128 * CT - 1) / (128 * CT)};
      c.n_blocks = 1;
      c.K2max = (fwd && tb.ks) ? tb.kpw : tb.K2;
      c.ks = tb.ks;
      c.nparts = tb.nparts;
      c.hyb = fwd ? tb.hyb : 0;
      c.ngmax = tb.ngmax;
      c.n_cols = p.binfo[tb.bi].n_cols;
      c.bi = tb.bi;
      c.gp_off = tb.gp_off;
      c.Kmax = tb.K;
      c.kcw = tb.kcw;
      c.kb2 = tb.kb2;
      c.cls = tb.cls;
      c.ntiles = tt.back();
      cudaError_t e1 = up(bl, &c.blocks);
      if (e1 == cudaSuccess) e1 = up(tt, &c.tiles);
      out->push_back(c);
      if (e1 != cudaSuccess) return e1;
    }
    return cudaSuccess;
  };
  if ((e = build_classes(p.tc_blocks, &d->tc, true)) != cudaSuccess) { free_tables(d); return e; }
  if ((e = build_classes(p.tcb_blocks, &d->tcb, false)) != cudaSuccess) { free_tables(d); return e; }
  std::vector<int32_t> kf;
  for (auto& f : p.L_fr) kf.push_back(std::min(f.j, p.log2F));
  UP(kf, kf_of);
  UP(p.hfr_H, hfr_H);
  {
    std::vector<int32_t> ru, ti;   // rows (u, rho); adjoint tiles (u, rho, first column)
    for (size_t u = 0; u < p.units.size(); ++u)
      for (int rho = 0; rho < p.units[u].rows_out; ++rho) {
        ru.push_back((int32_t)u);
        ru.push_back(rho);
        for (int64_t c0 = 0; c0 < p.binfo[p.units[u].bi].n_cols; c0 += 1024)   // kernels_fr.cu kPhiTCols
          ti.insert(ti.end(), {(int32_t)u, (int32_t)rho, (int32_t)c0});
      }
    d->phT_nrows = (int)(ru.size() / 2);
    d->phT_ntiles = (int64_t)(ti.size() / 3);
    UP(ru, phT_rows_u);
    UP(ti, phT_tiles);
  }
  if (!p.ph3_groups.empty()) {
    UP(p.ph3_groups, ph3_groups); UP(p.ph3_rows, ph3_rows); UP(p.ph3_atiles, ph3_atiles);
    d->ph3_ngroups = (int)(p.ph3_groups.size() / 8);
    d->ph3_natiles = (int64_t)(p.ph3_atiles.size() / 2);
    d->ph3_mask = p.ph3_mask;
  }
  std::vector<int32_t> nm;
  std::vector<int64_t> bt;
  d->Kmax = 0;
  for (size_t bi = 0; bi < p.blocks.size(); ++bi) {
    nm.push_back(p.blocks[bi].n1_max);
    d->Kmax = std::max(d->Kmax, p.blocks[bi].n1_max);
    // CUDA-core backward: 32-column tiles over all n1 rows; blocks on the tensor-core path: none
    const bool simt = route_of(p, bi, true) == kRouteSimt;
    bt.push_back(simt ? (p.binfo[bi].n_cols + 31) / 32 : 0);
    if (simt) d->Kmax_simt_bwd = std::max(d->Kmax_simt_bwd, p.blocks[bi].n1_max);
  }
  UP(nm, blk_nmax);
  t = prefix(bt); UP(t, bwd_tiles); d->bwd_ntiles = t.back();
  const int nfr1 = 1 + (int)p.psi_fr_plus.size();
  d->o2_start = p.units.empty() ? p.n_coef : p.paths[1 + nfr1].offset;
  d->n_o2 = p.n_coef - d->o2_start;
  std::vector<int64_t> uc, uo;
  for (auto& u : p.units) { uc.push_back(p.paths[u.path].offset - d->o2_start); uo.push_back(u.o_off); }
  UP(uc, ucoef); UP(uo, uo);
  std::vector<int32_t> cp(p.n_coef), pu(p.paths.size());
  for (size_t q = 0; q < p.paths.size(); ++q) {
    auto& pa = p.paths[q];
    for (int64_t i = 0; i < (int64_t)pa.rows * pa.frames; ++i) cp[pa.offset + i] = (int32_t)q;
    pu[q] = pa.order == 0 ? -2 : (pa.order == 1 ? -1 : (int32_t)((q - 1 - nfr1) / p.L_fr.size()));   // block
  }
  UP(cp, coef_path); UP(pu, path_owner_unit);
  {
    std::vector<int64_t> po;
    for (auto& pa : p.paths) po.push_back(pa.offset);
    po.push_back(p.n_coef);
    UP(po, path_off);
  }
  UP(p.L1_off, l1_off);
  std::vector<int32_t> k1;
  std::vector<int64_t> ut;
  for (size_t n = 0; n < p.psi1.size(); ++n) {
    k1.push_back(std::min(p.psi1[n].j, p.log2T));
    ut.push_back((p.L1[n] + 1023) / 1024);   // kernels_time.cu kU1AdjTile
  }
  UP(k1, n1_k1);
  t = prefix(ut); UP(t, u1adj_tiles); d->u1adj_ntiles = t.back();
  UP(p.gx_tile_start, gx_tile_start); UP(p.gx_list, gx_list);
  UP(p.o1_rlo, o1_rlo); UP(p.o1_nrows, o1_nrows);
  std::vector<float2> tw = fft_twiddle_table();
  UP(tw, tw);
  std::vector<double2> twd = fft_twiddle_table_d();
  UP(twd, twd);
  d->fftt.tw = d->tw;
  d->fftt.twd = d->twd;
  {
    std::vector<float2> pf = fft_pass_tables();
    std::vector<double2> pd = fft_pass_tables_d();
    float2* a = nullptr;
    double2* c = nullptr;
    if ((e = up(pf, &a)) != cudaSuccess || (e = up(pd, &c)) != cudaSuccess) {
      if (a) cudaFree(a);
      free_tables(d);
      return e;
    }
    d->fs_bufs.insert(d->fs_bufs.end(), {(void*)a, (void*)c});
    d->fftt.twp = a;
    d->fftt.twpd = c;
  }
  for (int lg = 13; lg <= 22 && (int64_t(1) << lg) <= p.N_pad; ++lg) {
    std::vector<float2> tf;
    std::vector<double2> td;
    fft_fourstep_table_f(lg, &tf);
    fft_fourstep_table_d(lg, &td);
    float2* a = nullptr;
    double2* c = nullptr;
    if ((e = up(tf, &a)) != cudaSuccess || (e = up(td, &c)) != cudaSuccess) {
      free_tables(d);
      return e;
    }
    d->fs_bufs.insert(d->fs_bufs.end(), {(void*)a, (void*)c});
    d->fftt.tw2_f[lg] = a; d->fftt.tw2_d[lg] = c;
  }
  d->maxLf = (int)p.P;
  // FFT route tables and block lists
  UP(p.fr_spec, fr_spec); UP(p.u_wts, u_wts); UP(p.u_wt_off, u_wt_off);
  for (int bw = 0; bw < 2; ++bw) {
    std::vector<int32_t> bl;
    std::vector<int64_t> cnt;
    for (size_t bi = 0; bi < p.blocks.size(); ++bi)
      if (route_of(p, bi, bw == 1) == kRouteFft) {
        bl.push_back((int32_t)bi);
        cnt.push_back(joint_fft_tiles(p.binfo[bi].n_cols));
      }
    FfList& L = bw ? d->ffb : d->ffw;
    L.nb = (int)bl.size();
    if (!bl.empty()) {
      t = prefix(cnt);
      if ((e = up(bl, &L.blist)) != cudaSuccess || (e = up(t, &L.tiles)) != cudaSuccess) {
        free_tables(d);
        return e;
      }
      L.ntiles = t.back();
    }
  }
#undef UP
  p.dev = d;
  return cudaSuccess;
}

static jtfs_status ensure_device(jtfs_plan_s* h) {
  int dev = -1;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->p.dev) {
    if (h->p.dev_id != dev) return fail(JTFS_ERR_STATE, "plan was prepared on another device");
    return JTFS_OK;
  }
  CK(upload(h->p));
  h->p.dev_id = dev;
  return JTFS_OK;
}

// ------------------------------------------------------------------------------ workspace layout
struct Layout {
  // per-signal sizes in bytes (each 256-aligned) of every buffer, in this order
  size_t xp, Xh, A, Z1, U1h, Y2, cs, ct, S1t, W1, V2, o, S, r, gS1t, g, loss, thr, Wk, gp;
  size_t per_signal() const {
    return xp + Xh + A + Z1 + U1h + Y2 + cs + ct + S1t + W1 + V2 + o + S + r + gS1t + g + loss + thr + Wk + gp;
  }
};
static size_t al(size_t b) { return (b + 255) / 256 * 256; }
static Layout layout(const Plan& p, int with_grad) {
  Layout L{};
  const int64_t nfr1 = 1 + (int64_t)p.psi_fr_plus.size();
  const int64_t N1 = (int64_t)p.psi1.size();
  // xp, Xh hold complex128 in the forward (float64 first layer), complex64 views in the backward;
  // A holds the complex128 layer-1 spectra (sum L1) or complex64 (sum Y2, sum L1)
  L.xp = al(p.N_pad * 16); L.Xh = al(p.N_pad * 16);
  L.A = al(std::max(2 * p.sumL1, p.sumY2) * 8);
  // Z1 and U1_hat share a stride; U1_hat holds the pair-packed float64 spectra (u1p_size complex128) in the
  // forward and g_hat_U1 (sum L1 complex64) in the backward
  L.Z1 = al(std::max(p.sumL1 * 8, p.u1p_size * 16)); L.U1h = L.Z1;
  L.Y2 = al(std::max<int64_t>(p.sumY2, 1) * 8);
  L.cs = al((1 + N1) * p.Ft * 8); L.ct = L.cs;
  L.S1t = al(N1 * p.Ft * 4);
  L.W1 = al(nfr1 * p.P * p.Ft * 8);
  L.V2 = al(nfr1 * p.P * p.frames * 4);
  L.o = al(std::max<int64_t>(p.o_size, 1) * 4);
  L.S = al(p.n_coef * 4); L.r = al(p.n_coef * 4);
  L.gS1t = al(N1 * p.Ft * 4);
  L.g = with_grad ? al(p.N * 4) : 0;
  L.loss = 256;   // k_loss partials (32 float64 per signal)
  L.thr = 256;
  L.Wk = al(std::max<int64_t>(p.ks_w_floats, 1) * 4);   // split-K blocks: complex W of every cell
  L.gp = with_grad ? al(std::max<int64_t>(p.gp_complex, 1) * 8) : 0;   // g_Y2 partials of filter groups
  return L;
}

struct Bufs {
  float2 *xp, *Xh, *A, *Z1, *U1h, *Y2, *cs, *ct, *W1;
  float *S1t, *V2, *o, *S, *r, *gS1t, *g, *loss, *thr, *Wk;
  float2* gp;
  // per-signal strides in elements
  int64_t s_xp, s_A, s_L1, s_Y2, s_c, s_S1t, s_W1, s_V2, s_o, s_S, s_g, s_Wk, s_gp;
};
static Bufs carve(const Plan& p, const Layout& L, char* base, int mb) {
  Bufs b{};
  char* q = base;
  auto take = [&](size_t per) { char* r = q; q += per * mb; return r; };
  b.xp = (float2*)take(L.xp); b.Xh = (float2*)take(L.Xh); b.A = (float2*)take(L.A); b.Z1 = (float2*)take(L.Z1);
  b.U1h = (float2*)take(L.U1h); b.Y2 = (float2*)take(L.Y2); b.cs = (float2*)take(L.cs); b.ct = (float2*)take(L.ct);
  b.S1t = (float*)take(L.S1t); b.W1 = (float2*)take(L.W1); b.V2 = (float*)take(L.V2); b.o = (float*)take(L.o);
  b.S = (float*)take(L.S); b.r = (float*)take(L.r); b.gS1t = (float*)take(L.gS1t); b.g = (float*)take(L.g);
  b.loss = (float*)take(L.loss);
  b.thr = (float*)take(L.thr);   // one float per signal (mb contiguous floats at the start)
  b.Wk = (float*)take(L.Wk);
  b.gp = (float2*)take(L.gp);
  // strides in complex64 units (complex128 views: half)
  b.s_xp = L.xp / 8; b.s_A = L.A / 8; b.s_L1 = L.Z1 / 8; b.s_Y2 = L.Y2 / 8; b.s_c = L.cs / 8;
  b.s_S1t = L.S1t / 4; b.s_W1 = L.W1 / 8; b.s_V2 = L.V2 / 4; b.s_o = L.o / 4; b.s_S = L.S / 4; b.s_g = L.g / 4;
  b.s_Wk = L.Wk / 4;
  b.s_gp = L.gp / 8;
  (void)p;
  return b;
}

static cudaError_t fft_rows(const Plan& p, const float2* in, int64_t in_sb, float2* out, int64_t out_sb,
                            int64_t off, int64_t count, int64_t L, int B, bool inv, cudaStream_t st) {
  Rows ri{in_sb, off, count, L}, ro{out_sb, off, count, L};
  return fft_launch(in, out, ri, ro, B, inv, p.dev->fftt, st);
}

PackGroups jtfs::pack_groups(const Plan& p) {
  PackGroups G{};
  G.n = (int)p.l1_groups.size();
  int64_t acc = 0;
  for (int g = 0; g < G.n; ++g) {
    const FftGroup& q = p.l1_groups[g];
    G.off[g] = q.off;
    G.count[g] = (int)q.count;
    int lg = 0;
    while ((int64_t(1) << lg) < q.L) ++lg;
    G.lgL[g] = lg;
    G.pstart[g] = acc;
    acc += ((q.count + 1) / 2) * q.L;
  }
  G.pstart[G.n] = acc;
  return G;
}

// Y2 row groups (one per second-order block) of the blocks a path shard owns
static std::vector<FftGroup> own_groups(const Plan& p, uint64_t own) {
  std::vector<FftGroup> g;
  for (size_t bi = 0; bi < p.y2_groups.size(); ++bi)
    if (owns_block(own, (int)bi)) g.push_back(p.y2_groups[bi]);
  return g;
}

// Forward of one micro-batch. stop: 0 = full; 1 = after U1 (in A); 2 = after S1t; 3 = after Y2.
static cudaError_t run_forward(const Plan& p, const float* x, int64_t sx, int mb, float* S, int64_t S_sb,
                               const Bufs& w, uint64_t own, cudaStream_t st, int stop = 0,
                               bool keep_w = false, int lane = 0) {
  const DeviceTables& d = *p.dev;
  cudaError_t e;
#define RET() if ((e = cudaGetLastError()) != cudaSuccess) return e
  // A1: reflect pad + FFT in float64
  double2* xpd = reinterpret_cast<double2*>(w.xp);
  double2* Xhd = reinterpret_cast<double2*>(w.Xh);
  double2* Ad = reinterpret_cast<double2*>(w.A);
  const int64_t sd = w.s_xp / 2, sAd = w.s_A / 2;
  launch_reflect_pad(x, sx, xpd, p, mb, st);
  {
    Rows ri{sd, 0, 1, p.N_pad}, ro{sd, 0, 1, p.N_pad};
    if ((e = fft_launch_dd(xpd, Xhd, ri, ro, mb, false, d.fftt, st))) return e;
  }
  // A2: layer 1: cdgmm + subsample_fourier (float64), ifft (float64 -> complex64 Z1),
  // modulus (-> float64 rows), fft (float64 -> complex64 U1_hat)
  launch_gather_dd(Xhd, sd, Ad, sAd, d.l1_jobs, d.l1_tiles, d.n_l1, d.l1_ntiles, d.spec_vals_d, mb, st);
  // Z1 rows longer than 4096 points stay in the four-step's T-layout (fft.cuh): every consumer of Z1 and
  // U1 up to the U1 FFT (which takes T-layout input) is elementwise
  if ((e = fft_groups_df(Ad, w.Z1, sAd, w.s_L1, p.l1_groups.data(), (int)p.l1_groups.size(), mb, true, d.fftt, st,
                         kLayoutToT)))
    return e;
  const PackGroups pg = pack_groups(p);
  launch_modulus_pack(w.Z1, w.s_L1, Ad, sAd, pg, mb, st);   // A: pair-packed complex128 rows (L1 layout)
  RET();
  if (stop == 1) return cudaSuccess;
  // U1_hat = FFT(U1) in float64, two real rows per complex FFT (pair packing), kept in float64 (the gathers
  // unpack the two spectra, so a row's bins must not carry its partner's rounding: DESIGN.md R22 precision)
  double2* U1hd = reinterpret_cast<double2*>(w.U1h);
  const int64_t sU1d = w.s_L1 / 2;
  if ((e = fft_groups_dd(Ad, U1hd, sAd, sU1d, p.l1_pgroups.data(), (int)p.l1_pgroups.size(), mb, false, d.fftt,
                         st, kLayoutFromT)))
    return e;
  // S0 and S1 time averages (Eq.3 time part)
  launch_gather_df(Xhd, sd, w.cs, w.s_c, d.s0_job, d.s0_tiles, 1, d.s0_ntiles, d.spec_vals, mb, st);
  launch_gather_df(U1hd, sU1d, w.cs + p.Ft, w.s_c, d.s1_jobs, d.s1_tiles, d.n_s1, d.s1_ntiles, d.spec_vals, mb, st);
  if ((e = fft_rows(p, w.cs, w.s_c, w.ct, w.s_c, 0, 1 + (int64_t)p.psi1.size(), p.Ft, mb, true, st))) return e;
  launch_s0_out(w.ct, w.s_c, S, S_sb, p, mb, st);
  launch_real_rows(w.ct, w.s_c, p.Ft, w.S1t, w.s_S1t, 0, (int64_t)p.psi1.size() * p.Ft, mb, st);
  RET();
  if (stop == 2) return cudaSuccess;
  // A3: order-1 frequential scattering (shard 0 only)
  if (own & kOwnOrder1) launch_o1_fwd(p, d, w.S1t, w.s_S1t, w.W1, w.s_W1, w.V2, w.s_V2, S, S_sb, mb, st);
  // A4: layer 2, width-first
  if (!p.blocks.empty()) {
    // path shards compute only their own blocks' Y2 (layer 1 is the only replicated stage)
    launch_gather_df(U1hd, sU1d, w.A, w.s_A, d.l2_jobs, d.l2_tiles, d.n_l2, d.l2_ntiles, d.spec_vals, mb, st, own);
    const std::vector<FftGroup> g2 = own_groups(p, own);
    if (!g2.empty() &&
        (e = fft_groups(w.A, w.Y2, w.s_A, w.s_Y2, g2.data(), (int)g2.size(), mb, true, d.fftt, st,
                        kLayoutFromT)))   // the gather left rows > 4096 points in T-layout
      return e;
    RET();
    if (stop == 3) return cudaSuccess;
    // A5: joint lambda_1 stage + phi_F; A6: phi_T
    prof_begin(st, 0 + 4 * lane);
    Fanout* fo = fanout_get(lane);
    fan_fork(fo, st);
    launch_joint_fft(p, d, false, w.Y2, w.s_Y2, w.o, w.s_o, nullptr, 0, nullptr, own, mb, fo->s[0]);
    launch_joint_fwd_tc(p, d, w.Y2, w.s_Y2, w.o, w.s_o, w.Wk, w.s_Wk, keep_w, w.thr, own, mb, fo->s + 1,
                        kFanStreams - 1);
    launch_joint_fwd(p, d, w.Y2, w.s_Y2, w.o, w.s_o, own, mb, fo->s[0]);
    fan_join(fo, st);
    prof_end(st, 0 + 4 * lane);
    launch_phiT_fwd(p, d, w.o, w.s_o, S, S_sb, own, mb, st);
  }
  RET();
  return cudaSuccess;
}

// Backward of one micro-batch (after run_forward + loss): r in w.r -> grad [mb][N] (stride sg)
static cudaError_t run_backward(const Plan& p, const Bufs& w, float* grad, int64_t sg, int mb, uint64_t own, cudaStream_t st, int lane = 0) {
  const DeviceTables& d = *p.dev;
  cudaError_t e;
  const int64_t N1 = (int64_t)p.psi1.size();
  if (!p.blocks.empty()) {
    // A7: phi_T adjoint (r -> g_o, reusing o), joint adjoint (-> g_Y2 in A)
    launch_phiT_adj(p, d, w.r, w.s_S, w.o, w.s_o, own, mb, st);
    if ((e = cudaMemsetAsync(w.A, 0, (size_t)w.s_A * 8 * mb, st))) return e;
    prof_begin(st, 2 + 4 * lane);
    Fanout* fo = fanout_get(lane);
    fan_fork(fo, st);
    launch_joint_fft(p, d, true, w.Y2, w.s_Y2, w.o, w.s_o, w.A, w.s_A, w.thr, own, mb, fo->s[0]);
    launch_joint_bwd_tc(p, d, w.Y2, w.s_Y2, w.o, w.s_o, w.A, w.s_A, w.Wk, w.s_Wk, w.gp, w.s_gp, w.thr, own, mb, fo->s + 1,
                        kFanStreams - 1);
    launch_joint_bwd(p, d, w.Y2, w.s_Y2, w.o, w.s_o, w.A, w.s_A, w.thr, own, mb, fo->s[0]);
    fan_join(fo, st);
    prof_end(st, 2 + 4 * lane);
    // FFT of g_Y2 rows -> G_Y (into Y2), own blocks only
    const std::vector<FftGroup> g2 = own_groups(p, own);
    if (!g2.empty() &&
        (e = fft_groups(w.A, w.Y2, w.s_A, w.s_Y2, g2.data(), (int)g2.size(), mb, false, d.fftt, st,
                        kLayoutToT)))   // spectra of rows > 4096 points left in T-layout (k_adj_gather_u1)
      return e;
  }
  // order-1 adjoint -> g_S1t ; G_S = FFT(g_S1t)
  // order 1 belongs to shard 0 (its forward W1/V2 exist only there): other shards contribute g_S1t = 0
  if (own & kOwnOrder1) {
    launch_o1_bwd(p, d, w.r, w.s_S, w.W1, w.s_W1, w.V2, w.s_V2, w.S1t, w.s_S1t, w.gS1t, w.s_S1t, w.thr, mb, st);
  } else if ((e = cudaMemsetAsync(w.gS1t, 0, (size_t)w.s_S1t * 4 * mb, st))) {
    return e;
  }
  launch_real_to_complex(w.gS1t, w.s_S1t, w.cs, w.s_c, N1 * p.Ft, mb, st);
  if ((e = fft_rows(p, w.cs, w.s_c, w.ct, w.s_c, 0, N1, p.Ft, mb, false, st))) return e;
  // A8: g_hat_U1 -> U1h ; g_U1 = Re IFFT -> A
  launch_adj_gather_u1(p, d, w.ct, w.s_c, w.Y2, w.s_Y2, w.U1h, w.s_L1, mb, st, own);
  if ((e = fft_groups(w.U1h, w.A, w.s_L1, w.s_A, p.l1_groups.data(), (int)p.l1_groups.size(), mb, true, d.fftt,
                      st, kLayoutToT)))   // g_U1 in T-layout, like Z1 (elementwise phase below)
    return e;
  // A9: modulus adjoint, FFT, layer-1 adjoint gather, IFFT, reflect adjoint
  launch_phase_mul(w.Z1, w.A, w.s_A, w.U1h, p.sumL1, w.s_L1, w.thr, mb, st);  // Z1, U1h share the L1 stride
  if ((e = fft_groups(w.U1h, w.A, w.s_L1, w.s_A, p.l1_groups.data(), (int)p.l1_groups.size(), mb, false, d.fftt,
                      st, kLayoutFromT)))   // T-layout g_Z1 -> natural spectrum
    return e;
  launch_adj_gather_x(p, d, w.A, w.s_A, w.Xh, w.s_xp, mb, st);
  if ((e = fft_rows(p, w.Xh, w.s_xp, w.xp, w.s_xp, 0, 1, p.N_pad, mb, true, st))) return e;
  launch_reflect_adj(w.xp, w.s_xp, grad, sg, p, mb, st);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------ ABI
extern "C" {

const char* jtfs_last_error(void) { return t_err.c_str(); }

void jtfs_prof_enable(int on) { jtfs::g_prof.store(on ? 1 : 0); }

jtfs_status jtfs_prof_read(int id, double* total_ms, int64_t* count) {
  if (!total_ms || !count) return fail(JTFS_ERR_SIZE, "NULL argument");
  std::lock_guard<std::mutex> lk(jtfs::g_prof_mu);
  // records of this id on every lane (id + 4 lane): the union of their [begin, end] intervals on the
  // device timeline, so concurrent lanes are not double counted
  std::vector<jtfs::ProfRec> keep, mine;
  for (auto& r : jtfs::g_prof_recs) (r.id % 4 == id ? mine : keep).push_back(r);
  std::vector<std::pair<double, double>> iv;
  for (auto& r : mine) {
    CK(cudaEventSynchronize(r.b));
    float t0 = 0, t1 = 0;
    CK(cudaEventElapsedTime(&t0, mine[0].a, r.a));
    CK(cudaEventElapsedTime(&t1, mine[0].a, r.b));
    iv.emplace_back(t0, t1);
  }
  std::sort(iv.begin(), iv.end());
  double tot = 0, cs = 0, ce = -1e300;
  for (auto& x : iv) {
    if (x.first > ce) {
      if (ce > cs) tot += ce - cs;
      cs = x.first;
      ce = x.second;
    } else if (x.second > ce) {
      ce = x.second;
    }
  }
  if (!iv.empty() && ce > cs) tot += ce - cs;
  for (auto& r : mine) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  jtfs::g_prof_recs.swap(keep);
  *total_ms = tot;
  *count = (int64_t)mine.size();
  return JTFS_OK;
}

jtfs_status jtfs_plan_cost(jtfs_plan_t plan, double* out, int64_t cap) {
  if (!plan || !out || cap < 8) return fail(JTFS_ERR_SIZE, "NULL argument or cap < 8");
  const Plan& p = plan->p;
  double c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  auto lg = [](double v) { return std::log2(v); };
  const double P = (double)p.P;
  // per-column FFT-route cost (FP32 flops, 5 L log2 L per complex FFT of length L)
  std::vector<double> ffw(p.blocks.size(), 0.0), ffb(p.blocks.size(), 0.0);
  for (auto& u : p.units) {
    const double Lf = (double)u.Lf, nr = (double)u.n_rows, ro = (double)u.rows_out;
    ffw[u.bi] += 4 * P + 5 * Lf * lg(Lf) + 4 * nr + 2 * ro * nr;                       // fold, IFFT, |.|, phi_F
    ffb[u.bi] += 4 * P + 10 * Lf * lg(Lf) + 2 * ro * nr + 8 * nr + 4 * P;             // + phase, FFT, accumulate
  }
  for (auto& u : p.units) {
    const double ncols = (double)p.binfo[u.bi].n_cols;
    const double cells = (double)u.n_rows * ncols;
    const int rf = route_of(p, u.bi, false), rb = route_of(p, u.bi, true);
    // tensor-core route: the complex contraction (8K flops per modulus value forward, 16K backward)
    if (rf == kRouteTc) c[0] += cells * 8.0 * u.n1_max;
    else if (rf == kRouteSimt) c[1] += cells * (8.0 * u.n1_max + 3.0 + 2.0 * u.rows_out);
    // split-K blocks: the backward reads W kept by the forward (GEMM2 only, 8K per cell)
    if (rb == kRouteTc) c[2] += cells * (p.blk_ks[u.bi] ? 8.0 : 16.0) * u.n1_max;
    else if (rb == kRouteSimt) c[3] += cells * (16.0 * u.n1_max + 6.0 + 2.0 * u.rows_out);
    c[4] += cells;
    c[5] += 2.0 * 4.0 * u.rows_out * ncols;   // o written (fwd) and g_o read (bwd)
  }
  for (size_t bi = 0; bi < p.blocks.size(); ++bi) {
    const double ncols = (double)p.binfo[bi].n_cols;
    if (route_of(p, bi, false) == kRouteFft) c[1] += ncols * (5 * P * lg(P) + ffw[bi]);
    if (route_of(p, bi, true) == kRouteFft) c[3] += ncols * (10 * P * lg(P) + ffb[bi]);
    c[5] += 3.0 * 8.0 * p.blocks[bi].n1_max * ncols;  // Y2 read fwd, read bwd, g_Y2 write
  }
  for (int i = 0; i < 8; ++i) out[i] = c[i];
  return JTFS_OK;
}

int64_t jtfs_launch_count(void) { return jtfs::g_launches.load(); }

jtfs_status jtfs_plan(int64_t N, int J, int Q, int J_fr, int Q_fr, int64_t T, int64_t F, jtfs_plan_t* out) {
  return jtfs_plan_q2(N, J, Q, 1, J_fr, Q_fr, T, F, out);
}

jtfs_status jtfs_plan_q2(int64_t N, int J, int Q, int Q2, int J_fr, int Q_fr, int64_t T, int64_t F,
                         jtfs_plan_t* out) {
  if (!out) return fail(JTFS_ERR_SIZE, "out is NULL");
  *out = nullptr;
  jtfs_plan_s* h = new (std::nothrow) jtfs_plan_s();
  if (!h) return fail(JTFS_ERR_OOM, "host allocation failed");
  std::string err;
  int rc;
  try {
    rc = make_plan(N, J, Q, J_fr, Q_fr, T, F, &h->p, &err, Q2);
  } catch (const std::bad_alloc&) {
    delete h;
    return fail(JTFS_ERR_OOM, "host allocation failed");
  }
  if (rc) {
    delete h;
    return fail(JTFS_ERR_CONFIG, err);
  }
  *out = h;
  t_err.clear();
  return JTFS_OK;
}

jtfs_status jtfs_plan_destroy(jtfs_plan_t plan) {
  if (!plan) return fail(JTFS_ERR_STATE, "NULL plan");
  delete plan;
  return JTFS_OK;
}

jtfs_status jtfs_plan_info(jtfs_plan_t plan, jtfs_plan_info_t* info) {
  if (!plan || !info) return fail(JTFS_ERR_STATE, "NULL argument");
  const Plan& p = plan->p;
  info->N = p.N; info->N_pad = p.N_pad; info->pad_left = p.pad_left; info->P = p.P; info->frames = p.frames;
  info->n_coef = p.n_coef; info->n_paths = (int64_t)p.paths.size();
  info->N1 = (int32_t)p.psi1.size(); info->N2 = (int32_t)p.psi2.size();
  info->N_fr = (int32_t)p.psi_fr_plus.size(); info->n_blocks = (int32_t)p.blocks.size();
  info->log2T = p.log2T; info->log2F = p.log2F;
  return JTFS_OK;
}

jtfs_status jtfs_plan_paths(jtfs_plan_t plan, jtfs_path_t* out, int64_t cap) {
  if (!plan || !out) return fail(JTFS_ERR_STATE, "NULL argument");
  if (cap < (int64_t)plan->p.paths.size()) return fail(JTFS_ERR_SIZE, "cap < n_paths");
  std::memcpy(out, plan->p.paths.data(), plan->p.paths.size() * sizeof(jtfs_path_t));
  return JTFS_OK;
}

static const std::vector<Filter>* bank(const Plan& p, int layer, std::vector<Filter>* tmp) {
  switch (layer) {
    case 0: return &p.psi1;
    case 1: return &p.psi2;
    case 2: return &p.L_fr;
    case 3: tmp->assign(1, p.phiT); return tmp;
    case 4: tmp->assign(1, p.phiF); return tmp;
  }
  return nullptr;
}

jtfs_status jtfs_plan_filters(jtfs_plan_t plan, int layer, double* xi, double* sigma, int32_t* j, int64_t cap,
                              int64_t* count) {
  if (!plan || !count) return fail(JTFS_ERR_STATE, "NULL argument");
  std::vector<Filter> tmp;
  auto* b = bank(plan->p, layer, &tmp);
  if (!b) return fail(JTFS_ERR_SIZE, "layer must be 0..4");
  *count = (int64_t)b->size();
  for (int64_t i = 0; i < std::min<int64_t>(cap, (int64_t)b->size()); ++i) {
    if (xi) xi[i] = (*b)[i].xi;
    if (sigma) sigma[i] = (*b)[i].sigma;
    if (j) j[i] = (*b)[i].j;
  }
  return JTFS_OK;
}

jtfs_status jtfs_plan_response(jtfs_plan_t plan, int layer, int idx, int k, double* out, int64_t cap) {
  if (!plan || !out) return fail(JTFS_ERR_STATE, "NULL argument");
  std::vector<Filter> tmp;
  auto* b = bank(plan->p, layer, &tmp);
  if (!b || idx < 0 || idx >= (int)b->size()) return fail(JTFS_ERR_SIZE, "bad layer/idx");
  int64_t L0 = (layer == 2 || layer == 4) ? plan->p.P : plan->p.N_pad;
  if (k < 0 || (L0 >> k) < 1 || cap < (L0 >> k)) return fail(JTFS_ERR_SIZE, "bad level or cap");
  std::vector<double> v;
  level_response((*b)[idx], L0, k, &v);
  std::memcpy(out, v.data(), v.size() * sizeof(double));
  return JTFS_OK;
}

jtfs_status jtfs_plan_prepare(jtfs_plan_t plan, jtfs_stream_t stream) {
  if (!plan) return fail(JTFS_ERR_STATE, "NULL plan");
  jtfs_status s = ensure_device(plan);
  if (s) return s;
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return JTFS_OK;
}

size_t jtfs_workspace_size(jtfs_plan_t plan, int64_t batch, int with_grad) {
  if (!plan || batch < 0) return 0;
  return layout(plan->p, with_grad).per_signal() * (size_t)batch;
}

// Path shards: whole second-order blocks go to shards by LPT over Plan::block_cost
// (largest first to the least-loaded shard, ties to the lower index; shard 0 starts with the order-1
// work), so a shard computes layer 2 / its adjoint only for its own blocks and layer 1 is the only
// replicated stage. Deterministic: every rank derives every rank's blocks.
constexpr int kMaxShards = 64;
static std::vector<int> block_owner(const Plan& p, int n_shards) {
  const int nb = (int)p.blocks.size();
  std::vector<int> owner(nb, 0), order(nb);
  for (int i = 0; i < nb; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return p.block_cost[a] > p.block_cost[b]; });
  std::vector<double> load(n_shards, 0.0);
  load[0] = p.order1_cost;
  for (int bi : order) {
    int s = 0;
    for (int k = 1; k < n_shards; ++k)
      if (load[k] < load[s]) s = k;
    owner[bi] = s;
    load[s] += p.block_cost[bi];
  }
  return owner;
}
static uint64_t shard_mask(const Plan& p, int shard, int n_shards) {
  if (n_shards <= 1) return kOwnAll;
  const std::vector<int> owner = block_owner(p, n_shards);
  uint64_t m = shard == 0 ? kOwnOrder1 : 0;
  for (size_t bi = 0; bi < owner.size(); ++bi)
    if (owner[bi] == shard) m |= 1ull << bi;
  return m;
}

static jtfs_status check_common(jtfs_plan_t plan, int64_t B, size_t ws_bytes, int with_grad, void* ws, int* mb) {
  if (!plan) return fail(JTFS_ERR_STATE, "NULL plan");
  if (B <= 0) return fail(JTFS_ERR_SIZE, "B must be > 0");
  if (!ws) return fail(JTFS_ERR_SIZE, "workspace is NULL");
  if (((uintptr_t)ws) % 256) return fail(JTFS_ERR_SIZE, "workspace must be 256-byte aligned");
  size_t per = layout(plan->p, with_grad).per_signal();
  int64_t m = (int64_t)(ws_bytes / per);
  if (m < 1) return fail(JTFS_ERR_SIZE, "workspace too small for one signal (need jtfs_workspace_size(plan,1,...))");
  *mb = (int)std::min<int64_t>(m, B);
  return ensure_device(plan);
}

static bool aligned16(const void* p) { return ((uintptr_t)p % 16) == 0; }

jtfs_status jtfs_forward(jtfs_plan_t plan, const float* x, int64_t B, float* S, void* ws, size_t ws_bytes,
                         jtfs_stream_t stream) {
  int mb;
  jtfs_status s = check_common(plan, B, ws_bytes, 0, ws, &mb);
  if (s) return s;
  if (!x || !S || !aligned16(x) || !aligned16(S)) return fail(JTFS_ERR_SIZE, "x/S NULL or not 16-byte aligned");
  const Plan& p = plan->p;
  Layout L = layout(p, 0);
  Bufs w = carve(p, L, (char*)ws, mb);
  for (int64_t b0 = 0; b0 < B; b0 += mb) {
    int n = (int)std::min<int64_t>(mb, B - b0);
    CK(run_forward(p, x + b0 * p.N, p.N, n, S + b0 * p.n_coef, p.n_coef, w, kOwnAll, (cudaStream_t)stream));
  }
  t_err.clear();
  return JTFS_OK;
}

static jtfs_status loss_grad_impl(jtfs_plan_t plan, const float* y, const float* St, int64_t B, float* loss,
                                  float* grad, int shard, int n_shards, void* ws, size_t ws_bytes, cudaStream_t st,
                                  jtfs_metamer_state* mstate, float momentum, float grow, float shrink) {
  int mb;
  jtfs_status s = check_common(plan, B, ws_bytes, 1, ws, &mb);
  if (s) return s;
  if (n_shards < 1 || n_shards > kMaxShards || shard < 0 || shard >= n_shards)
    return fail(JTFS_ERR_SIZE, "need 0 <= shard < n_shards <= 64");
  const Plan& p = plan->p;
  const uint64_t own = shard_mask(p, shard, n_shards);
  Layout L = layout(p, 1);
  // Optional two lanes (JTFS_LANES=2): each lane runs its own micro-batches on its own stream (forked from
  // and joined to `st`), so one lane's tensor-core joint stage can overlap the other's HBM-bound FFT /
  // gather stages. Per-signal results do not depend on the lane or micro-batch.
  const int lanes = (g_lanes > 1 && mb >= 2 && B >= 2) ? 2 : 1;
  const int mbl = mb / lanes;
  Fanout* fl = lanes > 1 ? fanout_get(kMaxLanes) : nullptr;   // lane streams: fl->s[0], fl->s[1] (own slot)
  if (lanes > 1) {
    cudaEventRecord(fl->fork, st);
    for (int l = 0; l < lanes; ++l) cudaStreamWaitEvent(fl->s[l], fl->fork, 0);
  }
  for (int l = 0; l < lanes; ++l) {
    cudaStream_t ls = lanes > 1 ? fl->s[l] : st;
    Bufs w = carve(p, L, (char*)ws + (size_t)l * mbl * L.per_signal(), mbl);
    for (int64_t b0 = (int64_t)l * mbl; b0 < B; b0 += (int64_t)lanes * mbl) {
    int n = (int)std::min<int64_t>(mbl, B - b0);
    // R22 dead zone first: the forward's phase store (split-K blocks) decides it on the final W
    launch_mod_threshold(y + b0 * p.N, p.N, kEpsMod, w.thr, n, ls);
    CK(run_forward(p, y + b0 * p.N, p.N, n, w.S, w.s_S, w, own, ls, 0, true, l));
    float* lossp = mstate ? mstate->loss + b0 : loss + b0;
    launch_loss(p, *p.dev, w.S, w.s_S, St + b0 * p.n_coef, p.n_coef, w.r, w.s_S, lossp, (double*)w.loss, own, n, ls);
    float* gp = mstate ? w.g : grad + b0 * p.N;
    int64_t sg = mstate ? w.s_g : p.N;
    CK(run_backward(p, w, gp, sg, n, own, ls, l));
    if (mstate) {
      launch_metamer(mstate->y + b0 * p.N, mstate->u + b0 * p.N, mstate->y_prev + b0 * p.N,
                     mstate->g_prev + b0 * p.N, mstate->mu + b0, mstate->loss_prev + b0, lossp,
                     mstate->accepted + b0, mstate->active ? mstate->active + b0 : nullptr, gp, sg, p.N, n,
                     momentum, grow, shrink, ls);
      CK(cudaGetLastError());
    }
    }
  }
  if (lanes > 1)
    for (int l = 0; l < lanes; ++l) {
      cudaEventRecord(fl->join[l], fl->s[l]);
      cudaStreamWaitEvent(st, fl->join[l], 0);
    }
  t_err.clear();
  return JTFS_OK;
}

jtfs_status jtfs_loss_grad(jtfs_plan_t plan, const float* y, const float* S_target, int64_t B, float* loss,
                           float* grad, int shard, int n_shards, void* ws, size_t ws_bytes, jtfs_stream_t stream) {
  if (!y || !S_target || !loss || !grad) return fail(JTFS_ERR_SIZE, "NULL data pointer");
  if (!aligned16(y) || !aligned16(S_target) || !aligned16(grad))
    return fail(JTFS_ERR_SIZE, "y/S_target/grad must be 16-byte aligned");
  return loss_grad_impl(plan, y, S_target, B, loss, grad, shard, n_shards, ws, ws_bytes, (cudaStream_t)stream,
                        nullptr, 0, 0, 0);
}

jtfs_status metamer_step(jtfs_plan_t plan, jtfs_metamer_state* st, const float* S_target, int64_t B,
                         float momentum, float grow, float shrink, void* ws, size_t ws_bytes, jtfs_stream_t stream) {
  if (!st || !st->y || !st->u || !st->y_prev || !st->g_prev || !st->mu || !st->loss_prev || !st->loss ||
      !st->accepted || !S_target)
    return fail(JTFS_ERR_SIZE, "NULL state or target pointer");
  jtfs_status s = loss_grad_impl(plan, st->y, S_target, B, nullptr, nullptr, 0, 1, ws, ws_bytes,
                                 (cudaStream_t)stream, st, momentum, grow, shrink);
  if (s == JTFS_OK) st->iter += 1;
  return s;
}

size_t jtfs_host_staging_size(jtfs_plan_t plan, int64_t B, int with_grad) {
  if (!plan || B < 0) return 0;
  const Plan& p = plan->p;
  size_t s = al(B * p.N * 4) + al(B * p.n_coef * 4) + al(B * 4);
  if (with_grad) s += al(B * p.N * 4);
  return s;
}

jtfs_status jtfs_loss_grad_host(jtfs_plan_t plan, const float* y_host, const float* S_target_host, int64_t B,
                                float* loss_host, float* grad_host, void* ws, size_t ws_bytes, jtfs_stream_t stream) {
  if (!plan) return fail(JTFS_ERR_STATE, "NULL plan");
  if (!y_host || !S_target_host || !loss_host || !grad_host) return fail(JTFS_ERR_SIZE, "NULL host pointer");
  const Plan& p = plan->p;
  size_t stg = jtfs_host_staging_size(plan, B, 1);
  if (ws_bytes < stg) return fail(JTFS_ERR_SIZE, "workspace smaller than the host staging");
  char* q = (char*)ws;
  float* y = (float*)q; q += al(B * p.N * 4);
  float* St = (float*)q; q += al(B * p.n_coef * 4);
  float* loss = (float*)q; q += al(B * 4);
  float* grad = (float*)q; q += al(B * p.N * 4);
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(y, y_host, B * p.N * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(St, S_target_host, B * p.n_coef * 4, cudaMemcpyHostToDevice, st));
  jtfs_status s = loss_grad_impl(plan, y, St, B, loss, grad, 0, 1, q, ws_bytes - stg, st, nullptr, 0, 0, 0);
  if (s) return s;
  CK(cudaMemcpyAsync(loss_host, loss, B * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(grad_host, grad, B * p.N * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return JTFS_OK;
}

jtfs_status jtfs_debug_fft(jtfs_plan_t plan, const void* in, void* out, int64_t L, int64_t count, int64_t B,
                           int inverse, int dbl, jtfs_stream_t stream) {
  if (!plan || !in || !out) return fail(JTFS_ERR_SIZE, "NULL argument");
  jtfs_status s = ensure_device(plan);
  if (s) return s;
  const Plan& p = plan->p;
  if (L < 2 || (L & (L - 1)) || L > p.N_pad || count < 1 || B < 1)
    return fail(JTFS_ERR_SIZE, "need L a power of two in [2, N_pad], count >= 1, B >= 1");
  Rows ri{count * L, 0, count, L}, ro{count * L, 0, count, L};
  cudaError_t e = dbl ? fft_launch_dd((const double2*)in, (double2*)out, ri, ro, (int)B, inverse != 0, p.dev->fftt,
                                      (cudaStream_t)stream)
                      : fft_launch((const float2*)in, (float2*)out, ri, ro, (int)B, inverse != 0, p.dev->fftt,
                                   (cudaStream_t)stream);
  CK(e);
  t_err.clear();
  return JTFS_OK;
}

jtfs_status jtfs_check_finite(const float* x, int64_t n, jtfs_stream_t stream) {
  if (n < 0 || (n > 0 && !x)) return fail(JTFS_ERR_SIZE, "NULL array or n < 0");
  if (n == 0) return JTFS_OK;
  static thread_local std::vector<int32_t*> flags;   // one device flag per device and host thread
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if ((int)flags.size() <= dev) flags.resize(dev + 1, nullptr);
  if (!flags[dev]) CK(cudaMalloc(&flags[dev], sizeof(int32_t)));
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemsetAsync(flags[dev], 0, sizeof(int32_t), st));
  launch_check_finite(x, n, flags[dev], st);
  int32_t h = 0;
  CK(cudaMemcpyAsync(&h, flags[dev], sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h) return fail(JTFS_ERR_NUMERIC, "non-finite value (NaN or inf)");
  t_err.clear();
  return JTFS_OK;
}

jtfs_status jtfs_plan_shards(jtfs_plan_t plan, int n_shards, int32_t* block_owner_out, int64_t cap) {
  if (!plan || !block_owner_out) return fail(JTFS_ERR_SIZE, "NULL argument");
  if (n_shards < 1 || n_shards > kMaxShards) return fail(JTFS_ERR_SIZE, "need 1 <= n_shards <= 64");
  const Plan& p = plan->p;
  if (cap < (int64_t)p.blocks.size()) return fail(JTFS_ERR_SIZE, "cap < n_blocks");
  const std::vector<int> owner = block_owner(p, n_shards);
  for (size_t i = 0; i < owner.size(); ++i) block_owner_out[i] = owner[i];
  t_err.clear();
  return JTFS_OK;
}

jtfs_status jtfs_loss_report(jtfs_plan_t plan, const float* S, const float* S_target, int64_t B, float* per_path,
                             jtfs_stream_t stream) {
  if (!plan) return fail(JTFS_ERR_STATE, "NULL plan");
  if (B <= 0 || !S || !S_target || !per_path) return fail(JTFS_ERR_SIZE, "B <= 0 or NULL argument");
  jtfs_status s = ensure_device(plan);
  if (s) return s;
  launch_loss_report(plan->p, *plan->p.dev, S, S_target, per_path, (int)B, (cudaStream_t)stream);
  CK(cudaGetLastError());
  t_err.clear();
  return JTFS_OK;
}

jtfs_status jtfs_colored_noise(jtfs_plan_t plan, const float* S_target, const float* white, int64_t B, float* y0,
                               void* ws, size_t ws_bytes, jtfs_stream_t stream) {
  int mb;
  jtfs_status s = check_common(plan, B, ws_bytes, 0, ws, &mb);
  if (s) return s;
  if (!S_target || !white || !y0) return fail(JTFS_ERR_SIZE, "NULL argument");
  const Plan& p = plan->p;
  if ((p.psi1.size() + p.F - 1) / p.F > 1024) return fail(JTFS_ERR_CONFIG, "more than 1024 order-1 rows");
  Layout L = layout(p, 0);
  Bufs w = carve(p, L, (char*)ws, mb);
  cudaStream_t st = (cudaStream_t)stream;
  const DeviceTables& d = *p.dev;
  for (int64_t b0 = 0; b0 < B; b0 += mb) {
    const int n = (int)std::min<int64_t>(mb, B - b0);
    launch_cn_gains(p, d, S_target + b0 * p.n_coef, p.n_coef, w.S1t, w.s_S1t, n, st);
    launch_real_to_complex(white + b0 * p.N_pad, p.N_pad, w.xp, w.s_xp, p.N_pad, n, st);
    CK(fft_rows(p, w.xp, w.s_xp, w.Xh, w.s_xp, 0, 1, p.N_pad, n, false, st));
    launch_cn_shape(p, d, w.Xh, w.s_xp, w.S1t, w.s_S1t, n, st);
    CK(fft_rows(p, w.Xh, w.s_xp, w.xp, w.s_xp, 0, 1, p.N_pad, n, true, st));
    launch_cn_crop(p, w.xp, w.s_xp, white + b0 * p.N_pad, w.S1t, w.s_S1t, y0 + b0 * p.N, n, st);
    CK(cudaGetLastError());
  }
  t_err.clear();
  return JTFS_OK;
}

jtfs_status jtfs_debug_stage(jtfs_plan_t plan, int stage, const float* x, int64_t B, void* out, size_t out_bytes,
                             void* ws, size_t ws_bytes, jtfs_stream_t stream) {
  int mb;
  jtfs_status s = check_common(plan, B, ws_bytes, 0, ws, &mb);
  if (s) return s;
  if (mb < B) return fail(JTFS_ERR_SIZE, "debug stage needs the whole batch in one micro-batch");
  const Plan& p = plan->p;
  Layout L = layout(p, 0);
  Bufs w = carve(p, L, (char*)ws, mb);
  cudaStream_t st = (cudaStream_t)stream;
  const int n = (int)B;
  if (stage == 1) {
    if (out_bytes < (size_t)B * p.sumL1 * 4) return fail(JTFS_ERR_SIZE, "out too small");
    CK(run_forward(p, x, p.N, n, w.S, w.s_S, w, kOwnAll, st, 1));
    launch_unpack_u1(reinterpret_cast<const double2*>(w.A), w.s_A / 2, (float*)out, p.sumL1, pack_groups(p), p.sumL1,
                     n, st);
  } else if (stage == 2) {
    int64_t per = (int64_t)p.psi1.size() * p.Ft;
    if (out_bytes < (size_t)B * per * 4) return fail(JTFS_ERR_SIZE, "out too small");
    CK(run_forward(p, x, p.N, n, w.S, w.s_S, w, kOwnAll, st, 2));
    CK(cudaMemcpy2DAsync(out, per * 4, w.S1t, w.s_S1t * 4, per * 4, B, cudaMemcpyDeviceToDevice, st));
  } else if (stage == 3) {
    if (out_bytes < (size_t)B * p.sumY2 * 8) return fail(JTFS_ERR_SIZE, "out too small");
    CK(run_forward(p, x, p.N, n, w.S, w.s_S, w, kOwnAll, st, 3));
    if (p.sumY2 > 0)
      CK(cudaMemcpy2DAsync(out, p.sumY2 * 8, w.Y2, w.s_Y2 * 8, p.sumY2 * 8, B, cudaMemcpyDeviceToDevice, st));
  } else if (stage == 5 || stage == 6) {
    CK(run_forward(p, x, p.N, n, w.S, w.s_S, w, kOwnAll, st, 1));
    if (stage == 5) {   // X_hat, complex128 [B][N_pad]
      if (out_bytes < (size_t)B * p.N_pad * 16) return fail(JTFS_ERR_SIZE, "out too small");
      CK(cudaMemcpy2DAsync(out, p.N_pad * 16, w.Xh, w.s_xp * 8, p.N_pad * 16, B, cudaMemcpyDeviceToDevice, st));
    } else {            // Z1, complex64 [B][sum L1]
      if (out_bytes < (size_t)B * p.sumL1 * 8) return fail(JTFS_ERR_SIZE, "out too small");
      launch_untranspose_rows(w.Z1, w.s_L1, (float2*)out, p.sumL1, pack_groups(p), p.sumL1, (int)B, st);
    }
  } else if (stage == 4) {
    if (out_bytes < (size_t)B * p.n_coef * 4) return fail(JTFS_ERR_SIZE, "out too small");
    CK(run_forward(p, x, p.N, n, (float*)out, p.n_coef, w, kOwnAll, st, 0));
  } else {
    return fail(JTFS_ERR_SIZE, "stage must be 1..6");
  }
  CK(cudaGetLastError());
  return JTFS_OK;
}

}  // extern "C"
