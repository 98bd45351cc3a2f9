// libreax: C ABI + host orchestration of the B200 ReaxFF hot path.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared -Xcompiler -fPIC
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/reax.h"
#include "common.cuh"
#include "kernels.cuh"

using namespace rx;

namespace {

constexpr size_t ALIGN = 256;
constexpr int MAX_SPLIT = 8;
// CTAs per home block for the window kernels: small systems (c0/c1) have too
// few home blocks to fill 148 SMs, so each block's rows are split over
// several CTAs (each builds the same window)
// (measured on c1: the step is fastest with the nonbonded at 2 CTA-units per
// SM — one CTA per home block, leaving the side-stream bond chain room — and
// the list build at 4)
int choose_split(int nblock, int per_sm, const char* env) {
  if (const char* e = getenv(env)) per_sm = std::max(1, atoi(e));   // tuning experiments
  int target = 148 * per_sm;
  int s = (target + nblock - 1) / std::max(nblock, 1);
  return std::max(1, std::min(MAX_SPLIT, s));
}
constexpr int TPB = 256;

inline size_t align_up(size_t x) { return (x + ALIGN - 1) & ~(ALIGN - 1); }
inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

// ------------------------------------------------------------ window tables
bool forward_offset(int ox, int oy, int oz) {
  return oz > 0 || (oz == 0 && (oy > 0 || (oy == 0 && ox > 0)));
}

WindowTables make_tables() {
  WindowTables T;
  memset(&T, 0, sizeof(T));
  bool used[NWB] = {false};
  for (int h = 0; h < NHOME; ++h) {
    int hv[3] = {h % HB, (h / HB) % HB, h / (HB * HB)};
    for (int oz = -SR; oz <= SR; ++oz)
      for (int oy = -SR; oy <= SR; ++oy)
        for (int ox = -SR; ox <= SR; ++ox) {
          if (!(forward_offset(ox, oy, oz) || (ox == 0 && oy == 0 && oz == 0))) continue;
          int w = (hv[0] + SR + ox) + WB * ((hv[1] + SR + oy) + WB * (hv[2] + SR + oz));
          used[w] = true;
        }
  }
  T.nwu = 0;
  for (int w = 0; w < NWB; ++w) {
    T.widx[w] = -1;
    if (used[w]) {
      T.widx[w] = T.nwu;
      T.wu[T.nwu++] = w;
    }
  }
  if (T.nwu > NWU_MAX) abort();   // compile-time geometry constants are inconsistent
  for (int h = 0; h < NHOME; ++h) {
    int hv[3] = {h % HB, (h / HB) % HB, h / (HB * HB)};
    auto wk = [&](int ox, int oy, int oz) {
      return T.widx[(hv[0] + SR + ox) + WB * ((hv[1] + SR + oy) + WB * (hv[2] + SR + oz))];
    };
    T.home_k[h] = wk(0, 0, 0);
    for (int oz = -SR; oz <= SR; ++oz)
      for (int oy = -SR; oy <= SR; ++oy)
        for (int ox = -SR; ox <= SR; ++ox) {
          if (!(forward_offset(ox, oy, oz) || (ox == 0 && oy == 0 && oz == 0))) continue;
          int kk = wk(ox, oy, oz);
          T.mask[h][kk / 32] |= 1u << (kk % 32);
        }
    std::vector<std::pair<int, int>> runs;
    for (int oz = 0; oz <= SR; ++oz)
      for (int oy = -SR; oy <= SR; ++oy) {
        int oxa = -SR, oxb = SR;
        if (oz == 0 && oy < 0) continue;
        if (oz == 0 && oy == 0) oxa = 1;
        runs.push_back({wk(oxa, oy, oz), wk(oxb, oy, oz)});
      }
    T.nrun1[h] = (int)runs.size();
    if (T.nrun1[h] + 1 > 16) abort();   // k_nbr_build keeps the runs + own cell in lanes 0..15
    for (size_t q = 0; q < runs.size(); ++q) {
      T.run1_a[h][q] = runs[q].first;
      T.run1_b[h][q] = runs[q].second;
    }
    std::sort(runs.begin(), runs.end());
    std::vector<std::pair<int, int>> merged;
    for (auto& r : runs) {
      if (!merged.empty() && merged.back().second + 1 == r.first) merged.back().second = r.second;
      else merged.push_back(r);
    }
    T.nrun[h] = (int)merged.size();
    for (size_t q = 0; q < merged.size(); ++q) {
      T.run_a[h][q] = merged[q].first;
      T.run_b[h][q] = merged[q].second;
    }
  }
  return T;
}

std::mutex g_tab_mu;

// The dynamic shared memory limit is a per-function (process-wide) attribute:
// contexts with different window capacities only ever raise it.
template <typename F>
cudaError_t ensure_smem(F* func, size_t bytes) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, func);
  if (e != cudaSuccess) return e;
  if ((size_t)a.maxDynamicSharedSizeBytes >= bytes) return cudaSuccess;
  return cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}
bool g_tab_done[64] = {false};

cudaError_t ensure_tables() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_tab_mu);
  if (dev < 64 && g_tab_done[dev]) return cudaSuccess;
  WindowTables T = make_tables();
  e = cudaMemcpyToSymbol(c_win, &T, sizeof(T));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_win_wu, T.wu, sizeof(T.wu));   // per-thread (divergent) reads
  if (e == cudaSuccess && dev < 64) g_tab_done[dev] = true;
  return e;
}

// ------------------------------------------------------------------- grid
bool make_grid(const double box[3], double R, Grid& g) {
  for (int k = 0; k < 3; ++k) {
    double L = box[k];
    // sub-cell side strictly >= R/2 with a relative margin, so rounding in
    // floor(x/h) never separates two atoms within R by more than SR cells
    int nc = (int)std::floor(L / (0.5 * R * (1.0 + 1e-10)));
    if (nc < 1) nc = 1;
    g.nc[k] = nc;
    g.nb[k] = (nc + HB - 1) / HB;
    g.L[k] = L;
    g.h[k] = L / nc;
    g.inv_h[k] = nc / L;
  }
  long long ncell = (long long)g.nc[0] * g.nc[1] * g.nc[2];
  long long nblock = (long long)g.nb[0] * g.nb[1] * g.nb[2];
  if (ncell > (1LL << 30)) return false;
  g.ncell = (int)ncell;
  g.nblock = (int)nblock;
  return true;
}

bool finite_pos(double x) { return std::isfinite(x) && x > 0.0; }

// --------------------------------------------------------- validation (a1)
reax_status check_box_cut(const double box[3], const reax_cutoffs* cut) {
  if (!box || !cut) return REAX_ERR_ARG;
  if (!(finite_pos(cut->r_nonb) && finite_pos(cut->r_bond))) return REAX_ERR_CUTOFF;
  if (cut->r_bond > cut->r_nonb) return REAX_ERR_CUTOFF;
  if (!(cut->bo_cut > 0.0 && cut->bo_cut < 1.0)) return REAX_ERR_CUTOFF;
  for (int k = 0; k < 3; ++k) {
    // strictly greater than 2 r_nonb: every pair within r_nonb then has exactly
    // one periodic image within r_nonb (reading 18)
    if (!std::isfinite(box[k]) || !(box[k] > 2.0 * cut->r_nonb)) return REAX_ERR_BOX;
  }
  return REAX_OK;
}

// host copy of B1-B2 for the conservative candidate radius (bisection)
double host_bo_prime(double r, const reax_params* p, int ti, int tj) {
  int nt = p->ntypes, tp = ti * nt + tj;
  double r0s = 0.5 * (p->r_sigma[ti] + p->r_sigma[tj]);
  double r0p = 0.5 * (p->r_pi[ti] + p->r_pi[tj]);
  double r0pp = 0.5 * (p->r_pipi[ti] + p->r_pipi[tj]);
  return std::exp(p->p_bo1[tp] * std::pow(r / r0s, p->p_bo2[tp])) +
         std::exp(p->p_bo3[tp] * std::pow(r / r0p, p->p_bo4[tp])) +
         std::exp(p->p_bo5[tp] * std::pow(r / r0pp, p->p_bo6[tp]));
}

reax_status build_params(const reax_params* p, const reax_cutoffs* cut, DevParams& d) {
  if (!p) return REAX_ERR_ARG;
  int nt = p->ntypes;
  if (nt < 1 || nt > REAX_MAX_TYPES) return REAX_ERR_PARAM;
  const double* per_type[] = {p->r_sigma, p->r_pi, p->r_pipi, p->gamma, p->r_vdw, p->eps, p->alpha,
                              p->gamma_w, p->b131, p->b132, p->b133, p->val, p->val_boc};
  for (auto a : per_type) {
    if (!a) return REAX_ERR_ARG;
    for (int t = 0; t < nt; ++t)
      if (!std::isfinite(a[t])) return REAX_ERR_PARAM;
  }
  const double* per_pair[] = {p->p_bo1, p->p_bo2, p->p_bo3, p->p_bo4, p->p_bo5, p->p_bo6, p->De};
  for (auto a : per_pair) {
    if (!a) return REAX_ERR_ARG;
    for (int t = 0; t < nt * nt; ++t) {
      if (!std::isfinite(a[t])) return REAX_ERR_PARAM;
      if (a[t] != a[(t % nt) * nt + t / nt]) return REAX_ERR_PARAM;  // symmetric
    }
  }
  for (int t = 0; t < nt; ++t) {
    if (!(p->r_sigma[t] > 0 && p->r_pi[t] > 0 && p->r_pipi[t] > 0 && p->gamma[t] > 0 && p->r_vdw[t] > 0 &&
          p->eps[t] >= 0 && p->alpha[t] >= 0 && p->gamma_w[t] > 0 && p->b131[t] >= 0 && p->b132[t] >= 0 &&
          p->b133[t] >= 0 && p->val[t] > 0))
      return REAX_ERR_PARAM;
  }
  if (!(std::isfinite(p->p_boc1) && std::isfinite(p->p_boc2) && p->p_boc2 != 0.0 && p->p_vdw1 > 0 &&
        std::isfinite(p->p_vdw1) && std::isfinite(p->coulomb_c)))
    return REAX_ERR_PARAM;
  memset(&d, 0, sizeof(d));
  d.nt = nt;
  d.R = cut->r_nonb;
  d.R2 = cut->r_nonb * cut->r_nonb;
  d.rb2 = cut->r_bond * cut->r_bond;
  d.bo_cut = cut->bo_cut;
  d.p_vdw = p->p_vdw1;
  d.inv_p = 1.0 / p->p_vdw1;
  d.invR = 1.0 / cut->r_nonb;
  d.C = p->coulomb_c;
  d.p_boc1 = p->p_boc1;
  d.p_boc2 = p->p_boc2;
  // fp32 band: the fp32 r^2 error is < 3e-4 A^2 for |d| < 16 A;
  // the band is +-0.02 A^2 (scaled with R^2 for other cutoffs)
  double m = 0.02 * (d.R2 / 100.0);
  d.R2lo = (float)(d.R2 - m);
  d.R2hi = (float)(d.R2 + m);
  d.rcand2_max = -1.0f;
  for (int t = 0; t < nt; ++t) {
    d.val[t] = p->val[t];
    d.val_boc[t] = p->val_boc[t];
  }
  // tables of the nonbonded's exp/log (x86 long double: 64-bit mantissa)
  for (int j = 0; j < EXP_TBL; ++j) d.exp_tbl[j] = (double)exp2l((long double)j / (long double)EXP_TBL);
  for (int j = 0; j < LOG_TBL; ++j) {
    long double cj = 1.0L + ((long double)j + 0.5L) / (long double)LOG_TBL;
    double inv = (double)(1.0L / cj);
    d.log_tbl[2 * j] = inv;
    d.log_tbl[2 * j + 1] = (double)(-logl((long double)inv));
  }
  for (int a = 0; a < nt; ++a)
    for (int b = 0; b < nt; ++b) {
      int tp = a * nt + b;
      NBPair& c = d.nb[tp];
      double D = std::sqrt(p->eps[a] * p->eps[b]);
      double alpha = std::sqrt(p->alpha[a] * p->alpha[b]);
      double rvdw = 2.0 * std::sqrt(p->r_vdw[a] * p->r_vdw[b]);
      double gw = std::sqrt(p->gamma_w[a] * p->gamma_w[b]);
      double g = std::sqrt(p->gamma[a] * p->gamma[b]);
      c.D = D;
      c.ahalf = 0.5 * alpha;
      c.Dadr = D * alpha / rvdw;
      c.inv_rvdw = 1.0 / rvdw;
      c.gwmp = std::pow(gw, -p->p_vdw1);
      c.g3 = 1.0 / (g * g * g);
      BOPair& o = d.bo[tp];
      o.lr0[0] = std::log(0.5 * (p->r_sigma[a] + p->r_sigma[b]));
      o.lr0[1] = std::log(0.5 * (p->r_pi[a] + p->r_pi[b]));
      o.lr0[2] = std::log(0.5 * (p->r_pipi[a] + p->r_pipi[b]));
      o.pa[0] = p->p_bo1[tp]; o.pa[1] = p->p_bo3[tp]; o.pa[2] = p->p_bo5[tp];
      o.pb[0] = p->p_bo2[tp]; o.pb[1] = p->p_bo4[tp]; o.pb[2] = p->p_bo6[tp];
      o.pboc3 = std::sqrt(p->b132[a] * p->b132[b]);
      o.pboc4 = std::sqrt(p->b131[a] * p->b131[b]);
      o.pboc5 = std::sqrt(p->b133[a] * p->b133[b]);
      // conservative candidate radius: BO' is decreasing in r when p_bo(1,3,5) <= 0
      // and p_bo(2,4,6) >= 0; otherwise fall back to r_bond
      bool mono = p->p_bo1[tp] <= 0 && p->p_bo3[tp] <= 0 && p->p_bo5[tp] <= 0 && p->p_bo2[tp] >= 0 &&
                  p->p_bo4[tp] >= 0 && p->p_bo6[tp] >= 0;
      double rc = cut->r_bond;
      if (mono) {
        double lo = 1e-3, hi = cut->r_bond;
        if (host_bo_prime(hi, p, a, b) < cut->bo_cut) {
          if (host_bo_prime(lo, p, a, b) < cut->bo_cut) {
            rc = 0.0;
          } else {
            for (int it = 0; it < 200; ++it) {
              double mid = 0.5 * (lo + hi);
              if (host_bo_prime(mid, p, a, b) >= cut->bo_cut) lo = mid; else hi = mid;
            }
            rc = std::min(cut->r_bond, hi * (1.0 + 1e-6) + 1e-6);
          }
        }
      }
      d.rcand2[tp] = rc > 0.0 ? (float)(rc * rc + m) : -1.0f;
      d.rcand2_max = std::max(d.rcand2_max, d.rcand2[tp]);
    }
  return REAX_OK;
}

// ------------------------------------------------------------ capacities
void resolve_caps(int64_t n, const double box[3], const reax_cutoffs* cut, const reax_capacity* in,
                  reax_capacity& c) {
  reax_capacity z = {0, 0, 0, 0};
  if (!in) in = &z;
  double vol = box[0] * box[1] * box[2];
  double rho = vol > 0 ? (double)n / vol : 0.0;
  double R = cut->r_nonb;
  double mean = 2.0 * M_PI / 3.0 * rho * R * R * R;
  int rc = (int)std::ceil(1.3 * mean + 96.0);   // rows: about mean +- 5 sigma plus the own-cell part; overflow regrows
  rc = (rc + 31) / 32 * 32;
  c.row_cap = in->row_cap > 0 ? in->row_cap : std::min(rc, 65535);
  c.row_cap = std::min((c.row_cap + 7) & ~7, 65528);   // 16-byte rows (asynchronous row copies)
  c.cand_cap = in->cand_cap > 0 ? in->cand_cap : 16;
  c.bond_cap = in->bond_cap > 0 ? in->bond_cap : std::max<int64_t>(8 * n, 64);
  c.window_cap = in->window_cap > 0 ? in->window_cap : 2048;
  c.window_cap = (c.window_cap + 31) & ~31;   // vector zeroing of the shared F window
}

struct Layout {
  size_t off[40];
  size_t total;
};

// assigns WS pointers relative to base (base may be null to size)
size_t layout(int64_t n, const Grid& g, const reax_capacity& c, char* base, WS* w) {
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o = align_up(o + std::max<size_t>(bytes, 1));
    return base ? base + r : nullptr;
  };
  size_t N = (size_t)std::max<int64_t>(n, 1);
  // scan partials: atoms, cells or bond entries (the interaction-list scan runs over the bond list)
  size_t nscan = (size_t)nblk(std::max<int64_t>(std::max<int64_t>(N + 1, (int64_t)g.ncell + 1), c.bond_cap + 1), SCAN_TILE) + 2;
  WS t;
  t.cell_cnt = (int*)take(sizeof(int) * (g.ncell + 1));
  t.cell_start = (int*)take(sizeof(int) * (g.ncell + 1));
  t.cell_of = (int*)take(sizeof(int) * N);
  t.perm = (int*)take(sizeof(int) * N);
  t.iperm = (int*)take(sizeof(int) * N);
  t.spos = (double4*)take(sizeof(double4) * N);
  t.sloc = (float4*)take(sizeof(float4) * N);
  t.stype = (int*)take(sizeof(int) * N);
  t.nbr = (uint16_t*)take(sizeof(uint16_t) * N * (size_t)c.row_cap);
  t.nbr_len = (int*)take(sizeof(int) * N);
  t.wpack = (int*)take(sizeof(int) * WPACK_INTS * (size_t)g.nblock);
  t.wsinfo = (int2*)take(sizeof(int2) * (size_t)c.window_cap * (size_t)g.nblock);
  t.bc = (int*)take(sizeof(int) * N * (size_t)c.cand_cap);
  t.bc_len = (int*)take(sizeof(int) * N);
  t.bkey = (int*)take(sizeof(int) * (size_t)c.bond_cap);
  t.bown = (int*)take(sizeof(int) * (size_t)c.bond_cap);
  t.bc_raw = (double4*)take(sizeof(double4) * N * (size_t)c.cand_cap);
  t.bdeg = (int*)take(sizeof(int) * (N + 1));
  t.brow = (int*)take(sizeof(int) * (N + 1));
  t.bcol = (int*)take(sizeof(int) * (size_t)c.bond_cap);
  t.bmir = (int*)take(sizeof(int) * (size_t)c.bond_cap);
  t.bo = (double*)take(sizeof(double) * 8 * (size_t)c.bond_cap);
  t.delta = (double2*)take(sizeof(double2) * N);
  t.sf = (unsigned long long*)take(3 * sizeof(long long) * N);
  t.erow = (double2*)take(sizeof(double2) * std::max<size_t>(N, (size_t)g.nblock * MAX_SPLIT * NB_WARPS));
  t.epart = (double*)take(sizeof(double) * 2 * ((size_t)nblk((int64_t)std::max<int64_t>(N, 1), FIN_THREADS) + 1));   // k_finalize block partials
  t.ticket = (unsigned*)take(sizeof(unsigned) * 4);
  t.ucol = (int*)take(sizeof(int) * (size_t)c.bond_cap);
  t.ukey = (int*)take(sizeof(int) * (size_t)c.bond_cap);
  t.uown = (int*)take(sizeof(int) * (size_t)c.bond_cap);
  t.uraw = (double4*)take(sizeof(double4) * (size_t)c.bond_cap);
  t.scan_tmp = (long long*)take(sizeof(long long) * nscan);
  t.exp_off = (long long*)take(sizeof(long long) * (N + 1));
  t.lb_status = (unsigned long long*)take(sizeof(unsigned long long) *
                                          ((size_t)nblk(std::max<int64_t>((int64_t)N + 1, (int64_t)g.ncell + 1), LB_TILE) + 1));
  t.lb_ticket = (unsigned*)take(sizeof(unsigned) * 4);
  t.bin_ticket = (unsigned*)take(sizeof(unsigned) * 4);
  const size_t nplan = g.nblock <= NB_PLAN_MAX ? (size_t)g.nblock : 0;   // planned nonbonded units (small grids)
  t.blk_pairs = (int*)take(sizeof(int) * nplan);
  t.blkrow = (int*)take(sizeof(int) * nplan);
  t.units = (int*)take(sizeof(int) * NB_UNIT_SPLIT * nplan);
  t.nunits = (int*)take(sizeof(int) * 4);
  t.ilist_tot = (unsigned long long*)take(sizeof(unsigned long long) * 4);   // [2]: H-atom count (k_hb_collect)
  t.prm = (DevParams*)take(sizeof(DevParams));
  t.st = (Status*)take(sizeof(Status));
  t.h_pos = (double*)take(sizeof(double) * 3 * N);
  t.h_type = (int*)take(sizeof(int) * N);
  t.h_q = (double*)take(sizeof(double) * N);
  t.h_force = (double*)take(sizeof(double) * 3 * N);
  t.h_energy = (double*)take(sizeof(double) * 2);
  t.bep = (BEPair*)take(sizeof(BEPair) * NTP_MAX);
  t.bD = (double*)take(sizeof(double) * N);
  t.bde = t.uraw;   // per-entry bond-energy terms reuse the fill buffer (dead after k_bond_rank)
  if (w) *w = t;
  return o;
}

}  // namespace

// ===================================================================== ctx
struct reax_ctx {
  bool bound = false;
  char* ws_base = nullptr;
  size_t ws_bytes = 0;
  WS w{};
  Grid g{};
  int64_t n = 0;
  reax_capacity cap{};
  reax_cutoffs cut{};
  // pinned host
  Status* h_st = nullptr;
  DevParams* h_prm = nullptr;
  BEPair* h_bep = nullptr;   // staging of the bond-energy parameters (reax_bond_energy)
  size_t maxsm = 0;          // opt-in shared memory per block (bound device)
  bool bep_valid = false;    // device copy matches h_bep
  int bep_nt = 0;
  bool prm_valid = false;  // device copy matches *h_prm
  std::vector<double> prm_key;  // raw reax_params + cutoffs of the last successful build
  // state
  bool lists_ok = false;
  uint64_t list_gen = 0;      // reax_build_lists / reax_step calls (QEq H belongs to one list)
  const void* qeq_scratch = nullptr;
  uint64_t qeq_gen = 0;
  int64_t qeq_P = -1;
  bool qeq_unsorted = false;
  bool bonds_ok = false;
  const double* last_pos = nullptr;
  const int* last_type = nullptr;
  double last_box[3] = {0, 0, 0};
  bool async = false;
  reax_capacity need{};
  // timing
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pending[REAX_NKERNELS];
  double ms_acc[REAX_NKERNELS] = {0};
  int64_t launches_acc[REAX_NKERNELS] = {0};
  int launches_step = 0;
  int launches_cur = 0;
  int nsplit = 1;
  int nsplit_nbr = 1;
  // planned nonbonded units (k_nb_plan) for grids of at most NB_PLAN_MAX blocks
  bool nb_plan = false;
  int nb_slots = 0;     // resident nonbonded CTAs (SMs x NB_MINB)
  int nb_umax = 0;      // launched CTAs (>= planned units; the rest exit)
  float nb_frac = 1.2f; // unit target T = frac * pairs / slots (1.2: measured best at c1 of 0.8-1.5)
  float nb_grid_frac = 0.2f;   // launched units: nblock + grid_frac * slots / frac + 8 (c1 swept 0.12-0.6)
  // fork/join of reax_step (bond chain beside the nonbonded kernel)
  // reax_step_host replays one CUDA graph (copies in, step, copies out) per
  // unchanged (host buffers, box, parameters, workspace, mode)
  cudaGraphExec_t hg_exec = nullptr;
  std::vector<double> hg_key;
  const void* hg_ptr[5] = {};
  char* hg_ws = nullptr;
  bool hg_async = false;
  bool hg_off = getenv("REAX_NO_HOST_GRAPH") != nullptr;
  cudaStream_t side = nullptr;
  cudaStream_t cap_s = nullptr;   // capture stream of the reax_step_host graph
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // reax_step_host: host-to-device copies on their own stream, so that the
  // charges (needed only by the nonbonded kernel) and the types (needed from
  // the cell gather on) arrive while the binning and the list build run
  cudaStream_t copy_s = nullptr;
  cudaEvent_t ev_in0 = nullptr, ev_pos = nullptr, ev_type = nullptr, ev_q = nullptr;
  bool host_in = false;   // do_step: the inputs arrive through ev_pos / ev_type / ev_q
  bool serial = getenv("REAX_SERIAL") != nullptr;
  bool pdl = getenv("REAX_NO_PDL") == nullptr;   // programmatic dependent launch on the hot path
  // REAX_CHAIN_PRIO (measurement): 1 = the side-stream bond chain's kernels at
  // the device's greatest priority, -1 = that on grids without a nonbonded work
  // plan only; default 0 (the default priority).  c4: the step 77.33 -> 77.08 ms
  // with it, but the nonbonded kernel's span in the step 51.8 -> 56.2 ms (the
  // chain's CTAs are dispatched ahead of its pending ones); c1 0.227 -> 0.243 ms
  int chain_prio_env = getenv("REAX_CHAIN_PRIO") ? atoi(getenv("REAX_CHAIN_PRIO")) : 0;
  int prio_hi = 0, prio_lo = 0;   // the device's greatest and least stream priorities
};

namespace {

thread_local cudaError_t g_last_cuda = cudaSuccess;   // reax_last_cuda_error()
reax_status fail_cuda(cudaError_t e) {
  g_last_cuda = e;
  return REAX_ERR_CUDA;
}
reax_status cuda_err(cudaError_t e) { return e == cudaSuccess ? REAX_OK : fail_cuda(e); }

cudaEvent_t take_event(reax_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct Timer {
  reax_ctx* c;
  int k;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  int l0;
  // inside stream capture the events become external event-record nodes, so
  // a replayed graph still reports per-kernel times (reax_kernel_ms, peek mode)
  static void record(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    else cudaEventRecord(e, s);
  }
  Timer(reax_ctx* c_, int k_, cudaStream_t s_) : c(c_), k(k_), s(s_) {
    l0 = c->launches_cur;
    if (c->timing) {
      a = take_event(c);
      record(a, s);
    }
  }
  ~Timer() {
    c->launches_acc[k] += c->launches_cur - l0;
    if (c->timing) {
      cudaEvent_t b = take_event(c);
      record(b, s);
      c->ev_pending[k].push_back({a, b});
    }
  }
};

// REAX_DEBUG=1: report a failing launch (file:line) on stderr (diagnostics only)
const bool g_debug = getenv("REAX_DEBUG") != nullptr;
inline void launch_check(const char* file, int line) {
  if (!g_debug) return;
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) fprintf(stderr, "libreax: launch at %s:%d failed: %s\n", file, line, cudaGetErrorString(e));
}
#define LAUNCH(ctx) (++(ctx)->launches_cur, launch_check(__FILE__, __LINE__))

// Hot-path launches: programmatic dependent launch (each kernel starts with
// griddepcontrol.wait, so a successor's launch and block scheduling overlap
// its predecessor's tail; captured as programmatic edges in CUDA graphs)
template <typename... KArgs, typename... Args>
void launch_k(reax_ctx* c, void (*k)(KArgs...), int grid, int block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = c->pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (s == c->side) {   // kept by graph capture as the kernel node's priority
    const bool hi = c->chain_prio_env == 1 || (c->chain_prio_env < 0 && c->g.nblock > NB_PLAN_MAX);
    at[1].id = cudaLaunchAttributePriority;
    at[1].val.priority = hi ? c->prio_hi : c->prio_lo;
    cfg.numAttrs = 2;
  }
  cudaLaunchKernelEx(&cfg, k, args...);
}

// one-launch scan for the hot path (status cleared by the producing kernel)
cudaError_t scan1(reax_ctx* c, const int* in, int64_t n, int* out, unsigned long long* status, cudaStream_t s) {
  if (n <= 0) return cudaMemsetAsync(out, 0, sizeof(int), s);
  launch_k(c, k_scan_lookback, nblk(n, LB_TILE), LB_THREADS, 0, s, in, (int)n, out, status, c->w.lb_ticket);
  LAUNCH(c);
  return cudaGetLastError();
}

template <typename TI, typename TO>
cudaError_t scan(reax_ctx* c, const TI* in, int64_t n, TO* out, cudaStream_t s) {
  int nparts = nblk(n, SCAN_TILE);
  if (n <= 0) return cudaMemsetAsync(out, 0, sizeof(TO), s);
  k_scan_partial<TI><<<nparts, SCAN_THREADS, 0, s>>>(in, n, c->w.scan_tmp);
  LAUNCH(c);
  k_scan_top<<<1, SCAN_THREADS, 0, s>>>(c->w.scan_tmp, nparts);
  LAUNCH(c);
  k_scan_final<TI, TO><<<nparts, SCAN_THREADS, 0, s>>>(in, n, c->w.scan_tmp, out);
  LAUNCH(c);
  return cudaGetLastError();
}

reax_status interpret_status(reax_ctx* c, cudaStream_t s);

reax_status read_status(reax_ctx* c, cudaStream_t s, bool sync) {
  cudaError_t e = cudaMemcpyAsync(c->h_st, c->w.st, sizeof(Status), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return fail_cuda(e);
  if (!sync) return REAX_OK;
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail_cuda(e);
  return interpret_status(c, s);
}

// the status block read back into h_st (stream synchronised): OK, or the
// error it latched (the device copy is cleared for the next call)
reax_status interpret_status(reax_ctx* c, cudaStream_t s) {
  int f = c->h_st->flags & ~ST_QEQ_UNSORTED;   // informational: a QEq row left in fill order
  if (c->h_st->flags & ST_QEQ_UNSORTED) c->qeq_unsorted = true;
  if (f == 0) {
    if (c->h_st->flags) cudaMemsetAsync(c->w.st, 0, sizeof(Status), s);
    return REAX_OK;
  }
  if (f & (ST_ROW_OVF | ST_CAND_OVF | ST_BOND_OVF | ST_WIN_OVF)) {
    c->need = c->cap;
    if (f & ST_ROW_OVF) c->need.row_cap = std::max(c->cap.row_cap, (c->h_st->max_row + 32) / 32 * 32);
    if (f & ST_CAND_OVF) c->need.cand_cap = std::max(c->cap.cand_cap, c->h_st->max_cand + 4);
    if (f & ST_BOND_OVF) c->need.bond_cap = std::max<int64_t>(c->cap.bond_cap, c->h_st->bonds + 64);
    if (f & ST_WIN_OVF) c->need.window_cap = std::max(c->cap.window_cap, (c->h_st->max_window + 255) / 256 * 256);
    c->lists_ok = c->bonds_ok = false;
    cudaMemsetAsync(c->w.st, 0, sizeof(Status), s);
    return REAX_ERR_CAPACITY;
  }
  cudaMemsetAsync(c->w.st, 0, sizeof(Status), s);
  if (f & ST_TYPE) { c->lists_ok = c->bonds_ok = false; return REAX_ERR_ARG; }
  if (f & ST_HB_OVF) return REAX_ERR_CAPACITY;
  if (f & (ST_NONFINITE_IN | ST_NONFINITE_OUT)) return REAX_ERR_NONFINITE;
  return REAX_ERR_RANGE;
}

// raw parameter values (and cutoffs) as a flat key: rebuilding the tables
// (incl. the host bisection) only when something changed keeps per-call host
// cost to a memcmp, and keeps CUDA-graph capture free of synchronisation
bool params_key(const reax_params* p, const reax_cutoffs* cut, std::vector<double>& k) {
  if (!p || p->ntypes < 1 || p->ntypes > REAX_MAX_TYPES) return false;
  int nt = p->ntypes;
  k.clear();
  k.push_back(nt);
  const double* per_type[] = {p->r_sigma, p->r_pi, p->r_pipi, p->gamma, p->r_vdw, p->eps, p->alpha,
                              p->gamma_w, p->b131, p->b132, p->b133, p->val, p->val_boc};
  for (auto a : per_type) {
    if (!a) return false;
    k.insert(k.end(), a, a + nt);
  }
  const double* per_pair[] = {p->p_bo1, p->p_bo2, p->p_bo3, p->p_bo4, p->p_bo5, p->p_bo6, p->De};
  for (auto a : per_pair) {
    if (!a) return false;
    k.insert(k.end(), a, a + nt * nt);
  }
  double g[] = {p->p_boc1, p->p_boc2, p->p_vdw1, p->coulomb_c, cut->r_nonb, cut->r_bond, cut->bo_cut};
  k.insert(k.end(), g, g + 7);
  return true;
}

size_t nb_smem(int wcap, int row_cap, int nt);

reax_status upload_params(reax_ctx* c, const reax_params* p, const reax_cutoffs* cut, cudaStream_t s) {
  std::vector<double> key;
  if (!params_key(p, cut, key)) return p ? REAX_ERR_PARAM : REAX_ERR_ARG;
  // the nonbonded kernel's shared memory with this table's nt (bind checked
  // nt = 1): windows denser than that are unsupported (REAX_ERR_CAPACITY)
  if (nb_smem(c->cap.window_cap, c->cap.row_cap, p->ntypes) + sizeof(NBSmem) > c->maxsm) return REAX_ERR_CAPACITY;
  if (c->prm_valid && key.size() == c->prm_key.size() &&
      memcmp(key.data(), c->prm_key.data(), key.size() * sizeof(double)) == 0)
    return REAX_OK;
  DevParams d;
  reax_status r = build_params(p, cut, d);
  if (r != REAX_OK) return r;
  if (c->prm_valid && memcmp(&d, c->h_prm, sizeof(DevParams)) == 0) return REAX_OK;
  // the pinned staging buffer may still be read by an earlier async copy
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail_cuda(e);
  memcpy(c->h_prm, &d, sizeof(DevParams));
  e = cudaMemcpyAsync(c->w.prm, c->h_prm, sizeof(DevParams), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return fail_cuda(e);
  c->prm_valid = true;
  c->prm_key.swap(key);
  return REAX_OK;
}

size_t nbr_smem(int wcap, int row_cap = 0) {
  (void)row_cap;
  return (size_t)(wcap + 32) * (sizeof(float4) + sizeof(int) + 1) + 64;
}
size_t nb_smem(int wcap, int row_cap, int nt) {
  return sizeof(double) * (EXP_TBL + 2 * LOG_TBL) + sizeof(NBPair) * nt * nt + (size_t)wcap * (sizeof(int2) + 6 * sizeof(int)) +
         16 + (size_t)NB_WARPS * 2 * ((row_cap + 7) & ~7) * sizeof(uint16_t) + 64;
}
size_t exp_smem(int wcap) { return (size_t)wcap * sizeof(int) + 64; }

reax_status check_common(reax_ctx* c, int64_t n, const double box[3], const reax_cutoffs* cut) {
  if (!c) return REAX_ERR_ARG;
  if (!c->bound) return REAX_ERR_STATE;
  reax_status r = check_box_cut(box, cut);
  if (r != REAX_OK) return r;
  if (n != c->n) return REAX_ERR_STATE;
  if (cut->r_nonb != c->cut.r_nonb) return REAX_ERR_STATE;
  Grid g;
  if (!make_grid(box, cut->r_nonb, g)) return REAX_ERR_BOX;
  for (int k = 0; k < 3; ++k)
    if (g.nc[k] != c->g.nc[k]) return REAX_ERR_STATE;
  c->g = g;  // same topology; box lengths may differ slightly
  return REAX_OK;
}

// a1-a3: binning and the half list (+ bond candidates)
// host_in (reax_step_host): k_bin waits for the positions only (the type
// check moves to the cell gather), the cell gather for the types, and the
// charges are gathered later (launch_q_gather), after their copy
void launch_bin(reax_ctx* c, int N, const double* pos, const int* type, const double* q, int nt, cudaStream_t s) {
  const Grid& g = c->g;
  WS& w = c->w;
  {
    if (c->host_in) cudaStreamWaitEvent(s, c->ev_pos, 0);
    Timer t(c, 0, s);
    const int ctiles = nblk(g.ncell, LB_TILE);
    const bool fused_scan = g.ncell <= BIN_FUSED_SCAN_MAX;
    launch_k(c, k_bin, nblk(std::max<int64_t>(N, ctiles), TPB), TPB, 0, s, N, pos, c->host_in ? nullptr : type, g, nt,
             w.cell_of, w.cell_cnt, w.st, w.lb_status, ctiles, fused_scan ? w.cell_start : nullptr, w.bin_ticket);
    LAUNCH(c);
    if (!fused_scan) scan1(c, w.cell_cnt, g.ncell, w.cell_start, w.lb_status, s);
    launch_k(c, k_scatter, nblk(N, TPB), TPB, 0, s, N, w.cell_of, w.cell_start, w.cell_cnt, w.perm);
    LAUNCH(c);
    if (c->host_in) cudaStreamWaitEvent(s, c->ev_type, 0);
    launch_k(c, k_cell_gather, nblk((int64_t)g.ncell * 32, TPB), TPB, 0, s, g.ncell, w.cell_start, w.perm, pos, type,
             c->host_in ? nullptr : q, g, nt, w.iperm, w.spos, w.sloc, w.stype, w.st,
             c->nb_plan ? w.blk_pairs : nullptr, g.nblock, w.sf);
    LAUNCH(c);
  }
}

// host_in: the charges into the sorted records once their copy has landed
void launch_q_gather(reax_ctx* c, int N, const double* q, cudaStream_t s) {
  WS& w = c->w;
  cudaStreamWaitEvent(s, c->ev_q, 0);
  Timer t(c, 5, s);
  launch_k(c, k_q_gather, nblk(N, TPB), TPB, 0, s, N, q, w.perm, w.spos, w.st);
  LAUNCH(c);
}

// constants of the list build's candidate test (fp32 as the kernel would compute them)
RowTest make_rowtest(const DevParams& p, const Grid& g) {
  RowTest t;
  t.R2lo = p.R2lo;
  t.R2mid = 0.5f * (p.R2lo + p.R2hi);
  t.R2half = 0.5f * (p.R2hi - p.R2lo);
  t.Rt = sqrtf(p.R2hi) + 1e-3f;   // trimming radius (conservative)
  t.hy = (float)g.h[1];
  t.hz = (float)g.h[2];
  t.ihx = 1.0f / (float)g.h[0];
  t.rcmax = p.rcand2_max;
  t.R2 = p.R2;
  return t;
}

// a3-a4: the half list and the bond candidates
void launch_nbr(reax_ctx* c, cudaStream_t s) {
  const Grid& g = c->g;
  WS& w = c->w;
  Timer t(c, 1, s);
  launch_k(c, k_nbr_build, g.nblock * c->nsplit_nbr, NBR_THREADS, nbr_smem(c->cap.window_cap, c->cap.row_cap), s,
           g, w.cell_start, w.sloc, w.spos, w.prm, w.nbr, w.nbr_len, c->cap.row_cap, w.bc, w.bc_len,
           c->cap.cand_cap, c->cap.window_cap, c->nsplit_nbr, w.st, c->nb_plan ? w.blk_pairs : nullptr,
           make_rowtest(*c->h_prm, g), w.wpack, w.wsinfo);
  LAUNCH(c);
}

void launch_lists(reax_ctx* c, int N, const double* pos, const int* type, const double* q, int nt, cudaStream_t s) {
  launch_bin(c, N, pos, type, q, nt, s);
  launch_nbr(c, s);
}

// a4-a5: full bond list with BO' and Delta' (reads spos x/y/z, stype, bond candidates)
void launch_bonds(reax_ctx* c, int N, cudaStream_t s) {
  const Grid& g = c->g;
  WS& w = c->w;
  Timer t(c, 2, s);
  const int btiles = nblk(N, LB_TILE);
  launch_k(c, k_bond_eval, nblk(std::max<int64_t>(N, (int64_t)btiles * 32), TPB), TPB, 0, s, 
      N, w.spos, w.stype, g, w.prm, w.bc, w.bc_len, w.bc_raw, c->cap.cand_cap, w.bdeg, w.lb_status, btiles);
  LAUNCH(c);
  scan1(c, w.bdeg, N, w.brow, w.lb_status, s);
  launch_k(c, k_bond_fill, nblk(N, TPB), TPB, 0, s, N, w.bc, w.bc_len, c->cap.cand_cap, w.brow, w.perm, w.bdeg,
                                          w.ucol, w.ukey, w.uown, reinterpret_cast<long long*>(w.uraw), c->cap.bond_cap, w.st);
  LAUNCH(c);
  launch_k(c, k_bond_rank, 148 * 4, TPB, 0, s, w.brow, w.ucol, w.ukey, w.uown,
           reinterpret_cast<const long long*>(w.uraw), (const double4*)w.bc_raw, w.bcol, w.bkey, w.bown, w.bo,
                                     c->cap.bond_cap, w.st);
  LAUNCH(c);
  launch_k(c, k_bond_delta, nblk(N, TPB), TPB, 0, s, N, w.brow, w.stype, w.prm, w.bo, w.delta, c->cap.bond_cap);
  LAUNCH(c);
}

// a6: corrected bond orders
void launch_bond_correct(reax_ctx* c, cudaStream_t s) {
  Timer t(c, 3, s);
  launch_k(c, k_bond_correct, 148 * 8, TPB, 0, s, c->w.brow, c->w.perm, c->w.stype, c->w.prm, c->w.bcol, c->w.bkey,
                                         c->w.bown, c->w.bmir, c->w.bo, c->w.delta, c->cap.bond_cap, c->w.st);
  LAUNCH(c);
}

reax_status prep_build(reax_ctx* c, int64_t n, const double* pos, const int* type, const double box[3],
                       const reax_params* prm, const reax_cutoffs* cut, cudaStream_t s) {
  reax_status r = check_common(c, n, box, cut);
  if (r != REAX_OK) return r;
  if (n > 0 && (!pos || !type)) return REAX_ERR_ARG;
  r = upload_params(c, prm, cut, s);
  if (r != REAX_OK) return r;
  c->cut = *cut;
  c->lists_ok = c->bonds_ok = false;
  ++c->list_gen;
  return REAX_OK;
}

void note_build(reax_ctx* c, const double* pos, const int* type, const double box[3]) {
  c->last_pos = pos;
  c->last_type = type;
  memcpy(c->last_box, box, sizeof(c->last_box));
}

reax_status do_build_lists(reax_ctx* c, int64_t n, const double* pos, const int* type, const double box[3],
                           const reax_params* prm, const reax_cutoffs* cut, cudaStream_t s) {
  reax_status r = prep_build(c, n, pos, type, box, prm, cut, s);
  if (r != REAX_OK) return r;
  int N = (int)n;
  if (N > 0) {
    launch_lists(c, N, pos, type, nullptr, prm->ntypes, s);
    launch_bonds(c, N, s);
  }
  if (cudaError_t e_ = cudaGetLastError()) return fail_cuda(e_);
  note_build(c, pos, type, box);
  r = read_status(c, s, !c->async);
  if (r != REAX_OK) return r;
  c->lists_ok = true;
  return REAX_OK;
}

reax_status do_bond_orders(reax_ctx* c, const reax_params* prm, const reax_cutoffs* cut, cudaStream_t s) {
  if (!c) return REAX_ERR_ARG;
  if (!c->bound || !c->lists_ok) return REAX_ERR_STATE;
  reax_status r = upload_params(c, prm, cut, s);
  if (r != REAX_OK) return r;
  if (c->n > 0) launch_bond_correct(c, s);
  if (cudaError_t e_ = cudaGetLastError()) return fail_cuda(e_);
  c->bonds_ok = true;
  return REAX_OK;
}

// a7-a8: nonbonded energies and forces (reads the half list, spos, stype, perm/iperm)
// a7: one CTA per (home block, split)
void launch_nb(reax_ctx* c, int nt, cudaStream_t s) {
  const Grid& g = c->g;
  WS& w = c->w;
  if (c->nb_plan) {   // timed with "other", so the nonbonded group times k_nonbonded alone
    Timer tp(c, 5, s);
    launch_k(c, k_nb_plan, 1, PLAN_THREADS, 0, s, g.nblock, (const int*)w.blk_pairs, c->nb_slots, c->nb_frac, c->nb_umax,
             w.units, w.nunits, w.blkrow);
    LAUNCH(c);
  }
  Timer t(c, 4, s);
  launch_k(c, k_nonbonded, c->nb_plan ? c->nb_umax : g.nblock * c->nsplit, NB_THREADS,
           nb_smem(c->cap.window_cap, c->cap.row_cap, nt), s, nt, g, w.spos, w.prm, w.nbr, w.nbr_len,
           c->cap.row_cap, c->cap.window_cap, w.sf, w.erow, c->nsplit, w.st,
           c->nb_plan ? (const int*)w.units : nullptr, c->nb_plan ? (const int*)w.nunits : nullptr, w.blkrow,
           (const int*)w.wpack, (const int2*)w.wsinfo);
  LAUNCH(c);
}

// a8
void launch_finalize(reax_ctx* c, int N, double* force, double* energy, cudaStream_t s) {
  WS& w = c->w;
  Timer t(c, 5, s);
  // one energy partial per half-list row (sorted order), summed in fixed order
  launch_k(c, k_finalize, nblk(N, FIN_THREADS), FIN_THREADS, 0, s, N, w.iperm, w.sf, force, N,
           w.erow, w.epart, w.ticket, energy, 2, w.st);
  LAUNCH(c);
}

// q == nullptr: the charges were gathered by k_cell_gather (reax_step)
void launch_nonbonded(reax_ctx* c, int N, const double* q, double* force, double* energy, int nt, cudaStream_t s) {
  const Grid& g = c->g;
  WS& w = c->w;
  if (q) {
    Timer t(c, 5, s);
    launch_k(c, k_nb_prep, nblk(N, TPB), TPB, 0, s, N, q, w.perm, w.spos, w.sf, w.st);
    LAUNCH(c);
  }
  launch_nb(c, nt, s);
  launch_finalize(c, N, force, energy, s);
}

reax_status check_nonbonded(reax_ctx* c, int64_t n, const double* pos, const int* type, const double* q,
                            const double box[3], const reax_cutoffs* cut, double* force, double* energy) {
  reax_status r = check_common(c, n, box, cut);
  if (r != REAX_OK) return r;
  if (!c->lists_ok) return REAX_ERR_STATE;
  if (pos != c->last_pos || type != c->last_type || memcmp(box, c->last_box, sizeof(c->last_box)) != 0)
    return REAX_ERR_STATE;
  if (!energy || (n > 0 && (!q || !force))) return REAX_ERR_ARG;
  return REAX_OK;
}

reax_status do_nonbonded(reax_ctx* c, int64_t n, const double* pos, const int* type, const double* q,
                         const double box[3], const reax_params* prm, const reax_cutoffs* cut, double* force,
                         double* energy, cudaStream_t s) {
  reax_status r = check_nonbonded(c, n, pos, type, q, box, cut, force, energy);
  if (r != REAX_OK) return r;
  r = upload_params(c, prm, cut, s);
  if (r != REAX_OK) return r;
  if (n == 0) {
    if (cudaError_t e_ = cudaMemsetAsync(energy, 0, 2 * sizeof(double), s)) return fail_cuda(e_);
    return REAX_OK;
  }
  launch_nonbonded(c, (int)n, q, force, energy, prm->ntypes, s);
  if (cudaError_t e_ = cudaGetLastError()) return fail_cuda(e_);
  return read_status(c, s, !c->async);
}

// reax_step: lists on `s`, then a fork: the bond chain (a4-a6, small
// latency-bound kernels) runs on the context's side stream while the
// nonbonded kernel (a7-a8) runs on `s`; both only read the lists and the
// sorted atoms.  The join makes `s` wait for the side stream, so the call is
// stream-ordered on `s` as a whole (and capturable into one CUDA graph).
reax_status do_step(reax_ctx* c, int64_t n, const double* pos, const int* type, const double* q, const double box[3],
                    const reax_params* prm, const reax_cutoffs* cut, double* force, double* energy, cudaStream_t s) {
  reax_status r = prep_build(c, n, pos, type, box, prm, cut, s);
  if (r != REAX_OK) return r;
  if (!energy || (n > 0 && (!q || !force))) return REAX_ERR_ARG;
  const int N = (int)n;
  if (N == 0) {
    note_build(c, pos, type, box);
    c->lists_ok = c->bonds_ok = true;
    if (cudaError_t e_ = cudaMemsetAsync(energy, 0, 2 * sizeof(double), s)) return fail_cuda(e_);
    return REAX_OK;
  }
  // REAX_SERIAL=1 (measurement only): everything on `s`, so per-kernel event
  // times are not shared between concurrent kernels
  const bool fork = !c->serial;
  const int nt = prm->ntypes;
  launch_bin(c, N, pos, type, q, nt, s);
  launch_nbr(c, s);
  // fork: the bond chain (a4-a6, small latency-bound kernels) on the side
  // stream beside the nonbonded kernel (a7) on s; join; k_finalize (a8)
  cudaStream_t sb = s;
  if (fork) {
    if (cudaEventRecord(c->ev_fork, s) != cudaSuccess || cudaStreamWaitEvent(c->side, c->ev_fork, 0) != cudaSuccess)
      return fail_cuda(cudaGetLastError());
    sb = c->side;
  }
  launch_bonds(c, N, sb);
  launch_bond_correct(c, sb);
  if (c->host_in) launch_q_gather(c, N, q, s);
  launch_nb(c, nt, s);
  if (fork && (cudaEventRecord(c->ev_join, c->side) != cudaSuccess || cudaStreamWaitEvent(s, c->ev_join, 0) != cudaSuccess))
    return fail_cuda(cudaGetLastError());
  launch_finalize(c, N, force, energy, s);
  if (cudaError_t e_ = cudaGetLastError()) return fail_cuda(e_);
  note_build(c, pos, type, box);
  c->lists_ok = c->bonds_ok = true;
  r = read_status(c, s, !c->async);
  if (r != REAX_OK) c->lists_ok = c->bonds_ok = false;
  return r;
}

// NEXT-1: bond energy E1 and its forces at the bond set of the last
// reax_bond_orders / reax_step (reading 28)
reax_status do_bond_energy(reax_ctx* c, const reax_params* prm, const reax_bond_params* bp, double* force,
                           double* energy, cudaStream_t s) {
  if (!c || !prm || !bp || !energy) return REAX_ERR_ARG;
  if (!c->bound || !c->lists_ok || !c->bonds_ok) return REAX_ERR_STATE;
  if (c->n > 0 && !force) return REAX_ERR_ARG;
  const int nt = prm->ntypes;
  if (nt < 1 || nt > REAX_MAX_TYPES || !prm->De || !bp->De_pi || !bp->De_pipi || !bp->p_be1 || !bp->p_be2)
    return REAX_ERR_PARAM;
  const double* tab[5] = {prm->De, bp->De_pi, bp->De_pipi, bp->p_be1, bp->p_be2};
  for (int k = 0; k < 5; ++k)
    for (int t = 0; t < nt * nt; ++t) {
      const double v = tab[k][t];
      if (!std::isfinite(v) || v != tab[k][(t % nt) * nt + t / nt]) return REAX_ERR_PARAM;   // finite, symmetric
      if (k == 4 && !(v > 0.0)) return REAX_ERR_PARAM;                                    // BOs^p_be2: p_be2 > 0
    }
  reax_status r = upload_params(c, prm, &c->cut, s);
  if (r != REAX_OK) return r;
  if (c->n == 0) {
    if (cudaError_t e_ = cudaMemsetAsync(energy, 0, sizeof(double), s)) return fail_cuda(e_);
    return REAX_OK;
  }
  WS& w = c->w;
  bool same = c->bep_valid && c->bep_nt == nt;
  for (int t = 0; same && t < nt * nt; ++t) {
    const BEPair v{prm->De[t], bp->De_pi[t], bp->De_pipi[t], bp->p_be1[t], bp->p_be2[t]};
    same = memcmp(&v, &c->h_bep[t], sizeof(BEPair)) == 0;
  }
  if (!same) {   // the pinned staging is only rewritten when the table changes (it may back an in-flight copy)
    if (c->bep_valid && cudaStreamSynchronize(s) != cudaSuccess) return fail_cuda(cudaGetLastError());
    for (int t = 0; t < nt * nt; ++t) c->h_bep[t] = BEPair{prm->De[t], bp->De_pi[t], bp->De_pipi[t], bp->p_be1[t], bp->p_be2[t]};
    if (cudaError_t e_ = cudaMemcpyAsync(w.bep, c->h_bep, sizeof(BEPair) * nt * nt, cudaMemcpyHostToDevice, s))
      return fail_cuda(e_);
    c->bep_valid = true;
    c->bep_nt = nt;
  }
  const int N = (int)c->n;
  {
    Timer t(c, 6, s);
    launch_k(c, k_bond_energy_terms, 148 * 8, TPB, 0, s, w.perm, w.stype, w.spos, c->g, w.prm, w.bep, w.bcol, w.bkey,
             w.bown, w.bmir, w.bo, w.delta, w.bde, c->cap.bond_cap, w.st);
    LAUNCH(c);
    launch_k(c, k_bond_energy_rows, nblk(N, TPB), TPB, 0, s, N, w.brow, w.bde, w.bD, c->cap.bond_cap);
    LAUNCH(c);
    launch_k(c, k_bond_energy_out, nblk(N, FIN_THREADS), FIN_THREADS, 0, s, N, w.perm, w.spos, c->g, w.brow, w.bcol,
             w.bde, w.bD, c->cap.bond_cap, force, w.epart, w.ticket, energy, w.st);
    LAUNCH(c);
  }
  if (cudaError_t e_ = cudaGetLastError()) return fail_cuda(e_);
  return read_status(c, s, !c->async);
}

// NEXT-3: interaction lists (3-body angles, H-bonds) of the current bond
// list and positions (readings 30-31)
reax_status ilist_prepare(reax_ctx* c, const reax_ilist_params* p, IList& il) {
  if (!c || !p) return REAX_ERR_ARG;
  if (!c->bound || !c->lists_ok || !c->bonds_ok) return REAX_ERR_STATE;
  if (!(std::isfinite(p->thb_cut) && p->thb_cut >= 0.0 && std::isfinite(p->thb_cutsq) && p->thb_cutsq >= 0.0))
    return REAX_ERR_PARAM;
  const double hmin = std::min(c->g.h[0], std::min(c->g.h[1], c->g.h[2]));
  const double lmin = std::min(c->g.L[0], std::min(c->g.L[1], c->g.L[2]));
  // the H-bond search covers +-SR sub-cells; one periodic image within r_hb
  if (!(std::isfinite(p->r_hb) && p->r_hb > 0.0 && p->r_hb <= SR * hmin && 2.0 * p->r_hb < lmin)) return REAX_ERR_CUTOFF;
  if (p->h_type < 0 || p->h_type >= NT_MAX) return REAX_ERR_PARAM;
  il.thb_cut = p->thb_cut;
  il.thb_cutsq = p->thb_cutsq;
  il.r_hb2 = p->r_hb * p->r_hb;
  il.h_type = p->h_type;
  il.acc_mask = p->acceptor_mask;
  return REAX_OK;
}

reax_status do_ilist_counts(reax_ctx* c, const reax_ilist_params* p, int64_t* n_angles, int64_t* n_hbonds,
                            cudaStream_t s) {
  IList il;
  reax_status r = ilist_prepare(c, p, il);
  if (r != REAX_OK) return r;
  unsigned long long tot[2] = {0, 0};
  const int N = (int)c->n;
  if (N > 0) {
    WS& w = c->w;
    if (cudaError_t e_ = cudaMemsetAsync(w.ilist_tot, 0, 4 * sizeof(unsigned long long), s)) return fail_cuda(e_);
    k_ang_count<<<148 * 8, TPB, 0, s>>>(w.brow, w.bown, w.perm, w.bo, nullptr, nullptr, w.ilist_tot,
                                        c->cap.bond_cap, il, w.st);
    unsigned* hn = reinterpret_cast<unsigned*>(w.ilist_tot + 2);
    k_hb_collect<<<nblk(N, TPB), TPB, 0, s>>>(N, w.stype, w.brow, w.perm, il.h_type, w.bc_len, w.cell_of, hn);
    k_hb_list<<<148 * 8, HB_THREADS, 0, s>>>(w.cell_of, hn, c->g, w.cell_start, w.spos, w.stype, w.perm, il, w.bc_len,
                                             w.ilist_tot + 1, nullptr, nullptr, w.st);
    if (cudaError_t e_ = cudaGetLastError()) return fail_cuda(e_);
    if (cudaError_t e_ = cudaMemcpyAsync(tot, w.ilist_tot, sizeof(tot), cudaMemcpyDeviceToHost, s)) return fail_cuda(e_);
    if (cudaError_t e_ = cudaStreamSynchronize(s)) return fail_cuda(e_);
  }
  if (n_angles) *n_angles = (int64_t)tot[0];
  if (n_hbonds) *n_hbonds = (int64_t)tot[1];
  return REAX_OK;
}

reax_status do_ilist_lists(reax_ctx* c, const reax_ilist_params* p, int64_t* ang_off, int32_t* ang_k, int64_t* hb_off,
                           int32_t* hb_z, cudaStream_t s) {
  IList il;
  reax_status r = ilist_prepare(c, p, il);
  if (r != REAX_OK) return r;
  if (!ang_off || !hb_off) return REAX_ERR_ARG;
  const int N = (int)c->n;
  WS& w = c->w;
  if (N == 0) {
    if (cudaMemsetAsync(ang_off, 0, sizeof(int64_t), s) != cudaSuccess ||
        cudaMemsetAsync(hb_off, 0, sizeof(int64_t), s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
      return fail_cuda(cudaGetLastError());
    return REAX_OK;
  }
  int B = 0;
  if (cudaMemcpyAsync(&B, w.brow + N, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return fail_cuda(cudaGetLastError());
  // angles: exported row offsets of the bond list, per-entry counts at the
  // exported positions, prefix sum, fill
  k_export_bond_deg<<<nblk(N, TPB), TPB, 0, s>>>(N, w.iperm, w.brow, w.bc_len);
  if (scan<int, long long>(c, w.bc_len, N, w.exp_off, s) != cudaSuccess) return fail_cuda(cudaGetLastError());
  k_ang_count<<<148 * 8, TPB, 0, s>>>(w.brow, w.bown, w.perm, w.bo, w.exp_off, w.ucol, nullptr, c->cap.bond_cap, il,
                                      w.st);
  if (B > 0) {
    if (scan<int, long long>(c, w.ucol, B, reinterpret_cast<long long*>(ang_off), s) != cudaSuccess)
      return fail_cuda(cudaGetLastError());
    if (ang_k)
      k_ang_fill<<<148 * 8, TPB, 0, s>>>(w.brow, w.bown, w.perm, w.bkey, w.bo, w.exp_off,
                                         reinterpret_cast<const long long*>(ang_off), ang_k, c->cap.bond_cap, il, w.st);
  } else if (cudaMemsetAsync(ang_off, 0, sizeof(int64_t), s) != cudaSuccess) {
    return fail_cuda(cudaGetLastError());
  }
  // H-bonds: per-atom counts, prefix sum, fill
  unsigned* hn = reinterpret_cast<unsigned*>(w.ilist_tot + 2);
  if (cudaError_t e_ = cudaMemsetAsync(hn, 0, sizeof(unsigned), s)) return fail_cuda(e_);
  k_hb_collect<<<nblk(N, TPB), TPB, 0, s>>>(N, w.stype, w.brow, w.perm, il.h_type, w.bc_len, w.cell_of, hn);
  k_hb_list<<<148 * 8, HB_THREADS, 0, s>>>(w.cell_of, hn, c->g, w.cell_start, w.spos, w.stype, w.perm, il, w.bc_len,
                                           nullptr, nullptr, nullptr, w.st);
  if (scan<int, long long>(c, w.bc_len, N, reinterpret_cast<long long*>(hb_off), s) != cudaSuccess)
    return fail_cuda(cudaGetLastError());
  if (hb_z)
    k_hb_list<<<148 * 8, HB_THREADS, 0, s>>>(w.cell_of, hn, c->g, w.cell_start, w.spos, w.stype, w.perm, il, nullptr,
                                             nullptr, reinterpret_cast<const long long*>(hb_off), hb_z, w.st);
  if (cudaError_t e_ = cudaGetLastError()) return fail_cuda(e_);
  return read_status(c, s, true);
}

// NEXT-4: species analysis of the current corrected bond orders
// (reading 32).  Scratch layout (caller-owned):
struct SpLayout {
  size_t parent, isroot, comp, out_comp, rank, out_cnt, table, nsp, total;
  unsigned tsize;
};
SpLayout sp_layout(int64_t n, int nt) {
  SpLayout L;
  const size_t N = (size_t)std::max<int64_t>(n, 1);
  unsigned t = 1024;
  while ((size_t)t < 2 * N) t <<= 1;
  L.tsize = t;
  size_t o = 0;
  auto take = [&](size_t bytes) { const size_t at = o; o = (o + bytes + 255) & ~(size_t)255; return at; };
  L.parent = take(4 * N);
  L.isroot = take(4 * N);
  L.comp = take(4 * N * nt);
  L.out_comp = take(4 * N * nt);
  L.rank = take(8 * (N + 1));
  L.out_cnt = take(8 * N);
  L.table = take(8 * (size_t)t);
  L.nsp = take(16);
  L.total = o;
  return L;
}

reax_status do_species(reax_ctx* c, const double* thresh, void* scratch, size_t scratch_bytes, int32_t* mol_id,
                       int64_t* n_molecules, int32_t* sp_comp, int64_t* sp_count, int64_t sp_cap, int64_t* n_species,
                       cudaStream_t s) {
  if (!c || !n_molecules || !n_species) return REAX_ERR_ARG;
  if (!c->bound || !c->lists_ok || !c->bonds_ok || !c->prm_valid) return REAX_ERR_STATE;
  const int nt = c->h_prm->nt;
  const int N = (int)c->n;
  if (sp_cap < 0 || (sp_cap > 0 && (!sp_comp || !sp_count)) || (N > 0 && !mol_id)) return REAX_ERR_ARG;
  SpThr thr;
  for (int t = 0; t < nt * nt; ++t) {
    const double v = thresh ? thresh[t] : 0.3;
    if (!std::isfinite(v) || (thresh && v != thresh[(t % nt) * nt + t / nt])) return REAX_ERR_PARAM;
    thr.t[t] = v;
  }
  *n_molecules = 0;
  *n_species = 0;
  if (N == 0) return REAX_OK;
  const SpLayout L = sp_layout(N, nt);
  if (!scratch || scratch_bytes < L.total) return REAX_ERR_CAPACITY;
  if (((uintptr_t)scratch) % 256 != 0) return REAX_ERR_ARG;
  char* b = (char*)scratch;
  int* parent = (int*)(b + L.parent);
  int* isroot = (int*)(b + L.isroot);
  int* comp = (int*)(b + L.comp);
  int* out_comp = (int*)(b + L.out_comp);
  long long* rank = (long long*)(b + L.rank);
  long long* out_cnt = (long long*)(b + L.out_cnt);
  int2* table = (int2*)(b + L.table);
  unsigned* nsp = (unsigned*)(b + L.nsp);
  WS& w = c->w;
  {
    Timer t(c, 7, s);
    if (cudaMemsetAsync(comp, 0, 4 * (size_t)N * nt, s) != cudaSuccess ||
        cudaMemsetAsync(table, 0xff, 8 * (size_t)L.tsize, s) != cudaSuccess ||   // rep = -1 (and count -1, reset below)
        cudaMemsetAsync(nsp, 0, 16, s) != cudaSuccess)
      return fail_cuda(cudaGetLastError());
    k_sp_init<<<nblk(N, TPB), TPB, 0, s>>>(N, parent);
    LAUNCH(c);
    k_sp_union<<<148 * 8, TPB, 0, s>>>(w.brow, N, w.bown, w.bcol, w.bkey, w.perm, w.stype, w.bo, c->cap.bond_cap, nt,
                                        thr, parent);
    LAUNCH(c);
    k_sp_count<<<nblk(N, TPB), TPB, 0, s>>>(N, w.perm, w.stype, nt, parent, isroot, comp);
    LAUNCH(c);
    if (scan<int, long long>(c, isroot, N, rank, s) != cudaSuccess) return fail_cuda(cudaGetLastError());
    k_sp_label<<<nblk(N, TPB), TPB, 0, s>>>(N, parent, rank, mol_id, comp, nt, table, L.tsize - 1);
    LAUNCH(c);
    k_sp_collect<<<nblk(L.tsize, TPB), TPB, 0, s>>>(L.tsize, table, comp, nt, out_comp, out_cnt, nsp);
    LAUNCH(c);
  }
  if (cudaError_t e_ = cudaGetLastError()) return fail_cuda(e_);
  long long M = 0;
  unsigned S = 0;
  if (cudaMemcpyAsync(&M, rank + N, sizeof(long long), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaMemcpyAsync(&S, nsp, sizeof(unsigned), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return fail_cuda(cudaGetLastError());
  std::vector<int> hc((size_t)S * nt);
  std::vector<long long> hn(S);
  if (S > 0 && (cudaMemcpyAsync(hc.data(), out_comp, sizeof(int) * hc.size(), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                cudaMemcpyAsync(hn.data(), out_cnt, sizeof(long long) * S, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                cudaStreamSynchronize(s) != cudaSuccess))
    return fail_cuda(cudaGetLastError());
  // the table's slot order is arbitrary: species sorted by composition
  std::vector<unsigned> ord(S);
  for (unsigned k = 0; k < S; ++k) ord[k] = k;
  std::sort(ord.begin(), ord.end(), [&](unsigned x, unsigned y) {
    return std::lexicographical_compare(hc.begin() + (size_t)x * nt, hc.begin() + (size_t)(x + 1) * nt,
                                        hc.begin() + (size_t)y * nt, hc.begin() + (size_t)(y + 1) * nt);
  });
  for (unsigned k = 0; k < S && (int64_t)k < sp_cap; ++k) {
    for (int t = 0; t < nt; ++t) sp_comp[(size_t)k * nt + t] = hc[(size_t)ord[k] * nt + t];
    sp_count[k] = hn[ord[k]] + 1;   // the count word started at -1 (0xffffffff)
  }
  *n_molecules = M;
  *n_species = S;
  if ((int64_t)S > sp_cap) return REAX_ERR_CAPACITY;
  return read_status(c, s, true);
}

// NEXT-2: QEq (reading 33).  Caller-owned
// scratch (sorted order): row offsets, lower-segment counts and cursors, the
// doubly stored H (column, value), the interleaved CG vectors, partials.
struct QLayout {
  size_t off, lcnt, cur, hcol, hval, x, r, z, p, Ap, part, part2, stt, total;
};
QLayout qeq_layout(int64_t n, int64_t P) {
  QLayout L;
  const size_t N = (size_t)std::max<int64_t>(n, 1), E = (size_t)std::max<int64_t>(2 * P, 1);
  size_t o = 0;
  auto take = [&](size_t bytes) { const size_t at = o; o = (o + bytes + 255) & ~(size_t)255; return at; };
  L.off = take(8 * (N + 1));
  L.lcnt = take(4 * N);
  L.cur = take(4 * N);
  L.hcol = take(4 * E);
  L.hval = take(8 * E);
  L.x = take(16 * N);
  L.r = take(16 * N);
  L.z = take(16 * N);
  L.p = take(16 * N);
  L.Ap = take(16 * N);
  L.part = take(8 * 6 * QEQ_GRID);
  L.part2 = take(8 * 6 * QEQ_GRID);
  L.stt = take(sizeof(QEqState));
  L.total = o;
  return L;
}

reax_status half_pairs(reax_ctx* c, cudaStream_t s, int64_t* P) {
  long long p = 0;
  if (c->n > 0) {
    if (scan<int, long long>(c, c->w.nbr_len, c->n, c->w.exp_off, s) != cudaSuccess ||
        cudaMemcpyAsync(&p, c->w.exp_off + c->n, sizeof(long long), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return fail_cuda(cudaGetLastError());
  }
  *P = p;
  return REAX_OK;
}

reax_status do_qeq_build(reax_ctx* c, void* scratch, size_t bytes, cudaStream_t s) {
  if (!c) return REAX_ERR_ARG;
  if (!c->bound || !c->lists_ok || !c->prm_valid) return REAX_ERR_STATE;
  int64_t P = 0;
  reax_status r = half_pairs(c, s, &P);
  if (r != REAX_OK) return r;
  const QLayout L = qeq_layout(c->n, P);
  if (!scratch || bytes < L.total) return REAX_ERR_CAPACITY;
  if (((uintptr_t)scratch) % 256 != 0) return REAX_ERR_ARG;
  c->qeq_scratch = nullptr;
  const int N = (int)c->n;
  if (N > 0) {
    char* b = (char*)scratch;
    long long* off = (long long*)(b + L.off);
    int* lcnt = (int*)(b + L.lcnt);
    int* cur = (int*)(b + L.cur);
    WS& w = c->w;
    Timer t(c, 8, s);
    const size_t sm = (size_t)c->cap.window_cap * (sizeof(int) + 1) + 64;
    if (ensure_smem(k_qeq_hbuild, sm) != cudaSuccess) return fail_cuda(cudaGetLastError());
    if (cudaMemsetAsync(lcnt, 0, 4 * (size_t)N, s) != cudaSuccess ||
        cudaMemsetAsync(cur, 0, 4 * (size_t)N, s) != cudaSuccess)
      return fail_cuda(cudaGetLastError());
    k_qeq_hbuild<<<c->g.nblock, NBR_THREADS, sm, s>>>(c->g, w.cell_start, w.spos, w.stype, w.prm, w.nbr, w.nbr_len,
                                                      c->cap.row_cap, c->cap.window_cap, 0, lcnt, nullptr, nullptr,
                                                      nullptr, nullptr);
    LAUNCH(c);
    k_qeq_rowlen<<<nblk(N, TPB), TPB, 0, s>>>(N, w.nbr_len, lcnt);   // lcnt += len (row degree)
    LAUNCH(c);
    if (scan<int, long long>(c, lcnt, N, off, s) != cudaSuccess) return fail_cuda(cudaGetLastError());
    k_qeq_hbuild<<<c->g.nblock, NBR_THREADS, sm, s>>>(c->g, w.cell_start, w.spos, w.stype, w.prm, w.nbr, w.nbr_len,
                                                      c->cap.row_cap, c->cap.window_cap, 1, nullptr, off, cur,
                                                      (int*)(b + L.hcol), (double*)(b + L.hval));
    LAUNCH(c);
    k_qeq_sortlow<<<QEQ_GRID * 2, QEQ_SORT_THREADS, 0, s>>>(N, off, w.nbr_len, (int*)(b + L.hcol), (double*)(b + L.hval), w.st);
    LAUNCH(c);
  }
  if (cudaError_t e_ = cudaGetLastError()) return fail_cuda(e_);
  r = read_status(c, s, true);
  if (r != REAX_OK) return r;
  c->qeq_scratch = scratch;
  c->qeq_gen = c->list_gen;
  c->qeq_P = P;
  return REAX_OK;
}

reax_status qeq_types(reax_ctx* c, const double* chi, const double* eta, QEqType& ty) {
  const int nt = c->h_prm->nt;
  if (!eta) return REAX_ERR_ARG;
  memset(&ty, 0, sizeof(ty));
  for (int t = 0; t < nt; ++t) {
    if (!(std::isfinite(eta[t]) && eta[t] > 0.0)) return REAX_ERR_PARAM;
    if (chi && !std::isfinite(chi[t])) return REAX_ERR_PARAM;
    ty.eta[t] = eta[t];
    ty.chi[t] = chi ? chi[t] : 0.0;
  }
  return REAX_OK;
}

reax_status qeq_ready(reax_ctx* c, const void* scratch, size_t bytes, QLayout& L) {
  if (!c->bound || !c->lists_ok || !c->prm_valid) return REAX_ERR_STATE;
  if (!scratch || scratch != c->qeq_scratch || c->qeq_gen != c->list_gen) return REAX_ERR_STATE;
  L = qeq_layout(c->n, c->qeq_P);
  if (bytes < L.total) return REAX_ERR_CAPACITY;
  return REAX_OK;
}

reax_status do_qeq_matvec(reax_ctx* c, const double* eta, void* scratch, size_t bytes, const double* x0,
                          const double* x1, double* y0, double* y1, cudaStream_t s) {
  if (!c) return REAX_ERR_ARG;
  QLayout L;
  reax_status r = qeq_ready(c, scratch, bytes, L);
  if (r != REAX_OK) return r;
  QEqType ty;
  r = qeq_types(c, nullptr, eta, ty);
  if (r != REAX_OK) return r;
  const int N = (int)c->n;
  if (N == 0) return REAX_OK;
  if (!x0 || !x1 || !y0 || !y1) return REAX_ERR_ARG;
  char* b = (char*)scratch;
  double2* x = (double2*)(b + L.x);
  double2* y = (double2*)(b + L.Ap);
  WS& w = c->w;
  k_qeq_gather<<<QEQ_GRID, QEQ_THREADS, 0, s>>>(N, w.perm, x0, x1, x);
  k_qeq_spmv<<<QEQ_GRID, QEQ_THREADS, 0, s>>>(N, (const long long*)(b + L.off), (const int*)(b + L.hcol),
                                             (const double*)(b + L.hval), w.stype, ty, x, y, nullptr);
  k_qeq_scatter<<<QEQ_GRID, QEQ_THREADS, 0, s>>>(N, w.perm, y, y0, y1, (double*)(b + L.part));
  if (cudaError_t e_ = cudaGetLastError()) return fail_cuda(e_);
  if (cudaError_t e_ = cudaStreamSynchronize(s)) return fail_cuda(e_);
  return REAX_OK;
}

reax_status do_qeq_solve(reax_ctx* c, const double* chi, const double* eta, double tol, int maxiter, void* scratch,
                         size_t bytes, double* sv, double* tv, double* q, int32_t* iters, cudaStream_t s) {
  if (!c || !chi || !iters) return REAX_ERR_ARG;
  QLayout L;
  reax_status r = qeq_ready(c, scratch, bytes, L);
  if (r != REAX_OK) return r;
  QEqType ty;
  r = qeq_types(c, chi, eta, ty);
  if (r != REAX_OK) return r;
  if (!(std::isfinite(tol) && tol >= 0.0) || maxiter < 0) return REAX_ERR_ARG;
  iters[0] = iters[1] = 0;
  const int N = (int)c->n;
  if (N == 0) return REAX_OK;
  if (!sv || !tv || !q) return REAX_ERR_ARG;
  char* b = (char*)scratch;
  const long long* off = (const long long*)(b + L.off);
  const int* hcol = (const int*)(b + L.hcol);
  const double* hval = (const double*)(b + L.hval);
  double2 *x = (double2*)(b + L.x), *rr = (double2*)(b + L.r), *z = (double2*)(b + L.z), *p = (double2*)(b + L.p),
          *Ap = (double2*)(b + L.Ap);
  double *part = (double*)(b + L.part), *part2 = (double*)(b + L.part2);
  QEqState* stt = (QEqState*)(b + L.stt);
  WS& w = c->w;
  Timer tm(c, 8, s);
  k_qeq_gather<<<QEQ_GRID, QEQ_THREADS, 0, s>>>(N, w.perm, sv, tv, x);
  k_qeq_spmv<<<QEQ_GRID, QEQ_THREADS, 0, s>>>(N, off, hcol, hval, w.stype, ty, x, Ap, nullptr);
  k_qeq_start<<<QEQ_GRID, QEQ_THREADS, 0, s>>>(N, w.stype, ty, Ap, rr, z, p, part);
  k_qeq_start_state<<<1, QEQ_THREADS, 0, s>>>(part, tol, maxiter, stt);
  int act[2] = {1, 1};
  // the kernels of an iteration return at once when both systems have
  // converged, so the host reads the flags only every QEQ_CHECK iterations
  constexpr int QEQ_CHECK = 8;
  for (int it = 0; it < maxiter; ++it) {
    const int par = it & 1;
    if (it > 0 && it % QEQ_CHECK == 0) {
      if (cudaMemcpyAsync(act, &stt->active[par][0], sizeof(act), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
          cudaStreamSynchronize(s) != cudaSuccess)
        return fail_cuda(cudaGetLastError());
      if (!act[0] && !act[1]) break;
    }
    k_qeq_spmv<<<QEQ_GRID, QEQ_THREADS, 0, s>>>(N, off, hcol, hval, w.stype, ty, p, Ap, part, stt, par);
    k_qeq_update<<<QEQ_GRID, QEQ_THREADS, 0, s>>>(N, w.stype, ty, part, stt, par, x, rr, z, p, Ap, part2);
    k_qeq_direction<<<QEQ_GRID, QEQ_THREADS, 0, s>>>(N, part2, stt, par, tol, maxiter, z, p);
    c->launches_cur += 3;
  }
  k_qeq_scatter<<<QEQ_GRID, QEQ_THREADS, 0, s>>>(N, w.perm, x, sv, tv, part);
  k_qeq_charges<<<QEQ_GRID, QEQ_THREADS, 0, s>>>(N, part, sv, tv, q);
  if (cudaError_t e_ = cudaGetLastError()) return fail_cuda(e_);
  int it2[2] = {0, 0};
  if (cudaMemcpyAsync(it2, stt->iters, sizeof(it2), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaMemcpyAsync(act, &stt->active[maxiter & 1][0], sizeof(act), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return fail_cuda(cudaGetLastError());
  iters[0] = it2[0];
  iters[1] = it2[1];
  r = read_status(c, s, true);
  if (r != REAX_OK) return r;
  // not converged within maxiter (iterations stopped by the cap)
  double rr_h[2], bb_h[2];
  if (cudaMemcpy(rr_h, stt->rr, sizeof(rr_h), cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(bb_h, stt->bb, sizeof(bb_h), cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail_cuda(cudaGetLastError());
  for (int k = 0; k < 2; ++k)
    if (!(rr_h[k] <= tol * tol * bb_h[k])) return REAX_ERR_CONVERGENCE;
  return REAX_OK;
}

}  // namespace

// ==================================================================== ABI
extern "C" {

#ifdef REAX_TIMELINE
// measurement builds only: copy the CTA timeline (see TL_MARK) to host,
// [2][TL_MAX][4] unsigned 64-bit words; returns TL_MAX
int reax_timeline_read(void* host) {
  if (cudaMemcpyFromSymbol(host, g_tl, sizeof(g_tl)) != cudaSuccess) return -1;
  if (cudaMemcpyFromSymbol((char*)host + sizeof(g_tl), g_tl_span, sizeof(g_tl_span)) != cudaSuccess) return -1;
  return TL_MAX;
}
// reset the span stamps (first start = max, last end = 0)
int reax_timeline_reset(void) {
  unsigned long long v[8][2];
  for (int i = 0; i < 8; ++i) { v[i][0] = ~0ull; v[i][1] = 0ull; }
  return cudaMemcpyToSymbol(g_tl_span, v, sizeof(v)) == cudaSuccess ? 0 : -1;
}
#endif

const char* reax_last_cuda_error(void) { return cudaGetErrorString(g_last_cuda); }


const char* reax_status_str(reax_status s) {
  switch (s) {
    case REAX_OK: return "ok";
    case REAX_ERR_ARG: return "invalid argument";
    case REAX_ERR_BOX: return "box length must be finite and > 2 r_nonb";
    case REAX_ERR_CUTOFF: return "invalid cutoffs (need 0 < r_bond <= r_nonb, 0 < bo_cut < 1)";
    case REAX_ERR_PARAM: return "invalid parameter table";
    case REAX_ERR_CAPACITY: return "workspace capacity exceeded (see reax_required)";
    case REAX_ERR_NONFINITE: return "non-finite input or output";
    case REAX_ERR_CUDA: return "CUDA error";
    case REAX_ERR_STATE: return "invalid call sequence or binding";
    case REAX_ERR_RANGE: return "force contribution outside the fixed-point accumulator range (>= 65536 kcal/mol/A)";
    case REAX_ERR_CONVERGENCE: return "QEq not converged within maxiter";
  }
  return "unknown";
}

reax_status reax_create(reax_ctx** out) {
  if (!out) return REAX_ERR_ARG;
  *out = nullptr;
  if (ensure_tables() != cudaSuccess) return REAX_ERR_CUDA;
  reax_ctx* c = new reax_ctx();
  if (cudaHostAlloc((void**)&c->h_st, sizeof(Status), cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc((void**)&c->h_prm, sizeof(DevParams), cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc((void**)&c->h_bep, sizeof(BEPair) * NTP_MAX, cudaHostAllocDefault) != cudaSuccess) {
    if (c->h_prm) cudaFreeHost(c->h_prm);
    if (c->h_st) cudaFreeHost(c->h_st);
    delete c;
    return REAX_ERR_CUDA;
  }
  memset(c->h_st, 0, sizeof(Status));
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  c->prio_hi = prio_hi;
  c->prio_lo = prio_lo;
  // the side stream at the greatest priority; its kernels carry their own (launch attribute)
  bool ok = cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, prio_hi) == cudaSuccess &&
            cudaStreamCreateWithFlags(&c->cap_s, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) == cudaSuccess &&
            cudaStreamCreateWithFlags(&c->copy_s, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&c->ev_in0, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&c->ev_pos, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&c->ev_type, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&c->ev_q, cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    reax_destroy(c);
    return REAX_ERR_CUDA;
  }
  *out = c;
  return REAX_OK;
}

reax_status reax_destroy(reax_ctx* c) {
  if (!c) return REAX_ERR_ARG;
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  for (int k = 0; k < REAX_NKERNELS; ++k)
    for (auto& p : c->ev_pending[k]) {
      cudaEventDestroy(p.first);
      cudaEventDestroy(p.second);
    }
  if (c->h_st) cudaFreeHost(c->h_st);
  if (c->h_prm) cudaFreeHost(c->h_prm);
  if (c->h_bep) cudaFreeHost(c->h_bep);
  if (c->hg_exec) cudaGraphExecDestroy(c->hg_exec);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->cap_s) cudaStreamDestroy(c->cap_s);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->copy_s) cudaStreamDestroy(c->copy_s);
  for (cudaEvent_t e : {c->ev_in0, c->ev_pos, c->ev_type, c->ev_q})
    if (e) cudaEventDestroy(e);
  delete c;
  return REAX_OK;
}

reax_status reax_workspace_bytes(int64_t n, const double box[3], const reax_cutoffs* cut, const reax_capacity* cap,
                                 size_t* bytes, reax_capacity* cap_out) {
  if (!bytes || n < 0 || n >= (1LL << 31) - 1) return REAX_ERR_ARG;
  reax_status r = check_box_cut(box, cut);
  if (r != REAX_OK) return r;
  Grid g;
  if (!make_grid(box, cut->r_nonb, g)) return REAX_ERR_BOX;
  reax_capacity c;
  resolve_caps(n, box, cut, cap, c);
  *bytes = layout(n, g, c, nullptr, nullptr);
  if (cap_out) *cap_out = c;
  return REAX_OK;
}

reax_status reax_bind_workspace(reax_ctx* ctx, void* ws, size_t bytes, int64_t n, const double box[3],
                                const reax_cutoffs* cut, const reax_capacity* cap) {
  if (!ctx || !ws || n < 0 || n >= (1LL << 31) - 1) return REAX_ERR_ARG;
  reax_status r = check_box_cut(box, cut);
  if (r != REAX_OK) return r;
  Grid g;
  if (!make_grid(box, cut->r_nonb, g)) return REAX_ERR_BOX;
  reax_capacity c;
  resolve_caps(n, box, cut, cap, c);
  if (c.row_cap > 65535 || c.window_cap > 65535 || c.cand_cap < 1) return REAX_ERR_ARG;
  size_t need = layout(n, g, c, nullptr, nullptr);
  if (bytes < need) return REAX_ERR_CAPACITY;
  if (((uintptr_t)ws) % ALIGN != 0) return REAX_ERR_ARG;
  // shared memory limits of the window kernels
  int dev = 0, maxsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // shared memory of the window kernels: the nonbonded kernel's also holds
  // the nt*nt pair table, checked with the real nt when parameters arrive
  // (upload_params); here with nt = 1
  size_t s1 = nbr_smem(c.window_cap, c.row_cap) + sizeof(NbrSmem), s2 = nb_smem(c.window_cap, c.row_cap, 1) + sizeof(NBSmem);
  if ((size_t)maxsm < s1 || (size_t)maxsm < s2) return REAX_ERR_CAPACITY;
  size_t nb_attr = std::min<size_t>(nb_smem(c.window_cap, c.row_cap, NT_MAX), (size_t)maxsm - sizeof(NBSmem));
  if (ensure_smem(k_nbr_build, nbr_smem(c.window_cap, c.row_cap)) != cudaSuccess ||
      ensure_smem(k_nonbonded, nb_attr) != cudaSuccess ||
      ensure_smem(k_export_pairs, exp_smem(c.window_cap)) != cudaSuccess)
    return REAX_ERR_CUDA;

  // a graph captured by reax_step_host holds the old layout's offsets and
  // capacities: never replay it on the new workspace (even at the same base)
  if (ctx->hg_exec) {
    cudaGraphExecDestroy(ctx->hg_exec);
    ctx->hg_exec = nullptr;
  }
  ctx->hg_key.clear();
  memset(ctx->hg_ptr, 0, sizeof(ctx->hg_ptr));
  ctx->hg_ws = nullptr;
  ctx->maxsm = (size_t)maxsm;
  ctx->ws_base = (char*)ws;
  ctx->ws_bytes = bytes;
  layout(n, g, c, ctx->ws_base, &ctx->w);
  ctx->g = g;
  ctx->n = n;
  ctx->cap = c;
  ctx->nsplit = choose_split(g.nblock, 2, "REAX_CTAS_PER_SM");
  ctx->nsplit_nbr = choose_split(g.nblock, 4, "REAX_NBR_CTAS_PER_SM");
  if (const char* e = getenv("REAX_NBR_SPLIT")) ctx->nsplit_nbr = std::max(1, std::min(MAX_SPLIT, atoi(e)));
  {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    ctx->nb_slots = nsm * NB_MINB;
    const char* pe = getenv("REAX_NB_PLAN");   // "0": static grid (measurement)
    ctx->nb_plan = g.nblock > 0 && g.nblock <= NB_PLAN_MAX && !(pe && atoi(pe) == 0);
    if (const char* fe = getenv("REAX_NB_UNIT_FRAC")) ctx->nb_frac = std::max(0.05f, (float)atof(fe));
    if (const char* ge = getenv("REAX_NB_GRID_FRAC")) ctx->nb_grid_frac = std::max(0.0f, (float)atof(ge));
    // sum_b ceil(p_b / T) <= nblock + (sum p) / T ~ nblock + slots / frac (T = frac (sum p) / slots);
    // blocks below T stay whole, so plans need much less (c1: 515 of 343 + 296). The grid is kept
    // near that (its empty CTAs delay the dispatch of the side-stream kernels behind it); a plan that
    // does not fit is made coarser (k_nb_plan doubles T)
    ctx->nb_umax = (int)std::min<long long>((long long)NB_UNIT_SPLIT * g.nblock,
                                            g.nblock + (long long)std::ceil(ctx->nb_grid_frac * ctx->nb_slots / ctx->nb_frac) + 8);
  }
  ctx->cut = *cut;
  ctx->prm_valid = false;
  ctx->bep_valid = false;
  ctx->lists_ok = ctx->bonds_ok = false;
  // zero the counters that kernels keep self-cleaning
  cudaError_t e = cudaMemset(ctx->w.cell_cnt, 0, sizeof(int) * (g.ncell + 1));
  if (e == cudaSuccess) e = cudaMemset(ctx->w.bdeg, 0, sizeof(int) * (std::max<int64_t>(n, 1) + 1));
  if (e == cudaSuccess) e = cudaMemset(ctx->w.st, 0, sizeof(Status));
  // fixed-point force accumulators: zeroed by every gather (k_cell_gather, k_nb_prep) before a nonbonded pass
  if (e == cudaSuccess) e = cudaMemset(ctx->w.sf, 0, 3 * sizeof(long long) * std::max<int64_t>(n, 1));
  if (e == cudaSuccess) e = cudaMemset(ctx->w.ticket, 0, sizeof(unsigned) * 4);
  if (e == cudaSuccess) e = cudaMemset(ctx->w.lb_ticket, 0, sizeof(unsigned) * 4);
  if (e == cudaSuccess) e = cudaMemset(ctx->w.bin_ticket, 0, sizeof(unsigned) * 4);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return fail_cuda(e);
  ctx->bound = true;
  return REAX_OK;
}

reax_status reax_required(const reax_ctx* ctx, reax_capacity* need) {
  if (!ctx || !need) return REAX_ERR_ARG;
  *need = ctx->need;
  return REAX_OK;
}

reax_status reax_build_lists(reax_ctx* ctx, int64_t n, const double* pos, const int32_t* type, const double box[3],
                             const reax_params* params, const reax_cutoffs* cut, void* stream) {
  if (ctx) ctx->launches_cur = 0;
  reax_status r = do_build_lists(ctx, n, pos, type, box, params, cut, (cudaStream_t)stream);
  return r;
}

reax_status reax_bond_orders(reax_ctx* ctx, const reax_params* params, const reax_cutoffs* cut, void* stream) {
  return do_bond_orders(ctx, params, cut, (cudaStream_t)stream);
}

reax_status reax_bond_energy(reax_ctx* ctx, const reax_params* params, const reax_bond_params* bond_params,
                             double* force, double* energy, void* stream) {
  return do_bond_energy(ctx, params, bond_params, force, energy, (cudaStream_t)stream);
}

reax_status reax_nonbonded(reax_ctx* ctx, int64_t n, const double* pos, const int32_t* type, const double* q,
                           const double box[3], const reax_params* params, const reax_cutoffs* cut, double* force,
                           double* energy, void* stream) {
  return do_nonbonded(ctx, n, pos, type, q, box, params, cut, force, energy, (cudaStream_t)stream);
}

reax_status reax_step(reax_ctx* ctx, int64_t n, const double* pos, const int32_t* type, const double* q,
                      const double box[3], const reax_params* params, const reax_cutoffs* cut, double* force,
                      double* energy, void* stream) {
  if (!ctx) return REAX_ERR_ARG;
  ctx->launches_cur = 0;
  reax_status r = do_step(ctx, n, pos, type, q, box, params, cut, force, energy, (cudaStream_t)stream);
  ctx->launches_step = ctx->launches_cur;
  return r;
}

// copies in, reax_step, copies out (no synchronisation)
reax_status step_host_enqueue(reax_ctx* ctx, int64_t n, const double* pos, const int32_t* type, const double* q,
                              const double box[3], const reax_params* params, const reax_cutoffs* cut, double* force,
                              cudaStream_t s) {
  WS& w = ctx->w;
  // copies on the context's copy stream (positions, types, charges, each
  // followed by an event the step waits on where it first needs the array),
  // except in REAX_SERIAL mode; the step joins every event before it ends
  const bool overlap = n > 0 && !ctx->serial;
  cudaStream_t cs = overlap ? ctx->copy_s : s;
  if (n > 0) {
    if (overlap && (cudaEventRecord(ctx->ev_in0, s) != cudaSuccess || cudaStreamWaitEvent(cs, ctx->ev_in0, 0) != cudaSuccess))
      return fail_cuda(cudaGetLastError());
    if (cudaMemcpyAsync(w.h_pos, pos, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
        (overlap && cudaEventRecord(ctx->ev_pos, cs) != cudaSuccess) ||
        cudaMemcpyAsync(w.h_type, type, sizeof(int) * n, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
        (overlap && cudaEventRecord(ctx->ev_type, cs) != cudaSuccess) ||
        cudaMemcpyAsync(w.h_q, q, sizeof(double) * n, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
        (overlap && cudaEventRecord(ctx->ev_q, cs) != cudaSuccess))
      return fail_cuda(cudaGetLastError());
  }
  ctx->host_in = overlap;
  reax_status r = reax_step(ctx, n, w.h_pos, w.h_type, w.h_q, box, params, cut, w.h_force, w.h_energy, s);
  ctx->host_in = false;
  if (r != REAX_OK) {
    if (overlap) {   // an early return may leave the copy stream unjoined: join it
      cudaStreamWaitEvent(s, ctx->ev_q, 0);
    }
    return r;
  }
  if (n > 0 && cudaMemcpyAsync(force, w.h_force, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return fail_cuda(cudaGetLastError());
  return REAX_OK;
}

reax_status reax_step_host(reax_ctx* ctx, int64_t n, const double* pos, const int32_t* type, const double* q,
                           const double box[3], const reax_params* params, const reax_cutoffs* cut, double* force,
                           double* energy, void* stream) {
  if (!ctx) return REAX_ERR_ARG;
  if (!ctx->bound) return REAX_ERR_STATE;
  if (n != ctx->n) return REAX_ERR_STATE;
  if (!energy || (n > 0 && (!pos || !type || !q || !force))) return REAX_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  WS& w = ctx->w;
  std::vector<double> key;
  const bool keyed = n > 0 && !ctx->hg_off && box && params_key(params, cut, key);
  if (keyed) key.insert(key.end(), box, box + 3);
  const void* ptr[5] = {pos, type, q, force, energy};
  if (keyed && ctx->hg_exec && key == ctx->hg_key && memcmp(ptr, ctx->hg_ptr, sizeof(ptr)) == 0 &&
      ctx->hg_ws == ctx->ws_base && ctx->hg_async == ctx->async) {
    // the graph holds no parameter upload (the set was current at capture);
    // another call on this context may have uploaded a different set since
    // (a memcmp when nothing changed)
    reax_status ru = upload_params(ctx, params, cut, s);
    if (ru != REAX_OK) return ru;
    // replay: H2D copies, the whole step (side-stream fork included), D2H copies
    if (cudaError_t e_ = cudaGraphLaunch(ctx->hg_exec, s)) return fail_cuda(e_);
    if (cudaError_t e_ = cudaStreamSynchronize(s)) return fail_cuda(e_);
    return ctx->async ? REAX_OK : interpret_status(ctx, s);
  }
  // direct path (validates, sizes, reports errors); then capture the same
  // sequence for the next calls with these buffers
  reax_status r = step_host_enqueue(ctx, n, pos, type, q, box, params, cut, force, s);
  if (r != REAX_OK) return r;
  if (cudaMemcpyAsync(energy, w.h_energy, sizeof(double) * 2, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return fail_cuda(cudaGetLastError());
  if (cudaError_t e_ = cudaStreamSynchronize(s)) return fail_cuda(e_);
  if (!keyed) return REAX_OK;
  if (ctx->hg_exec) {
    cudaGraphExecDestroy(ctx->hg_exec);
    ctx->hg_exec = nullptr;
  }
  const bool was_async = ctx->async;
  ctx->async = true;   // no host synchronisation inside the captured step
  // captured on the context's own stream (the caller's may be the legacy
  // stream, which cannot be captured); replays are launched on the caller's.
  // The status block copy-back (read_status) is part of the captured step.
  cudaGraph_t graph = nullptr;
  cudaStream_t hs = ctx->cap_s;
  bool ok = cudaStreamBeginCapture(hs, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  if (ok) {
    r = step_host_enqueue(ctx, n, pos, type, q, box, params, cut, force, hs);
    ok = r == REAX_OK &&
         cudaMemcpyAsync(energy, w.h_energy, sizeof(double) * 2, cudaMemcpyDeviceToHost, hs) == cudaSuccess;
    ok = (cudaStreamEndCapture(hs, &graph) == cudaSuccess) && ok && graph;
  }
  ctx->async = was_async;
  if (ok) ok = cudaGraphInstantiate(&ctx->hg_exec, graph, 0) == cudaSuccess;
  if (graph) cudaGraphDestroy(graph);
  if (!ok) {   // not capturable here: keep the direct path
    ctx->hg_exec = nullptr;
    ctx->hg_off = true;
    cudaGetLastError();
    return REAX_OK;
  }
  ctx->hg_key.swap(key);
  memcpy(ctx->hg_ptr, ptr, sizeof(ptr));
  ctx->hg_ws = ctx->ws_base;
  ctx->hg_async = was_async;
  return REAX_OK;
}

reax_status reax_set_async(reax_ctx* ctx, int enable) {
  if (!ctx) return REAX_ERR_ARG;
  ctx->async = enable != 0;
  return REAX_OK;
}

reax_status reax_check(reax_ctx* ctx, void* stream) {
  if (!ctx) return REAX_ERR_ARG;
  if (!ctx->bound) return REAX_ERR_STATE;
  return read_status(ctx, (cudaStream_t)stream, true);
}

reax_status reax_set_timing(reax_ctx* ctx, int enable) {
  if (!ctx) return REAX_ERR_ARG;
  ctx->timing = enable != 0;
  return REAX_OK;
}

reax_status reax_kernel_ms(reax_ctx* ctx, double ms[REAX_NKERNELS], int64_t launches[REAX_NKERNELS], int reset) {
  if (!ctx) return REAX_ERR_ARG;
  if (reset == 2) {  // peek: elapsed time of the recorded events, left in place (graph replays)
    for (int k = 0; k < REAX_NKERNELS; ++k) {
      double t = 0.0;
      for (auto& p : ctx->ev_pending[k]) {
        if (cudaError_t e_ = cudaEventSynchronize(p.second)) return fail_cuda(e_);
        float f = 0.f;
        if (cudaError_t e_ = cudaEventElapsedTime(&f, p.first, p.second)) return fail_cuda(e_);
        t += f;
      }
      if (ms) ms[k] = t;
      if (launches) launches[k] = ctx->launches_acc[k];
    }
    return REAX_OK;
  }
  for (int k = 0; k < REAX_NKERNELS; ++k) {
    for (auto& p : ctx->ev_pending[k]) {
      if (cudaError_t e_ = cudaEventSynchronize(p.second)) return fail_cuda(e_);
      float t = 0.f;
      cudaEventElapsedTime(&t, p.first, p.second);
      ctx->ms_acc[k] += t;
      ctx->ev_pool.push_back(p.first);
      ctx->ev_pool.push_back(p.second);
    }
    ctx->ev_pending[k].clear();
    if (ms) ms[k] = ctx->ms_acc[k];
    if (launches) launches[k] = ctx->launches_acc[k];
    if (reset) {
      ctx->ms_acc[k] = 0;
      ctx->launches_acc[k] = 0;
    }
  }
  return REAX_OK;
}

int32_t reax_launches_per_step(const reax_ctx* ctx) { return ctx ? ctx->launches_step : 0; }

reax_status reax_selftest_math(reax_ctx* ctx, int64_t n, const double* x, double* out, const reax_params* params,
                               const reax_cutoffs* cut, void* stream) {
  if (!ctx || n < 0 || (n > 0 && (!x || !out))) return REAX_ERR_ARG;
  if (!ctx->bound) return REAX_ERR_STATE;
  cudaStream_t s = (cudaStream_t)stream;
  reax_status r = upload_params(ctx, params, cut, s);
  if (r != REAX_OK) return r;
  if (n > 0) k_selftest_math<<<nblk(n, TPB), TPB, 0, s>>>((int)n, x, out, ctx->w.prm);
  if (cudaError_t e_ = cudaGetLastError()) return fail_cuda(e_);
  if (cudaError_t e_ = cudaStreamSynchronize(s)) return fail_cuda(e_);
  return REAX_OK;
}

reax_status reax_qeq_bytes(reax_ctx* ctx, size_t* bytes, void* stream) {
  if (!ctx || !bytes) return REAX_ERR_ARG;
  if (!ctx->bound || !ctx->lists_ok) return REAX_ERR_STATE;
  int64_t P = 0;
  reax_status r = half_pairs(ctx, (cudaStream_t)stream, &P);
  if (r != REAX_OK) return r;
  *bytes = qeq_layout(ctx->n, P).total;
  return REAX_OK;
}

reax_status reax_qeq_build(reax_ctx* ctx, void* scratch, size_t scratch_bytes, void* stream) {
  return do_qeq_build(ctx, scratch, scratch_bytes, (cudaStream_t)stream);
}

reax_status reax_qeq_matvec(reax_ctx* ctx, const double* eta, void* scratch, size_t scratch_bytes, const double* x_s,
                            const double* x_t, double* y_s, double* y_t, void* stream) {
  return do_qeq_matvec(ctx, eta, scratch, scratch_bytes, x_s, x_t, y_s, y_t, (cudaStream_t)stream);
}

reax_status reax_qeq_solve(reax_ctx* ctx, const double* chi, const double* eta, double tol, int32_t maxiter,
                           void* scratch, size_t scratch_bytes, double* s, double* t, double* q, int32_t* iters,
                           void* stream) {
  return do_qeq_solve(ctx, chi, eta, tol, maxiter, scratch, scratch_bytes, s, t, q, iters, (cudaStream_t)stream);
}

reax_status reax_species_bytes(int64_t n, int32_t ntypes, size_t* bytes) {
  if (!bytes || n < 0 || ntypes < 1 || ntypes > REAX_MAX_TYPES) return REAX_ERR_ARG;
  *bytes = sp_layout(n, ntypes).total;
  return REAX_OK;
}

reax_status reax_species(reax_ctx* ctx, const double* bo_threshold, void* scratch, size_t scratch_bytes,
                         int32_t* mol_id, int64_t* n_molecules, int32_t* species_comp, int64_t* species_count,
                         int64_t species_cap, int64_t* n_species, void* stream) {
  return do_species(ctx, bo_threshold, scratch, scratch_bytes, mol_id, n_molecules, species_comp, species_count,
                    species_cap, n_species, (cudaStream_t)stream);
}

reax_status reax_interaction_counts(reax_ctx* ctx, const reax_ilist_params* params, int64_t* n_angles,
                                    int64_t* n_hbonds, void* stream) {
  return do_ilist_counts(ctx, params, n_angles, n_hbonds, (cudaStream_t)stream);
}

reax_status reax_interaction_lists(reax_ctx* ctx, const reax_ilist_params* params, int64_t* ang_off, int32_t* ang_k,
                                   int64_t* hb_off, int32_t* hb_z, void* stream) {
  return do_ilist_lists(ctx, params, ang_off, ang_k, hb_off, hb_z, (cudaStream_t)stream);
}

reax_status reax_pair_count(reax_ctx* ctx, int64_t* n_half_pairs, int64_t* n_bond_entries, void* stream) {
  if (!ctx) return REAX_ERR_ARG;
  if (!ctx->bound || !ctx->lists_ok) return REAX_ERR_STATE;
  cudaStream_t s = (cudaStream_t)stream;
  int N = (int)ctx->n;
  long long P = 0;
  int B = 0;
  if (N > 0) {
    if (scan<int, long long>(ctx, ctx->w.nbr_len, N, ctx->w.exp_off, s) != cudaSuccess) return REAX_ERR_CUDA;
    if (cudaMemcpyAsync(&P, ctx->w.exp_off + N, sizeof(long long), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(&B, ctx->w.brow + N, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return REAX_ERR_CUDA;
  }
  if (n_half_pairs) *n_half_pairs = P;
  if (n_bond_entries) *n_bond_entries = B;
  return REAX_OK;
}

reax_status reax_export_pairs(reax_ctx* ctx, int32_t* pi, int32_t* pj, void* stream) {
  if (!ctx || !pi || !pj) return REAX_ERR_ARG;
  if (!ctx->bound || !ctx->lists_ok) return REAX_ERR_STATE;
  cudaStream_t s = (cudaStream_t)stream;
  int N = (int)ctx->n;
  if (N == 0) return REAX_OK;
  if (scan<int, long long>(ctx, ctx->w.nbr_len, N, ctx->w.exp_off, s) != cudaSuccess) return REAX_ERR_CUDA;
  k_export_pairs<<<ctx->g.nblock, NBR_THREADS, exp_smem(ctx->cap.window_cap), s>>>(
      ctx->g, ctx->w.cell_start, ctx->w.perm, ctx->w.nbr, ctx->w.nbr_len, ctx->cap.row_cap, ctx->cap.window_cap,
      ctx->w.exp_off, 0, pi, pj, nullptr, nullptr);
  if (cudaError_t e_ = cudaGetLastError()) return fail_cuda(e_);
  if (cudaError_t e_ = cudaStreamSynchronize(s)) return fail_cuda(e_);
  return REAX_OK;
}

reax_status reax_export_nbr_digest(reax_ctx* ctx, int64_t* cnt, uint64_t* dig, void* stream) {
  if (!ctx || !cnt || !dig) return REAX_ERR_ARG;
  if (!ctx->bound || !ctx->lists_ok) return REAX_ERR_STATE;
  cudaStream_t s = (cudaStream_t)stream;
  int N = (int)ctx->n;
  if (N == 0) return REAX_OK;
  if (cudaMemsetAsync(cnt, 0, sizeof(int64_t) * N, s) != cudaSuccess ||
      cudaMemsetAsync(dig, 0, sizeof(uint64_t) * N, s) != cudaSuccess)
    return REAX_ERR_CUDA;
  k_export_pairs<<<ctx->g.nblock, NBR_THREADS, exp_smem(ctx->cap.window_cap), s>>>(
      ctx->g, ctx->w.cell_start, ctx->w.perm, ctx->w.nbr, ctx->w.nbr_len, ctx->cap.row_cap, ctx->cap.window_cap,
      nullptr, 1, nullptr, nullptr, (unsigned long long*)cnt, (unsigned long long*)dig);
  if (cudaError_t e_ = cudaGetLastError()) return fail_cuda(e_);
  if (cudaError_t e_ = cudaStreamSynchronize(s)) return fail_cuda(e_);
  return REAX_OK;
}

reax_status reax_export_bonds(reax_ctx* ctx, int64_t* brow, int32_t* bcol, int32_t* mirror, double* bo, double* delta,
                              void* stream) {
  if (!ctx) return REAX_ERR_ARG;
  if (!ctx->bound || !ctx->lists_ok) return REAX_ERR_STATE;
  if (bo && !ctx->bonds_ok) return REAX_ERR_STATE;
  cudaStream_t s = (cudaStream_t)stream;
  int N = (int)ctx->n;
  if (N == 0) {
    if (brow && cudaMemsetAsync(brow, 0, sizeof(int64_t), s) != cudaSuccess) return REAX_ERR_CUDA;
    return cudaStreamSynchronize(s) == cudaSuccess ? REAX_OK : REAX_ERR_CUDA;
  }
  WS& w = ctx->w;
  // original-order row offsets; bc_len is free scratch outside a step
  k_export_bond_deg<<<nblk(N, TPB), TPB, 0, s>>>(N, w.iperm, w.brow, w.bc_len);
  if (scan<int, long long>(ctx, w.bc_len, N, w.exp_off, s) != cudaSuccess) return REAX_ERR_CUDA;
  k_export_bonds<<<nblk(N + 1, TPB), TPB, 0, s>>>(N, w.iperm, w.perm, w.brow, w.bcol, w.bmir, w.bo, ctx->cap.bond_cap, w.delta,
                                                 w.exp_off, brow, bcol, mirror, bo, delta);
  if (cudaError_t e_ = cudaGetLastError()) return fail_cuda(e_);
  if (cudaError_t e_ = cudaStreamSynchronize(s)) return fail_cuda(e_);
  return REAX_OK;
}

}  // extern "C"
