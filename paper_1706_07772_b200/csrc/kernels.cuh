// Device kernels of the ReaxFF hot path (arXiv:1706.07772 ReaxC-OMP kernels,
// re-designed for B200).  Included once, by reax.cu.
#pragma once
#include "common.cuh"

namespace rx {

__constant__ WindowTables c_win;
// copy of c_win.wu in global memory: read with one index per thread (a
// divergent constant-bank read would serialise over the warp)
__device__ int g_win_wu[NWB];

__device__ __forceinline__ void set_flag(Status* st, int f) { atomicOr(&st->flags, f); }

// Programmatic dependent launch (the hot path is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): every such kernel
// waits for its predecessor's memory before touching global memory; small
// kernels let their successor launch right away (its blocks then wait here).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// CTA timeline instrumentation (measurement builds only, -DREAX_TIMELINE):
// per CTA of k_nbr_build (kind 0) and k_nonbonded (kind 1), the SM and the
// global-timer stamps at start, end of setup and end; read by
// reax_timeline_read (tools/timeline.py).
#ifdef REAX_TIMELINE
constexpr int TL_MAX = 1 << 16;
__device__ unsigned long long g_tl[2][TL_MAX][8];   // 0 start, 1 setup done, 2 end, 3 SM | work << 16, 4-7 kernel phases
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void tl_mark(int kind, int slot, unsigned long long work = 0) {
  if (threadIdx.x == 0 && blockIdx.x < TL_MAX) {
    unsigned sm;
    asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
    g_tl[kind][blockIdx.x][slot] = tl_now();
    if (slot == 0) {
      g_tl[kind][blockIdx.x][6] = ~0ull;
      g_tl[kind][blockIdx.x][7] = 0ull;
    }
    if (slot == 1) g_tl[kind][blockIdx.x][3] = sm | (work << 16);   // SM, work units of the CTA
  }
}
#define TL_MARK(kind, slot, ...) tl_mark(kind, slot, ##__VA_ARGS__)
// per-warp extremes (slot 6: first warp done, atomicMin; slot 7: last warp done)
__device__ __forceinline__ void tl_warp_done(int kind) {
  if ((threadIdx.x & 31) == 0 && blockIdx.x < TL_MAX) {
    const unsigned long long t = tl_now();
    atomicMin(&g_tl[kind][blockIdx.x][6], t);
    atomicMax(&g_tl[kind][blockIdx.x][7], t);
  }
}
#define TL_WARP_DONE(kind) tl_warp_done(kind)
// first CTA start (before griddepcontrol.wait) / last CTA end of the step's
// other kernels (id: tools/timeline.py SPANS)
__device__ unsigned long long g_tl_span[8][2];
struct TLSpan {
  int id;
  __device__ __forceinline__ explicit TLSpan(int i) : id(i) {
    if (threadIdx.x == 0) atomicMin(&g_tl_span[id][0], tl_now());
  }
  __device__ __forceinline__ ~TLSpan() {
    if (threadIdx.x == 0) atomicMax(&g_tl_span[id][1], tl_now());
  }
};
#define TL_SPAN(id) TLSpan tl_span_(id)
#else
#define TL_MARK(kind, slot, ...) ((void)0)
#define TL_WARP_DONE(kind) ((void)0)
#define TL_SPAN(id) ((void)0)
#endif

// a1: x <- x - L floor(x/L), a result equal to L (or below 0 by rounding) -> 0.
// Explicitly rounded operations keep it bit-identical to any IEEE scalar code.
__device__ __forceinline__ double wrap_coord(double x, double L) {
  double w = __dsub_rn(x, __dmul_rn(L, floor(__ddiv_rn(x, L))));
  return (w >= L || w < 0.0) ? 0.0 : w;
}

// ===================================================================== scan
// Exclusive prefix sum in 3 launches (block partials, top, final); T in/out.
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <typename TI>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_partial(const TI* in, int64_t n, long long* part) {
  __shared__ long long red[32];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  long long s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    int64_t i = base + threadIdx.x + (int64_t)k * SCAN_THREADS;
    if (i < n) s += (long long)in[i];
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    long long v = red[threadIdx.x];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
  }
}

// single block: exclusive scan of nparts partials in place; total -> part[nparts]
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_top(long long* part, int nparts) {
  __shared__ long long warp_tot[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nparts; base += SCAN_THREADS) {
    int i = base + threadIdx.x;
    long long v = i < nparts ? part[i] : 0;
    long long x = v;
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
      long long t = warp_tot[lane];
      for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;
    }
    __syncthreads();
    long long incl = x + (w > 0 ? warp_tot[w - 1] : 0) + carry;
    if (i < nparts) part[i] = incl - v;
    __syncthreads();
    if (threadIdx.x == SCAN_THREADS - 1) carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) part[nparts] = carry;
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_final(const TI* in, int64_t n, const long long* part, TO* out) {
  __shared__ long long warp_tot[32];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // each thread owns SCAN_ITEMS consecutive elements
  int64_t i0 = base + (int64_t)threadIdx.x * SCAN_ITEMS;
  long long v[SCAN_ITEMS];
  long long s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    v[k] = (i0 + k < n) ? (long long)in[i0 + k] : 0;
    s += v[k];
  }
  long long x = s;
  for (int o = 1; o < 32; o <<= 1) {
    long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    long long t = warp_tot[lane];
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;
  }
  __syncthreads();
  long long run = part[blockIdx.x] + x - s + (w > 0 ? warp_tot[w - 1] : 0);
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    if (i0 + k < n) out[i0 + k] = (TO)run;
    run += v[k];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = (TO)part[gridDim.x];
}

// Single-pass exclusive scan (decoupled look-back): tiles get ids from a
// ticket counter (forward progress), publish their aggregate, then look back
// over predecessors until an inclusive prefix is found.  status[] and the
// ticket must be zero on entry (the producing kernel clears them).
constexpr int LB_THREADS = 512;
constexpr int LB_ITEMS = 8;
constexpr int LB_TILE = LB_THREADS * LB_ITEMS;
constexpr unsigned long long LB_AGG = 1ull << 62, LB_PRE = 2ull << 62, LB_MASK = (1ull << 62) - 1;

__global__ void __launch_bounds__(LB_THREADS) k_scan_lookback(const int* __restrict__ in, int n, int* __restrict__ out,
                                                              unsigned long long* __restrict__ status,
                                                              unsigned* __restrict__ ticket) {
  TL_SPAN(1);
  pdl_wait();
  pdl_trigger();
  __shared__ int tile_id;
  __shared__ long long warp_tot[LB_THREADS / 32];
  __shared__ long long excl_tile;
  if (threadIdx.x == 0) tile_id = (int)atomicAdd(ticket, 1u);
  __syncthreads();
  const int t = tile_id;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i0 = (int64_t)t * LB_TILE + (int64_t)threadIdx.x * LB_ITEMS;
  int v[LB_ITEMS];
  long long sum = 0;
#pragma unroll
  for (int q = 0; q < LB_ITEMS; ++q) {
    v[q] = (i0 + q < n) ? in[i0 + q] : 0;
    sum += v[q];
  }
  long long x = sum;
  for (int o = 1; o < 32; o <<= 1) {
    long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    long long y = lane < LB_THREADS / 32 ? warp_tot[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      long long z = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += z;
    }
    if (lane < LB_THREADS / 32) warp_tot[lane] = y;
    long long agg = __shfl_sync(0xffffffffu, y, LB_THREADS / 32 - 1);
    if (lane == 0) {
      volatile unsigned long long* vs = status;
      if (t == 0) {
        vs[0] = LB_PRE | (unsigned long long)agg;
        excl_tile = 0;
      } else {
        vs[t] = LB_AGG | (unsigned long long)agg;
        long long acc = 0;
        int p = t - 1;
        for (;;) {
          unsigned long long s;
          do { s = vs[p]; } while ((s >> 62) == 0);
          acc += (long long)(s & LB_MASK);
          if ((s >> 62) == 2) break;
          --p;
        }
        __threadfence();
        vs[t] = LB_PRE | (unsigned long long)(acc + agg);
        excl_tile = acc;
      }
      if (t == (int)gridDim.x - 1) *ticket = 0u;  // ready for the next call
    }
  }
  __syncthreads();
  long long run = excl_tile + x - sum + (w > 0 ? warp_tot[w - 1] : 0);
#pragma unroll
  for (int q = 0; q < LB_ITEMS; ++q) {
    if (i0 + q < n) out[i0 + q] = (int)run;
    run += v[q];
  }
  if (t == (int)gridDim.x - 1 && threadIdx.x == LB_THREADS - 1) out[n] = (int)(excl_tile + warp_tot[LB_THREADS / 32 - 1]);
}

// clears a look-back status array (run by the kernel before the scan)
__device__ __forceinline__ void clear_status(unsigned long long* status, int ntiles) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ntiles) status[i] = 0ull;
}

// ================================================================ a1-a2 bin
// wrap, validate, sub-cell id, histogram
// (small grids: BIN_FUSED_SCAN_MAX cells or fewer) the last k_bin block to
// finish turns the histogram into cell_start itself, saving the scan launch
constexpr int BIN_FUSED_SCAN_MAX = 4096;
__global__ void __launch_bounds__(256) k_bin(int n, const double* __restrict__ pos, const int* __restrict__ type, Grid g,
                      int nt, int* __restrict__ cell_of, int* __restrict__ cell_cnt, Status* st,
                      unsigned long long* __restrict__ scan_status, int scan_tiles, int* __restrict__ cell_start,
                      unsigned* __restrict__ ticket) {
  pdl_wait();
  pdl_trigger();
  clear_status(scan_status, scan_tiles);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    int c[3];
    bool bad = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double x = pos[3 * (int64_t)i + k];
      bad |= !isfinite(x);
      double w = isfinite(x) ? wrap_coord(x, g.L[k]) : 0.0;
      int ck = (int)(w * g.inv_h[k]);
      c[k] = ck >= g.nc[k] ? g.nc[k] - 1 : ck;
    }
    if (bad) set_flag(st, ST_NONFINITE_IN);
    if (type) {   // else checked by the cell gather (reax_step_host: the types arrive later)
      int t = type[i];
      if (t < 0 || t >= nt) set_flag(st, ST_TYPE);
    }
    int cid = (c[2] * g.nc[1] + c[1]) * g.nc[0] + c[0];
    cell_of[i] = cid;
    atomicAdd(&cell_cnt[cid], 1);
  }
  if (!cell_start) return;   // separate scan
  __shared__ bool last;
  __shared__ int warp_sum[8];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // exclusive scan of the ncell counts by this block: thread t owns a
  // contiguous segment of m cells (all its loads in flight at once), a block
  // scan of the segment sums, then the segment's prefixes
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int m = (g.ncell + 255) / 256;
  const int k0 = threadIdx.x * m;
  constexpr int MSEG = BIN_FUSED_SCAN_MAX / 256;
  int v[MSEG];
  int seg = 0;
#pragma unroll
  for (int q = 0; q < MSEG; ++q) {
    v[q] = (q < m && k0 + q < g.ncell) ? __ldcg(cell_cnt + k0 + q) : 0;
    seg += v[q];
  }
  int x = seg;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sum[w] = x;
  __syncthreads();
  int run = x - seg;
  for (int q = 0; q < w; ++q) run += warp_sum[q];
  int carry = 0;
  for (int q = 0; q < 8; ++q) carry += warp_sum[q];
#pragma unroll
  for (int q = 0; q < MSEG; ++q) {
    if (q < m && k0 + q < g.ncell) cell_start[k0 + q] = run;
    run += v[q];
  }
  if (threadIdx.x == 0) {
    cell_start[g.ncell] = carry;
    *ticket = 0u;   // ready for the next call
  }
}

// counting-sort scatter; cell_cnt returns to zero (ready for the next call)
__global__ void k_scatter(int n, const int* __restrict__ cell_of, const int* __restrict__ cell_start,
                          int* __restrict__ cell_cnt, int* __restrict__ perm) {
  pdl_wait();
  pdl_trigger();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = cell_of[i];
  int r = atomicSub(&cell_cnt[c], 1) - 1;
  perm[cell_start[c] + r] = i;
}

// sort key of a coordinate: the wrapped value (non-finite -> 0, flagged by k_bin)
__device__ __forceinline__ double wrap_key(double x, double L) { return isfinite(x) ? wrap_coord(x, L) : 0.0; }

// Per cell (one warp): order the cell's atoms by x (rank sort in registers;
// deterministic), then gather the sorted arrays.
// One atom record of the sorted arrays (sorted position sp, staged record v,
// input index i, cell cc)
__device__ __forceinline__ void gather_one(int sp, int i, const double4& v, int t, const int (&cc)[3], const Grid& g,
                                           int nt, bool has_q, int* __restrict__ perm, int* __restrict__ iperm,
                                           double4* __restrict__ spos, float4* __restrict__ sloc,
                                           int* __restrict__ stype, Status* st, unsigned long long* __restrict__ sf) {
  const double x[3] = {v.x, v.y, v.z};
  double w[3];
  float l[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    w[d] = isfinite(x[d]) ? wrap_coord(x[d], g.L[d]) : 0.0;
    l[d] = (float)(w[d] - cc[d] * g.h[d]);
  }
  if (t < 0 || t >= nt) {   // flagged (also by k_bin when it had the types); clamp keeps every table index valid
    set_flag(st, ST_TYPE);
    t = 0;
  }
  const double qs = has_q ? v.w : 0.0;   // reax_step: charges staged by k_scatter (reax_nonbonded: k_nb_prep)
  if (has_q && !isfinite(qs)) set_flag(st, ST_NONFINITE_IN);
  perm[sp] = i;
  spos[sp] = make_double4(w[0], w[1], w[2], qs);
  sloc[sp] = make_float4(l[0], l[1], l[2], __int_as_float(t));
  stype[sp] = t;
  iperm[i] = sp;
  // the fixed-point force accumulators of this step start at zero (one 24-byte record per atom)
  sf[3 * (int64_t)sp] = 0ull;
  sf[3 * (int64_t)sp + 1] = 0ull;
  sf[3 * (int64_t)sp + 2] = 0ull;
}

// Warp per cell: order the cell's atoms by (wrapped x, original index) —
// deterministic, and every run of cells along x is then x-sorted, which lets
// the list build cut each run to the x-window of a row by binary search —
// and write the sorted arrays.  Each lane reads its atom's input record once
// (scattered) and writes it to its sorted position.
__device__ __forceinline__ double4 in_rec(const double* __restrict__ pos, const double* __restrict__ qin, int i) {
  return make_double4(pos[3 * (int64_t)i], pos[3 * (int64_t)i + 1], pos[3 * (int64_t)i + 2], qin ? qin[i] : 0.0);
}
__global__ void k_cell_gather(int ncell, const int* __restrict__ cell_start, int* __restrict__ perm,
                              const double* __restrict__ pos, const int* __restrict__ type,
                              const double* __restrict__ qin, Grid g, int nt,
                              int* __restrict__ iperm, double4* __restrict__ spos, float4* __restrict__ sloc,
                              int* __restrict__ stype, Status* st,
                              int* __restrict__ blk_pairs, int nblock, unsigned long long* __restrict__ sf) {
  pdl_wait();
  pdl_trigger();
  if (blk_pairs) {   // per-block pair counts of the next list build start at zero
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < nblock) blk_pairs[t] = 0;
  }
  int c = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  int lane = threadIdx.x & 31;
  if (c >= ncell) return;
  const int a = cell_start[c], b = cell_start[c + 1], m = b - a;
  const int cc[3] = {c % g.nc[0], (c / g.nc[0]) % g.nc[1], c / (g.nc[0] * g.nc[1])};
  if (m <= 32) {
    const int v = lane < m ? perm[a + lane] : 0x7fffffff;
    const double4 r = lane < m ? in_rec(pos, qin, v) : make_double4(0.0, 0.0, 0.0, 0.0);
    const int t = lane < m ? type[v] : 0;
    const double xv = wrap_key(r.x, g.L[0]);
    int rank = 0;
    for (int q = 0; q < m; ++q) {
      const int vq = __shfl_sync(0xffffffffu, v, q);
      const double xq = __shfl_sync(0xffffffffu, xv, q);
      rank += (xq < xv) || (xq == xv && vq < v);
    }
    __syncwarp();   // every lane has read its perm entry before any is overwritten
    if (lane < m) gather_one(a + rank, v, r, t, cc, g, nt, qin != nullptr, perm, iperm, spos, sloc, stype, st, sf);
  } else {   // rare (Poisson tail): serial insertion sort of the input indices, scratch in the cell's force records
    unsigned long long* key = sf + 3 * (int64_t)a;   // key q at key[3 q]; zeroed by gather_one afterwards
    for (int q = lane; q < m; q += 32) key[3 * q] = (unsigned long long)(unsigned)perm[a + q];
    __syncwarp();
    if (lane == 0) {
      for (int q = 1; q < m; ++q) {
        const unsigned long long kv = key[3 * q];
        const int vv = (int)kv;
        const double xv = wrap_key(pos[3 * (int64_t)vv], g.L[0]);
        int u = q - 1;
        while (u >= 0) {
          const unsigned long long ku = key[3 * u];
          const double xu = wrap_key(pos[3 * (int64_t)(int)ku], g.L[0]);
          if (!(xu > xv || (xu == xv && (int)ku > vv))) break;
          key[3 * (u + 1)] = ku;
          --u;
        }
        key[3 * (u + 1)] = kv;
      }
    }
    __syncwarp();
    for (int q = lane; q < m; q += 32) {
      const int i = (int)key[3 * q];
      gather_one(a + q, i, in_rec(pos, qin, i), type[i], cc, g, nt, qin != nullptr, perm, iperm, spos, sloc, stype, st,
                 sf);
    }
  }
}

// ======================================================== window of a block
// Shared-memory description of a home block's neighbour window.
struct WinSmem {
  int start[NWU_MAX];       // first sorted atom of each used window cell
  int cnt[NWU_MAX];
  int slot[NWU_MAX + 1];    // slot base (prefix of cnt)
  double4 shift[NWU_MAX];   // periodic image shift (0 or +-L) of each window cell (x, y, z, 0)
  int shc[NWU_MAX];         // the same as a code: sum over axes a of (m_a + 1) << 2a, m_a in {-1, 0, 1}
  int home_ok[NHOME];       // home sub-cell exists (odd nc leaves the last block partial)
  int has_shift;            // some window cell is a periodic image
};

// Fill WinSmem for block b (all threads participate). Returns total slots.
__device__ int build_window(WinSmem& W, int b, const Grid& g, const int* __restrict__ cell_start) {
  // b = home block index
  int bx = b % g.nb[0], by = (b / g.nb[0]) % g.nb[1], bz = b / (g.nb[0] * g.nb[1]);
  int base[3] = {bx * HB, by * HB, bz * HB};
  int nwu = c_win.nwu;
  int my_shift = 0;
  // home sub-cells that exist (an odd cell count per axis leaves the last
  // block partial): only the union of their half stencils is staged
  unsigned hok = 0;
#pragma unroll
  for (int h = 0; h < NHOME; ++h)
    hok |= ((base[0] + h % HB < g.nc[0]) && (base[1] + (h / HB) % HB < g.nc[1]) && (base[2] + h / (HB * HB) < g.nc[2]))
               ? (1u << h) : 0u;
  for (int k = threadIdx.x; k < nwu; k += blockDim.x) {
    int code = 0;
    bool need = false;
#pragma unroll
    for (int h = 0; h < NHOME; ++h) need |= ((hok >> h) & 1u) && ((c_win.mask[h][k >> 5] >> (k & 31)) & 1u);
    int wb = __ldg(g_win_wu + k);
    int wv[3] = {wb % WB, (wb / WB) % WB, wb / (WB * WB)};
    int cc[3];
    double sh[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      int u = base[a] + wv[a] - SR;          // unwrapped sub-cell, in [-SR, nc + HB + SR - 2]
      // floor(u / nc) in {-1, 0, 1}: nc >= 4 (L > 2 r_nonb, sub-cells >= r_nonb / 2)
      int m = u < 0 ? -1 : (u >= g.nc[a] ? 1 : 0);
      cc[a] = u - m * g.nc[a];
      sh[a] = m == 0 ? 0.0 : (m > 0 ? g.L[a] : -g.L[a]);
      code |= (m + 1) << (2 * a);
      my_shift |= need && (m != 0);
    }
    W.shift[k] = make_double4(sh[0], sh[1], sh[2], 0.0);
    W.shc[k] = code;
    int cid = (cc[2] * g.nc[1] + cc[1]) * g.nc[0] + cc[0];
    int s0 = cell_start[cid];
    W.start[k] = s0;
    W.cnt[k] = need ? cell_start[cid + 1] - s0 : 0;
  }
  if (threadIdx.x < NHOME) W.home_ok[threadIdx.x] = (hok >> threadIdx.x) & 1u;
  const int any_shift = __syncthreads_or(my_shift);
  if (threadIdx.x == 0) W.has_shift = any_shift;
  if (threadIdx.x < 32) {  // warp 0: exclusive scan over <= 216 counts
    int carry = 0;
    for (int k0 = 0; k0 < nwu; k0 += 32) {
      int k = k0 + threadIdx.x;
      int v = k < nwu ? W.cnt[k] : 0;
      int x = v;
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if ((int)threadIdx.x >= o) x += y;
      }
      if (k < nwu) W.slot[k] = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (threadIdx.x == 0) W.slot[nwu] = carry;
  }
  __syncthreads();
  return W.slot[nwu];
}

// The window of a home block as the list build made it, for the nonbonded
// kernel (which then skips its own window build and slot-info staging):
// {W, home_ok bits, has_shift, 0}, start[NWU_MAX], cnt[NWU_MAX],
// slot[NWU_MAX + 1], shift codes[NWU_MAX] per block in `wpack`, and the
// slot info {sorted atom, window cell | type << 8} of every slot in `wsinfo`
// (window_cap entries per block); then the lengths of the block's first
// WP_MAXROWS rows in home order (written by the list-build CTA that made the
// row).
constexpr int WP_MAXROWS = 256;
constexpr int WP_START = 4, WP_CNT = WP_START + NWU_MAX, WP_SLOT = WP_CNT + NWU_MAX, WP_SHC = WP_SLOT + NWU_MAX + 1;
constexpr int WP_LEN = (WP_SHC + NWU_MAX + 3) & ~3;
constexpr int WPACK_INTS = WP_LEN + WP_MAXROWS;
__device__ void win_store(const WinSmem& W, int Wslots, int* __restrict__ wp) {
  const int nwu = c_win.nwu;
  for (int t = threadIdx.x; t < WP_LEN; t += blockDim.x) {
    int v = 0;
    if (t == 0) v = Wslots;
    else if (t == 1) {
      for (int h = 0; h < NHOME; ++h) v |= W.home_ok[h] ? 1 << h : 0;
    } else if (t == 2) v = W.has_shift;
    else if (t >= WP_START && t < WP_START + nwu) v = W.start[t - WP_START];
    else if (t >= WP_CNT && t < WP_CNT + nwu) v = W.cnt[t - WP_CNT];
    else if (t >= WP_SLOT && t <= WP_SLOT + nwu) v = W.slot[t - WP_SLOT];
    else if (t >= WP_SHC && t < WP_SHC + nwu) v = W.shc[t - WP_SHC];
    wp[t] = v;
  }
}
// the inverse (all threads; ends with __syncthreads), row lengths into
// lens[WP_MAXROWS]; returns W.  NT threads: every load is issued before any
// is used (one round trip).
template <int NT>
__device__ int win_load(WinSmem& W, const Grid& g, const int* __restrict__ wp, int* lens) {
  constexpr int PER = (WPACK_INTS + NT - 1) / NT;
  const int nwu = c_win.nwu;
  int v[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int t = threadIdx.x + u * NT;
    v[u] = t < WPACK_INTS ? wp[t] : 0;
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int t = threadIdx.x + u * NT;
    if (t >= WPACK_INTS) break;
    if (t >= WP_LEN) lens[t - WP_LEN] = v[u];
    else if (t == 1) {
      for (int h = 0; h < NHOME; ++h) W.home_ok[h] = (v[u] >> h) & 1;
    } else if (t == 2) W.has_shift = v[u];
    else if (t >= WP_START && t < WP_START + nwu) W.start[t - WP_START] = v[u];
    else if (t >= WP_CNT && t < WP_CNT + nwu) W.cnt[t - WP_CNT] = v[u];
    else if (t >= WP_SLOT && t <= WP_SLOT + nwu) W.slot[t - WP_SLOT] = v[u];
    else if (t >= WP_SHC && t < WP_SHC + nwu) {
      const int k = t - WP_SHC;
      double sh[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int m = ((v[u] >> (2 * a)) & 3) - 1;
        sh[a] = m == 0 ? 0.0 : (m > 0 ? g.L[a] : -g.L[a]);
      }
      W.shift[k] = make_double4(sh[0], sh[1], sh[2], 0.0);
      W.shc[k] = v[u];
    }
  }
  __syncthreads();
  return W.slot[nwu];   // W (the slot total, also when the list build found W > window_cap)
}

// rows of the block: home sub-cell h, slot range [slot[home_k[h]], slot[home_k[h]+1])
__device__ __forceinline__ bool row_of(const WinSmem& W, int r, int& h, int& si) {
  for (h = 0; h < NHOME; ++h) {
    if (!W.home_ok[h]) continue;
    int k = c_win.home_k[h];
    int c = W.cnt[k];
    if (r < c) {
      si = W.slot[k] + r;
      return true;
    }
    r -= c;
  }
  return false;
}

__device__ __forceinline__ int warp_find(int incl, int t) {
  // largest q with excl(q) <= t, where incl is the lane's inclusive prefix
  int q = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    int v = __shfl_sync(0xffffffffu, incl, q + step - 1);
    if (t >= v) q += step;
  }
  return q;
}

// ========================================================= a3-a4 list build
constexpr int NBR_THREADS = 256;

// per (home sub-cell, forward run): the run's window cells and the
// block-frame origin of its first cell (staged per CTA: the constant-bank
// tables would be read with a different index per lane, which serialises)
struct RunInfo {
  short ka, kb, wxa, pad;
  float oy, oz;
};

struct NbrSmem {
  WinSmem W;
  RunInfo run[NHOME][MAX_RUNS];
  float rcand2[NTP_MAX];
  int gbase[NHOME + 1];   // first row group of each home sub-cell (groups of NBR_G rows)
  int rbase[NHOME];       // first row (block order) of each home sub-cell
  int ncs[NBR_THREADS / 32][8];   // per warp: bond-candidate counters of its group's rows
  int next_row;
  int pairs;                      // half-list entries of this CTA's rows (nonbonded work plan)
};

// Per-kernel constants of the half-list candidate test, made on the host
// (make_rowtest in reax.cu) and passed by value: the kernel reads them from the
// constant bank, so they hold no registers in the chunk loop.
struct RowTest {
  float R2lo, R2mid, R2half, Rt, hy, hz, ihx;   // band [R2lo, R2lo + 2 R2half] = [R2lo, R2hi]
  float rcmax;                                  // largest bond-candidate radius^2 (fp32, conservative)
  double R2;
};
#ifndef NBR_GROUP
#define NBR_GROUP 3   // measured at 4 CTAs/SM, 64 registers (c4): 3 rows 18.13 ms, 2 rows 18.53, 4 rows 18.84 (spills)
#endif
constexpr int NBR_G = NBR_GROUP;   // rows sharing one candidate stream

__device__ __forceinline__ float4 lds_f4(unsigned a) {   // explicit 32-bit shared address (no per-use re-derivation)
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

// A group of up to NBR_G consecutive rows (atoms) of one home sub-cell,
// tested by one warp (Write Lists).  The atoms of a cell are
// x-sorted, so the rows of a group are x-neighbours and share one candidate
// stream: the forward runs of the sub-cell's half stencil, each cut first to
// the cells meeting [x_min - w, x_max + w] and then, the run being x-sorted,
// to that x-window by binary search (w = sqrt(R^2 - d_yz^2), d_yz the
// smallest distance of the group's atoms to the run's y-z cross-section, so
// no partner is ever cut), then the own cell after the group's first row.
// The runs + own cell fit lanes 0..15 (empty intervals included), so stream
// position p -> slot is a 4-step binary search over the lane-held interval
// offsets (the interval of p is the largest q with excl(q) <= p): no
// compaction, no vote.  Each lane loads one candidate (32 per step) and tests
// it against every row of the group held in registers (bare coordinates; rows
// beyond nrow are parked at -1e30 so they never test true): r^2 in fp32
// against a band of +-m around R^2 (~70x the fp32 error bound), the band
// settled by the exact FMA-free fp64 test (bit-identical to the oracle's
// r^2); accepted window slots of row r are compacted with one ballot per row
// and stored coalesced.  The rare candidates below the conservative BO' =
// bo_cut radius (~3 per row) are appended per lane through a shared-memory
// counter of the row (no warp vote; their order is irrelevant because
// k_bond_rank sorts each bond row); the rare paths re-read what they need
// (row type, atom index, bond row) from shared memory, so the hot loop
// carries only coordinates, row pointers and lengths.  len[r] may exceed
// row_cap (the caller flags it).
__device__ __forceinline__ void nbr_group_stream(const WinSmem& W, const RunInfo* __restrict__ runs, int Wslots,
                                                 const float4* __restrict__ cand, const int* __restrict__ cand_j,
                                                 const unsigned char* __restrict__ cand_k,
                                                 const double4* __restrict__ spos, int si0, int nrow, int h,
                                                 const RowTest& rt, uint16_t* __restrict__ nbr, int row_cap,
                                                 int* __restrict__ bc, int cand_cap, const float* __restrict__ rc2,
                                                 int nt, int* ncs, int (&len)[NBR_G]) {
  constexpr int G = NBR_G;
  const int lane = threadIdx.x & 31;
  if (lane < G) ncs[lane] = 0;   // per-row bond-candidate counters (shared, this warp's)
  __syncwarp();
  const unsigned lt_mask = (1u << lane) - 1u;
  float rx[G], ry[G], rz[G];
  uint16_t* rowp[G];
  float xmin = 1e30f, xmax = -1e30f;
#pragma unroll
  for (int r = 0; r < G; ++r) {
    len[r] = 0;
    if (r < nrow) {
      const float4 c = cand[si0 + r];
      rx[r] = c.x; ry[r] = c.y; rz[r] = c.z;
      rowp[r] = nbr + (int64_t)cand_j[si0 + r] * row_cap;
      xmin = fminf(xmin, c.x);
      xmax = fmaxf(xmax, c.x);
    } else {
      rx[r] = ry[r] = rz[r] = -1e30f;   // r^2 overflows to inf (also against the +1e30 sentinel)
      rowp[r] = nbr;
    }
  }
  const int kh = c_win.home_k[h];
  const int ownlo = W.slot[kh];
  // ---- intervals: lane q < nrun cuts run q, lane nrun takes the own cell
  const int nrun = c_win.nrun1[h];
  int ia = 0, il = 0;
  if (lane < nrun) {
    const RunInfo ru = runs[lane];
    const int ka = ru.ka, kb = ru.kb;
    const int wxa = ru.wxa;   // x cell offset (block frame) of the run's first cell
    float d2min = 1e30f;
#pragma unroll
    for (int r = 0; r < G; ++r) {
      if (r < nrow) {
        const float dy = fmaxf(0.f, fmaxf(ru.oy - ry[r], ry[r] - (ru.oy + rt.hy)));
        const float dz = fmaxf(0.f, fmaxf(ru.oz - rz[r], rz[r] - (ru.oz + rt.hz)));
        d2min = fminf(d2min, dy * dy + dz * dz);
      }
    }
    const float w2 = rt.Rt * rt.Rt - d2min;
    if (w2 >= 0.f) {
      const float w = sqrtf(w2) + 1e-3f;
      const int c0 = max(wxa, (int)floorf((xmin - w) * rt.ihx));
      const int c1 = min(wxa + (kb - ka), (int)floorf((xmax + w) * rt.ihx));
      if (c0 <= c1) {
        const int lo = W.slot[ka + (c0 - wxa)], hi = W.slot[ka + (c1 - wxa) + 1];
        const float xlo = xmin - w, xhi = xmax + w;
        int l = lo, u = hi;
        while (l < u) {
          const int mid = (l + u) >> 1;
          if (cand[mid].x < xlo) l = mid + 1; else u = mid;
        }
        int l2 = l, u2 = hi;
        while (l2 < u2) {
          const int mid = (l2 + u2) >> 1;
          if (cand[mid].x <= xhi) l2 = mid + 1; else u2 = mid;
        }
        ia = l;
        il = l2 - l;
      }
    }
  } else if (lane == nrun) {
    ia = si0 + 1;
    il = W.slot[kh + 1] - ia;
  }
  int inc = il;
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  const int total = __shfl_sync(0xffffffffu, inc, 15);
  const int excl = inc - il;
  const int shift = ia - excl;   // slot = p + shift inside the lane's interval
  // own-cell partners of row r: slots after si0 + r only.  The stream holds
  // the own cell from si0 + 1 on, so the only slots to exclude for row r are
  // the group's rows si0 + 1 .. si0 + r: ok(r) <=> (unsigned)(slot - si0 - 1) >= r
  const unsigned cand_s = (unsigned)__cvta_generic_to_shared(cand);
  for (int p0 = 0; p0 < total; p0 += 32) {
    const int p = p0 + lane;
    int q = 0;
#pragma unroll
    for (int step = 8; step >= 1; step >>= 1)
      if (__shfl_sync(0xffffffffu, excl, q + step) <= p) q += step;
    const int sh = __shfl_sync(0xffffffffu, shift, q);
    const int slot = p < total ? p + sh : Wslots;   // Wslots (window_cap, a kernel constant): sentinel at 1e30
    const float4 c = lds_f4(cand_s + 16u * (unsigned)slot);
    const unsigned tself = (unsigned)(slot - si0 - 1);
    float r2v[G];
    unsigned mk[G];
    bool rare = false;
#pragma unroll
    for (int r = 0; r < G; ++r) {
      const float dx = c.x - rx[r], dy = c.y - ry[r], dz = c.z - rz[r];
      r2v[r] = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
      const bool ok = tself >= (unsigned)r;
      mk[r] = __ballot_sync(0xffffffffu, ok & (r2v[r] < rt.R2lo));
      // rare: inside the fp32 band around R^2 (settled exactly below) or a
      // possible bond candidate (rcmax < R2lo); bitwise, so no branches
      rare |= ok & ((fabsf(r2v[r] - rt.R2mid) <= rt.R2half) | (r2v[r] <= rt.rcmax));
    }
    if (__any_sync(0xffffffffu, rare)) {
      const int tj = __float_as_int(c.w);
#pragma unroll
      for (int r = 0; r < G; ++r) {
        const bool ok = tself >= (unsigned)r;
        bool in = ((mk[r] >> lane) & 1u) != 0u;
        if (ok && !in && fabsf(r2v[r] - rt.R2mid) <= rt.R2half) {
          // exact, FMA-free fp64 decision (bit-identical to the oracle's r^2)
          const int k = cand_k[slot];
          const double4 xi = spos[cand_j[si0 + r]];
          const double4 xj = spos[cand_j[slot]];
          const double4 sw = W.shift[k];
          const double ex = __dadd_rn(__dsub_rn(xj.x, xi.x), sw.x);
          const double ey = __dadd_rn(__dsub_rn(xj.y, xi.y), sw.y);
          const double ez = __dadd_rn(__dsub_rn(xj.z, xi.z), sw.z);
          const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez));
          in = d2 <= rt.R2;
        } else if (in && r2v[r] <= rc2[__float_as_int(cand[si0 + r].w) * nt + tj]) {
          const int pc = atomicAdd(ncs + r, 1);   // per-lane append, no warp vote
          if (pc < cand_cap) bc[(int64_t)cand_j[si0 + r] * cand_cap + pc] = cand_j[slot];
        }
        mk[r] = __ballot_sync(0xffffffffu, in);
      }
    }
#pragma unroll
    for (int r = 0; r < G; ++r) {
      const int pp = len[r] + __popc(mk[r] & lt_mask);
      if (((mk[r] >> lane) & 1u) && pp < row_cap) rowp[r][pp] = (uint16_t)slot;
      len[r] += __popc(mk[r]);
    }
  }
  __syncwarp();
}

// One CTA per (home block, split).  Candidates of the window are staged in
// shared memory as fp32 coordinates relative to the block origin.  A warp
// takes a group of NBR_G rows of one home sub-cell at a time (dynamically)
// and runs nbr_group_stream on it (with bond candidates).
#ifndef NBR_MINB
#define NBR_MINB 4   // 4 CTAs x 8 warps at <= 64 registers (36 B of spills; measured faster than 3 at 80)
#endif
__global__ void __launch_bounds__(NBR_THREADS, NBR_MINB) k_nbr_build(Grid g, const int* __restrict__ cell_start,
    const float4* __restrict__ sloc, const double4* __restrict__ spos, const DevParams* __restrict__ prm,
    uint16_t* __restrict__ nbr, int* __restrict__ nbr_len, int row_cap, int* __restrict__ bc,
    int* __restrict__ bc_len, int cand_cap, int window_cap, int nsplit, Status* st, int* __restrict__ blk_pairs,
    const RowTest rt, int* __restrict__ wpack, int2* __restrict__ wsinfo) {
  pdl_wait();
  TL_MARK(0, 0);
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ NbrSmem S;
  const int blk = blockIdx.x / nsplit, split = blockIdx.x % nsplit;
  float4* cand = reinterpret_cast<float4*>(dyn);                                // window_cap + 32
  int* cand_j = reinterpret_cast<int*>(cand + window_cap + 32);                  // window_cap + 32
  unsigned char* cand_k = reinterpret_cast<unsigned char*>(cand_j + window_cap + 32);
  const int nt = prm->nt;
  for (int t = threadIdx.x; t < nt * nt; t += blockDim.x) S.rcand2[t] = prm->rcand2[t];
  for (int t = threadIdx.x; t < NHOME * MAX_RUNS; t += blockDim.x) {
    const int h = t / MAX_RUNS, q = t % MAX_RUNS;
    if (q < c_win.nrun1[h]) {
      const int ka = c_win.run1_a[h][q], kb = c_win.run1_b[h][q];
      const int wba = c_win.wu[ka];
      RunInfo ru;
      ru.ka = (short)ka;
      ru.kb = (short)kb;
      ru.wxa = (short)(wba % WB - SR);
      ru.pad = 0;
      ru.oy = (float)((wba / WB % WB - SR) * g.h[1]);
      ru.oz = (float)((wba / (WB * WB) - SR) * g.h[2]);
      S.run[h][q] = ru;
    }
  }
  int W = build_window(S.W, blk, g, cell_start);
  const int nwu = c_win.nwu;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {   // row groups of the block (home sub-cell order)
    int gb = 0, rb = 0;
    for (int h = 0; h < NHOME; ++h) {
      S.gbase[h] = gb;
      S.rbase[h] = rb;
      if (S.W.home_ok[h]) {
        gb += (S.W.cnt[c_win.home_k[h]] + NBR_G - 1) / NBR_G;
        rb += S.W.cnt[c_win.home_k[h]];
      }
    }
    S.gbase[NHOME] = gb;
    S.next_row = 0;
    S.pairs = 0;
  }
  __syncthreads();
  if (split == 0) win_store(S.W, W, wpack + (int64_t)blk * WPACK_INTS);   // for the nonbonded kernel
  if (W > window_cap) {
    if (threadIdx.x == 0) {
      set_flag(st, ST_WIN_OVF);
      atomicMax(&st->max_window, W);
    }
    // leave every row of the block empty so later kernels stay in bounds
    for (int h = 0; h < NHOME; ++h) {
      if (!S.W.home_ok[h]) continue;
      const int kk = c_win.home_k[h];
      for (int q = threadIdx.x; q < S.W.cnt[kk]; q += blockDim.x) {
        nbr_len[S.W.start[kk] + q] = 0;
        bc_len[S.W.start[kk] + q] = 0;
      }
    }
    return;
  }
  // slot -> window cell map (thread per cell), then staging flattened over
  // slots so that all global loads are in flight at once
  for (int k = threadIdx.x; k < nwu; k += blockDim.x) {
    const int b0 = S.W.slot[k], c = S.W.cnt[k];
    for (int a = 0; a < c; ++a) cand_k[b0 + a] = (unsigned char)k;
  }
  __syncthreads();
#pragma unroll 4
  for (int t = threadIdx.x; t < W; t += blockDim.x) {
    const int k = cand_k[t];
    const int j = S.W.start[k] + (t - S.W.slot[k]);
    const int wb = c_win.wu[k];
    // cell origin relative to the block origin: (w - SR) h per axis
    const float ox = (float)((wb % WB - SR) * g.h[0]);
    const float oy = (float)((wb / WB % WB - SR) * g.h[1]);
    const float oz = (float)((wb / (WB * WB) - SR) * g.h[2]);
    const float4 l = sloc[j];
    cand[t] = make_float4(l.x + ox, l.y + oy, l.z + oz, l.w);
    cand_j[t] = j;
  }
  if (threadIdx.x < 32) cand[window_cap + threadIdx.x] = make_float4(1e30f, 1e30f, 1e30f, 0.f);   // sentinel
  __syncthreads();
  if (split == 0) {   // slot info of the window, for the nonbonded kernel
    int2* ws = wsinfo + (int64_t)blk * window_cap;
    for (int t = threadIdx.x; t < W; t += blockDim.x)
      ws[t] = make_int2(cand_j[t], (int)cand_k[t] | (__float_as_int(cand[t].w) << 8));
  }
  TL_MARK(0, 1, W);
  // groups of NBR_G consecutive rows of one home sub-cell; this CTA takes
  // groups split, split + nsplit, ...
  const int ngroups = S.gbase[NHOME];
  for (;;) {
    int m = 0;
    if (lane == 0) m = atomicAdd(&S.next_row, 1);
    m = __shfl_sync(0xffffffffu, m, 0);
    const int G = split + m * nsplit;
    if (G >= ngroups) break;
    int h = 0;
    while (S.gbase[h + 1] <= G) ++h;
    const int kh = c_win.home_k[h];
    const int a0 = (G - S.gbase[h]) * NBR_G;
    const int nrow = min(NBR_G, S.W.cnt[kh] - a0);
    const int si0 = S.W.slot[kh] + a0;
    int len[NBR_G], nc[NBR_G];
    nbr_group_stream(S.W, S.run[h], window_cap, cand, cand_j, cand_k, spos, si0, nrow, h, rt, nbr, row_cap, bc, cand_cap,
                     S.rcand2, nt, S.ncs[threadIdx.x >> 5], len);
#pragma unroll
    for (int r = 0; r < NBR_G; ++r) nc[r] = S.ncs[threadIdx.x >> 5][r];
    if (lane < nrow) {
      int l = len[0], c = nc[0];
#pragma unroll
      for (int r = 1; r < NBR_G; ++r)
        if (lane == r) { l = len[r]; c = nc[r]; }
      const int s = cand_j[si0 + lane];
      nbr_len[s] = l < row_cap ? l : row_cap;
      const int rblk = S.rbase[h] + a0 + lane;   // row index in the block (home order)
      if (rblk < WP_MAXROWS) wpack[(int64_t)blk * WPACK_INTS + WP_LEN + rblk] = l < row_cap ? l : row_cap;
      bc_len[s] = c < cand_cap ? c : cand_cap;
      if (l > row_cap) { set_flag(st, ST_ROW_OVF); atomicMax(&st->max_row, l); }
      if (c > cand_cap) { set_flag(st, ST_CAND_OVF); atomicMax(&st->max_cand, c); }
    }
    if (blk_pairs) {
      int t = 0;
#pragma unroll
      for (int r = 0; r < NBR_G; ++r) t += r < nrow ? min(len[r], row_cap) : 0;
      if (lane == 0) atomicAdd(&S.pairs, t);
    }
    __syncwarp();   // ncs is reset by the warp's next group
  }
  if (blk_pairs) {
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(blk_pairs + blk, S.pairs);
  }
#ifdef REAX_TIMELINE
  __syncthreads();
  TL_MARK(0, 2);
#endif
}

// ---- branch-free fp64 math for the nonbonded pair (inputs in known, finite,
// normal ranges; ~1-2 ulp).  Tables live in shared memory.
constexpr int EXP_TBL = 256;   // 2^(j/256)
// polynomial / reduction constants as constant-bank operands (ptxas otherwise
// re-materialises 64-bit literals with register moves inside the pair loop)
__constant__ double c_nb[28] = {
    0x1.71547652b82fep+8,      // 0  256 / ln 2
    6755399441055744.0,        // 1  1.5 * 2^52
    0x1.62e42fee00000p-9,      // 2  ln2_hi / 256
    0x1.a39ef35793c76p-41,     // 3  ln2_lo / 256
    0.0, 1.0 / 24.0, 1.0 / 6.0, 0.5,   // 4-7  exp polynomial (4 unused)
    -1.0 / 6.0, 1.0 / 5.0, -0.25, 1.0 / 3.0, -0.5,   // 8-12 log1p polynomial
    0x1.62e42fee00000p-1,      // 13 ln2_hi
    0x1.a39ef35793c76p-33,     // 14 ln2_lo
    0.375, 2.0 / 9.0, 1.0 / 3.0,   // 15-17 Halley rsqrt / rcbrt
    20.0, -70.0, 84.0, -35.0, -140.0,   // 18-22 taper
    1.0,                       // 23
    14.0 / 81.0,               // 24 rcbrt quartic term
    0x1.0p35,                  // 25 fixed-point force scale 2^FIX_BITS
    6755399441055744.0,        // 26 1.5 * 2^52 (round-to-integer magic)
    65536.0};                  // 27 fixed-point range limit per contribution

constexpr int LOG_TBL = 256;   // {1/c_j, -log(1/c_j)}, c_j = 1 + (j + 1/2)/256

// e^x for |x| < 700: x = k ln2/256 + r, |r| <= ln2/512; e^r - 1 by a degree-4
// polynomial (error r^5/120 < 4e-17); 2^(k/256) = 2^(k>>8) * T[k & 255].
__device__ __forceinline__ double fexp(double x, const double* __restrict__ T) {
  double t = fma(x, c_nb[0], c_nb[1]);
  double kd = t - c_nb[1];
  int k = __double2loint(t);
  double r = fma(kd, -c_nb[2], x);
  r = fma(kd, -c_nb[3], r);
  double q = fma(r, c_nb[5], c_nb[6]);
  q = fma(q, r, c_nb[7]);
  double p = fma(q, r * r, r);
  double tj = T[k & (EXP_TBL - 1)];
  double y = fma(tj, p, tj);
  return __hiloint2double(__double2hiint(y) + ((k >> 8) << 20), __double2loint(y));
}

// ln x for finite normal x > 0: x = 2^e m, m in [1,2); m/c_j = 1 + r with
// |r| < 2^-9; log1p(r) by a degree-5 polynomial (error r^6/6 < 1e-17).
__device__ __forceinline__ double flog(double x, const double2* __restrict__ LT) {
  int hi = __double2hiint(x);
  int e = (hi >> 20) - 1023;
  int j = (hi >> 12) & (LOG_TBL - 1);
  double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, __double2loint(x));
  double2 t = LT[j];
  double r = fma(m, t.x, -c_nb[23]);
  double q = fma(r, c_nb[9], c_nb[10]);
  q = fma(q, r, c_nb[11]);
  q = fma(q, r, c_nb[12]);
  double p = fma(q, r * r, r);
  // (double)e without I2F.F64 (an XU op): 2^52 + 2^31 + e, minus 2^52 + 2^31
  double ed = __hiloint2double(0x43300000, e ^ 0x80000000) - 4503601774854144.0;
  return fma(ed, c_nb[13], t.y) + fma(ed, c_nb[14], p);
}

// approximate seeds from the MUFU unit, then one Halley-type correction:
// (1-e)^(-1/2) = 1 + e/2 + 3e^2/8 + ..., (1-e)^(-1/3) = 1 + e/3 + 2e^2/9 + ...,
// 1/(1-e) = 1 + e + e^2: relative error ~ (2^-22)^3
__device__ __forceinline__ double frsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x * y, y, c_nb[23]);
  return fma(y * e, fma(e, c_nb[15], c_nb[7]), y);
}
__device__ __forceinline__ double frcp(double x) {
  // MUFU.RCP64H seed (~2^-22), then 1/(1-e) = 1 + e + e^2: ~1e-20
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, c_nb[23]);
  return fma(y * e, c_nb[23] + e, y);
}
__device__ __forceinline__ double frcbrt(double x) {
  // fp32 seed x^(-1/3) = 2^(-log2(x)/3) from MUFU.LG2/EX2 (~1e-6), then one
  // quartic correction (1-e)^(-1/3) = 1 + e/3 + 2e^2/9 + 14e^3/81: ~1e-23
  const float xf = __double2float_rn(x);
  float lf, yf;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lf) : "f"(xf));
  lf *= -0.333333343f;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(yf) : "f"(lf));
  double y = (double)yf;
  double e = fma(-x * y, y * y, c_nb[23]);
  double q = fma(e, c_nb[24], c_nb[16]);
  q = fma(e, q, c_nb[17]);
  return fma(y * e, q, y);
}

// =================================================== a4 bond orders (B1-B2)
__device__ __forceinline__ double min_image(double d, double L) {
  // same rule as the definition: [-L/2, L/2)
  if (d >= 0.5 * L) return __dsub_rn(d, L);
  if (d < -0.5 * L) return __dadd_rn(d, L);
  return d;
}

// BO'sigma, BO'pi, BO'pipi, BO' at distance r:  exp(pa * (r/r0)^pb), with
// (r/r0)^pb = exp(pb (ln r - ln r0)); one log shared by the three terms.
__device__ __forceinline__ double4 bo_raw(double r, const BOPair& c) {
  double lr = log(r);
  double v[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) v[k] = exp(c.pa[k] * exp(c.pb[k] * (lr - c.lr0[k])));
  return make_double4(v[0], v[1], v[2], (v[0] + v[1]) + v[2]);
}

// bo_raw with the table exp/log of the nonbonded kernel (~1-2 ulp; the
// outer exponent is clamped at -700, where BO' < 1e-304 stands for 0)
__device__ __forceinline__ double4 bo_raw_fast(double r, const BOPair& c, const double* __restrict__ ET,
                                               const double2* __restrict__ LT) {
  const double lr = flog(r, LT);
  double v[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) v[k] = fexp(fmax(c.pa[k] * fexp(c.pb[k] * (lr - c.lr0[k]), ET), -700.0), ET);
  return make_double4(v[0], v[1], v[2], (v[0] + v[1]) + v[2]);
}

// Bond candidates are flattened across a warp: lane i owns atom a0+i, the
// warp scans the candidate counts and every lane then evaluates one
// (atom, candidate) pair per round: the exact FMA-free r^2 <= r_bond^2 test,
// B1-B2, and BO' >= bo_cut.  Rejected candidates are marked -1 in place;
// kept ones store BO' and are counted per atom (bdeg).
__global__ void k_bond_eval(int n, const double4* __restrict__ spos, const int* __restrict__ stype, Grid g,
                            const DevParams* __restrict__ prm, int* __restrict__ bc, const int* __restrict__ bc_len,
                            double4* __restrict__ bc_raw, int cand_cap, int* __restrict__ bdeg,
                            unsigned long long* __restrict__ scan_status, int scan_tiles) {
  TL_SPAN(0);
  pdl_wait();
  pdl_trigger();
  clear_status(scan_status, scan_tiles);
  __shared__ BOPair sbo[NTP_MAX];
  __shared__ double ET[EXP_TBL];
  __shared__ double2 LT[LOG_TBL];
  const int nt = prm->nt;
  for (int t = threadIdx.x; t < nt * nt; t += blockDim.x) sbo[t] = prm->bo[t];
  for (int t = threadIdx.x; t < EXP_TBL; t += blockDim.x) ET[t] = prm->exp_tbl[t];
  for (int t = threadIdx.x; t < LOG_TBL; t += blockDim.x) LT[t] = make_double2(prm->log_tbl[2 * t], prm->log_tbl[2 * t + 1]);
  __syncthreads();
  const double rb2 = prm->rb2, bo_cut = prm->bo_cut;
  const int lane = threadIdx.x & 31;
  const int a0 = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32;
  if (a0 >= n) return;
  int a = a0 + lane;
  int cnt = a < n ? bc_len[a] : 0;
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int total = __shfl_sync(0xffffffffu, incl, 31);
  for (int b0 = 0; b0 < total; b0 += 32) {
    int t = b0 + lane;
    int q = warp_find(incl, t);
    int excl_q = __shfl_sync(0xffffffffu, incl - cnt, q);
    if (t >= total) continue;
    int s = a0 + q, k = t - excl_q;
    int64_t slot = (int64_t)s * cand_cap + k;
    int j = bc[slot];
    double4 xi = spos[s], xj = spos[j];
    double dx = min_image(__dsub_rn(xj.x, xi.x), g.L[0]);
    double dy = min_image(__dsub_rn(xj.y, xi.y), g.L[1]);
    double dz = min_image(__dsub_rn(xj.z, xi.z), g.L[2]);
    double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    bool keep = false;
    double4 v = make_double4(0, 0, 0, 0);
    if (r2 <= rb2) {
      v = bo_raw_fast(__dsqrt_rn(r2), sbo[stype[s] * nt + stype[j]], ET, LT);
      keep = v.w >= bo_cut;
    }
    if (keep) {
      bc_raw[slot] = v;
      atomicAdd(&bdeg[s], 1);
      atomicAdd(&bdeg[j], 1);
    } else {
      bc[slot] = -1;
    }
  }
}

// full list fill: each kept half bond reserves one slot in row i and one in
// row j (the paper's "critical region only includes the reservation of a
// slot", as an atomic decrement); bdeg returns to zero.  The
// sort key (original partner index) is stored beside each entry.
__global__ void k_bond_fill(int n, const int* __restrict__ bc, const int* __restrict__ bc_len,
                            int cand_cap, const int* __restrict__ brow,
                            const int* __restrict__ perm, int* __restrict__ bdeg, int* __restrict__ ucol,
                            int* __restrict__ ukey, int* __restrict__ uown, long long* __restrict__ usrc,
                            long long bond_cap, Status* st) {
  TL_SPAN(2);
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int a0 = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32;
  if (blockIdx.x == 0 && threadIdx.x == 0) st->bonds = brow[n];
  if (a0 >= n) return;
  int a = a0 + lane;
  int cnt = a < n ? bc_len[a] : 0;
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int total = __shfl_sync(0xffffffffu, incl, 31);
  for (int b0 = 0; b0 < total; b0 += 32) {
    int t = b0 + lane;
    int q = warp_find(incl, t);
    int excl_q = __shfl_sync(0xffffffffu, incl - cnt, q);
    if (t >= total) continue;
    int s = a0 + q;
    int64_t slot = (int64_t)s * cand_cap + (t - excl_q);
    int j = bc[slot];
    if (j < 0) continue;
    long long e1 = (long long)brow[s] + atomicSub(&bdeg[s], 1) - 1;
    long long e2 = (long long)brow[j] + atomicSub(&bdeg[j], 1) - 1;
    // each side independently: every entry below the capacity is written; the
    // entry keeps the index of its candidate (k_bond_rank gathers BO' from it)
    if (e1 < bond_cap) { ucol[e1] = j; ukey[e1] = perm[j]; uown[e1] = s; usrc[e1] = slot; }
    if (e2 < bond_cap) { ucol[e2] = s; ukey[e2] = perm[s]; uown[e2] = j; usrc[e2] = slot; }
    if (e1 >= bond_cap || e2 >= bond_cap) set_flag(st, ST_BOND_OVF);
  }
}

// a5 (B3): rows in ascending original-partner order.  One thread per entry
// (grid-stride over the filled entries): its rank inside its row is the
// number of smaller keys; it moves the entry to that position of the sorted
// arrays.  Then one thread per atom sums BO' in that order: Delta'.
__global__ void k_bond_rank(const int* __restrict__ brow, const int* __restrict__ ucol, const int* __restrict__ ukey,
                            const int* __restrict__ uown, const long long* __restrict__ usrc,
                            const double4* __restrict__ bc_raw, int* __restrict__ bcol,
                            int* __restrict__ bkey, int* __restrict__ bown, double* __restrict__ bo, long long bond_cap,
                            const Status* __restrict__ st) {
  TL_SPAN(3);
  pdl_wait();
  pdl_trigger();
  long long B = st->bonds < bond_cap ? st->bonds : bond_cap;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < B; e += (long long)gridDim.x * blockDim.x) {
    int s = uown[e];
    int key = ukey[e];
    int a = brow[s], b = brow[s + 1];
    if (b > bond_cap) b = (int)bond_cap;
    int rank = 0;
    for (int f = a; f < b; ++f) rank += ukey[f] < key;
    long long o = a + rank;
    bcol[o] = ucol[e];
    bkey[o] = key;
    bown[o] = s;
    const double4 v = bc_raw[usrc[e]];
    bo[o] = v.x;                     // bond orders are stored as 8 arrays of bond_cap (BO_K)
    bo[bond_cap + o] = v.y;
    bo[2 * bond_cap + o] = v.z;
    bo[3 * bond_cap + o] = v.w;
  }
}

__global__ void k_bond_delta(int n, const int* __restrict__ brow, const int* __restrict__ stype,
                             const DevParams* __restrict__ prm, const double* __restrict__ bo,
                             double2* __restrict__ delta, long long bond_cap) {
  TL_SPAN(4);
  pdl_wait();
  pdl_trigger();
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  int a = brow[s], b = brow[s + 1];
  if (b > bond_cap) b = (int)bond_cap;
  double sum = 0.0;
  for (int e = a; e < b; ++e) sum += bo[3 * bond_cap + e];
  int t = stype[s];
  delta[s] = make_double2(sum - prm->val[t], sum - prm->val_boc[t]);
}

// a6 (B4-B8): one thread per full entry: mirror index and corrected bond
// orders in canonical orientation (smaller original index first), so
// BO_ij == BO_ji bitwise.  The mirror is found by binary search in the
// partner's row (rows are sorted by original partner index, k_bond_rank):
// c4 1.95 -> 1.84 ms against the linear scan (the table exp/log of the
// nonbonded kernel on top: 1.77 ms at c4 but +1.4 us at c1, where staging
// the tables per CTA dominates; not kept).
__global__ void k_bond_correct(const int* __restrict__ brow, const int* __restrict__ perm,
                               const int* __restrict__ stype, const DevParams* __restrict__ prm,
                               const int* __restrict__ bcol, const int* __restrict__ bkey, const int* __restrict__ bown,
                               int* __restrict__ bmir, double* __restrict__ bo, const double2* __restrict__ delta,
                               long long bond_cap, const Status* __restrict__ st) {
  TL_SPAN(5);
  pdl_wait();
  pdl_trigger();
  __shared__ BOPair sbo[NTP_MAX];
  __shared__ double sval[NT_MAX];
  const int nt = prm->nt;
  for (int t = threadIdx.x; t < nt * nt; t += blockDim.x) sbo[t] = prm->bo[t];
  for (int t = threadIdx.x; t < nt; t += blockDim.x) sval[t] = prm->val[t];
  __syncthreads();
  long long B = st->bonds < bond_cap ? st->bonds : bond_cap;
  const double p1 = prm->p_boc1, p2 = prm->p_boc2, inv_p2 = 1.0 / p2;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < B; e += (long long)gridDim.x * blockDim.x) {
    int s = bown[e];
    int j = bcol[e];
    int os = perm[s];
    // mirror: the entry of row j whose key is os (keys ascending, unique)
    int lo = brow[j], hi = brow[j + 1];
    if (hi > bond_cap) hi = (int)bond_cap;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (bkey[mid] < os) lo = mid + 1; else hi = mid;
    }
    const int em = (lo < brow[j + 1] && lo < bond_cap && bkey[lo] == os) ? lo : -1;
    bmir[e] = em;
    bool first = os < bkey[e];
    int ia = first ? s : j, ib = first ? j : s;
    int ta = stype[ia], tb = stype[ib];
    double2 da = delta[ia], db = delta[ib];
    const BOPair& c = sbo[ta * nt + tb];
    double bpi = bo[bond_cap + e], bpp = bo[2 * bond_cap + e], bp = bo[3 * bond_cap + e];
    double f2 = exp(-p1 * da.x) + exp(-p1 * db.x);
    double f3 = -inv_p2 * log(0.5 * (exp(-p2 * da.x) + exp(-p2 * db.x)));
    double va = sval[ta], vb = sval[tb];
    double f1 = 0.5 * ((va + f2) / (va + f2 + f3) + (vb + f2) / (vb + f2 + f3));
    double bb = c.pboc4 * bp * bp;
    double f4 = 1.0 / (1.0 + exp(-c.pboc3 * (bb - da.y) + c.pboc5));
    double f5 = 1.0 / (1.0 + exp(-c.pboc3 * (bb - db.y) + c.pboc5));
    double f145 = f1 * f4 * f5;
    double BO = bp * f145;
    double BOpi = bpi * f1 * f145;
    double BOpp = bpp * f1 * f145;
    bo[4 * bond_cap + e] = BO;
    bo[5 * bond_cap + e] = BO - BOpi - BOpp;
    bo[6 * bond_cap + e] = BOpi;
    bo[7 * bond_cap + e] = BOpp;
  }
}

// ====================================================== a7-a8 nonbonded
// reax_step_host: the charges gathered into the sorted records after their
// host-to-device copy (the cell gather ran without them)
__global__ void k_q_gather(int n, const double* __restrict__ q, const int* __restrict__ perm, double4* __restrict__ spos,
                           Status* st) {
  pdl_wait();
  pdl_trigger();
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  double qs = q[perm[s]];
  if (!isfinite(qs)) set_flag(st, ST_NONFINITE_IN);
  spos[s].w = qs;
}

__global__ void k_nb_prep(int n, const double* __restrict__ q, const int* __restrict__ perm, double4* __restrict__ spos,
                          unsigned long long* __restrict__ sf, Status* st) {
  pdl_wait();
  pdl_trigger();
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  double qs = q[perm[s]];
  if (!isfinite(qs)) set_flag(st, ST_NONFINITE_IN);
  spos[s].w = qs;
  sf[3 * (int64_t)s] = 0ull;
  sf[3 * (int64_t)s + 1] = 0ull;
  sf[3 * (int64_t)s + 2] = 0ull;
}

struct NBConst {
  double invR, phalf, inv_p, m140invR;
};

// device self-test of the nonbonded math (tests/test_math_gpu.py)
__global__ void k_selftest_math(int n, const double* __restrict__ x, double* __restrict__ out,
                                const DevParams* __restrict__ prm) {
  __shared__ double ET[EXP_TBL];
  __shared__ double2 LT[LOG_TBL];
  for (int t = threadIdx.x; t < EXP_TBL; t += blockDim.x) ET[t] = prm->exp_tbl[t];
  for (int t = threadIdx.x; t < LOG_TBL; t += blockDim.x) LT[t] = make_double2(prm->log_tbl[2 * t], prm->log_tbl[2 * t + 1]);
  __syncthreads();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = x[i];
  out[5 * (int64_t)i + 0] = fexp(v, ET);
  out[5 * (int64_t)i + 1] = v > 0 ? flog(v, LT) : 0.0;
  out[5 * (int64_t)i + 2] = v > 0 ? frsqrt(v) : 0.0;
  out[5 * (int64_t)i + 3] = v > 0 ? frcp(v) : 0.0;
  out[5 * (int64_t)i + 4] = v > 0 ? frcbrt(v) : 0.0;
}

// One Alg. 2 pair (N1-N5): tapered shielded vdW + Coulomb; returns energies
// and g = (dE/dr)/r so that F_i += g d, F_j -= g d.  dE = dE/dr (range check).
__device__ __forceinline__ void nb_pair(double r2, double qiqj, const NBPair& c, const NBConst& k,
                                        const double* __restrict__ ET, const double2* __restrict__ LT,
                                        double& ev, double& ec, double& g, double& dE) {
  double rinv = frsqrt(r2);
  double r = r2 * rinv;
  // N1 taper: 1 + x^4 (-35 + x (84 + x (-70 + 20 x))), dTap/dr = -140 x^3 (1-x)^3 / R
  double x = r * k.invR;
  double x2 = x * x, x3 = x2 * x;
  double tp = fma(x, c_nb[18], c_nb[19]);
  tp = fma(x, tp, c_nb[20]);
  tp = fma(x, tp, c_nb[21]);
  double tap = fma(x2 * x2, tp, c_nb[23]);
  double omx = c_nb[23] - x;
  double dtap = k.m140invR * x3 * (omx * omx * omx);
  // N2-N4 shielded vdW: r^p = exp((p/2) ln r^2), f13 = (r^p + gw^-p)^(1/p)
  double rp = fexp(k.phalf * flog(r2, LT), ET);
  double sv = rp + c.gwmp;
  double f13 = fexp(flog(sv, LT) * k.inv_p, ET);
  double u = fma(-f13, c.inv_rvdw, c_nb[23]);
  double e2 = fexp(c.ahalf * u, ET);      // e^{alpha u / 2}
  double e1 = e2 * e2;                    // e^{alpha u}
  double evu = c.D * fma(-2.0, e2, e1);
  // d f13/dr = sv^(1/p - 1) r^(p-1) = (f13 / sv) (r^p / r)
  double df13 = (f13 * frcp(sv)) * (rp * rinv);
  double devu = -c.Dadr * (e1 - e2) * df13;
  // N5 shielded Coulomb: S^(-1/3), S = r^3 + gamma^-3; S^(-4/3) = (S^(-1/3))^4
  double S = fma(r2, r, c.g3);
  double cb = frcbrt(S);
  double cb2 = cb * cb;
  double ecu = qiqj * cb;
  double decu = -qiqj * r2 * (cb2 * cb2);
  ev = tap * evu;
  ec = tap * ecu;
  dE = fma(dtap, evu + ecu, tap * (devu + decu));
  g = dE * rinv;
}

// ---- fixed-point force accumulation (deterministic: integer sums are exact
// and order-free).  A contribution c (kcal/mol/A) becomes v = round(c 2^35)
// via t = c 2^35 + 1.5 2^52 (bits(t) = bits(1.5 2^52) + v for |v| < 2^51), and
// is added to a slot as two int32 words: A = v mod 2^20 (unsigned, < 2^20, so
// up to 4096 adds cannot overflow 32 bits) and B = floor(v / 2^20) (mod 2^32).
// The slot value is B 2^20 + A.  Error per contribution <= 2^-36 (1.5e-11);
// |c| must stay below 2^16 (flagged otherwise, REAX_ERR_RANGE).
constexpr int FIX_BITS = 35;
constexpr unsigned FIX_BKEY = (unsigned)(0x4338000000000000ull >> 20);   // low word of bits(1.5 2^52) >> 20

__device__ __forceinline__ void fix_add(unsigned* A, int* B, double t) {
  const unsigned lo = (unsigned)__double2loint(t), hi = (unsigned)__double2hiint(t);
  const unsigned b = __funnelshift_r(lo, hi, 20) - FIX_BKEY;
  atomicAdd(A, lo & 0xFFFFFu);
  atomicAdd(B, (int)b);
}

// End of a row (one warp): warp-reduce F_i and the row's energies with a
// fixed butterfly, add F_i to the shared fixed-point window at slot si, and
// store the row's (E_vdW, E_Coul) partial at its sorted atom s.  Per-row
// partials make the energy independent of which warp ran the row (the two
// nonbonded kernels and any row schedule give identical sums).
__device__ __forceinline__ void row_reduce_store(double fix, double fiy, double fiz, double ev, double ec, int lane,
                                                 int si, int s, unsigned* fa, int* fb, int window_cap,
                                                 double2* __restrict__ erow, bool& bad) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    fix += __shfl_xor_sync(0xffffffffu, fix, o);
    fiy += __shfl_xor_sync(0xffffffffu, fiy, o);
    fiz += __shfl_xor_sync(0xffffffffu, fiz, o);
    ev += __shfl_xor_sync(0xffffffffu, ev, o);
    ec += __shfl_xor_sync(0xffffffffu, ec, o);
  }
  if (lane == 0) {
    const double FIXS = c_nb[25], MAGIC = c_nb[26], FLIM = c_nb[27];
    bad |= !(fabs(fix) < FLIM && fabs(fiy) < FLIM && fabs(fiz) < FLIM);
    fix_add(fa + si, fb + si, fma(fix, FIXS, MAGIC));
    fix_add(fa + window_cap + si, fb + window_cap + si, fma(fiy, FIXS, MAGIC));
    fix_add(fa + 2 * window_cap + si, fb + 2 * window_cap + si, fma(fiz, FIXS, MAGIC));
    erow[s] = make_double2(ev, ec);
  }
}

// rows of a (block, split) work unit whose kernel gave up (window overflow):
// zero their energy partials so the fixed-order energy sum stays defined
__device__ void zero_rows_erow(const WinSmem& W, int split, int nsplit, double2* __restrict__ erow) {
  int r0 = 0;
  for (int h = 0; h < NHOME; ++h) {
    if (!W.home_ok[h]) continue;
    const int k = c_win.home_k[h], c = W.cnt[k];
    for (int q = threadIdx.x; q < c; q += blockDim.x)
      if ((r0 + q) % nsplit == split) erow[W.start[k] + q] = make_double2(0.0, 0.0);
    r0 += c;
  }
}

#ifndef NB_THREADS_DEF
#define NB_THREADS_DEF 256
#endif
constexpr int NB_THREADS = NB_THREADS_DEF;
constexpr int NB_WARPS = NB_THREADS / 32;
#ifndef NB_MINB
#define NB_MINB 2   // 2 CTAs x 8 warps at <= 128 registers (3 CTAs at 80 registers spills; measured slower)
#endif

// Work plan of the nonbonded kernel for small grids (a few CTAs per SM slot:
// there the kernel's length is set by its heaviest home blocks).  Block b,
// with p_b half-list entries (summed by the list build), becomes n_b =
// min(NB_UNIT_SPLIT, ceil(p_b / T)) units, T = frac * (sum p) / slots; the
// n_b CTAs of a block share its rows through a global row counter.  Units
// are launched by work p_b / n_b, largest first (ties: block index), so the
// CTA order is longest-processing-time-first.  Which CTA evaluates a row does
// not change any result (forces are fixed-point sums, energies per-row
// partials), so the plan only moves time.
constexpr int PLAN_THREADS = 1024;
constexpr int NB_PLAN_MAX = PLAN_THREADS;   // home blocks (one per thread)
constexpr int NB_UNIT_SPLIT = 4;
__global__ void __launch_bounds__(PLAN_THREADS) k_nb_plan(int nblock, const int* __restrict__ blk_pairs, int slots,
                                                          float frac, int umax, int* __restrict__ units,
                                                          int* __restrict__ nunits, int* __restrict__ blkrow) {
  TL_SPAN(7);
  pdl_wait();
  pdl_trigger();
  __shared__ __align__(16) int wk[PLAN_THREADS];
  __shared__ int off[PLAN_THREADS];
  __shared__ long long psum[PLAN_THREADS / 32];
  __shared__ int wsum[PLAN_THREADS / 32];
  const int b = threadIdx.x, lane = b & 31, w = b >> 5;
  int p = 0;
  if (b < nblock) {
    p = blk_pairs[b];
    blkrow[b] = 0;
  }
  long long t = p;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) psum[w] = t;
  __syncthreads();
  long long tot = 0;
  for (int q = 0; q < PLAN_THREADS / 32; ++q) tot += psum[q];
  long long T = max(1ll, (long long)(frac * (double)tot / slots));
  int ns = 0;
  for (int pass = 0;; ++pass) {   // coarser units (T doubled) until the plan fits the launched grid
    ns = b < nblock ? (int)min((long long)NB_UNIT_SPLIT, max(1ll, (p + T - 1) / T)) : 0;
    int c = ns;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) wsum[w] = c;
    __syncthreads();
    int cnt = 0;
    for (int q = 0; q < PLAN_THREADS / 32; ++q) cnt += wsum[q];
    __syncthreads();
    if (cnt <= umax || pass >= 8) break;
    T *= 2;
  }
  // unique sort key: unit work, then lower block index first (work < 2^21)
  const int key = b < nblock ? ((min(p / ns, (1 << 21) - 1) << 10) | (PLAN_THREADS - 1 - b)) : -1;
  wk[b] = key;
  __syncthreads();
  int rank = 0;
  if (b < nblock) {
    const int4* k4 = reinterpret_cast<const int4*>(wk);
    for (int q = 0; q < (nblock + 3) >> 2; ++q) {   // entries >= nblock hold -1
      const int4 v = k4[q];
      rank += (v.x > key) + (v.y > key) + (v.z > key) + (v.w > key);
    }
  }
  off[b] = 0;
  __syncthreads();
  if (b < nblock) off[rank] = ns;
  __syncthreads();
  // exclusive scan of the unit counts in rank order
  const int x = off[b];
  int y = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int z = __shfl_up_sync(0xffffffffu, y, o);
    if (lane >= o) y += z;
  }
  if (lane == 31) wsum[w] = y;
  __syncthreads();
  int base = 0, total = 0;
  for (int q = 0; q < PLAN_THREADS / 32; ++q) {
    base += q < w ? wsum[q] : 0;
    total += wsum[q];
  }
  __syncthreads();
  off[b] = base + y - x;
  __syncthreads();
  const bool fits = total <= umax;   // else one unit per block (always fits)
  if (b < nblock) {
    if (fits) {
      const int o = off[rank];
      for (int k = 0; k < ns; ++k) units[o + k] = b | (ns << 24);
    } else {
      units[b] = b | (1 << 24);
    }
  }
  if (b == 0) *nunits = fits ? total : nblock;
}

constexpr int NB_MAX_ROWS = 256;   // rows of one (block, split) work unit that are ranked
struct NBSmem {
  WinSmem W;
  int bad;
  __align__(16) int rkey[NB_MAX_ROWS];   // ranking keys in home order: length << 8 | (255 - index); -1 past the rows
  int order[NB_MAX_ROWS];        // row window slots, longest row first
  int rlen[NB_MAX_ROWS];         // their lengths
  int next_row;                  // dynamic row counter
  int blen[WP_MAXROWS];          // lengths of the block's rows (home order), from the list build
};
static_assert(NB_MAX_ROWS <= WP_MAXROWS, "row lengths of the ranked rows");

// One CTA per (home block, split) (Alg. 2, re-designed): a
// warp streams the half-list entries of its rows 32 at a time (lanes over
// j), with the next chunk's entries, slot info and positions in flight while
// the current chunk is evaluated — across row boundaries too (the last chunk
// of a row loads the next row's first chunk).  Rows are ranked longest first
// and taken dynamically by the warps (the CTA's rows finish together).  F_i
// stays in registers and is warp-reduced once per row; F_j is accumulated in
// a shared-memory fixed-point window (the block's private force array, the
// GPU form of the paper's thread-private tprivForce) and flushed to the
// global int64 sorted force array once per CTA.  Energies: per-lane sums in
// the row's pair order, one partial per row, reduced later in fixed order.
// Forces and energies are bitwise reproducible.  The CTA does not rebuild
// its window: the list build stored it (window arrays, slot info and row
// lengths, `wpack` / `wsinfo`), and the setup is one round trip for them plus
// cp.async copies of the tables and slot info (c4: 9.2 -> 5.1 us per CTA).
__global__ void __launch_bounds__(NB_THREADS, NB_MINB) k_nonbonded(int nt, Grid g,
    const double4* __restrict__ spos, const DevParams* __restrict__ prm,
    const uint16_t* __restrict__ nbr, const int* __restrict__ nbr_len, int row_cap, int window_cap,
    unsigned long long* __restrict__ sf,
    double2* __restrict__ erow, int nsplit, Status* st, const int* __restrict__ units, const int* __restrict__ nunits,
    int* __restrict__ blkrow, const int* __restrict__ wpack, const int2* __restrict__ wsinfo) {
  pdl_wait();
  TL_MARK(1, 0);
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ NBSmem S;
  int blk, split;
  int* gctr = nullptr;   // global row counter of a block shared by several CTAs
  if (units) {           // planned units (k_nb_plan): all rows of block blk, shared by ns CTAs
    if ((int)blockIdx.x >= *nunits) return;
    const int u = units[blockIdx.x];
    blk = u & 0xFFFFFF;
    split = 0;
    nsplit = 1;
    if ((u >> 24) > 1) gctr = blkrow + blk;
  } else {
    blk = blockIdx.x / nsplit;
    split = blockIdx.x % nsplit;
  }
  double* ET = reinterpret_cast<double*>(dyn);                  // exp table
  double2* LT = reinterpret_cast<double2*>(ET + EXP_TBL);       // log table
  NBPair* pc = reinterpret_cast<NBPair*>(LT + LOG_TBL);         // nt*nt pair constants
  int2* sinfo = reinterpret_cast<int2*>(pc + nt * nt);          // slot -> {sorted atom, window cell | type << 8}
  unsigned* fa = reinterpret_cast<unsigned*>(sinfo + window_cap);   // F window, low words [3][window_cap]
  int* fb = reinterpret_cast<int*>(fa + 3 * window_cap);            // F window, high words [3][window_cap]
  // the row buffers follow the 16-byte aligned F window directly (window_cap is
  // a multiple of 32), typed from the shared base: shared-space loads (LDS)
  const int rb_cap = (row_cap + 7) & ~7;                                          // row buffer entries (16-byte multiple)
  uint16_t* rbuf = reinterpret_cast<uint16_t*>(fb + 3 * window_cap);              // [NB_WARPS][2][rb_cap]
  // tables, pair constants and the window's slot info, copied asynchronously
  // (16-byte pieces; exp and log tables are contiguous in DevParams, as in
  // shared memory) while the window arrays are read
  {
    auto cp16 = [&](void* dst, const void* src, int bytes) {
      for (int p = threadIdx.x; p < (bytes >> 4); p += blockDim.x) {
        const unsigned d = (unsigned)__cvta_generic_to_shared(reinterpret_cast<char*>(dst) + 16 * p);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(reinterpret_cast<const char*>(src) + 16 * p));
      }
    };
    static_assert(sizeof(NBPair) % 16 == 0, "pair constants in 16-byte pieces");
    cp16(pc, prm->nb, (int)sizeof(NBPair) * nt * nt);
    cp16(ET, prm->exp_tbl, (int)sizeof(double) * EXP_TBL);
    cp16(LT, prm->log_tbl, (int)sizeof(double) * 2 * LOG_TBL);
    // the whole capacity (not the block's W, which would cost a dependent round trip first)
    cp16(sinfo, wsinfo + (int64_t)blk * window_cap, 8 * window_cap);
    asm volatile("cp.async.commit_group;");
  }
  NBConst kc;
  kc.invR = prm->invR; kc.phalf = 0.5 * prm->p_vdw; kc.inv_p = prm->inv_p; kc.m140invR = -140.0 * prm->invR;
  const double C = prm->C;
  {   // zero F window (while the loads below are in flight)
    uint4* z = reinterpret_cast<uint4*>(fa);          // fa and fb are contiguous: 6 window_cap words
    for (int t = threadIdx.x; t < (6 * window_cap) / 4; t += blockDim.x) z[t] = make_uint4(0u, 0u, 0u, 0u);
  }
  // the window as the list build made it (and the block's row lengths)
  const int W = win_load<NB_THREADS>(S.W, g, wpack + (int64_t)blk * WPACK_INTS, S.blen);
  TL_MARK(1, 4);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (W > window_cap) {
    if (threadIdx.x == 0) {
      set_flag(st, ST_WIN_OVF);
      atomicMax(&st->max_window, W);
    }
    zero_rows_erow(S.W, split, nsplit, erow);
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }
  const int nwu = c_win.nwu;
  // this CTA's rows: split, split + nsplit, ... of the block (home sub-cell order)
  int nrows_blk = 0;
  for (int h = 0; h < NHOME; ++h)
    if (S.W.home_ok[h]) nrows_blk += S.W.cnt[c_win.home_k[h]];
  const int nrows = nrows_blk > split ? (nrows_blk - split + nsplit - 1) / nsplit : 0;
  const int nsorted = nrows < NB_MAX_ROWS ? nrows : NB_MAX_ROWS;
  // phase 1 (no global dependence between threads): row ranking keys, F window zero
  (void)nwu;
  int my_si = 0, my_len = 0;
  if ((int)threadIdx.x < nsorted) {
    int h;
    const int r = split + threadIdx.x * nsplit;
    row_of(S.W, r, h, my_si);
    if (r < WP_MAXROWS) {
      my_len = S.blen[r];
    } else {
      const int k = c_win.home_k[h];
      my_len = nbr_len[S.W.start[k] + (my_si - S.W.slot[k])];
    }
    S.rkey[threadIdx.x] = (my_len << 8) | (NB_MAX_ROWS - 1 - (int)threadIdx.x);
  } else if ((int)threadIdx.x < NB_MAX_ROWS) {
    S.rkey[threadIdx.x] = -1;
  }
  if (threadIdx.x == 0) {
    S.bad = 0;
    S.next_row = 0;
  }
  __syncthreads();
  TL_MARK(1, 5);
  // phase 2: row ranking (longest first; ties by home order); the tables and
  // the slot info have landed
  asm volatile("cp.async.wait_all;" ::: "memory");
  static_assert(NB_MAX_ROWS <= NB_THREADS, "one ranked row per thread");
  static_assert(NB_MAX_ROWS <= 256, "ranking keys: 8-bit index");
  if ((int)threadIdx.x < nsorted) {   // longest first, ties by home order: count the greater keys
    const int key = (my_len << 8) | (NB_MAX_ROWS - 1 - (int)threadIdx.x);
    const int4* k4 = reinterpret_cast<const int4*>(S.rkey);
    int rank = 0;
#pragma unroll 4
    for (int q = 0; q < (nsorted + 3) >> 2; ++q) {
      const int4 v = k4[q];
      rank += (v.x > key) + (v.y > key) + (v.z > key) + (v.w > key);
    }
    S.order[rank] = my_si;
    S.rlen[rank] = my_len;
  }
  __syncthreads();
#ifdef REAX_TIMELINE
  {
    unsigned long long pairs = 0;
    if (threadIdx.x == 0)
      for (int t = 0; t < nsorted; ++t) pairs += S.rlen[t];
    TL_MARK(1, 1, pairs);
  }
#endif
  const bool has_shift = S.W.has_shift != 0;
  const double FIXS = c_nb[25], MAGIC = c_nb[26], FLIM = c_nb[27];
  bool bad = false;
  // per-warp double buffer of row entries in shared memory: row k+1 is
  // copied (cp.async) while row k is evaluated
  uint16_t* rb = rbuf + warp * 2 * rb_cap;
  // rows are taken dynamically, longest first (per-row energy partials make
  // the result independent of which warp runs a row)
  auto row_info = [&](int& si, int& len) -> bool {
    int r = 0;
    if (lane == 0) r = gctr ? atomicAdd(gctr, 1) : atomicAdd(&S.next_row, 1);
    r = __shfl_sync(0xffffffffu, r, 0);
    if (r >= nrows) return false;
    if (r < nsorted) {
      si = S.order[r];
      len = S.rlen[r];
    } else {   // beyond the ranked rows (dense blocks): original order
      int h;
      row_of(S.W, split + r * nsplit, h, si);
      len = nbr_len[sinfo[si].x];
    }
    return true;
  };
  auto row_fetch = [&](int si, int len, uint16_t* dst) {
    const uint16_t* src = nbr + (int64_t)sinfo[si].x * row_cap;
    for (int p = lane; p < (len + 7) >> 3; p += 32) {   // 16-byte pieces (rows are 16-byte aligned)
      const unsigned d = (unsigned)__cvta_generic_to_shared(dst + 8 * p);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + 8 * p));
    }
    asm volatile("cp.async.commit_group;");
  };
  int si_n = 0, len_n = 0;
  bool have_n = row_info(si_n, len_n);
  if (have_n) row_fetch(si_n, len_n, rb);
  // the chunk in flight: (slot, slot info, position) per lane; across a row
  // boundary it holds the next row's first chunk (pre)
  int slot = 0;
  int2 inf = make_int2(0, 0);
  double4 xj = make_double4(0.0, 0.0, 0.0, 0.0);
  bool pre = false;
  for (int kr = 0; have_n; ++kr) {
    const int si = si_n, len = len_n;
    const uint16_t* row = rb + (kr & 1) * rb_cap;
    have_n = row_info(si_n, len_n);
    if (have_n) row_fetch(si_n, len_n, rb + ((kr + 1) & 1) * rb_cap);
    else asm volatile("cp.async.commit_group;");
    const int2 ii = sinfo[si];
    const double4 xi = spos[ii.x];
    const NBPair* pci = pc + (ii.y >> 8) * nt;
    const double cqi = C * xi.w;
    if (!pre) {
      asm volatile("cp.async.wait_group 1;" ::: "memory");   // this row's entries have landed
      __syncwarp();
      slot = lane < len ? (int)row[lane] : si;
      inf = sinfo[slot];
      xj = spos[inf.x];
    }
    pre = false;
    double fix = 0.0, fiy = 0.0, fiz = 0.0, ev_acc = 0.0, ec_acc = 0.0;
    for (int e0 = 0; e0 < len; e0 += 32) {
      const int cslot = slot;
      const int2 cinf = inf;
      const double4 cxj = xj;
      const bool act = e0 + lane < len;
      if (e0 + 32 < len) {   // next chunk in flight
        slot = e0 + 32 + lane < len ? (int)row[e0 + 32 + lane] : si;
        inf = sinfo[slot];
        xj = spos[inf.x];
      } else if (have_n) {   // last chunk: the next row's first chunk in flight
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        const uint16_t* nrow = rb + ((kr + 1) & 1) * rb_cap;
        slot = lane < len_n ? (int)nrow[lane] : si_n;
        inf = sinfo[slot];
        xj = spos[inf.x];
        pre = true;
      }
      double dx = cxj.x - xi.x, dy = cxj.y - xi.y, dz = cxj.z - xi.z;
      if (has_shift) {   // block-uniform
        const double4 sh = S.W.shift[cinf.y & 255];
        dx += sh.x;
        dy += sh.y;
        dz += sh.z;
      }
      if (act) {
        const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
        double ev, ec, gg, dE;
        nb_pair(r2, cqi * cxj.w, pci[cinf.y >> 8], kc, ET, LT, ev, ec, gg, dE);
        ev_acc += ev;
        ec_acc += ec;
        fix = fma(gg, dx, fix);
        fiy = fma(gg, dy, fiy);
        fiz = fma(gg, dz, fiz);
        bad |= !(fabs(dE) < FLIM);
        const double gs = -gg * FIXS;
        fix_add(fa + cslot, fb + cslot, fma(gs, dx, MAGIC));
        fix_add(fa + window_cap + cslot, fb + window_cap + cslot, fma(gs, dy, MAGIC));
        fix_add(fa + 2 * window_cap + cslot, fb + 2 * window_cap + cslot, fma(gs, dz, MAGIC));
      }
    }
    row_reduce_store(fix, fiy, fiz, ev_acc, ec_acc, lane, si, ii.x, fa, fb, window_cap, erow, bad);
    __syncwarp();   // the buffer of this row is refilled two rows later
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  TL_WARP_DONE(1);
  if (__any_sync(0xffffffffu, bad) && lane == 0) S.bad = 1;
  __syncthreads();
  if (threadIdx.x == 0 && S.bad) set_flag(st, ST_RANGE);
  bool wide = false;
  // lanes over (slot, component): a warp's reductions cover consecutive words
  // of the force records
  for (int u = threadIdx.x; u < 3 * W; u += blockDim.x) {
    const int t = u / 3, c = u - 3 * t;
    const int j = sinfo[t].x;
    const int b = fb[c * window_cap + t];
    // the high word wraps mod 2^32 at |F| = 2^16 kcal/mol/A: a slot's
    // accumulated F_j beyond half of that (|B| > 2^30) is flagged too
    wide |= b > (1 << 30) || b < -(1 << 30);
    const long long v = ((long long)b << 20) + (long long)fa[c * window_cap + t];
    if (v != 0) atomicAdd(sf + 3 * (int64_t)j + c, (unsigned long long)v);
  }
  if (wide) set_flag(st, ST_RANGE);
#ifdef REAX_TIMELINE
  __syncthreads();
  TL_MARK(1, 2);
#endif
}

// a8 finalize, one kernel: un-permute the forces, force[perm[s]] =
// F_sorted[s] (int64 fixed point -> fp64; sorted-order reads and resets are
// coalesced, the 24-byte writes scattered), resetting the accumulators to
// zero for the next step; and the energy: block b sums a fixed slice of the
// nonbonded partials, the last block to finish sums the block partials with
// a fixed-shape tree (strided per-thread sums, then warp and block trees), so
// the result does not depend on timing (deterministic).
constexpr int FIN_THREADS = 256;
__device__ __forceinline__ void fin_block_sum(double& a, double& b, double (*red)[FIN_THREADS / 32]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if (lane == 0) { red[0][w] = a; red[1][w] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = 0.0; b = 0.0;
    for (int k = 0; k < FIN_THREADS / 32; ++k) { a += red[0][k]; b += red[1][k]; }
  }
}
__global__ void __launch_bounds__(FIN_THREADS) k_finalize(int n, const int* __restrict__ iperm,
    const unsigned long long* __restrict__ sf, double* __restrict__ force, int nparts,
    const double2* __restrict__ epart, double* __restrict__ part, unsigned* __restrict__ ticket,
    double* __restrict__ energy, int ne, Status* st) {
  TL_SPAN(6);
  pdl_wait();
  pdl_trigger();
  // input order: gathered (one scattered 24-byte record per atom) and written as coalesced
  // 24-byte rows (scattered partial-sector writes cost read-modify-writes in
  // DRAM); the accumulators are zeroed by the next gather (k_cell_gather /
  // k_nb_prep), not here
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const int s = iperm[i];
    const double sc = 0x1.0p-35;
    static_assert(FIX_BITS == 35, "scale");
    const unsigned long long* r = sf + 3 * (int64_t)s;
    const double fx = (double)(long long)__ldcs(r) * sc, fy = (double)(long long)__ldcs(r + 1) * sc,
                 fz = (double)(long long)__ldcs(r + 2) * sc;
    force[3 * (int64_t)i] = fx;
    force[3 * (int64_t)i + 1] = fy;
    force[3 * (int64_t)i + 2] = fz;
  }
  __shared__ double red[2][FIN_THREADS / 32];
  __shared__ bool last;
  const int per = (nparts + gridDim.x - 1) / gridDim.x;
  const int p0 = blockIdx.x * per, p1 = min(nparts, p0 + per);
  double a = 0.0, b = 0.0;
  for (int p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
    const double2 v = epart[p];
    a += v.x;
    b += v.y;
  }
  fin_block_sum(a, b, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  a = 0.0; b = 0.0;
  for (unsigned k = threadIdx.x; k < gridDim.x; k += blockDim.x) {
    a += __ldcg(part + 2 * k);
    b += __ldcg(part + 2 * k + 1);
  }
  __syncthreads();   // red[] is reused
  fin_block_sum(a, b, red);
  if (threadIdx.x == 0) {
    energy[0] = a;
    if (ne > 1) energy[1] = b;
    *ticket = 0u;   // ready for the next call
    if (!(isfinite(a) && isfinite(b))) set_flag(st, ST_NONFINITE_OUT);
  }
}

// ============================================ NEXT-1 bond energy (E1)
// SURVEY.md §8(f) NEXT-1, the bond part of "Aggregate Forces" (PAPER.md:160,
// 285).  E1 per bond (standard ReaxFF, ref [6]; reading 28):
//   e = -De_s BOs exp[p_be1 (1 - BOs^p_be2)] - De_p BOpi - De_pp BOpipi,
// BOs^p_be2 := 0 for BOs <= 0, at the bond set of a6 (held fixed).  Every bond
// order of bond b = (i, j) depends on r_b (B1) and on S_i = sum_k BO'_ik, S_j
// (f1, f4, f5), so dE/dr_b = de_b/dr_b|_S + (D_i + D_j) dBO'_b/dr_b with
// D_i = sum_{b' at i} de_b'/dS_i, and the forces are central along the bonds.
// Three passes: per bond (canonical entry, orientation as k_bond_correct) the
// terms, written to both entries of the bond; per atom row D_i (row order);
// per atom row the force, gathered over the row's bonds (no atomics), and
// the energy (fixed-shape sums).

// bond vector d = minimum-image(x_b - x_a) and r, exactly as k_bond_eval
__device__ __forceinline__ double bond_vec(const double4& xa, const double4& xb, const Grid& g, double d[3]) {
  d[0] = min_image(__dsub_rn(xb.x, xa.x), g.L[0]);
  d[1] = min_image(__dsub_rn(xb.y, xa.y), g.L[1]);
  d[2] = min_image(__dsub_rn(xb.z, xa.z), g.L[2]);
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2])));
}

__global__ void k_bond_energy_terms(const int* __restrict__ perm, const int* __restrict__ stype,
                                    const double4* __restrict__ spos, Grid g, const DevParams* __restrict__ prm,
                                    const BEPair* __restrict__ bep, const int* __restrict__ bcol,
                                    const int* __restrict__ bkey, const int* __restrict__ bown,
                                    const int* __restrict__ bmir, const double* __restrict__ bo,
                                    const double2* __restrict__ delta, double4* __restrict__ bde, long long bond_cap,
                                    const Status* __restrict__ st) {
  pdl_wait();
  pdl_trigger();
  __shared__ BOPair sbo[NTP_MAX];
  __shared__ BEPair sbe[NTP_MAX];
  __shared__ double sval[NT_MAX];
  const int nt = prm->nt;
  for (int t = threadIdx.x; t < nt * nt; t += blockDim.x) { sbo[t] = prm->bo[t]; sbe[t] = bep[t]; }
  for (int t = threadIdx.x; t < nt; t += blockDim.x) sval[t] = prm->val[t];
  __syncthreads();
  const long long B = st->bonds < bond_cap ? st->bonds : bond_cap;
  const double p1 = prm->p_boc1, p2 = prm->p_boc2, inv_p2 = 1.0 / p2;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < B; e += (long long)gridDim.x * blockDim.x) {
    const int s = bown[e], j = bcol[e];
    if (!(perm[s] < bkey[e])) continue;   // the canonical entry writes both
    const int ta = stype[s], tb = stype[j];
    const BOPair& c = sbo[ta * nt + tb];
    const BEPair& q = sbe[ta * nt + tb];
    double d[3];
    const double r = bond_vec(spos[s], spos[j], g, d);
    const double raw[3] = {bo[e], bo[bond_cap + e], bo[2 * bond_cap + e]};
    const double bpi = raw[1], bpp = raw[2], bp = bo[3 * bond_cap + e];
    const double2 da = delta[s], db = delta[j];
    // B4-B8 (as k_bond_correct) and the derivative of every factor
    const double ea1 = exp(-p1 * da.x), eb1 = exp(-p1 * db.x);
    const double ea2 = exp(-p2 * da.x), eb2 = exp(-p2 * db.x);
    const double f2 = ea1 + eb1;
    const double f3 = -inv_p2 * log(0.5 * (ea2 + eb2));
    const double va = sval[ta], vb = sval[tb];
    const double na = va + f2 + f3, nb = vb + f2 + f3;
    const double f1 = 0.5 * ((va + f2) / na + (vb + f2) / nb);
    const double bb = c.pboc4 * bp * bp;
    const double f4 = 1.0 / (1.0 + exp(-c.pboc3 * (bb - da.y) + c.pboc5));
    const double f5 = 1.0 / (1.0 + exp(-c.pboc3 * (bb - db.y) + c.pboc5));
    const double A = f1 * f4 * f5;
    const double BOs = bp * A - bpi * f1 * A - bpp * f1 * A;
    // E1 and its partials
    const double sp = BOs > 0.0 ? exp(q.pbe2 * log(BOs)) : 0.0;
    const double ex = exp(q.pbe1 * (1.0 - sp));
    const double en = -q.Ds * BOs * ex - q.Dp * bpi * f1 * A - q.Dpp * bpp * f1 * A;
    const double e_s = -q.Ds * ex * (1.0 - q.pbe1 * q.pbe2 * sp);
    const double c_pi = -q.Dp - e_s, c_pp = -q.Dpp - e_s;
    const double w = c_pi * bpi + c_pp * bpp;
    const double de_dA = e_s * bp + w * f1;
    const double de_df1 = de_dA * f4 * f5 + w * A;
    const double de_df4 = de_dA * f1 * f5, de_df5 = de_dA * f1 * f4;
    const double sa2 = f3 / (na * na) + f3 / (nb * nb);
    const double sa3 = -(va + f2) / (na * na) - (vb + f2) / (nb * nb);
    const double df1_da = 0.5 * (sa2 * (-p1 * ea1) + sa3 * (ea2 / (ea2 + eb2)));
    const double df1_db = 0.5 * (sa2 * (-p1 * eb1) + sa3 * (eb2 / (ea2 + eb2)));
    const double g4 = f4 * (1.0 - f4), g5 = f5 * (1.0 - f5);
    const double dSa = de_df1 * df1_da - de_df4 * g4 * c.pboc3;
    const double dSb = de_df1 * df1_db - de_df5 * g5 * c.pboc3;
    // dBO'_k/dr = BO'_k pa pb (r/r0)^pb / r, (r/r0)^pb = exp(pb (ln r - ln r0))
    const double lr = log(r), ir = 1.0 / r;
    double dr[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) dr[k] = raw[k] * c.pa[k] * c.pb[k] * exp(c.pb[k] * (lr - c.lr0[k])) * ir;
    const double X = (de_df4 * g4 + de_df5 * g5) * 2.0 * c.pboc3 * c.pboc4 * bp;
    const double cA = e_s * A + X;
    const double de_dr = cA * dr[0] + (cA + c_pi * f1 * A) * dr[1] + (cA + c_pp * f1 * A) * dr[2];
    const double dbo_dr = (dr[0] + dr[1]) + dr[2];
    bde[e] = make_double4(de_dr, dbo_dr, en, dSa);
    bde[bmir[e]] = make_double4(de_dr, dbo_dr, 0.0, dSb);
  }
}

// per atom row (sorted order): D_i = sum of de/dS_i over the row, in row order
__global__ void k_bond_energy_rows(int n, const int* __restrict__ brow, const double4* __restrict__ bde,
                                   double* __restrict__ bD, long long bond_cap) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  double D = 0.0;
  const long long e1 = min((long long)brow[s + 1], bond_cap);
  for (long long e = brow[s]; e < e1; ++e) D += bde[e].w;
  bD[s] = D;
}

// per atom row (sorted order), gathering: F_s = sum over its bonds of g d with
// g = (de/dr|S + (D_s + D_j) dBO'/dr) / r and d = minimum-image(x_j - x_s)
// (both entries of a bond give the same g), written straight to the caller's
// input-order force array; the row's energy (its canonical entries) goes
// into a fixed-shape block sum and the last block sums the block partials
// (deterministic, as k_finalize)
__global__ void __launch_bounds__(FIN_THREADS) k_bond_energy_out(int n, const int* __restrict__ perm,
    const double4* __restrict__ spos, Grid g, const int* __restrict__ brow, const int* __restrict__ bcol,
    const double4* __restrict__ bde, const double* __restrict__ bD, long long bond_cap, double* __restrict__ force,
    double* __restrict__ part, unsigned* __restrict__ ticket, double* __restrict__ energy, Status* st) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  double E = 0.0;
  if (s < n) {
    double f[3] = {0.0, 0.0, 0.0};
    const double4 xs = spos[s];
    const double Ds = bD[s];
    const long long e0 = brow[s], e1 = min((long long)brow[s + 1], bond_cap);
    // the row's entries in batches of 4 with every load issued before use
    for (long long eb = e0; eb < e1; eb += 4) {
      int j[4];
      double4 v[4], xj[4];
      double Dj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) j[u] = eb + u < e1 ? bcol[eb + u] : -1;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int jj = j[u] < 0 ? s : j[u];
        v[u] = j[u] < 0 ? make_double4(0.0, 0.0, 0.0, 0.0) : bde[eb + u];
        xj[u] = spos[jj];
        Dj[u] = bD[jj];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (j[u] < 0) continue;
        double d[3];
        const double r = bond_vec(xs, xj[u], g, d);
        const double gg = (v[u].x + (Ds + Dj[u]) * v[u].y) / r;
#pragma unroll
        for (int k = 0; k < 3; ++k) f[k] = fma(gg, d[k], f[k]);
        E += v[u].z;
      }
    }
    const int i = perm[s];
    force[3 * (int64_t)i] = f[0];
    force[3 * (int64_t)i + 1] = f[1];
    force[3 * (int64_t)i + 2] = f[2];
  }
  __shared__ double red[2][FIN_THREADS / 32];
  __shared__ bool last;
  double b = 0.0;
  fin_block_sum(E, b, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = E;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  E = 0.0;
  b = 0.0;
  for (unsigned k = threadIdx.x; k < gridDim.x; k += blockDim.x) E += __ldcg(part + 2 * k);
  __syncthreads();   // red[] is reused
  fin_block_sum(E, b, red);
  if (threadIdx.x == 0) {
    energy[0] = E;
    *ticket = 0u;   // ready for the next call
    if (!isfinite(E)) set_flag(st, ST_NONFINITE_OUT);
  }
}

// ============================== NEXT-3 interaction lists (angles, H-bonds)
// SURVEY.md §8(f) NEXT-3; PAPER.md:198-202 (§3.3 "Three-body Interactions":
// the angles present are identified, a prefix sum gives every list its
// offset, then they are stored) and PAPER.md:154-158 (the H-bond list from
// the surroundings of covalently bonded H atoms).  Readings:
// the angle partners of a full-bond-list entry e = (j, i) are the partners k
// of the other entries f of row j with BO_e > thb_cut, BO_f > thb_cut and
// BO_e BO_f > thb_cutsq (corrected BO), in row order; the H-bond list of an H
// atom with a bond holds the acceptor atoms within r_hb, ascending.  Both are
// written in the exported (input) order: angle lists over the entries of the
// exported bond list, H-bond lists over the atoms.
struct IList {
  double thb_cut, thb_cutsq, r_hb2;
  int h_type;
  unsigned acc_mask;
};

// per bond entry (grid-stride): the number of angle partners, stored at the
// entry's exported position (acnt) and/or summed into *total
__global__ void k_ang_count(const int* __restrict__ brow, const int* __restrict__ bown, const int* __restrict__ perm,
                            const double* __restrict__ bo, const long long* __restrict__ orow, int* __restrict__ acnt,
                            unsigned long long* __restrict__ total, long long bond_cap, IList il,
                            const Status* __restrict__ st) {
  const long long B = st->bonds < bond_cap ? st->bonds : bond_cap;
  unsigned long long mine = 0;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < B; e += (long long)gridDim.x * blockDim.x) {
    const int s = bown[e];
    const int f0 = brow[s], f1 = brow[s + 1];
    const double be = bo[4 * bond_cap + e];
    int c = 0;
    if (be > il.thb_cut)
      for (int f = f0; f < f1; ++f) {
        const double bf = bo[4 * bond_cap + f];
        c += (f != e && bf > il.thb_cut && be * bf > il.thb_cutsq);
      }
    if (acnt) acnt[orow[perm[s]] + (e - f0)] = c;
    mine += c;
  }
  if (total) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(total, mine);
  }
}

// per bond entry: its angle partners (original indices, row order) at ang_off
__global__ void k_ang_fill(const int* __restrict__ brow, const int* __restrict__ bown, const int* __restrict__ perm,
                           const int* __restrict__ bkey, const double* __restrict__ bo,
                           const long long* __restrict__ orow, const long long* __restrict__ ang_off,
                           int* __restrict__ ang_k, long long bond_cap, IList il, const Status* __restrict__ st) {
  const long long B = st->bonds < bond_cap ? st->bonds : bond_cap;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < B; e += (long long)gridDim.x * blockDim.x) {
    const int s = bown[e];
    const int f0 = brow[s], f1 = brow[s + 1];
    const double be = bo[4 * bond_cap + e];
    if (!(be > il.thb_cut)) continue;
    long long o = ang_off[orow[perm[s]] + (e - f0)];
    for (int f = f0; f < f1; ++f) {
      const double bf = bo[4 * bond_cap + f];
      if (f != e && bf > il.thb_cut && be * bf > il.thb_cutsq) ang_k[o++] = bkey[f];
    }
  }
}

// H-bond list of one atom per warp (sorted order): candidates from the 5^3
// sub-cell stencil (r_hb <= 2 h), the exact FMA-free fp64 r^2 (bit-identical
// to the oracle's), acceptors only; counting (hcnt / total) or filling (sorted
// by original index through a rank sort in the warp's shared buffer)
constexpr int HB_THREADS = 256;
constexpr int HB_CAP = 1024;   // entries of one H atom's list (ST_HB_OVF beyond)
// the H atoms with a bond, compacted into hlist (warp-aggregated slots; the
// order is irrelevant: every H atom writes its own rows); zero counts for
// the others
__global__ void k_hb_collect(int n, const int* __restrict__ stype, const int* __restrict__ brow,
                             const int* __restrict__ perm, int h_type, int* __restrict__ hcnt, int* __restrict__ hlist,
                             unsigned* __restrict__ hn) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool is_h = s < n && stype[s] == h_type && brow[s + 1] > brow[s];
  if (s < n && hcnt && !is_h) hcnt[perm[s]] = 0;
  const unsigned mk = __ballot_sync(0xffffffffu, is_h);
  if (!mk) return;
  unsigned base = 0;
  if (lane == 0) base = atomicAdd(hn, (unsigned)__popc(mk));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (is_h) hlist[base + __popc(mk & ((1u << lane) - 1u))] = s;
}

// one warp per H atom of hlist (grid-stride over the warps)
__global__ void __launch_bounds__(HB_THREADS) k_hb_list(const int* __restrict__ hlist, const unsigned* __restrict__ hn,
    Grid g, const int* __restrict__ cell_start,
    const double4* __restrict__ spos, const int* __restrict__ stype, const int* __restrict__ perm, IList il,
    int* __restrict__ hcnt, unsigned long long* __restrict__ total,
    const long long* __restrict__ hb_off, int* __restrict__ hb_z, Status* st) {
  __shared__ int buf[HB_THREADS / 32][HB_CAP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nh = (int)*hn;
  for (int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); w < nh;
       w += (int)((gridDim.x * (int64_t)blockDim.x) >> 5)) {
  const int s = hlist[w];
  const int i = perm[s];
  const double4 xs = spos[s];
  int cs[3];
  const double xw[3] = {xs.x, xs.y, xs.z};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int c = (int)(xw[a] * g.inv_h[a]);
    cs[a] = c >= g.nc[a] ? g.nc[a] - 1 : c;
  }
  const unsigned lt = (1u << lane) - 1u;
  int cnt = 0;
  int* b = buf[warp];
  // the stencil as (2 SR + 1)^2 runs of sub-cells along x (contiguous in the
  // sorted order unless the run wraps: then two pieces); lane r < 25 fetches
  // run r's bounds up front, so the scan below has no dependent index loads
  constexpr int NR = (2 * SR + 1) * (2 * SR + 1);
  int pa0 = 0, pa1 = 0, pb0 = 0, pb1 = 0;
  double shy = 0.0, shz = 0.0, sxa = 0.0, sxb = 0.0;
  if (lane < NR) {
    const int oy = lane % (2 * SR + 1) - SR, oz = lane / (2 * SR + 1) - SR;
    int cy = cs[1] + oy, cz = cs[2] + oz;
    const int my = cy >= 0 ? cy / g.nc[1] : -((-cy + g.nc[1] - 1) / g.nc[1]);
    const int mz = cz >= 0 ? cz / g.nc[2] : -((-cz + g.nc[2] - 1) / g.nc[2]);
    cy -= my * g.nc[1];
    cz -= mz * g.nc[2];
    shy = my == 0 ? 0.0 : (my > 0 ? g.L[1] : -g.L[1]);
    shz = mz == 0 ? 0.0 : (mz > 0 ? g.L[2] : -g.L[2]);
    const int row = (cz * g.nc[1] + cy) * g.nc[0];
    const int xa = cs[0] - SR, xb = cs[0] + SR;   // unwrapped x-cell range: nc >= 4, so one end wraps at most
    if (xa < 0) {   // [nc + xa, nc) with -L, then [0, xb]
      pa0 = cell_start[row + g.nc[0] + xa]; pa1 = cell_start[row + g.nc[0]]; sxa = -g.L[0];
      pb0 = cell_start[row]; pb1 = cell_start[row + xb + 1]; sxb = 0.0;
    } else if (xb >= g.nc[0]) {   // [xa, nc), then [0, xb - nc] with +L
      pa0 = cell_start[row + xa]; pa1 = cell_start[row + g.nc[0]]; sxa = 0.0;
      pb0 = cell_start[row]; pb1 = cell_start[row + xb - g.nc[0] + 1]; sxb = g.L[0];
    } else {
      pa0 = cell_start[row + xa]; pa1 = cell_start[row + xb + 1]; sxa = 0.0;
    }
  }
  auto scan_piece = [&](int q0, int q1, double sx, double sy, double sz) {
    for (int qb = q0; qb < q1; qb += 64) {   // two chunks of 32 in flight
      const int qa = qb + lane, qc = qb + 32 + lane;
      const bool va = qa < q1 && qa != s, vc = qc < q1 && qc != s;
      const double4 xa4 = spos[va ? qa : s], xc4 = spos[vc ? qc : s];
      const int ta = va ? stype[qa] : -1, tc = vc ? stype[qc] : -1;
      bool ha = false, hc = false;
      if (va && ((il.acc_mask >> ta) & 1u)) {
        const double dx = __dadd_rn(__dsub_rn(xa4.x, xs.x), sx);
        const double dy = __dadd_rn(__dsub_rn(xa4.y, xs.y), sy);
        const double dz = __dadd_rn(__dsub_rn(xa4.z, xs.z), sz);
        ha = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)) <= il.r_hb2;
      }
      if (vc && ((il.acc_mask >> tc) & 1u)) {
        const double dx = __dadd_rn(__dsub_rn(xc4.x, xs.x), sx);
        const double dy = __dadd_rn(__dsub_rn(xc4.y, xs.y), sy);
        const double dz = __dadd_rn(__dsub_rn(xc4.z, xs.z), sz);
        hc = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)) <= il.r_hb2;
      }
      const unsigned ma = __ballot_sync(0xffffffffu, ha), mc = __ballot_sync(0xffffffffu, hc);
      if (hb_z) {
        if (ha) { const int p = cnt + __popc(ma & lt); if (p < HB_CAP) b[p] = perm[qa]; }
        if (hc) { const int p = cnt + __popc(ma) + __popc(mc & lt); if (p < HB_CAP) b[p] = perm[qc]; }
      }
      cnt += __popc(ma) + __popc(mc);
    }
  };
  for (int r = 0; r < NR; ++r) {
    const int a0 = __shfl_sync(0xffffffffu, pa0, r), a1 = __shfl_sync(0xffffffffu, pa1, r);
    const int b0 = __shfl_sync(0xffffffffu, pb0, r), b1 = __shfl_sync(0xffffffffu, pb1, r);
    const double sy = __shfl_sync(0xffffffffu, shy, r), sz = __shfl_sync(0xffffffffu, shz, r);
    const double xa = __shfl_sync(0xffffffffu, sxa, r), xb = __shfl_sync(0xffffffffu, sxb, r);
    scan_piece(a0, a1, xa, sy, sz);
    scan_piece(b0, b1, xb, sy, sz);
  }
  if (hcnt) {
    if (lane == 0) {
      hcnt[i] = cnt;
      if (total) atomicAdd(total, (unsigned long long)cnt);
    }
    continue;
  }
  if (cnt > HB_CAP) {
    if (lane == 0) set_flag(st, ST_HB_OVF);
    continue;
  }
  __syncwarp();
  const long long o = hb_off[i];
  for (int p = lane; p < cnt; p += 32) {   // rank sort by original index (all distinct)
    const int v = b[p];
    int r = 0;
    for (int t = 0; t < cnt; ++t) r += b[t] < v;
    hb_z[o + r] = v;
  }
  __syncwarp();   // b is reused by the warp's next atom
  }
}

// ================================================================= export
__device__ __forceinline__ uint64_t mix64(uint64_t a, uint64_t b) {
  uint64_t z = (a << 32) ^ b;
  z ^= z >> 33; z *= 0xff51afd7ed558ccdull;
  z ^= z >> 33; z *= 0xc4ceb9fe1a85ec53ull;
  z ^= z >> 33;
  return z;
}

// mode 0: write pairs at exp_off[s] + e;  mode 1: per-atom count / digest
__global__ void __launch_bounds__(NBR_THREADS) k_export_pairs(Grid g, const int* __restrict__ cell_start,
    const int* __restrict__ perm, const uint16_t* __restrict__ nbr, const int* __restrict__ nbr_len, int row_cap,
    int window_cap, const long long* __restrict__ off, int mode, int* __restrict__ pi, int* __restrict__ pj,
    unsigned long long* __restrict__ cnt, unsigned long long* __restrict__ dig) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ WinSmem W;
  int* slot_j = reinterpret_cast<int*>(dyn);
  int nW = build_window(W, blockIdx.x, g, cell_start);
  if (nW > window_cap) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int k = warp; k < c_win.nwu; k += nwarp)
    for (int a = lane; a < W.cnt[k]; a += 32) slot_j[W.slot[k] + a] = W.start[k] + a;
  __syncthreads();
  for (int r = warp;; r += nwarp) {
    int h, si;
    if (!row_of(W, r, h, si)) break;
    int s = slot_j[si];
    int len = nbr_len[s];
    int oi = perm[s];
    for (int e = lane; e < len; e += 32) {
      int oj = perm[slot_j[nbr[(int64_t)s * row_cap + e]]];
      int a = oi < oj ? oi : oj, b = oi < oj ? oj : oi;
      if (mode == 0) {
        long long o = off[s] + e;
        pi[o] = a;
        pj[o] = b;
      } else {
        unsigned long long hsh = mix64((uint64_t)a, (uint64_t)b);
        atomicAdd(&cnt[a], 1ull); atomicAdd(&cnt[b], 1ull);
        atomicAdd(&dig[a], hsh); atomicAdd(&dig[b], hsh);
      }
    }
  }
}

__global__ void k_export_bond_deg(int n, const int* __restrict__ iperm, const int* __restrict__ brow, int* __restrict__ deg) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int s = iperm[i];
  deg[i] = brow[s + 1] - brow[s];
}

__global__ void k_export_bonds(int n, const int* __restrict__ iperm, const int* __restrict__ perm,
                               const int* __restrict__ brow, const int* __restrict__ bcol, const int* __restrict__ bmir,
                               const double* __restrict__ bo, long long bcap, const double2* __restrict__ delta,
                               const long long* __restrict__ orow, int64_t* __restrict__ out_row, int* __restrict__ out_col,
                               int* __restrict__ out_mir, double* __restrict__ out_bo, double* __restrict__ out_delta) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  if (out_row) out_row[i] = orow[i];
  if (i == n) return;
  int s = iperm[i];
  long long o0 = orow[i];
  for (int e = brow[s]; e < brow[s + 1]; ++e) {
    long long o = o0 + (e - brow[s]);
    int j = bcol[e];
    if (out_col) out_col[o] = perm[j];
    if (out_mir) {
      int em = bmir[e];
      out_mir[o] = (int)(orow[perm[j]] + (em - brow[j]));
    }
    if (out_bo)
      for (int q = 0; q < 8; ++q) out_bo[8 * o + q] = bo[q * bcap + e];
  }
  if (out_delta) {
    out_delta[2 * (int64_t)i] = delta[s].x;
    out_delta[2 * (int64_t)i + 1] = delta[s].y;
  }
}

// ====================================================== NEXT-4 species analysis
// PAPER.md:217-221 (§3.4): bonds with BO > threshold (per type pair, default
// 0.3) join atoms into molecules labelled by their smallest global (input)
// index, renumbered 1..M in label order; species = molecules with the same
// atom count per element (type).  GPU form: a lock-free union-find over the
// bond list in input-index space (a root is only ever hooked under a smaller
// root, so every tree's root is its smallest index and the final labels do
// not depend on the order of the unions), a scan of the roots for the
// renumbering, per-root composition counters, and an open-addressing hash
// table keyed by the composition vector for the census (the host sorts the
// few distinct species).
struct SpThr {
  double t[NT_MAX * NT_MAX];
};

__device__ __forceinline__ int sp_find(int* P, int x) {
  for (;;) {   // path halving; P[x] <= x always, so every shortcut is an ancestor
    const int p = __ldcg(P + x);
    if (p == x) return x;
    const int g = __ldcg(P + p);
    if (g != p) P[x] = g;
    x = g;
  }
}

__global__ void k_sp_init(int n, int* __restrict__ parent) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) parent[i] = i;
}

// one canonical entry (original i < j) per bond: unite(i, j) if BO > thr
__global__ void k_sp_union(const int* __restrict__ brow, int n, const int* __restrict__ bown,
                           const int* __restrict__ bcol, const int* __restrict__ bkey, const int* __restrict__ perm,
                           const int* __restrict__ stype, const double* __restrict__ bo, long long bcap, int nt,
                           SpThr thr, int* parent) {
  const int B = brow[n];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < B; e += gridDim.x * blockDim.x) {
    const int so = bown[e];
    int a = perm[so], b = bkey[e];
    if (a >= b) continue;
    if (!(bo[4 * bcap + e] > thr.t[stype[so] * nt + stype[bcol[e]]])) continue;
    for (;;) {
      a = sp_find(parent, a);
      b = sp_find(parent, b);
      if (a == b) break;
      if (a > b) { const int t = a; a = b; b = t; }
      const int old = atomicCAS(parent + b, b, a);   // hook the larger root under the smaller
      if (old == b) break;
      b = old;
    }
  }
}

// after all unions: parent[i] = root (the component's smallest index);
// isroot for the renumbering scan; per-root composition counts
__global__ void k_sp_count(int n, const int* __restrict__ perm, const int* __restrict__ stype, int nt, int* parent,
                           int* __restrict__ isroot, int* __restrict__ comp) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    const int i = perm[s];
    const int r = sp_find(parent, i);
    isroot[i] = r == i;
    atomicAdd(comp + (int64_t)r * nt + stype[s], 1);
  }
}

__device__ __forceinline__ uint64_t sp_hash(const int* __restrict__ c, int nt) {
  uint64_t h = 0x9E3779B97F4A7C15ull;
  for (int t = 0; t < nt; ++t) {
    h ^= (uint64_t)(unsigned)c[t] + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
  }
  return h;
}

// mol_id[i] = 1 + rank of root(i) (exclusive scan of isroot); roots insert
// their composition into the species table (rep = a root holding that
// composition, cnt = molecules)
__global__ void k_sp_label(int n, const int* __restrict__ parent, const long long* __restrict__ rank,
                           int* __restrict__ mol_id, const int* __restrict__ comp, int nt, int2* table,
                           unsigned mask) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    // read-only walk to the root (no kernel writes parent any more; a root
    // written by one thread of k_sp_count may have been overwritten there by
    // another thread's path halving with an ancestor, so parent[i] itself
    // need not be the root)
    int r = i;
    for (int p = parent[r]; p != r; p = parent[r]) r = p;
    mol_id[i] = (int)rank[r] + 1;
    if (r != i) continue;
    const int* ci = comp + (int64_t)i * nt;
    unsigned h = (unsigned)sp_hash(ci, nt) & mask;
    for (;;) {
      const int old = atomicCAS(&table[h].x, -1, i);
      bool same = old == -1;
      if (!same) {
        const int* co = comp + (int64_t)old * nt;
        same = true;
        for (int t = 0; t < nt; ++t) same &= co[t] == ci[t];
      }
      if (same) {
        atomicAdd(&table[h].y, 1);
        break;
      }
      h = (h + 1) & mask;
    }
  }
}

__global__ void k_sp_collect(unsigned size, const int2* __restrict__ table, const int* __restrict__ comp, int nt,
                             int* __restrict__ out_comp, long long* __restrict__ out_cnt, unsigned* nsp) {
  for (unsigned h = blockIdx.x * blockDim.x + threadIdx.x; h < size; h += gridDim.x * blockDim.x) {
    const int2 v = table[h];
    if (v.x < 0) continue;
    const unsigned k = atomicAdd(nsp, 1u);
    for (int t = 0; t < nt; ++t) out_comp[(int64_t)k * nt + t] = comp[(int64_t)v.x * nt + t];
    out_cnt[k] = v.y;
  }
}

// ================================================================ NEXT-2 QEq
// PAPER.md:204-208 (§3.3 "QEq"): H_ii = eta_i, H_ij = C Tap(r) (r^3 +
// gamma_ij^-3)^(-1/3) over the half list ("only unique, non-zero elements ...
// computed", from the neighbour list, rows placed by an atom-based prefix
// sum), then "a diagonally preconditioned parallel CG solver" run on the two
// systems H s = -chi and H t = -1 concurrently ("combines the sparse matrix
// multiplication and orthogonalization computations for the two linear
// systems"): one pass over H per iteration serves both right-hand sides.
//
// GPU layout (sorted atom order): every unique H_ij is computed once, from
// the half list, and stored twice — in row i's upper segment (the half-list
// row, in its order) and in row j's lower segment — so that the SpMV is a
// pure gather (warp per row, no atomics, fixed summation order).  The lower
// segments are filled through per-row atomic cursors and then sorted by
// column, which makes every SpMV, and so the whole solve, deterministic.
// Vectors of the two systems are interleaved (double2: s-system, t-system).
constexpr int QEQ_THREADS = 256;
constexpr int QEQ_GRID = 148 * 8;     // fixed grid: the reduction shape never changes
constexpr int QEQ_SORT_CAP = 768;     // lower segment entries sorted in shared memory per warp
constexpr int QEQ_SORT_THREADS = 128;

struct QEqState {
  double rz[2][2];      // [parity][system]
  double bb[2];         // ||b||^2
  double rr[2];         // ||r||^2 after the last update
  int active[2][2];     // [parity][system]
  int iters[2];
};

__device__ __forceinline__ double qeq_H(double r, double g3, double C, double invR) {
  const double x = r * invR;
  const double x2 = x * x;
  const double tap = fma(x2 * x2, fma(x, fma(x, fma(x, 20.0, -70.0), 84.0), -35.0), 1.0);
  return C * tap * rcbrt(fma(r * r, r, g3));
}

// mode 0: lower-segment counts lcnt[j] (+1 per half entry with partner j);
// mode 1: H values into the upper (row s, position off[s] + e) and lower
// (row j, off[j] + len[j] + cursor) segments
__global__ void __launch_bounds__(NBR_THREADS) k_qeq_hbuild(Grid g, const int* __restrict__ cell_start,
    const double4* __restrict__ spos, const int* __restrict__ stype, const DevParams* __restrict__ prm,
    const uint16_t* __restrict__ nbr, const int* __restrict__ nbr_len, int row_cap, int window_cap, int mode,
    int* __restrict__ lcnt, const long long* __restrict__ off, int* __restrict__ cur, int* __restrict__ hcol,
    double* __restrict__ hval) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ WinSmem W;
  int* slot_j = reinterpret_cast<int*>(dyn);
  unsigned char* slot_k = reinterpret_cast<unsigned char*>(slot_j + window_cap);
  const int nW = build_window(W, blockIdx.x, g, cell_start);
  if (nW > window_cap) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int k = warp; k < c_win.nwu; k += nwarp)
    for (int a = lane; a < W.cnt[k]; a += 32) {
      slot_j[W.slot[k] + a] = W.start[k] + a;
      slot_k[W.slot[k] + a] = (unsigned char)k;
    }
  __syncthreads();
  const double C = prm->C, invR = prm->invR;
  const int nt = prm->nt;
  for (int r = warp;; r += nwarp) {
    int h, si;
    if (!row_of(W, r, h, si)) break;
    const int s = slot_j[si];
    const int len = nbr_len[s];
    const double4 xi = spos[s];
    const int ti = stype[s];
    for (int e = lane; e < len; e += 32) {
      const int t = nbr[(int64_t)s * row_cap + e];
      const int j = slot_j[t];
      if (mode == 0) {
        atomicAdd(lcnt + j, 1);
        continue;
      }
      const double4 xj = spos[j];
      const double4 sh = W.shift[slot_k[t]];
      const double dx = xj.x + sh.x - xi.x, dy = xj.y + sh.y - xi.y, dz = xj.z + sh.z - xi.z;
      const double rr = sqrt(fma(dz, dz, fma(dy, dy, dx * dx)));
      const double v = qeq_H(rr, prm->nb[ti * nt + stype[j]].g3, C, invR);
      const long long u = off[s] + e;
      hcol[u] = j;
      hval[u] = v;
      const long long l = off[j] + nbr_len[j] + atomicAdd(cur + j, 1);
      hcol[l] = s;
      hval[l] = v;
    }
  }
}

__global__ void k_qeq_rowlen(int n, const int* __restrict__ len, int* __restrict__ deg) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) deg[i] += len[i];
}

// sort every lower segment by column (warp per row, rank sort in shared memory)
__global__ void __launch_bounds__(QEQ_SORT_THREADS) k_qeq_sortlow(int n, const long long* __restrict__ off,
                                                            const int* __restrict__ nbr_len, int* __restrict__ hcol,
                                                            double* __restrict__ hval, Status* st) {
  __shared__ int sc[QEQ_SORT_THREADS / 32][QEQ_SORT_CAP];
  __shared__ double sv[QEQ_SORT_THREADS / 32][QEQ_SORT_CAP];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nw = gridDim.x * (QEQ_SORT_THREADS / 32);
  for (int row = blockIdx.x * (QEQ_SORT_THREADS / 32) + w; row < n; row += nw) {
    const long long a = off[row] + nbr_len[row], b = off[row + 1];
    const int m = (int)(b - a);
    if (m <= 1) continue;
    if (m > QEQ_SORT_CAP) {   // left in fill order: correct, not reproducible
      if (lane == 0) set_flag(st, ST_QEQ_UNSORTED);
      continue;
    }
    for (int k = lane; k < m; k += 32) {
      sc[w][k] = hcol[a + k];
      sv[w][k] = hval[a + k];
    }
    __syncwarp();
    for (int k = lane; k < m; k += 32) {
      const int key = sc[w][k];
      int rank = 0;
      for (int q = 0; q < m; ++q) rank += sc[w][q] < key;   // columns of a row are distinct
      hcol[a + rank] = key;
      hval[a + rank] = sv[w][k];
    }
    __syncwarp();
  }
}

// fixed-shape block sum of K doubles per thread -> part[blockIdx.x * K + k]
template <int K>
__device__ __forceinline__ void qeq_block_sum(double (&v)[K], double* __restrict__ part) {
  __shared__ double red[K][QEQ_THREADS / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    if (lane == 0) red[k][w] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double t = 0.0;
    for (int q = 0; q < QEQ_THREADS / 32; ++q) t += red[threadIdx.x][q];
    part[blockIdx.x * K + threadIdx.x] = t;
  }
}

// every block reduces the QEQ_GRID partials of K values in the same fixed
// order (so all blocks see identical scalars): out[k] = sum_b part[b*K + k]
template <int K>
__device__ __forceinline__ void qeq_total(const double* __restrict__ part, double (&out)[K]) {
  __shared__ double red[K][QEQ_THREADS / 32];
  __shared__ double tot[K];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double v = 0.0;
    for (int b = threadIdx.x; b < QEQ_GRID; b += QEQ_THREADS) v += part[b * K + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[k][w] = v;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double t = 0.0;
    for (int q = 0; q < QEQ_THREADS / 32; ++q) t += red[threadIdx.x][q];
    tot[threadIdx.x] = t;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = tot[k];
  __syncthreads();
}

struct QEqType {
  double eta[NT_MAX], chi[NT_MAX];
};

// y = H x for both systems (warp per row, fixed order); with part, also the
// partial dots x . y of both systems
__global__ void __launch_bounds__(QEQ_THREADS) k_qeq_spmv(int n, const long long* __restrict__ off,
    const int* __restrict__ hcol, const double* __restrict__ hval, const int* __restrict__ stype, QEqType ty,
    const double2* __restrict__ x, double2* __restrict__ y, double* __restrict__ part,
    const QEqState* __restrict__ stt = nullptr, int par = 0) {
  if (stt && !stt->active[par][0] && !stt->active[par][1]) return;   // both systems converged
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nw = gridDim.x * (QEQ_THREADS / 32);
  double d[2] = {0.0, 0.0};
  for (int row = blockIdx.x * (QEQ_THREADS / 32) + w; row < n; row += nw) {
    const long long a = off[row], b = off[row + 1];
    double a0 = 0.0, a1 = 0.0;
    // four entries per lane in flight (the same per-lane order as a plain
    // stride-32 loop): the column loads, then the dependent gathers
    for (long long e = a + lane; e < b; e += 128) {
      double v[4];
      int c[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const long long q = e + 32 * u;
        v[u] = q < b ? __ldcs(hval + q) : 0.0;
        c[u] = q < b ? __ldcs(hcol + q) : row;
      }
      double2 xc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) xc[u] = x[c[u]];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a0 = fma(v[u], xc[u].x, a0);
        a1 = fma(v[u], xc[u].y, a1);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    }
    if (lane == 0) {
      const double2 xr = x[row];
      const double et = ty.eta[stype[row]];
      const double2 yr = make_double2(fma(et, xr.x, a0), fma(et, xr.y, a1));
      y[row] = yr;
      d[0] = fma(xr.x, yr.x, d[0]);
      d[1] = fma(xr.y, yr.y, d[1]);
    }
  }
  if (part) qeq_block_sum<2>(d, part);
}

// start: x from the guesses (input order -> sorted), done by k_qeq_gather;
// r = b - Ax, z = r / eta, p = z; partials {r.z (2), r.r (2), b.b (2)}
__global__ void __launch_bounds__(QEQ_THREADS) k_qeq_gather(int n, const int* __restrict__ perm,
    const double* __restrict__ s0, const double* __restrict__ t0, double2* __restrict__ x) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int o = perm[i];
    x[i] = make_double2(s0[o], t0[o]);
  }
}

__global__ void __launch_bounds__(QEQ_THREADS) k_qeq_start(int n, const int* __restrict__ stype, QEqType ty,
    const double2* __restrict__ Ax, double2* __restrict__ r, double2* __restrict__ z, double2* __restrict__ p,
    double* __restrict__ part) {
  double v[6] = {0, 0, 0, 0, 0, 0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int t = stype[i];
    const double b0 = -ty.chi[t], b1 = -1.0, ie = 1.0 / ty.eta[t];
    const double2 ax = Ax[i];
    const double2 rr = make_double2(b0 - ax.x, b1 - ax.y);
    const double2 zz = make_double2(rr.x * ie, rr.y * ie);
    r[i] = rr;
    z[i] = zz;
    p[i] = zz;
    v[0] = fma(rr.x, zz.x, v[0]);
    v[1] = fma(rr.y, zz.y, v[1]);
    v[2] = fma(rr.x, rr.x, v[2]);
    v[3] = fma(rr.y, rr.y, v[3]);
    v[4] = fma(b0, b0, v[4]);
    v[5] = fma(b1, b1, v[5]);
  }
  qeq_block_sum<6>(v, part);
}

// one block: the start scalars
__global__ void __launch_bounds__(QEQ_THREADS) k_qeq_start_state(const double* __restrict__ part, double tol,
                                                                 int maxiter, QEqState* stt) {
  double t[6];
  qeq_total<6>(part, t);
  if (threadIdx.x == 0) {
    for (int c = 0; c < 2; ++c) {
      stt->rz[0][c] = t[c];
      stt->rr[c] = t[2 + c];
      stt->bb[c] = t[4 + c];
      stt->active[0][c] = maxiter > 0 && t[2 + c] > tol * tol * t[4 + c];
      stt->iters[c] = 0;
    }
  }
}

// alpha = r.z / p.Ap (from the spmv partials) for the active systems;
// x += alpha p, r -= alpha Ap, z = r / eta; partials {r.z (2), r.r (2)}
__global__ void __launch_bounds__(QEQ_THREADS) k_qeq_update(int n, const int* __restrict__ stype, QEqType ty,
    const double* __restrict__ part_pap, const QEqState* __restrict__ stt, int par, double2* __restrict__ x,
    double2* __restrict__ r, double2* __restrict__ z, const double2* __restrict__ p, const double2* __restrict__ Ap,
    double* __restrict__ part) {
  if (!stt->active[par][0] && !stt->active[par][1]) return;   // both systems converged
  double pap[2];
  qeq_total<2>(part_pap, pap);
  const double al0 = stt->active[par][0] ? stt->rz[par][0] / pap[0] : 0.0;
  const double al1 = stt->active[par][1] ? stt->rz[par][1] / pap[1] : 0.0;
  double v[4] = {0, 0, 0, 0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double ie = 1.0 / ty.eta[stype[i]];
    const double2 pi = p[i], api = Ap[i];
    double2 xi = x[i], ri = r[i];
    xi.x = fma(al0, pi.x, xi.x);
    xi.y = fma(al1, pi.y, xi.y);
    ri.x = fma(-al0, api.x, ri.x);
    ri.y = fma(-al1, api.y, ri.y);
    const double2 zi = make_double2(ri.x * ie, ri.y * ie);
    x[i] = xi;
    r[i] = ri;
    z[i] = zi;
    v[0] = fma(ri.x, zi.x, v[0]);
    v[1] = fma(ri.y, zi.y, v[1]);
    v[2] = fma(ri.x, ri.x, v[2]);
    v[3] = fma(ri.y, ri.y, v[3]);
  }
  qeq_block_sum<4>(v, part);
}

// beta = r.z (new) / r.z (old); p = z + beta p; block 0 advances the state
// (iteration counts, convergence ||r|| <= tol ||b||, the next r.z)
__global__ void __launch_bounds__(QEQ_THREADS) k_qeq_direction(int n, const double* __restrict__ part_rz,
    QEqState* stt, int par, double tol, int maxiter, const double2* __restrict__ z, double2* __restrict__ p) {
  const int a0 = stt->active[par][0], a1 = stt->active[par][1];
  if (!a0 && !a1) {   // both converged: only carry the flags to the next parity
    __syncthreads();  // every block has read the flags before block 0 writes the other parity
    if (blockIdx.x == 0 && threadIdx.x == 0) stt->active[par ^ 1][0] = stt->active[par ^ 1][1] = 0;
    return;
  }
  double t[4];
  qeq_total<4>(part_rz, t);
  const double be0 = a0 ? t[0] / stt->rz[par][0] : 0.0;
  const double be1 = a1 ? t[1] / stt->rz[par][1] : 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double2 zi = z[i];
    double2 pi = p[i];
    pi.x = fma(be0, pi.x, zi.x);
    pi.y = fma(be1, pi.y, zi.y);
    p[i] = pi;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int act[2] = {a0, a1};
    for (int c = 0; c < 2; ++c) {   // (parity par^1 is read only by the next iteration's kernels)
      stt->active[par ^ 1][c] = 0;
      if (!act[c]) continue;
      stt->rz[par ^ 1][c] = t[c];
      stt->rr[c] = t[2 + c];
      stt->iters[c] += 1;
      stt->active[par ^ 1][c] = stt->iters[c] < maxiter && t[2 + c] > tol * tol * stt->bb[c];
    }
  }
}

// s, t back to input order; partials {sum s, sum t}
__global__ void __launch_bounds__(QEQ_THREADS) k_qeq_scatter(int n, const int* __restrict__ perm,
    const double2* __restrict__ x, double* __restrict__ s, double* __restrict__ t, double* __restrict__ part) {
  double v[2] = {0.0, 0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double2 xi = x[i];
    const int o = perm[i];
    s[o] = xi.x;
    t[o] = xi.y;
    v[0] += xi.x;
    v[1] += xi.y;
  }
  qeq_block_sum<2>(v, part);
}

// q = s - (sum s / sum t) t (input order)
__global__ void __launch_bounds__(QEQ_THREADS) k_qeq_charges(int n, const double* __restrict__ part,
    const double* __restrict__ s, const double* __restrict__ t, double* __restrict__ q) {
  double tot[2];
  qeq_total<2>(part, tot);
  const double mu = tot[0] / tot[1];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) q[i] = fma(-mu, t[i], s[i]);
}

}  // namespace rx
