/* ============================================================================
 * CPU ORACLE for the ReaxFF list / bond-order / nonbonded hot path
 * (arXiv:1706.07772, ReaxC-OMP).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_1706_07772_b200/) never links, imports or executes it, and the two
 * share no code, headers, tables or constants.
 *
 * Plain, slow, obviously correct: scalar IEEE fp64, compiled with
 * -O2 -ffp-contract=off (no FMA contraction, no fast-math), glibc libm,
 * every loop in the order the definition states.  Row-parallel with POSIX
 * threads (SURVEY.md §8(c) "std::thread over atom rows"):
 * every atom row is computed on its own, in a fixed order, and writes only
 * its own outputs; per-row Neumaier partials are combined in row order after
 * the parallel pass.  Results are therefore bitwise independent of the
 * thread count T (tests/test_oracle_threads.py pins 1 vs T).
 *
 * What it computes (the reading adopted in DESIGN.md):
 *   O1 minimum image, half-open [-L/2, L/2)
 *   O2 half neighbour list r^2 <= r_nonb^2            PAPER.md:152 (§3.3)
 *   O3 uncorrected bond orders B1-B2, full bond list  PAPER.md:154-158 (§3.3); north_star
 *   O4 Delta' per atom (B3)                           PAPER.md:37 (§2.1 over/under-coordination)
 *   O5 corrected bond orders f1..f5 (B4-B8)           PAPER.md:160 (§3.3); north_star
 *   O6 tapered shielded vdW + Coulomb (N1-N6),
 *      Alg. 1/Alg. 2 pair loop with F_i += f, F_k -= f PAPER.md:87-110 (Alg. 1), 162-196 (Alg. 2)
 *   O8 (NEXT-1) bond energy E1 and its forces through the bond-order
 *      derivatives (the bond part of "Aggregate Forces")  PAPER.md:160, 285 (§3.3, Table 2)
 *   O9 (NEXT-3) valence-angle (3-body) and hydrogen-bond interaction lists
 *                                                       PAPER.md:154-158, 198-202 (§3.3)
 *
 * PARITY NOTE.  PAPER.md states no ReaxFF equations (it cites refs [6,7],
 * PAPER.md:37); the functional forms B1-B8 / N1-N6 are the standard published
 * ReaxFF forms as restated in SURVEY.md §8(c).  Every function below is pinned
 * by tests (brute force, closed forms, special cases, finite differences,
 * invariants), but whether these forms are what "the paper" computes is
 * parity unpinned (no in-paper worked example exists).  DESIGN.md lists every
 * reading taken.
 * ==========================================================================*/
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* ---------------------------------------------------------------- a1 / O1 */

/* a1: x <- x - L*floor(x/L); a result equal to L is mapped to 0. */
void orc_wrap(int64_t n, const double* pos, const double box[3], double* out) {
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      double x = pos[3 * i + k], L = box[k];
      double w = x - L * floor(x / L);
      if (w >= L || w < 0.0) w = 0.0;
      out[3 * i + k] = w;
    }
}

/* O1: per axis d = x_j - x_i wrapped into [-L/2, L/2). */
double orc_min_image(double d, double L) {
  if (d >= 0.5 * L) d -= L;
  else if (d < -0.5 * L) d += L;
  return d;
}

/* r^2 = (dx*dx + dy*dy) + dz*dz, products separately rounded (no FMA). */
static double orc_dist2(const double* pos, int64_t i, int64_t j, const double box[3], double d[3]) {
  for (int k = 0; k < 3; ++k) d[k] = orc_min_image(pos[3 * j + k] - pos[3 * i + k], box[k]);
  return (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2];
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* ------------------------------------------------------ row-parallel driver */

/* Rows [0, n) are dealt to T threads in chunks of ORC_CHUNK through an atomic
 * counter.  fn(i, ctx, scratch) writes only row i's outputs, so the result is
 * the same for every T and every dealing. */
#define ORC_CHUNK 64
typedef void (*orc_row_fn)(int64_t i, void* ctx, void* scratch);
typedef struct {
  int64_t n, next;
  orc_row_fn fn;
  void* ctx;
  size_t scratch;
} orc_job;

static void* orc_worker(void* arg) {
  orc_job* J = (orc_job*)arg;
  void* scr = J->scratch ? malloc(J->scratch) : NULL;
  for (;;) {
    int64_t a = __atomic_fetch_add(&J->next, (int64_t)ORC_CHUNK, __ATOMIC_RELAXED);
    if (a >= J->n) break;
    int64_t b = a + ORC_CHUNK < J->n ? a + ORC_CHUNK : J->n;
    for (int64_t i = a; i < b; ++i) J->fn(i, J->ctx, scr);
  }
  free(scr);
  return NULL;
}

static void orc_par_rows(int64_t n, int T, orc_row_fn fn, void* ctx, size_t scratch) {
  orc_job J = {n, 0, fn, ctx, scratch};
  pthread_t th[256];
  int started = 0;
  if (T > 256) T = 256;
  for (int t = 1; t < T && n > ORC_CHUNK; ++t)
    if (pthread_create(&th[started], NULL, orc_worker, &J) == 0) ++started;
  orc_worker(&J);
  for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
}

/* Cell grid for O2: cells of side L/floor(L/(Rc(1+1e-9))) per axis, strictly
 * wider than Rc, so rounding in floor(x/side) never puts two atoms within Rc
 * more than one cell apart; the atoms of each cell in ascending index
 * (counting sort).  maxcand bounds the candidates of any row. */
typedef struct {
  int nc[3];
  int64_t ncell, maxcand;
  int64_t* start; /* ncell + 1 */
  int64_t* atom;  /* n, cell-major */
  int32_t* cell;  /* 3n */
} orc_grid;

/* the deduplicated neighbour cells of cell cc (c0 has 2 cells per axis, so
 * -1 and +1 name the same cell) */
static int orc_grid_nbcells(const orc_grid* G, const int32_t* cc, int64_t nb[27]) {
  int nnb = 0;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int cx = ((cc[0] + dx) % G->nc[0] + G->nc[0]) % G->nc[0];
        int cy = ((cc[1] + dy) % G->nc[1] + G->nc[1]) % G->nc[1];
        int cz = ((cc[2] + dz) % G->nc[2] + G->nc[2]) % G->nc[2];
        int64_t c = ((int64_t)cz * G->nc[1] + cy) * G->nc[0] + cx;
        int dup = 0;
        for (int m = 0; m < nnb; ++m) dup |= (nb[m] == c);
        if (!dup) nb[nnb++] = c;
      }
  return nnb;
}

static void orc_grid_build(orc_grid* G, int64_t n, const double* pos, const double box[3], double Rc) {
  for (int k = 0; k < 3; ++k) {
    G->nc[k] = (int)floor(box[k] / (Rc * (1.0 + 1e-9)));
    if (G->nc[k] < 1) G->nc[k] = 1;
  }
  G->ncell = (int64_t)G->nc[0] * G->nc[1] * G->nc[2];
  G->start = (int64_t*)calloc((size_t)G->ncell + 1, sizeof(int64_t));
  G->atom = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  G->cell = (int32_t*)malloc(sizeof(int32_t) * 3 * (size_t)(n > 0 ? n : 1));
  int64_t* cid = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = 0;
    for (int k = 2; k >= 0; --k) {
      int ck = (int)floor(pos[3 * i + k] / (box[k] / G->nc[k]));
      if (ck >= G->nc[k]) ck = G->nc[k] - 1;
      if (ck < 0) ck = 0;
      G->cell[3 * i + k] = ck;
      c = c * G->nc[k] + ck;
    }
    cid[i] = c;
    G->start[c + 1]++;
  }
  for (int64_t c = 0; c < G->ncell; ++c) G->start[c + 1] += G->start[c];
  int64_t* fill = (int64_t*)calloc((size_t)G->ncell, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) G->atom[G->start[cid[i]] + fill[cid[i]]++] = i;
  G->maxcand = 1;
  for (int64_t c = 0; c < G->ncell; ++c) {
    int32_t cc[3] = {(int32_t)(c % G->nc[0]), (int32_t)((c / G->nc[0]) % G->nc[1]),
                     (int32_t)(c / ((int64_t)G->nc[0] * G->nc[1]))};
    int64_t nb[27], s = 0;
    int nnb = orc_grid_nbcells(G, cc, nb);
    for (int m = 0; m < nnb; ++m) s += G->start[nb[m] + 1] - G->start[nb[m]];
    if (s > G->maxcand) G->maxcand = s;
  }
  free(cid);
  free(fill);
}

static void orc_grid_free(orc_grid* G) {
  free(G->start);
  free(G->atom);
  free(G->cell);
}

/* Row i of the list at radius^2 R2 from the grid: every j != i (with half,
 * only j > i) in the neighbour cells with min-image r^2 <= R2, ascending. */
static int64_t orc_grid_row(const orc_grid* G, int64_t i, const double* pos, const double box[3], double R2,
                            int half, int32_t* out) {
  int64_t nb[27], len = 0;
  double d[3];
  int nnb = orc_grid_nbcells(G, &G->cell[3 * i], nb);
  for (int m = 0; m < nnb; ++m)
    for (int64_t a = G->start[nb[m]]; a < G->start[nb[m] + 1]; ++a) {
      int64_t j = G->atom[a];
      if (j == i || (half && j < i)) continue;
      if (orc_dist2(pos, i, j, box, d) <= R2) out[len++] = (int32_t)j;
    }
  qsort(out, (size_t)len, sizeof(int32_t), cmp_i32);
  return len;
}

/* ---------------------------------------------------------------- O2 list */

/* Brute force: every unordered pair i<j with min-image r^2 <= R^2, emitted as
 * canonical CSR (rows i ascending, j > i ascending).  This is the plain
 * definition ("exactly the pairs with minimum-image distance <=
 * r_nonb, each once with i<j").  Returns the pair count; writes at most cap. */
int64_t orc_half_list_brute(int64_t n, const double* pos, const double box[3], double R,
                            int64_t* rowoff, int32_t* col, int64_t cap) {
  double R2 = R * R, d[3];
  int64_t p = 0;
  for (int64_t i = 0; i < n; ++i) {
    rowoff[i] = p;
    for (int64_t j = i + 1; j < n; ++j)
      if (orc_dist2(pos, i, j, box, d) <= R2) {
        if (p < cap) col[p] = (int32_t)j;
        ++p;
      }
  }
  rowoff[n] = p;
  return p;
}

/* Cell-list version of the same set (O2), row-parallel: a counting pass
 * gives every row's length, a serial prefix sum the offsets, a fill pass the
 * rows (each j > i with r^2 <= R^2 in the deduplicated neighbour cells of the
 * grid above, ascending).  SPEC.md:155: "each thread writing disjoint row
 * ranges after a counting pass".  rowoff is written always, col only if the
 * total fits cap.  Returns the pair count. */
typedef struct {
  const orc_grid* G;
  const double* pos;
  const double* box;
  double R2;
  int64_t* len;
  const int64_t* rowoff;
  int32_t* col;
} orc_hl_ctx;

static void orc_hl_count(int64_t i, void* c, void* scr) {
  orc_hl_ctx* H = (orc_hl_ctx*)c;
  H->len[i] = orc_grid_row(H->G, i, H->pos, H->box, H->R2, 1, (int32_t*)scr);
}

static void orc_hl_fill(int64_t i, void* c, void* scr) {
  orc_hl_ctx* H = (orc_hl_ctx*)c;
  int64_t m = orc_grid_row(H->G, i, H->pos, H->box, H->R2, 1, (int32_t*)scr);
  memcpy(H->col + H->rowoff[i], scr, sizeof(int32_t) * (size_t)m);
}

int64_t orc_half_list_cells(int64_t n, const double* pos, const double box[3], double R,
                            int64_t* rowoff, int32_t* col, int64_t cap, int T) {
  orc_grid G;
  orc_grid_build(&G, n, pos, box, R);
  int64_t* len = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  orc_hl_ctx H = {&G, pos, box, R * R, len, rowoff, col};
  size_t scr = sizeof(int32_t) * (size_t)G.maxcand;
  orc_par_rows(n, T, orc_hl_count, &H, scr);
  int64_t p = 0;
  for (int64_t i = 0; i < n; ++i) {
    rowoff[i] = p;
    p += len[i];
  }
  rowoff[n] = p;
  if (p <= cap) orc_par_rows(n, T, orc_hl_fill, &H, scr);
  free(len);
  orc_grid_free(&G);
  return p;
}

/* Per-atom digest straight from the grid (c3/c4, no stored list): for each
 * atom, the number of pairs it belongs to (its full neighbour count) and the
 * sum of mix64(min, max) over them mod 2^64. */
static uint64_t orc_mix64(uint64_t a, uint64_t b);
typedef struct {
  const orc_grid* G;
  const double* pos;
  const double* box;
  double R2;
  int64_t* cnt;
  uint64_t* dig;
} orc_dg_ctx;

static void orc_dg_row(int64_t i, void* c, void* scr) {
  orc_dg_ctx* D = (orc_dg_ctx*)c;
  int32_t* row = (int32_t*)scr;
  int64_t m = orc_grid_row(D->G, i, D->pos, D->box, D->R2, 0, row);
  uint64_t h = 0;
  for (int64_t a = 0; a < m; ++a) {
    uint64_t j = (uint64_t)row[a], ii = (uint64_t)i;
    h += orc_mix64(ii < j ? ii : j, ii < j ? j : ii);
  }
  D->cnt[i] = m;
  D->dig[i] = h;
}

void orc_digest_cells(int64_t n, const double* pos, const double box[3], double R, int64_t* cnt, uint64_t* dig,
                      int T) {
  orc_grid G;
  orc_grid_build(&G, n, pos, box, R);
  orc_dg_ctx D = {&G, pos, box, R * R, cnt, dig};
  orc_par_rows(n, T, orc_dg_row, &D, sizeof(int32_t) * (size_t)G.maxcand);
  orc_grid_free(&G);
}

/* Per-atom digest for large configs: for each atom, the
 * number of pairs it belongs to and sum of mix64(min,max) mod 2^64. */
static uint64_t orc_mix64(uint64_t a, uint64_t b) {
  uint64_t z = (a << 32) ^ b;
  z ^= z >> 33; z *= 0xff51afd7ed558ccdull;
  z ^= z >> 33; z *= 0xc4ceb9fe1a85ec53ull;
  z ^= z >> 33;
  return z;
}
void orc_digest(int64_t n, const int64_t* rowoff, const int32_t* col, int64_t* cnt, uint64_t* dig) {
  for (int64_t i = 0; i < n; ++i) { cnt[i] = 0; dig[i] = 0; }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = rowoff[i]; p < rowoff[i + 1]; ++p) {
      int64_t j = col[p];
      uint64_t h = orc_mix64((uint64_t)(i < j ? i : j), (uint64_t)(i < j ? j : i));
      cnt[i] += 1; cnt[j] += 1; dig[i] += h; dig[j] += h;
    }
}
uint64_t orc_mix64_pub(uint64_t a, uint64_t b) { return orc_mix64(a, b); }

/* ------------------------------------------------------------ O3 bond orders */

/* B1-B2 for one pair at distance r (north_star: "uncorrected bond orders
 * BO'sigma/pi/pipi", combining rule
 * r0_ij = (r_i + r_j)/2, reading 9).  out = {BO'sigma, BO'pi, BO'pipi, BO'}. */
void orc_bo_raw(double r, int ti, int tj, const orc_params* P, double out[4]) {
  int nt = P->ntypes, tp = ti * nt + tj;
  double r0s = 0.5 * (P->r_sigma[ti] + P->r_sigma[tj]);
  double r0p = 0.5 * (P->r_pi[ti] + P->r_pi[tj]);
  double r0pp = 0.5 * (P->r_pipi[ti] + P->r_pipi[tj]);
  double bs = exp(P->p_bo1[tp] * pow(r / r0s, P->p_bo2[tp]));
  double bp = exp(P->p_bo3[tp] * pow(r / r0p, P->p_bo4[tp]));
  double bpp = exp(P->p_bo5[tp] * pow(r / r0pp, P->p_bo6[tp]));
  out[0] = bs;
  out[1] = bp;
  out[2] = bpp;
  out[3] = (bs + bp) + bpp; /* B2, summed in this order */
}

/* O3: for every canonical pair (i < j) with r <= r_bond (r^2 <= r_bond^2),
 * BO' from B1-B2; a bond iff BO' >= bo_cut (reading 2A).  Emits the FULL
 * list (both i->j and j->i, "requires the bond list to be a
 * full list with both i-j and j-i bonds available") as CSR with rows sorted by
 * j, plus the mirror index.  bo: [B][4].  Returns B (entries);
 * writes nothing past cap.
 * The canonical candidates of row i are its half-list row (hrow/hcol) or,
 * with hrow == NULL, the j > i of the cell grid at r_bond (large systems, no
 * stored half list).  Two row-parallel passes evaluate B1-B2 (count, then
 * fill per-row kept lists); the full list is then assembled serially in
 * canonical (i asc, j asc) order: row i receives partners j < i (from
 * earlier rows, ascending i) before its own partners j > i (ascending), so
 * every row ends sorted by j. */
typedef struct {
  const double* pos;
  const int32_t* type;
  const double* box;
  const orc_params* P;
  double rb2, bo_cut;
  const int64_t* hrow;
  const int32_t* hcol;
  const orc_grid* G;
  int64_t* kcnt;      /* kept canonical bonds of row i */
  const int64_t* koff;
  int32_t* kj;
  double* kv;         /* [K][4] */
} orc_bd_ctx;

static void orc_bd_row(int64_t i, orc_bd_ctx* C, int32_t* cand, int fill) {
  double d[3], v[4];
  int64_t m, k = 0;
  const int32_t* row;
  if (C->hrow) {
    row = C->hcol + C->hrow[i];
    m = C->hrow[i + 1] - C->hrow[i];
  } else {
    m = orc_grid_row(C->G, i, C->pos, C->box, C->rb2, 1, cand);
    row = cand;
  }
  for (int64_t a = 0; a < m; ++a) {
    int64_t j = row[a];
    double r2 = orc_dist2(C->pos, i, j, C->box, d);
    if (r2 > C->rb2) continue;
    orc_bo_raw(sqrt(r2), C->type[i], C->type[j], C->P, v);
    if (v[3] < C->bo_cut) continue;
    if (fill) {
      int64_t e = C->koff[i] + k;
      C->kj[e] = (int32_t)j;
      for (int t = 0; t < 4; ++t) C->kv[4 * e + t] = v[t];
    }
    ++k;
  }
  if (!fill) C->kcnt[i] = k;
}
static void orc_bd_count(int64_t i, void* c, void* scr) { orc_bd_row(i, (orc_bd_ctx*)c, (int32_t*)scr, 0); }
static void orc_bd_fill(int64_t i, void* c, void* scr) { orc_bd_row(i, (orc_bd_ctx*)c, (int32_t*)scr, 1); }

int64_t orc_bonds(int64_t n, const double* pos, const int32_t* type, const double box[3],
                  const orc_params* P, double r_bond, double bo_cut, const int64_t* hrow,
                  const int32_t* hcol, int64_t* brow, int32_t* bcol, int32_t* bmirror,
                  double* bo, int64_t cap, int T) {
  size_t n1 = (size_t)(n > 0 ? n : 1);
  orc_grid G = {{0, 0, 0}, 0, 1, NULL, NULL, NULL};
  if (!hrow) orc_grid_build(&G, n, pos, box, r_bond);
  int64_t* kcnt = (int64_t*)calloc(n1, sizeof(int64_t));
  int64_t* koff = (int64_t*)calloc(n1 + 1, sizeof(int64_t));
  orc_bd_ctx C = {pos, type, box, P, r_bond * r_bond, bo_cut, hrow, hcol, &G, kcnt, koff, NULL, NULL};
  size_t scr = hrow ? 0 : sizeof(int32_t) * (size_t)G.maxcand;
  orc_par_rows(n, T, orc_bd_count, &C, scr);
  for (int64_t i = 0; i < n; ++i) koff[i + 1] = koff[i] + kcnt[i];
  int64_t K = koff[n];
  /* full degrees: own canonical bonds + appearances as the partner */
  int64_t* deg = (int64_t*)calloc(n1, sizeof(int64_t));
  C.kj = (int32_t*)malloc(sizeof(int32_t) * (size_t)(K > 0 ? K : 1));
  C.kv = (double*)malloc(sizeof(double) * 4 * (size_t)(K > 0 ? K : 1));
  orc_par_rows(n, T, orc_bd_fill, &C, scr);
  for (int64_t i = 0; i < n; ++i) {
    deg[i] += kcnt[i];
    for (int64_t e = koff[i]; e < koff[i + 1]; ++e) deg[C.kj[e]]++;
  }
  brow[0] = 0;
  for (int64_t i = 0; i < n; ++i) brow[i + 1] = brow[i] + deg[i];
  int64_t B = brow[n];
  if (B <= cap) {
    int64_t* fill = (int64_t*)calloc(n1, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i)
      for (int64_t k = koff[i]; k < koff[i + 1]; ++k) {
        int64_t j = C.kj[k];
        int64_t ei = brow[i] + fill[i]++, ej = brow[j] + fill[j]++;
        bcol[ei] = (int32_t)j; bcol[ej] = (int32_t)i;
        bmirror[ei] = (int32_t)ej; /* mirror = absolute entry index of j->i */
        bmirror[ej] = (int32_t)ei;
        for (int t = 0; t < 4; ++t) { bo[4 * ei + t] = C.kv[4 * k + t]; bo[4 * ej + t] = C.kv[4 * k + t]; }
      }
    free(fill);
  }
  free(deg); free(kcnt); free(koff); free(C.kj); free(C.kv);
  if (!hrow) orc_grid_free(&G);
  return B;
}

/* O4 / B3: Delta'_i = sum_j BO'_ij - Val_i and Delta'boc_i = sum_j BO'_ij - Val^boc_i,
 * the sum over the kept bonds of row i in ascending j (readings 4, 6). */
void orc_delta(int64_t n, const int32_t* type, const orc_params* P, const int64_t* brow,
               const double* bo, double* delta) {
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t e = brow[i]; e < brow[i + 1]; ++e) s += bo[4 * e + 3];
    delta[2 * i] = s - P->val[type[i]];
    delta[2 * i + 1] = s - P->val_boc[type[i]];
  }
}

/* B4-B8 for one bond (i,j) given its BO' terms and the two atoms' Delta'.
 * out = {BO, BOsigma, BOpi, BOpipi}; f (optional) = {f1, f2, f3, f4, f5}. */
void orc_bo_corr_pair(const double raw[4], double di, double dboci, double dj, double dbocj,
                      int ti, int tj, const orc_params* P, double out[4], double* f) {
  int tp = ti * P->ntypes + tj;
  double p1 = P->p_boc1, p2 = P->p_boc2;
  double vi = P->val[ti], vj = P->val[tj];
  double pboc3 = sqrt(P->b132[ti] * P->b132[tj]);
  double pboc4 = sqrt(P->b131[ti] * P->b131[tj]);
  double pboc5 = sqrt(P->b133[ti] * P->b133[tj]);
  (void)tp;
  double bo = raw[3];
  double f2 = exp(-p1 * di) + exp(-p1 * dj);                                    /* B4 */
  double f3 = -(1.0 / p2) * log(0.5 * (exp(-p2 * di) + exp(-p2 * dj)));         /* B5 */
  double f1 = 0.5 * ((vi + f2) / (vi + f2 + f3) + (vj + f2) / (vj + f2 + f3));  /* B6 */
  double f4 = 1.0 / (1.0 + exp(-pboc3 * (pboc4 * bo * bo - dboci) + pboc5));    /* B7 */
  double f5 = 1.0 / (1.0 + exp(-pboc3 * (pboc4 * bo * bo - dbocj) + pboc5));
  double BO = bo * f1 * f4 * f5;                                                /* B8 */
  double BOpi = raw[1] * f1 * f1 * f4 * f5;
  double BOpipi = raw[2] * f1 * f1 * f4 * f5;
  out[0] = BO;
  out[1] = BO - BOpi - BOpipi; /* reading 5 */
  out[2] = BOpi;
  out[3] = BOpipi;
  if (f) { f[0] = f1; f[1] = f2; f[2] = f3; f[3] = f4; f[4] = f5; }
}

/* O5: B4-B8 once per unordered bond in canonical orientation (i < j, so f4
 * uses Delta'boc_i and f5 uses Delta'boc_j) and mirrored to both entries, so
 * BO_ij == BO_ji bitwise.  corr: [B][4]. */
void orc_bo_correct(int64_t n, const int32_t* type, const orc_params* P, const int64_t* brow,
                    const int32_t* bcol, const int32_t* bmirror, const double* bo,
                    const double* delta, double* corr) {
  double out[4];
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = brow[i]; e < brow[i + 1]; ++e) {
      int64_t j = bcol[e];
      if (j < i) continue;
      orc_bo_corr_pair(&bo[4 * e], delta[2 * i], delta[2 * i + 1], delta[2 * j], delta[2 * j + 1],
                       type[i], type[j], P, out, NULL);
      int64_t em = bmirror[e];
      for (int k = 0; k < 4; ++k) { corr[4 * e + k] = out[k]; corr[4 * em + k] = out[k]; }
    }
}

/* -------------------------------------------------------------- O6 nonbonded */

/* N1: 7th-order taper in x = r/R (inner radius 0, reading 14), and dTap/dr. */
void orc_taper(double r, double R, double* tap, double* dtap) {
  double x = r / R;
  double x2 = x * x, x3 = x2 * x, x4 = x3 * x, x5 = x4 * x, x6 = x5 * x, x7 = x6 * x;
  *tap = 1.0 - 35.0 * x4 + 84.0 * x5 - 70.0 * x6 + 20.0 * x7;
  *dtap = -140.0 * x3 * (1.0 - x) * (1.0 - x) * (1.0 - x) / R;
}

/* N2-N4: shielded vdW (untapered) e_v and de_v/dr for one pair.
 * Combining rules (reading 9): D = sqrt(eps_i eps_j), alpha = sqrt(alpha_i alpha_j),
 * r_vdW = 2 sqrt(r_vdw_i r_vdw_j), gamma_w = sqrt(gamma_w_i gamma_w_j). */
void orc_vdw(double r, int ti, int tj, const orc_params* P, double* ev, double* dev) {
  double D = sqrt(P->eps[ti] * P->eps[tj]);
  double alpha = sqrt(P->alpha[ti] * P->alpha[tj]);
  double rvdw = 2.0 * sqrt(P->r_vdw[ti] * P->r_vdw[tj]);
  double gw = sqrt(P->gamma_w[ti] * P->gamma_w[tj]);
  double p = P->p_vdw1;
  double sv = pow(r, p) + pow(gw, -p);
  double f13 = pow(sv, 1.0 / p);                                   /* N2 */
  double u = 1.0 - f13 / rvdw;
  double e1 = exp(alpha * u), e2 = exp(0.5 * alpha * u);
  *ev = D * (e1 - 2.0 * e2);                                       /* N3 */
  double df13 = pow(sv, 1.0 / p - 1.0) * pow(r, p - 1.0);          /* d f13 / dr */
  *dev = -D * (alpha / rvdw) * (e1 - e2) * df13;                   /* N4 (untapered part) */
}

/* N5 (untapered): shielded Coulomb kernel k(r) = S^(-1/3), S = r^3 + gamma_ij^-3,
 * gamma_ij = sqrt(gamma_i gamma_j); returns k and dk/dr. */
void orc_coulomb_kernel(double r, int ti, int tj, const orc_params* P, double* k, double* dk) {
  double g = sqrt(P->gamma[ti] * P->gamma[tj]);
  double S = r * r * r + pow(g, -3.0);
  *k = pow(S, -1.0 / 3.0);
  *dk = -r * r * pow(S, -4.0 / 3.0);
}

/* One Alg. 2 pair ("evdW, fvdW <- vdWaals(atom[i], atom[k]);
 * eClmb, fClmb <- Coulomb(atom[i], atom[k])"): tapered energies and the total
 * dE/dr.  e[0] = Tap*e_v, e[1] = C q_i q_j Tap S^(-1/3). */
void orc_pair(double r, int ti, int tj, double qi, double qj, const orc_params* P, double R,
              double e[2], double* dEdr) {
  double tap, dtap, ev, dev, k, dk;
  orc_taper(r, R, &tap, &dtap);
  orc_vdw(r, ti, tj, P, &ev, &dev);
  orc_coulomb_kernel(r, ti, tj, P, &k, &dk);
  double cqq = P->coulomb_c * qi * qj;
  e[0] = tap * ev;
  e[1] = cqq * tap * k;
  double dEv = dtap * ev + tap * dev;      /* N4 */
  double dEc = cqq * (dtap * k + tap * dk); /* N5 */
  *dEdr = dEv + dEc;
}

/* Neumaier compensated summation. */
typedef struct { double s, c; } orc_ksum;
static void ks_add(orc_ksum* a, double x) {
  double t = a->s + x;
  if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
  else a->c += (x - t) + a->s;
  a->s = t;
}

/* O6: Alg. 1 / Alg. 2 over the canonical half list:
 * E += e(i,k); f = g*d with g = (dE/dr)/r and d = minimum-image(x_k - x_i);
 * gForce[i] += f; gForce[k] -= f (Alg. 2 line 12 read as "-=", reading 20).
 * Energies use Neumaier sums in canonical pair order.  E = {E_vdW, E_Coul}. */
void orc_nonbonded(int64_t n, const double* pos, const int32_t* type, const double* q,
                   const double box[3], const orc_params* P, double R, const int64_t* hrow,
                   const int32_t* hcol, double E[2], double* F) {
  orc_ksum ev = {0, 0}, ec = {0, 0};
  double d[3], e[2], dEdr;
  for (int64_t i = 0; i < 3 * n; ++i) F[i] = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = hrow[i]; p < hrow[i + 1]; ++p) {
      int64_t k = hcol[p];
      double r = sqrt(orc_dist2(pos, i, k, box, d));
      orc_pair(r, type[i], type[k], q[i], q[k], P, R, e, &dEdr);
      ks_add(&ev, e[0]);
      ks_add(&ec, e[1]);
      double g = dEdr / r;
      for (int m = 0; m < 3; ++m) {
        F[3 * i + m] += g * d[m];
        F[3 * k + m] -= g * d[m];
      }
    }
  E[0] = ev.s + ev.c;
  E[1] = ec.s + ec.c;
}

/* O6, row-parallel (the form every evaluation uses; orc_nonbonded above is
 * Alg. 2's scatter loop literally, kept as its cross-check).  Each atom row a
 * visits its FULL neighbour set from the cell grid in ascending b and gathers
 * F_a = sum_b g_ab d_ab with d_ab = minimum-image(x_b - x_a), g_ab =
 * (dE/dr)/r — the same F = -grad E as the scatter F_i += f, F_k -= f, each
 * pair seen from both of its atoms; the energy of row a is the Neumaier sum
 * of e(a, b) over b > a (each pair once).  The row energies are combined in
 * row order with a Neumaier sum (reading 22: any order within tolerance). */
typedef struct {
  const orc_grid* G;
  const double *pos, *box, *q;
  const int32_t* type;
  const orc_params* P;
  double R;
  double* F;
  double* Erow; /* [n][2] */
} orc_nb_ctx;

static void orc_nb_row(int64_t a, void* c, void* scr) {
  orc_nb_ctx* C = (orc_nb_ctx*)c;
  int32_t* row = (int32_t*)scr;
  int64_t m = orc_grid_row(C->G, a, C->pos, C->box, C->R * C->R, 0, row);
  orc_ksum ev = {0, 0}, ec = {0, 0};
  double f[3] = {0.0, 0.0, 0.0}, d[3], e[2], dEdr;
  for (int64_t t = 0; t < m; ++t) {
    int64_t b = row[t];
    double r = sqrt(orc_dist2(C->pos, a, b, C->box, d));
    orc_pair(r, C->type[a], C->type[b], C->q[a], C->q[b], C->P, C->R, e, &dEdr);
    double g = dEdr / r;
    for (int k = 0; k < 3; ++k) f[k] += g * d[k];
    if (b > a) {
      ks_add(&ev, e[0]);
      ks_add(&ec, e[1]);
    }
  }
  for (int k = 0; k < 3; ++k) C->F[3 * a + k] = f[k];
  C->Erow[2 * a] = ev.s + ev.c;
  C->Erow[2 * a + 1] = ec.s + ec.c;
}

void orc_nonbonded_rows(int64_t n, const double* pos, const int32_t* type, const double* q,
                        const double box[3], const orc_params* P, double R, double E[2], double* F, int T) {
  orc_grid G;
  orc_grid_build(&G, n, pos, box, R);
  double* Erow = (double*)malloc(sizeof(double) * 2 * (size_t)(n > 0 ? n : 1));
  orc_nb_ctx C = {&G, pos, box, q, type, P, R, F, Erow};
  orc_par_rows(n, T, orc_nb_row, &C, sizeof(int32_t) * (size_t)G.maxcand);
  orc_ksum ev = {0, 0}, ec = {0, 0};
  for (int64_t a = 0; a < n; ++a) {
    ks_add(&ev, Erow[2 * a]);
    ks_add(&ec, Erow[2 * a + 1]);
  }
  E[0] = ev.s + ev.c;
  E[1] = ec.s + ec.c;
  free(Erow);
  orc_grid_free(&G);
}

/* ------------------------------------------ per-atom brute force (large N) */

/* All j != i with min-image r^2 <= R^2 (the FULL neighbour set of atom i),
 * ascending; O(N).  Used to sample c3/c4 outputs one atom at a time. */
int64_t orc_atom_neighbors(int64_t i, int64_t n, const double* pos, const double box[3], double R,
                           int32_t* out, int64_t cap) {
  double R2 = R * R, d[3];
  int64_t m = 0;
  for (int64_t j = 0; j < n; ++j)
    if (j != i && orc_dist2(pos, i, j, box, d) <= R2) {
      if (m < cap) out[m] = (int32_t)j;
      ++m;
    }
  return m;
}

/* Force on atom i and its pair-energy share (1/2 of each of its pairs),
 * brute force over all j.  F = sum_j g_ij d_ij (the F_i += f side of Alg. 1). */
void orc_atom_force(int64_t i, int64_t n, const double* pos, const int32_t* type, const double* q,
                    const double box[3], const orc_params* P, double R, double F[3], double Ehalf[2]) {
  double R2 = R * R, d[3], e[2], dEdr;
  orc_ksum a = {0, 0}, b = {0, 0};
  F[0] = F[1] = F[2] = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    if (j == i) continue;
    double r2 = orc_dist2(pos, i, j, box, d);
    if (r2 > R2) continue;
    double r = sqrt(r2);
    orc_pair(r, type[i], type[j], q[i], q[j], P, R, e, &dEdr);
    ks_add(&a, 0.5 * e[0]);
    ks_add(&b, 0.5 * e[1]);
    double g = dEdr / r;
    for (int m = 0; m < 3; ++m) F[m] += g * d[m];
  }
  Ehalf[0] = a.s + a.c;
  Ehalf[1] = b.s + b.c;
}

/* Bonds of atom i by brute force: partners (ascending), BO' terms, and the
 * atom's Delta' — O(N) per call. */
int64_t orc_atom_bonds(int64_t i, int64_t n, const double* pos, const int32_t* type,
                       const double box[3], const orc_params* P, double r_bond, double bo_cut,
                       int32_t* partner, double* raw, double* delta, int64_t cap) {
  double rb2 = r_bond * r_bond, d[3], v[4];
  int64_t m = 0;
  double s = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    if (j == i) continue;
    double r2 = orc_dist2(pos, i, j, box, d);
    if (r2 > rb2) continue;
    orc_bo_raw(sqrt(r2), type[i < j ? i : j], type[i < j ? j : i], P, v);
    if (v[3] < bo_cut) continue;
    if (m < cap) {
      partner[m] = (int32_t)j;
      for (int k = 0; k < 4; ++k) raw[4 * m + k] = v[k];
    }
    s += v[3];
    ++m;
  }
  delta[0] = s - P->val[type[i]];
  delta[1] = s - P->val_boc[type[i]];
  return m;
}

/* ------------------------------------------------------- O8 bond energy (NEXT-1)
 * the bond energy of the corrected bond orders and its
 * forces through the chain rule of B1-B8 (the bond part of "Aggregate Forces",
 * PAPER.md:160, 285).  Form (standard ReaxFF, ref [6]; reading 28):
 *   (E1) e_ij = -De_s BOs exp[p_be1 (1 - BOs^p_be2)] - De_p BOpi - De_pp BOpipi,
 *        BOs^p_be2 := 0 for BOs <= 0,
 * summed once per bond (canonical i < j).  Bonds are those of O3 (reading 2A:
 * BO' >= bo_cut), held fixed: E is differentiated at a fixed bond set.
 * Every bond order of bond b = (i, j) depends on its own distance r_b (B1) and
 * on the sums S_i = sum_k BO'_ik, S_j (through Delta'_i = S_i - Val_i and
 * Delta'boc_i = S_i - Val^boc_i in f1, f4, f5).  Hence
 *   dE/dr_b = de_b/dr_b |_S + (D_i + D_j) dBO'_b/dr_b,   D_i = sum_{b' ni i} de_b'/dS_i,
 * and the forces are central along each bond: F_i += g d, F_j -= g d with
 * g = (dE/dr_b)/r_b, d = minimum-image(x_j - x_i) (F = -grad E, as O6). */

/* d/dr of the three B1 terms at distance r: out = {dBO'sigma, dBO'pi, dBO'pipi}/dr,
 * from BO'_k = exp(pa (r/r0)^pb): dBO'_k/dr = BO'_k pa pb (r/r0)^pb / r. */
static void orc_bo_raw_dr(double r, int ti, int tj, const orc_params* P, const double raw[4], double out[3]) {
  int nt = P->ntypes, tp = ti * nt + tj;
  double r0[3] = {0.5 * (P->r_sigma[ti] + P->r_sigma[tj]), 0.5 * (P->r_pi[ti] + P->r_pi[tj]),
                  0.5 * (P->r_pipi[ti] + P->r_pipi[tj])};
  double pa[3] = {P->p_bo1[tp], P->p_bo3[tp], P->p_bo5[tp]};
  double pb[3] = {P->p_bo2[tp], P->p_bo4[tp], P->p_bo6[tp]};
  for (int k = 0; k < 3; ++k) out[k] = raw[k] * pa[k] * pb[k] * pow(r / r0[k], pb[k]) / r;
}

/* One bond (i, j) in canonical orientation: its energy e (E1) and the partial
 * derivatives de/dr|_S (at fixed S_i, S_j), de/dS_i, de/dS_j, plus dBO'/dr.
 * Follows B4-B8 as orc_bo_corr_pair and differentiates each factor:
 *   f2 = e^{-p1 Di} + e^{-p1 Dj}           df2/dDi = -p1 e^{-p1 Di}
 *   f3 = -(1/p2) ln(1/2 (e^{-p2 Di} + e^{-p2 Dj}))
 *                                          df3/dDi = e^{-p2 Di} / (e^{-p2 Di} + e^{-p2 Dj})
 *   f1 = 1/2 (u_i + u_j), u_a = (V_a + f2)/(V_a + f2 + f3)
 *                                          du_a/df2 = f3 / (V_a+f2+f3)^2,
 *                                          du_a/df3 = -(V_a + f2) / (V_a+f2+f3)^2
 *   f4 = 1/(1 + e^{z4}), z4 = -p3 (p4 BO'^2 - Dboc_i) + p5
 *                                          df4/dBO' = f4 (1-f4) 2 p3 p4 BO',  df4/dS_i = -f4 (1-f4) p3
 *   BO = BO' A, BOpi = BO'pi f1 A, BOpipi = BO'pipi f1 A, A = f1 f4 f5, BOs = BO - BOpi - BOpipi. */
void orc_bond_energy_pair(double r, const double raw[4], double di, double dboci, double dj, double dbocj,
                          int ti, int tj, const orc_params* P, const orc_bond_params* Q, double out[5]) {
  int tp = ti * P->ntypes + tj;
  double p1 = P->p_boc1, p2 = P->p_boc2;
  double vi = P->val[ti], vj = P->val[tj];
  double p3 = sqrt(P->b132[ti] * P->b132[tj]);
  double p4 = sqrt(P->b131[ti] * P->b131[tj]);
  double p5 = sqrt(P->b133[ti] * P->b133[tj]);
  double bpi = raw[1], bpp = raw[2], bo = raw[3];
  /* B4-B8 */
  double ei1 = exp(-p1 * di), ej1 = exp(-p1 * dj);
  double ei2 = exp(-p2 * di), ej2 = exp(-p2 * dj);
  double f2 = ei1 + ej1;
  double f3 = -(1.0 / p2) * log(0.5 * (ei2 + ej2));
  double ni = vi + f2 + f3, nj = vj + f2 + f3;
  double f1 = 0.5 * ((vi + f2) / ni + (vj + f2) / nj);
  double f4 = 1.0 / (1.0 + exp(-p3 * (p4 * bo * bo - dboci) + p5));
  double f5 = 1.0 / (1.0 + exp(-p3 * (p4 * bo * bo - dbocj) + p5));
  double A = f1 * f4 * f5;
  double BO = bo * A, BOpi = bpi * f1 * A, BOpp = bpp * f1 * A;
  double BOs = BO - BOpi - BOpp;
  /* E1 and its partials in BOs, BOpi, BOpipi */
  double Ds = Q->De_s[tp], Dp = Q->De_p[tp], Dpp = Q->De_pp[tp], b1 = Q->p_be1[tp], b2 = Q->p_be2[tp];
  double sp = BOs > 0.0 ? pow(BOs, b2) : 0.0;
  double ex = exp(b1 * (1.0 - sp));
  double e = -Ds * BOs * ex - Dp * BOpi - Dpp * BOpp;
  double e_s = -Ds * ex * (1.0 - b1 * b2 * sp);
  double c_bo = e_s, c_pi = -Dp - e_s, c_pp = -Dpp - e_s;   /* de/dBO, de/dBOpi, de/dBOpipi */
  /* through A = f1 f4 f5 and the explicit f1 of BOpi, BOpipi */
  double w = c_pi * bpi + c_pp * bpp;
  double de_dA = c_bo * bo + w * f1;
  double de_df1 = de_dA * f4 * f5 + w * A;
  double de_df4 = de_dA * f1 * f5;
  double de_df5 = de_dA * f1 * f4;
  /* f1 in Delta'_i, Delta'_j */
  double du_i_df2 = f3 / (ni * ni), du_i_df3 = -(vi + f2) / (ni * ni);
  double du_j_df2 = f3 / (nj * nj), du_j_df3 = -(vj + f2) / (nj * nj);
  double df2_di = -p1 * ei1, df2_dj = -p1 * ej1;
  double df3_di = ei2 / (ei2 + ej2), df3_dj = ej2 / (ei2 + ej2);
  double df1_di = 0.5 * ((du_i_df2 + du_j_df2) * df2_di + (du_i_df3 + du_j_df3) * df3_di);
  double df1_dj = 0.5 * ((du_i_df2 + du_j_df2) * df2_dj + (du_i_df3 + du_j_df3) * df3_dj);
  /* f4, f5 in S (through Delta'boc) and in BO' */
  double df4_dS = -f4 * (1.0 - f4) * p3, df5_dS = -f5 * (1.0 - f5) * p3;
  double df4_dbo = f4 * (1.0 - f4) * 2.0 * p3 * p4 * bo, df5_dbo = f5 * (1.0 - f5) * 2.0 * p3 * p4 * bo;
  double de_dSi = de_df1 * df1_di + de_df4 * df4_dS;
  double de_dSj = de_df1 * df1_dj + de_df5 * df5_dS;
  /* direct r dependence at fixed S: each raw term of BO, BOpi, BOpipi, and BO' in f4, f5 */
  double dr[3];
  orc_bo_raw_dr(r, ti, tj, P, raw, dr);
  double X = de_df4 * df4_dbo + de_df5 * df5_dbo;   /* de/dBO' through f4, f5 */
  double de_dr = (c_bo * A + X) * dr[0] + (c_bo * A + c_pi * f1 * A + X) * dr[1] +
                 (c_bo * A + c_pp * f1 * A + X) * dr[2];
  out[0] = e;
  out[1] = de_dr;
  out[2] = de_dSi;
  out[3] = de_dSj;
  out[4] = (dr[0] + dr[1]) + dr[2];   /* dBO'/dr */
}

/* O8: E1 over the bonds of O3, row-parallel.  Pass 1 (per atom row a, bonds
 * in row order): D_a = sum over a's bonds of de_b/dS_a, each bond evaluated
 * in canonical orientation (i, j) = (min, max) so that de/dS_i is out[2] and
 * de/dS_j out[3]; the row's energy is the Neumaier sum of e over its
 * partners b > a (each bond once), rows combined in row order.  Pass 2: F_a
 * = sum_b g d_ab, g = (de/dr + (D_i + D_j) dBO'/dr)/r, d_ab =
 * minimum-image(x_b - x_a) — the scatter F_i += g d_ij, F_j -= g d_ij seen
 * from each atom.  raw: [B][4] BO' terms of O3; delta: [n][2] of O4;
 * forces [n][3] overwritten. */
typedef struct {
  const double *pos, *box, *raw, *delta;
  const int32_t *type, *bcol;
  const int64_t* brow;
  const orc_params* P;
  const orc_bond_params* Q;
  double *D, *Erow, *F;
} orc_be_ctx;

static void orc_be_eval(const orc_be_ctx* C, int64_t a, int64_t e, double d[3], double* r, double out[5]) {
  int64_t b = C->bcol[e], i = a < b ? a : b, j = a < b ? b : a;
  *r = sqrt(orc_dist2(C->pos, a, b, C->box, d));
  orc_bond_energy_pair(*r, &C->raw[4 * e], C->delta[2 * i], C->delta[2 * i + 1], C->delta[2 * j],
                       C->delta[2 * j + 1], C->type[i], C->type[j], C->P, C->Q, out);
}

static void orc_be_row1(int64_t a, void* c, void* scr) {
  orc_be_ctx* C = (orc_be_ctx*)c;
  double d[3], r, out[5], D = 0.0;
  orc_ksum E = {0.0, 0.0};
  (void)scr;
  for (int64_t e = C->brow[a]; e < C->brow[a + 1]; ++e) {
    int64_t b = C->bcol[e];
    orc_be_eval(C, a, e, d, &r, out);
    D += a < b ? out[2] : out[3];
    if (b > a) ks_add(&E, out[0]);
  }
  C->D[a] = D;
  C->Erow[a] = E.s + E.c;
}

static void orc_be_row2(int64_t a, void* c, void* scr) {
  orc_be_ctx* C = (orc_be_ctx*)c;
  double d[3], r, out[5], f[3] = {0.0, 0.0, 0.0};
  (void)scr;
  for (int64_t e = C->brow[a]; e < C->brow[a + 1]; ++e) {
    int64_t b = C->bcol[e], i = a < b ? a : b, j = a < b ? b : a;
    orc_be_eval(C, a, e, d, &r, out);
    double g = (out[1] + (C->D[i] + C->D[j]) * out[4]) / r;
    for (int k = 0; k < 3; ++k) f[k] += g * d[k];
  }
  for (int k = 0; k < 3; ++k) C->F[3 * a + k] = f[k];
}

void orc_bond_energy(int64_t n, const double* pos, const int32_t* type, const double box[3],
                     const orc_params* P, const orc_bond_params* Q, const int64_t* brow,
                     const int32_t* bcol, const double* raw, const double* delta, double* force,
                     double* energy, int T) {
  size_t n1 = (size_t)(n > 0 ? n : 1);
  double* D = (double*)calloc(n1, sizeof(double));
  double* Erow = (double*)calloc(n1, sizeof(double));
  orc_be_ctx C = {pos, box, raw, delta, type, bcol, brow, P, Q, D, Erow, force};
  orc_par_rows(n, T, orc_be_row1, &C, 0);
  orc_par_rows(n, T, orc_be_row2, &C, 0);
  orc_ksum E = {0.0, 0.0};
  for (int64_t a = 0; a < n; ++a) ks_add(&E, Erow[a]);
  *energy = E.s + E.c;
  free(D);
  free(Erow);
}

/* ------------------------------------------------ O9 interaction lists (NEXT-3)
 * SURVEY.md §8(f) NEXT-3; PAPER.md:198-202 (§3.3 "Three-body Interactions":
 * angles are identified, a prefix sum gives the offsets, then they are
 * stored) and PAPER.md:154-158 (the hydrogen-bond list built from the
 * surroundings of covalently bonded H atoms).  Readings:
 *   angles   for every entry e = (j, i) of the full bond list (central atom j),
 *            the partners k of the other entries f = (j, k), f != e, of row j,
 *            kept iff BO_e > thb_cut, BO_f > thb_cut and BO_e BO_f > thb_cutsq
 *            (BO = corrected total bond order, a6), in row order (k ascending);
 *   H-bonds  for every atom i of type h_type with at least one bond, the atoms
 *            z != i of an acceptor type (bit type(z) of acc_mask) with
 *            minimum-image r_iz^2 <= r_hb^2 (FMA-free, as O2), z ascending.
 * Both lists are CSR: off[0] = 0, off[row+1] = off[row] + count (int64). */

/* angles over the bond CSR (rows i ascending, entries sorted by j), BO from
 * corr[B][4] (BO = corr[4e]).  Writes ang_off[B+1] always, ang_k up to cap;
 * returns the total. */
int64_t orc_angles(int64_t n, const int64_t* brow, const int32_t* bcol, const double* corr, double thb_cut,
                   double thb_cutsq, int64_t* ang_off, int32_t* ang_k, int64_t cap) {
  int64_t t = 0;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t e = brow[j]; e < brow[j + 1]; ++e) {
      ang_off[e] = t;
      double be = corr[4 * e];
      if (!(be > thb_cut)) continue;
      for (int64_t f = brow[j]; f < brow[j + 1]; ++f) {
        if (f == e) continue;
        double bf = corr[4 * f];
        if (bf > thb_cut && be * bf > thb_cutsq) {
          if (t < cap) ang_k[t] = bcol[f];
          ++t;
        }
      }
    }
  ang_off[brow[n]] = t;
  return t;
}

/* H-bond lists by brute force over all atom pairs (the definition).  Writes
 * hb_off[n+1] always, hb_z up to cap; returns the total. */
int64_t orc_hbonds(int64_t n, const double* pos, const int32_t* type, const double box[3], const int64_t* brow,
                   double r_hb, int32_t h_type, uint32_t acc_mask, int64_t* hb_off, int32_t* hb_z, int64_t cap) {
  double d[3], r2max = r_hb * r_hb;
  int64_t t = 0;
  for (int64_t i = 0; i < n; ++i) {
    hb_off[i] = t;
    if (type[i] != h_type || brow[i + 1] == brow[i]) continue;
    for (int64_t z = 0; z < n; ++z) {
      if (z == i || !((acc_mask >> type[z]) & 1u)) continue;
      if (orc_dist2(pos, i, z, box, d) <= r2max) {
        if (t < cap) hb_z[t] = (int32_t)z;
        ++t;
      }
    }
  }
  hb_off[n] = t;
  return t;
}

/* O9 for one atom (sampled checks at large sizes): the H-bond list of atom i
 * by brute force; has_bond says whether i has a bond.  Returns the count,
 * writes up to cap partners ascending. */
int64_t orc_atom_hbonds(int64_t i, int64_t n, const double* pos, const int32_t* type, const double box[3],
                        int has_bond, double r_hb, int32_t h_type, uint32_t acc_mask, int32_t* out, int64_t cap) {
  double d[3], r2max = r_hb * r_hb;
  int64_t t = 0;
  if (type[i] != h_type || !has_bond) return 0;
  for (int64_t z = 0; z < n; ++z) {
    if (z == i || !((acc_mask >> type[z]) & 1u)) continue;
    if (orc_dist2(pos, i, z, box, d) <= r2max) {
      if (t < cap) out[t] = (int32_t)z;
      ++t;
    }
  }
  return t;
}

/* O9 H-bond lists from the cell grid at r_hb, row-parallel (the same set as
 * orc_hbonds' O(N^2) definition, which pins it; c3/c4).  Count pass, serial
 * offsets, fill pass; rows ascending in z. */
typedef struct {
  const orc_grid* G;
  const double *pos, *box;
  const int32_t* type;
  const int64_t* brow;
  double r2;
  int32_t h_type;
  uint32_t acc_mask;
  int64_t* cnt;
  const int64_t* off;
  int32_t* z;
} orc_hb_ctx;

static void orc_hb_row(int64_t i, orc_hb_ctx* C, int32_t* row, int fill) {
  int64_t t = 0;
  if (C->type[i] == C->h_type && C->brow[i + 1] > C->brow[i]) {
    int64_t m = orc_grid_row(C->G, i, C->pos, C->box, C->r2, 0, row);
    for (int64_t a = 0; a < m; ++a)
      if ((C->acc_mask >> C->type[row[a]]) & 1u) {
        if (fill) C->z[C->off[i] + t] = row[a];
        ++t;
      }
  }
  if (!fill) C->cnt[i] = t;
}
static void orc_hb_count(int64_t i, void* c, void* s) { orc_hb_row(i, (orc_hb_ctx*)c, (int32_t*)s, 0); }
static void orc_hb_fill(int64_t i, void* c, void* s) { orc_hb_row(i, (orc_hb_ctx*)c, (int32_t*)s, 1); }

int64_t orc_hbonds_cells(int64_t n, const double* pos, const int32_t* type, const double box[3], const int64_t* brow,
                         double r_hb, int32_t h_type, uint32_t acc_mask, int64_t* hb_off, int32_t* hb_z, int64_t cap,
                         int T) {
  orc_grid G;
  orc_grid_build(&G, n, pos, box, r_hb);
  int64_t* cnt = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
  orc_hb_ctx C = {&G, pos, box, type, brow, r_hb * r_hb, h_type, acc_mask, cnt, hb_off, hb_z};
  size_t scr = sizeof(int32_t) * (size_t)G.maxcand;
  orc_par_rows(n, T, orc_hb_count, &C, scr);
  int64_t t = 0;
  for (int64_t i = 0; i < n; ++i) {
    hb_off[i] = t;
    t += cnt[i];
  }
  hb_off[n] = t;
  if (t <= cap) orc_par_rows(n, T, orc_hb_fill, &C, scr);
  free(cnt);
  orc_grid_free(&G);
  return t;
}

/* ------------------------------------------- O10 species analysis (NEXT-4)
 * PAPER.md:217-221 (§3.4, the in situ species algorithm), step by step:
 *  1. "A pair of atoms ... are deemed to be bonded if the bond order value
 *     between the two atoms is larger than a threshold specified for this
 *     interaction type (default value is 0.3).  A molecule ID, that is the
 *     smaller value of the two global IDs, is assigned to the pair of atoms.
 *     This process is repeated until every atom has been assigned a molecule
 *     ID": label[i] = i, then sweeps over the bonds (canonical i < j, BO =
 *     the corrected total bond order of a6, BO > thresh[ti][tj] strictly)
 *     setting both labels to the smaller one, until a sweep changes nothing
 *     (the label is then the smallest global ID of the connected component).
 *  2. "Sorting is performed for all molecule IDs and molecule IDs are
 *     reassigned from 1 to M": mol_id[i] = 1 + rank of label[i] among the
 *     distinct labels in ascending order.
 *  3. "counting the number of atoms of each element.  Molecules with the same
 *     number of atoms per element are identified as the same species" (the
 *     element of an atom is its type).
 *  4. "each distinct species and their counts": species sorted by their
 *     composition vector (count of type 0, then type 1, ...) ascending.
 * Global IDs are the 0-based input indices.  corr: [B][4] (corr[4e] = BO).
 * Writes mol_id[n]; up to cap species (sp_comp [cap][ntypes], sp_count);
 * *n_species = the number of distinct species.  Returns M. */
static int orc_sp_nt;
static int orc_cmp_comp(const void* a, const void* b) {
  const int32_t *x = (const int32_t*)a, *y = (const int32_t*)b;
  for (int t = 0; t < orc_sp_nt; ++t)
    if (x[t] != y[t]) return x[t] < y[t] ? -1 : 1;
  return 0;
}

int64_t orc_species(int64_t n, const int32_t* type, int ntypes, const int64_t* brow, const int32_t* bcol,
                    const double* corr, const double* thresh, int32_t* mol_id, int32_t* sp_comp, int64_t* sp_count,
                    int64_t cap, int64_t* n_species) {
  size_t n1 = (size_t)(n > 0 ? n : 1);
  int64_t* label = (int64_t*)malloc(sizeof(int64_t) * n1);
  for (int64_t i = 0; i < n; ++i) label[i] = i;
  for (int changed = 1; changed;) { /* step 1 */
    changed = 0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t e = brow[i]; e < brow[i + 1]; ++e) {
        int64_t j = bcol[e];
        if (j <= i || !(corr[4 * e] > thresh[type[i] * ntypes + type[j]])) continue;
        int64_t m = label[i] < label[j] ? label[i] : label[j];
        if (label[i] != m || label[j] != m) {
          label[i] = label[j] = m;
          changed = 1;
        }
      }
  }
  int64_t* rank = (int64_t*)malloc(sizeof(int64_t) * n1); /* step 2 */
  for (int64_t i = 0; i < n; ++i) rank[i] = 0;
  for (int64_t i = 0; i < n; ++i) rank[label[i]] = 1;
  int64_t M = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t isroot = rank[i];
    rank[i] = M;
    M += isroot;
  }
  for (int64_t i = 0; i < n; ++i) mol_id[i] = (int32_t)(rank[label[i]] + 1);
  int32_t* comp = (int32_t*)calloc((size_t)(M > 0 ? M : 1) * (size_t)ntypes, sizeof(int32_t)); /* step 3 */
  for (int64_t i = 0; i < n; ++i) comp[(int64_t)(mol_id[i] - 1) * ntypes + type[i]]++;
  orc_sp_nt = ntypes; /* step 4 */
  qsort(comp, (size_t)M, sizeof(int32_t) * (size_t)ntypes, orc_cmp_comp);
  int64_t S = 0;
  for (int64_t m = 0; m < M; ++m) {
    if (m == 0 || orc_cmp_comp(&comp[m * ntypes], &comp[(m - 1) * ntypes]) != 0) {
      if (S < cap) {
        memcpy(&sp_comp[S * ntypes], &comp[m * ntypes], sizeof(int32_t) * (size_t)ntypes);
        sp_count[S] = 0;
      }
      ++S;
    }
    if (S - 1 < cap) sp_count[S - 1]++;
  }
  *n_species = S;
  free(label);
  free(rank);
  free(comp);
  return M;
}

/* ------------------------------------------------------- O11 QEq (NEXT-2)
 * PAPER.md:204-208 (§3.3 "QEq"): charges minimise
 *   E(q) = sum_i (chi_i q_i + 1/2 eta_i q_i^2) + sum_{i<j} H_ij q_i q_j
 * subject to sum_i q_i = 0 (reading 33).  With Lagrange multipliers
 * this gives "two linear systems of equations ... with a common kernel H, an
 * N x N sparse matrix": H s = -chi, H t = -1, and q = s - (sum s / sum t) t.
 * H_ii = eta_i; H_ij = C Tap(r_ij) (r_ij^3 + gamma_ij^-3)^(-1/3) for the pairs
 * of the half list ("a truncated electrostatics interaction"; the shielded
 * Coulomb kernel of N5 without the charges, orc_taper x orc_coulomb_kernel),
 * stored once per unordered pair ("only unique, non-zero elements of the
 * sparse matrix are computed and stored").  Solved by "a diagonally
 * preconditioned ... CG solver" (Jacobi-PCG, preconditioner 1/eta_i), each
 * system from its initial guess to ||b - H x|| <= tol ||b|| (PAPER.md:243:
 * QEq tolerance 1e-6). */

/* H_ij of every canonical pair (hval[P], aligned with hcol). */
void orc_qeq_H(int64_t n, const double* pos, const int32_t* type, const double box[3], const orc_params* P,
               double R, const int64_t* hrow, const int32_t* hcol, double* hval) {
  double d[3], tap, dtap, k, dk;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = hrow[i]; p < hrow[i + 1]; ++p) {
      int64_t j = hcol[p];
      double r = sqrt(orc_dist2(pos, i, j, box, d));
      orc_taper(r, R, &tap, &dtap);
      orc_coulomb_kernel(r, type[i], type[j], P, &k, &dk);
      hval[p] = P->coulomb_c * tap * k;
    }
}

/* y = H x over the half-stored H: y_i = eta_i x_i + sum_{j in row i} H_ij x_j,
 * and y_j += H_ij x_i for each stored (i, j). */
void orc_qeq_spmv(int64_t n, const double* eta_atom, const int64_t* hrow, const int32_t* hcol, const double* hval,
                  const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) y[i] = eta_atom[i] * x[i];
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = hrow[i]; p < hrow[i + 1]; ++p) {
      int64_t j = hcol[p];
      y[i] += hval[p] * x[j];
      y[j] += hval[p] * x[i];
    }
}

static double orc_dot(int64_t n, const double* a, const double* b) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* Jacobi-PCG on H x = b from the initial x (in/out); returns the iterations. */
int orc_qeq_pcg(int64_t n, const double* eta_atom, const int64_t* hrow, const int32_t* hcol, const double* hval,
                const double* b, double* x, double tol, int maxiter) {
  size_t n1 = (size_t)(n > 0 ? n : 1);
  double *r = (double*)malloc(sizeof(double) * n1), *z = (double*)malloc(sizeof(double) * n1);
  double *p = (double*)malloc(sizeof(double) * n1), *Ap = (double*)malloc(sizeof(double) * n1);
  orc_qeq_spmv(n, eta_atom, hrow, hcol, hval, x, Ap);
  for (int64_t i = 0; i < n; ++i) {
    r[i] = b[i] - Ap[i];
    z[i] = r[i] / eta_atom[i];
    p[i] = z[i];
  }
  double bn = sqrt(orc_dot(n, b, b)), rz = orc_dot(n, r, z);
  int it = 0;
  while (it < maxiter && sqrt(orc_dot(n, r, r)) > tol * bn) {
    orc_qeq_spmv(n, eta_atom, hrow, hcol, hval, p, Ap);
    double alpha = rz / orc_dot(n, p, Ap);
    for (int64_t i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * Ap[i];
      z[i] = r[i] / eta_atom[i];
    }
    double rz1 = orc_dot(n, r, z), beta = rz1 / rz;
    rz = rz1;
    for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    ++it;
  }
  free(r); free(z); free(p); free(Ap);
  return it;
}

/* The whole QEq: H, then s (H s = -chi), t (H t = -1) from the guesses in
 * s, t (in/out), q = s - (sum s / sum t) t.  chi, eta per type.  iters[2]. */
void orc_qeq(int64_t n, const double* pos, const int32_t* type, const double box[3], const orc_params* P,
             double R, const int64_t* hrow, const int32_t* hcol, const double* chi, const double* eta, double tol,
             int maxiter, double* s, double* t, double* q, int* iters) {
  size_t n1 = (size_t)(n > 0 ? n : 1);
  int64_t np = hrow[n];
  double* hval = (double*)malloc(sizeof(double) * (size_t)(np > 0 ? np : 1));
  double *ea = (double*)malloc(sizeof(double) * n1), *bs = (double*)malloc(sizeof(double) * n1),
         *bt = (double*)malloc(sizeof(double) * n1);
  orc_qeq_H(n, pos, type, box, P, R, hrow, hcol, hval);
  for (int64_t i = 0; i < n; ++i) {
    ea[i] = eta[type[i]];
    bs[i] = -chi[type[i]];
    bt[i] = -1.0;
  }
  iters[0] = orc_qeq_pcg(n, ea, hrow, hcol, hval, bs, s, tol, maxiter);
  iters[1] = orc_qeq_pcg(n, ea, hrow, hcol, hval, bt, t, tol, maxiter);
  double ss = 0.0, st = 0.0;
  for (int64_t i = 0; i < n; ++i) { ss += s[i]; st += t[i]; }
  double mu = ss / st;
  for (int64_t i = 0; i < n; ++i) q[i] = s[i] - mu * t[i];
  free(hval); free(ea); free(bs); free(bt);
}
