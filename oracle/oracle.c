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
 * single thread, every loop in the order the definition states.
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

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* Cell-list version of the same set (O2): cells of side L/floor(L/(R(1+1e-9)))
 * per axis (strictly wider than R, so rounding in floor(x/side) can never put
 * two atoms within R more than one cell apart),
 * the set of neighbour cells deduplicated (c0 has 2 cells per axis, so -1 and
 * +1 name the same cell), candidate j > i kept iff r^2 <= R^2. */
int64_t orc_half_list_cells(int64_t n, const double* pos, const double box[3], double R,
                            int64_t* rowoff, int32_t* col, int64_t cap) {
  int nc[3];
  for (int k = 0; k < 3; ++k) {
    nc[k] = (int)floor(box[k] / (R * (1.0 + 1e-9)));
    if (nc[k] < 1) nc[k] = 1;
  }
  int64_t ncell = (int64_t)nc[0] * nc[1] * nc[2];
  int64_t* head = (int64_t*)malloc(sizeof(int64_t) * ncell);
  int64_t* next = (int64_t*)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  int32_t* cell = (int32_t*)malloc(sizeof(int32_t) * 3 * (n > 0 ? n : 1));
  int32_t* row = (int32_t*)malloc(sizeof(int32_t) * (n > 0 ? n : 1));
  for (int64_t c = 0; c < ncell; ++c) head[c] = -1;
  for (int64_t i = n - 1; i >= 0; --i) {
    int64_t c = 0;
    for (int k = 2; k >= 0; --k) {
      int ck = (int)floor(pos[3 * i + k] / (box[k] / nc[k]));
      if (ck >= nc[k]) ck = nc[k] - 1;
      if (ck < 0) ck = 0;
      cell[3 * i + k] = ck;
      c = c * nc[k] + ck;
    }
    next[i] = head[c];
    head[c] = i;
  }
  double R2 = R * R, d[3];
  int64_t p = 0;
  for (int64_t i = 0; i < n; ++i) {
    rowoff[i] = p;
    /* deduplicated neighbour cells */
    int64_t nb[27];
    int nnb = 0;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          int cx = ((cell[3 * i] + dx) % nc[0] + nc[0]) % nc[0];
          int cy = ((cell[3 * i + 1] + dy) % nc[1] + nc[1]) % nc[1];
          int cz = ((cell[3 * i + 2] + dz) % nc[2] + nc[2]) % nc[2];
          int64_t c = ((int64_t)cz * nc[1] + cy) * nc[0] + cx;
          int dup = 0;
          for (int m = 0; m < nnb; ++m) dup |= (nb[m] == c);
          if (!dup) nb[nnb++] = c;
        }
    int64_t len = 0;
    for (int m = 0; m < nnb; ++m)
      for (int64_t j = head[nb[m]]; j >= 0; j = next[j])
        if (j > i && orc_dist2(pos, i, j, box, d) <= R2) row[len++] = (int32_t)j;
    qsort(row, (size_t)len, sizeof(int32_t), cmp_i32);
    for (int64_t m = 0; m < len; ++m) {
      if (p < cap) col[p] = row[m];
      ++p;
    }
  }
  rowoff[n] = p;
  free(head); free(next); free(cell); free(row);
  return p;
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

/* O3: for every canonical pair of the half list with r <= r_bond (r^2 <=
 * r_bond^2), BO' from B1-B2; a bond iff BO' >= bo_cut (reading 2A).  Emits the
 * FULL list (both i->j and j->i, "requires the bond list to be a
 * full list with both i-j and j-i bonds available") as CSR with rows sorted by
 * j, plus the mirror index.  bo: [B][4].  Returns B (entries);
 * writes nothing past cap. */
int64_t orc_bonds(int64_t n, const double* pos, const int32_t* type, const double box[3],
                  const orc_params* P, double r_bond, double bo_cut, const int64_t* hrow,
                  const int32_t* hcol, int64_t* brow, int32_t* bcol, int32_t* bmirror,
                  double* bo, int64_t cap) {
  double rb2 = r_bond * r_bond, d[3], v[4];
  int64_t* deg = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
  /* pass 1: count kept bonds per atom */
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = hrow[i]; p < hrow[i + 1]; ++p) {
      int64_t j = hcol[p];
      double r2 = orc_dist2(pos, i, j, box, d);
      if (r2 > rb2) continue;
      orc_bo_raw(sqrt(r2), type[i], type[j], P, v);
      if (v[3] >= bo_cut) { deg[i]++; deg[j]++; }
    }
  brow[0] = 0;
  for (int64_t i = 0; i < n; ++i) brow[i + 1] = brow[i] + deg[i];
  int64_t B = brow[n];
  if (B > cap) { free(deg); return B; }
  /* pass 2: fill.  Canonical pairs are visited in (i asc, j asc) order, so row
   * i receives partners j < i (from earlier rows, ascending i) before its own
   * partners j > i (ascending): every row ends sorted by j. */
  int64_t* fill = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = hrow[i]; p < hrow[i + 1]; ++p) {
      int64_t j = hcol[p];
      double r2 = orc_dist2(pos, i, j, box, d);
      if (r2 > rb2) continue;
      orc_bo_raw(sqrt(r2), type[i], type[j], P, v);
      if (v[3] < bo_cut) continue;
      int64_t ei = brow[i] + fill[i]++, ej = brow[j] + fill[j]++;
      bcol[ei] = (int32_t)j; bcol[ej] = (int32_t)i;
      bmirror[ei] = (int32_t)ej; /* mirror = absolute entry index of j->i */
      bmirror[ej] = (int32_t)ei;
      for (int k = 0; k < 4; ++k) { bo[4 * ei + k] = v[k]; bo[4 * ej + k] = v[k]; }
    }
  free(deg); free(fill);
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

/* O8: E1 over the bonds of O3 (canonical i < j, ascending), Neumaier-summed;
 * forces [n][3] (overwritten) by the two passes stated above: D_i summed over
 * the canonical bonds in order, then g per bond.  raw: [B][4] BO' terms of
 * O3; delta: [n][2] of O4. */
void orc_bond_energy(int64_t n, const double* pos, const int32_t* type, const double box[3],
                     const orc_params* P, const orc_bond_params* Q, const int64_t* brow,
                     const int32_t* bcol, const double* raw, const double* delta, double* force,
                     double* energy) {
  double* D = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  orc_ksum E = {0.0, 0.0};
  double d[3], out[5];
  for (int64_t k = 0; k < 3 * n; ++k) force[k] = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = brow[i]; e < brow[i + 1]; ++e) {
      int64_t j = bcol[e];
      if (j < i) continue;
      double r = sqrt(orc_dist2(pos, i, j, box, d));
      orc_bond_energy_pair(r, &raw[4 * e], delta[2 * i], delta[2 * i + 1], delta[2 * j], delta[2 * j + 1],
                           type[i], type[j], P, Q, out);
      ks_add(&E, out[0]);
      D[i] += out[2];
      D[j] += out[3];
    }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = brow[i]; e < brow[i + 1]; ++e) {
      int64_t j = bcol[e];
      if (j < i) continue;
      double r = sqrt(orc_dist2(pos, i, j, box, d));
      orc_bond_energy_pair(r, &raw[4 * e], delta[2 * i], delta[2 * i + 1], delta[2 * j], delta[2 * j + 1],
                           type[i], type[j], P, Q, out);
      double g = (out[1] + (D[i] + D[j]) * out[4]) / r;
      for (int k = 0; k < 3; ++k) {
        force[3 * i + k] += g * d[k];
        force[3 * j + k] -= g * d[k];
      }
    }
  *energy = E.s + E.c;
  free(D);
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
