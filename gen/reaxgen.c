/* Seeded synthetic input generator for the ReaxFF hot path.
 *
 * INPUT ONLY.  This module holds none of the method's arithmetic: it draws
 * positions, types, charges and the synthetic parameter table that BOTH the
 * oracle (oracle/) and the CUDA library (paper_1706_07772_b200/) consume.
 *
 * Recipe (SURVEY.md §8(d) generator spec):
 *   RNG      SplitMix64, u = (next() >> 11) * 2^-53 in [0,1).
 *   seeds    positions+charges of config k: 1706077720 + k; parameters: 1706077720.
 *   atoms    sequential random addition: candidate (u*Lx, u*Ly, u*Lz) accepted iff
 *            its minimum-image squared distance to every accepted atom is >= dmin^2
 *            (dmin = 0.9 A), checked through a hash grid of cells >= 2*dmin.
 *   types    pattern[k mod 29], pattern = 5 C, 8 H, 4 N, 12 O (C=0,H=1,N=2,O=3):
 *            the C5H8N4O12 (PETN) formula unit of the paper's benchmark
 *            ("The PETN crystal benchmark").
 *   charges  q_k = u - 0.5 drawn after all positions, then minus their
 *            (Neumaier-compensated) mean so the system is neutral.
 *   params   per type C,H,N,O in this order: r_sigma, r_pi, r_pipi, gamma, r_vdw,
 *            eps, alpha, gamma_w, b131, b132, b133; then per type pair t1<=t2
 *            (lexicographic): p_bo1..p_bo6, De.  Ranges: BASELINE.json configs[0]
 *            plus SURVEY.md §8(c) point 10.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { uint64_t s; } sm64;

static uint64_t sm64_next(sm64* g) {
  uint64_t z = (g->s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static double sm64_u(sm64* g) { return (double)(sm64_next(g) >> 11) * 0x1.0p-53; }

/* exposed for tests: first k draws of u for a seed */
void gen_uniforms(uint64_t seed, int64_t k, double* out) {
  sm64 g = {seed};
  for (int64_t i = 0; i < k; ++i) out[i] = sm64_u(&g);
}

static double gen_min_image(double d, double L) {
  if (d >= 0.5 * L) d -= L;
  else if (d < -0.5 * L) d += L;
  return d;
}

/* Returns number of candidates drawn (>= n) or -1 on failure (too dense / OOM).
 * pos: n*3 row-major, type: n, q: n. */
int64_t gen_system(uint64_t seed, int64_t n, const double box[3], double dmin,
                   double* pos, int32_t* type, double* q, int64_t max_tries) {
  static const int32_t pattern[29] = {0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 1, 1, 1, 2, 2,
                                      2, 2, 3, 3, 3, 3, 3, 3, 3, 3, 3, 3, 3, 3};
  sm64 g = {seed};
  int nc[3];
  double inv_h[3];
  for (int k = 0; k < 3; ++k) {
    nc[k] = (int)floor(box[k] / (2.0 * dmin));
    if (nc[k] < 3) nc[k] = 1; /* tiny box: single cell, brute force */
    if (nc[k] > 2048) nc[k] = 2048;
    inv_h[k] = nc[k] / box[k];
  }
  int64_t ncell = (int64_t)nc[0] * nc[1] * nc[2];
  int32_t* head = (int32_t*)malloc(sizeof(int32_t) * ncell);
  int32_t* next = (int32_t*)malloc(sizeof(int32_t) * (n > 0 ? n : 1));
  if (!head || !next) { free(head); free(next); return -1; }
  for (int64_t c = 0; c < ncell; ++c) head[c] = -1;
  double d2min = dmin * dmin;
  int64_t accepted = 0, tries = 0;
  while (accepted < n) {
    if (tries >= max_tries) { free(head); free(next); return -1; }
    ++tries;
    double x[3];
    int ci[3];
    for (int k = 0; k < 3; ++k) {
      x[k] = sm64_u(&g) * box[k];
      if (x[k] >= box[k]) x[k] = 0.0;
      int c = (int)(x[k] * inv_h[k]);
      if (c >= nc[k]) c = nc[k] - 1;
      ci[k] = c;
    }
    int ok = 1;
    int rx = nc[0] >= 3 ? 1 : 0, ry = nc[1] >= 3 ? 1 : 0, rz = nc[2] >= 3 ? 1 : 0;
    for (int dz = -rz; dz <= rz && ok; ++dz)
      for (int dy = -ry; dy <= ry && ok; ++dy)
        for (int dx = -rx; dx <= rx && ok; ++dx) {
          int cx = (ci[0] + dx + nc[0]) % nc[0], cy = (ci[1] + dy + nc[1]) % nc[1],
              cz = (ci[2] + dz + nc[2]) % nc[2];
          int64_t c = ((int64_t)cz * nc[1] + cy) * nc[0] + cx;
          for (int32_t a = head[c]; a >= 0; a = next[a]) {
            double ddx = gen_min_image(pos[3 * a] - x[0], box[0]);
            double ddy = gen_min_image(pos[3 * a + 1] - x[1], box[1]);
            double ddz = gen_min_image(pos[3 * a + 2] - x[2], box[2]);
            if (ddx * ddx + ddy * ddy + ddz * ddz < d2min) { ok = 0; break; }
          }
        }
    if (!ok) continue;
    int64_t c = ((int64_t)ci[2] * nc[1] + ci[1]) * nc[0] + ci[0];
    pos[3 * accepted] = x[0];
    pos[3 * accepted + 1] = x[1];
    pos[3 * accepted + 2] = x[2];
    next[accepted] = head[c];
    head[c] = (int32_t)accepted;
    ++accepted;
  }
  free(head);
  free(next);
  for (int64_t k = 0; k < n; ++k) type[k] = pattern[k % 29];
  /* charges after positions; neutralise with a Neumaier-compensated mean */
  double s = 0.0, comp = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    q[k] = sm64_u(&g) - 0.5;
    double t = s + q[k];
    if (fabs(s) >= fabs(q[k])) comp += (s - t) + q[k];
    else comp += (q[k] - t) + s;
    s = t;
  }
  double mean = n > 0 ? (s + comp) / (double)n : 0.0;
  for (int64_t k = 0; k < n; ++k) q[k] -= mean;
  return tries;
}

/* Synthetic C/H/N/O parameter table.
 * per_type: [ntypes][11] = r_sigma, r_pi, r_pipi, gamma, r_vdw, eps, alpha,
 *                          gamma_w, b131, b132, b133
 * per_pair: [ntypes][ntypes][7] = p_bo1..p_bo6, De (symmetric, filled both ways) */
void gen_params(uint64_t seed, int ntypes, double* per_type, double* per_pair) {
  static const double lo_t[11] = {0.9, 1.1, 1.0, 0.5, 1.5, 0.05, 9.0, 1.5, 2.0, 1.0, 0.5};
  static const double hi_t[11] = {1.5, 1.3, 1.2, 1.0, 2.1, 0.20, 12.0, 8.0, 10.0, 10.0, 10.0};
  static const double lo_p[7] = {-0.15, 5.0, -0.35, 5.0, -0.45, 10.0, 50.0};
  static const double hi_p[7] = {-0.05, 9.0, -0.10, 12.0, -0.20, 40.0, 150.0};
  sm64 g = {seed};
  for (int t = 0; t < ntypes; ++t)
    for (int k = 0; k < 11; ++k) per_type[t * 11 + k] = lo_t[k] + (hi_t[k] - lo_t[k]) * sm64_u(&g);
  for (int a = 0; a < ntypes; ++a)
    for (int b = a; b < ntypes; ++b)
      for (int k = 0; k < 7; ++k) {
        double v = lo_p[k] + (hi_p[k] - lo_p[k]) * sm64_u(&g);
        per_pair[(a * ntypes + b) * 7 + k] = v;
        per_pair[(b * ntypes + a) * 7 + k] = v;
      }
}

/* Bond-energy parameters (NEXT-1; reading 28),
 * drawn from their own seed so the table above is unchanged.
 * per_pair: [ntypes][ntypes][4] = De_pi, De_pipi, p_be1, p_be2 per type pair
 * t1 <= t2 (lexicographic), symmetric.  De_sigma is the table's De. */
void gen_bond_params(uint64_t seed, int ntypes, double* per_pair) {
  static const double lo[4] = {20.0, 10.0, -0.8, 0.2};
  static const double hi[4] = {100.0, 80.0, 0.5, 1.0};
  sm64 g = {seed};
  for (int a = 0; a < ntypes; ++a)
    for (int b = a; b < ntypes; ++b)
      for (int k = 0; k < 4; ++k) {
        double v = lo[k] + (hi[k] - lo[k]) * sm64_u(&g);
        per_pair[(a * ntypes + b) * 4 + k] = v;
        per_pair[(b * ntypes + a) * 4 + k] = v;
      }
}
