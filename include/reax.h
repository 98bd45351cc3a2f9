/* libreax — C ABI of the B200-native ReaxFF list / bond-order / nonbonded hot path.
 *
 * The operations are the re-threaded ReaxC-OMP kernels of Aktulga et al.,
 * arXiv:1706.07772:
 *   reax_build_lists  "Write Lists" + bond part of "Init. Forces"
 *                     (§3.3; Table 2 rows PAPER.md:279-280)
 *   reax_bond_orders  "Bond Orders" (§3.3, 281)
 *   reax_nonbonded    "Non-Bonded Forces", Alg. 2
 *   reax_step         the three above, in order
 * Functional forms: SURVEY.md §8(c) B1-B8 / N1-N6 (the paper cites ReaxFF
 * refs [6,7], without stating equations; DESIGN.md lists every
 * reading taken).
 *
 * Conventions
 *   Units      A, e, kcal/mol, kcal/mol/A.  All arithmetic fp64.
 *   Memory     pointers marked [dev] are CUDA device memory owned by the caller
 *              (typically torch tensors); [host] are host memory.  Inputs are
 *              read-only and never retained past a call; outputs are
 *              overwritten, never accumulated.
 *   Workspace  the library never allocates device memory in a compute call.
 *              The caller allocates reax_workspace_bytes() bytes (e.g.
 *              torch.empty(bytes, dtype=uint8, device='cuda')) and binds it;
 *              the ctx only holds views into it (plus a few bytes of pinned
 *              host memory for status read-back, allocated by reax_create).
 *   Streams    every call is stream-ordered on `stream` (a cudaStream_t passed
 *              as void*; NULL = legacy default stream).  One ctx per stream;
 *              calls on different ctxs may run concurrently.
 *   Errors     argument / box / cutoff / parameter errors are detected on the
 *              host and returned before any launch.  Device-detected errors
 *              (non-finite input, type out of range, capacity overflow) are
 *              latched in a device status block: in synchronous mode (the
 *              default) reax_build_lists / reax_nonbonded / reax_step read it
 *              back once per call and return the error; in asynchronous mode
 *              (reax_set_async(ctx, 1), no host sync, CUDA-graph capturable)
 *              the caller collects them with reax_check().  No call aborts or
 *              prints.  After REAX_ERR_CAPACITY, reax_required() reports the
 *              capacities needed; rebind a larger workspace and retry.
 */
#ifndef REAX_H
#define REAX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  REAX_OK = 0,
  REAX_ERR_ARG = 1,       /* null pointer, n < 0, type out of range, size mismatch */
  REAX_ERR_BOX = 2,       /* a box length not finite or not > 2 r_nonb */
  REAX_ERR_CUTOFF = 3,    /* r_bond > r_nonb, r <= 0, or bo_cut not in (0,1) */
  REAX_ERR_PARAM = 4,     /* non-finite or out-of-domain parameter */
  REAX_ERR_CAPACITY = 5,  /* workspace too small; see reax_required().  Also, with
                             no regrow that clears it, when one home block's neighbour window
                             exceeds the per-CTA shared memory (~3x the PETN density) */
  REAX_ERR_NONFINITE = 6, /* NaN/Inf in positions, charges or computed energies */
  REAX_ERR_CUDA = 7,      /* a CUDA runtime error */
  REAX_ERR_STATE = 8,     /* call order / binding violated (no workspace, stale lists) */
  REAX_ERR_RANGE = 9      /* a pair force |dE/dr| or a row force component >= 65536 kcal/mol/A, or
                             one CTA's accumulated partial force on a window atom beyond 32768
                             kcal/mol/A: outside the fixed-point force accumulator (2^-35
                             resolution); results are then undefined */,
  REAX_ERR_CONVERGENCE = 10 /* QEq: a system not converged to tol within maxiter (results are the
                               last iterates) */
} reax_status;

#define REAX_MAX_TYPES 16

/* r_nonb: nonbonded cutoff (10 A); r_bond: bond cutoff (5 A); bo_cut: bond
 * order cut (0.01) — BASELINE.json north_star. */
typedef struct {
  double r_nonb, r_bond, bo_cut;
} reax_cutoffs;

/* Force-field parameter table (all [host], read during the call only).
 * Per type, length ntypes: r_sigma, r_pi, r_pipi (bond radii, A), gamma
 * (Coulomb shielding, 1/A), r_vdw (A), eps (kcal/mol), alpha, gamma_w (vdW
 * shielding, 1/A), b131/b132/b133 (over-coordination correction: p_boc4 =
 * sqrt(b131_i b131_j), p_boc3 = sqrt(b132_i b132_j), p_boc5 = sqrt(b133_i b133_j)),
 * val, val_boc (valences).  Per type pair, ntypes*ntypes row-major and
 * symmetric: p_bo1..p_bo6 (bond-order exponents), De (bond energy; unused on
 * this path, validated only).  Globals: p_boc1, p_boc2 (f2/f3), p_vdw1 (vdW
 * shielding power), coulomb_c (332.0638 kcal A/(mol e^2)).  Combining rules:
 * DESIGN.md reading 9. */
typedef struct {
  int32_t ntypes;
  const double *r_sigma, *r_pi, *r_pipi, *gamma, *r_vdw, *eps, *alpha, *gamma_w, *b131, *b132,
      *b133, *val, *val_boc;
  const double *p_bo1, *p_bo2, *p_bo3, *p_bo4, *p_bo5, *p_bo6, *De;
  double p_boc1, p_boc2, p_vdw1, coulomb_c;
} reax_params;

/* Bond-energy parameters (NEXT-1), per type pair [host],
 * ntypes*ntypes row-major, symmetric: De_pi, De_pipi (kcal/mol), p_be1,
 * p_be2 (> 0).  De_sigma is reax_params.De.  DESIGN.md reading 28. */
typedef struct {
  const double *De_pi, *De_pipi, *p_be1, *p_be2;
} reax_bond_params;

typedef struct reax_ctx reax_ctx;

/* Capacities of a bound workspace.  Zero fields mean "library default". */
typedef struct {
  int32_t row_cap;    /* max half-list entries per atom row (default from density) */
  int32_t cand_cap;   /* max bond candidates per atom (default 16) */
  int64_t bond_cap;   /* max full bond-list entries (default 8 n) */
  int32_t window_cap; /* max atoms in one home block's neighbour window (default 2048) */
} reax_capacity;

/* Text of the CUDA error behind the last REAX_ERR_CUDA returned on this host
 * thread ("no error" if none).  Static storage; never NULL. */
const char* reax_last_cuda_error(void);

const char* reax_status_str(reax_status s);

reax_status reax_create(reax_ctx** out);
reax_status reax_destroy(reax_ctx* ctx);

/* Workspace size for n atoms in `box` [host, 3] with `cut` and `cap` (NULL or
 * zero fields = defaults).  *bytes receives the size; *cap_out (optional)
 * the resolved capacities. */
reax_status reax_workspace_bytes(int64_t n, const double box[3], const reax_cutoffs* cut,
                                 const reax_capacity* cap, size_t* bytes, reax_capacity* cap_out);
/* Bind `ws` [dev] of `bytes` bytes for (n, box, cut, cap).  Later calls must
 * use the same n and a box giving the same cell grid, else REAX_ERR_STATE. */
reax_status reax_bind_workspace(reax_ctx* ctx, void* ws, size_t bytes, int64_t n,
                                const double box[3], const reax_cutoffs* cut,
                                const reax_capacity* cap);
/* After REAX_ERR_CAPACITY: the capacities that would have sufficed. */
reax_status reax_required(const reax_ctx* ctx, reax_capacity* need);

/* a1-a4: validate, wrap x <- x - L floor(x/L), counting-sort the atoms into
 * cells of side >= r_nonb/2, build the half neighbour list (every pair with
 * minimum-image r^2 <= r_nonb^2 exactly once; FMA-free fp64 decision) and the
 * bond candidates, then the FULL bond list with BO'sigma/pi/pipi (B1-B2;
 * bond iff BO' >= bo_cut and r <= r_bond) and mirror indices.
 * pos [dev] n*3 fp64 row-major; type [dev] n int32 in [0, ntypes). */
reax_status reax_build_lists(reax_ctx* ctx, int64_t n, const double* pos, const int32_t* type,
                             const double box[3], const reax_params* params,
                             const reax_cutoffs* cut, void* stream);

/* a5-a6: Delta'_i = sum_j BO'_ij - Val_i (B3) and corrected bond orders
 * BO, BOsigma, BOpi, BOpipi via f1, f4, f5 (B4-B8), bitwise symmetric.
 * Precondition: reax_build_lists on this ctx. */
reax_status reax_bond_orders(reax_ctx* ctx, const reax_params* params, const reax_cutoffs* cut,
                             void* stream);

/* NEXT-1: bond energy and its forces — the bond part of "Aggregate Forces"
 * (§3.3, Table 2 row PAPER.md:285).  Per bond of the current
 * bond list (each unordered bond once), from the corrected bond orders of a6
 * (standard ReaxFF form, reading 28):
 *   E1  e = -De_s BOs exp[p_be1 (1 - BOs^p_be2)] - De_pi BOpi - De_pipi BOpipi
 * (BOs^p_be2 := 0 for BOs <= 0).  Forces F = -dE_bond/dx at the fixed bond
 * set, through the bond-order derivatives: every bond order depends on its
 * r (B1) and on Delta'_i, Delta'_j (f1, f4, f5, B4-B7), so each bond carries a
 * central force (dE/dr_b)/r_b d with dE/dr_b = de_b/dr_b|_Delta +
 * (D_i + D_j) dBO'_b/dr_b, D_i = sum over i's bonds of de/dDelta'_i.
 * Precondition: reax_bond_orders (or reax_step) on this ctx; the parameters
 * must be those of that build.  force [dev] n*3 fp64 (overwritten, input
 * order); energy [dev] 1 fp64 {E_bond} (overwritten).  REAX_ERR_PARAM for a
 * non-finite or asymmetric table or p_be2 <= 0. */
reax_status reax_bond_energy(reax_ctx* ctx, const reax_params* params, const reax_bond_params* bond_params,
                             double* force, double* energy, void* stream);

/* NEXT-3: interaction lists of the current bond list and
 * positions — the valence-angle (3-body) list and the hydrogen-bond list
 * (§3.3: "we first identify which angles are
 * present ... a per-atom prefix sum is computed ... then computed and stored
 * using the global array offsets").  Readings:
 *   angles   for every entry e = (j, i) of the exported full bond list
 *            (reax_export_bonds order), the partners k of the other entries
 *            f = (j, k) of row j with BO_e > thb_cut, BO_f > thb_cut and
 *            BO_e BO_f > thb_cutsq (corrected total BO), in row order;
 *   H-bonds  for every atom i of type h_type with at least one bond, the atoms
 *            z != i whose type t has bit t set in acceptor_mask and whose
 *            minimum-image distance is <= r_hb (exact fp64 test), ascending.
 * Defaults (LAMMPS ReaxFF style): thb_cut 0.001, thb_cutsq 0.00001, r_hb
 * 7.5 A, H = type 1, acceptors N, O = types 2, 3.  r_hb must be <= 2 sub-cell
 * sides (>= r_nonb) and < L/2 (REAX_ERR_CUTOFF). */
typedef struct {
  double thb_cut, thb_cutsq, r_hb;
  int32_t h_type;
  uint32_t acceptor_mask;
} reax_ilist_params;

/* List sizes (synchronises): n_angles 3-body entries, n_hbonds H-bond entries.
 * Precondition: reax_bond_orders (or reax_step) on this ctx. */
reax_status reax_interaction_counts(reax_ctx* ctx, const reax_ilist_params* params, int64_t* n_angles,
                                    int64_t* n_hbonds, void* stream);
/* The lists as CSR in input order (synchronises): ang_off [dev] B+1 int64 over
 * the exported bond entries, ang_k [dev] n_angles int32 (partner k), hb_off
 * [dev] n+1 int64 over the atoms, hb_z [dev] n_hbonds int32 (acceptor z).
 * ang_k / hb_z may be NULL (offsets only).  REAX_ERR_CAPACITY if one H atom has
 * more than 1024 H-bond partners. */
reax_status reax_interaction_lists(reax_ctx* ctx, const reax_ilist_params* params, int64_t* ang_off, int32_t* ang_k,
                                   int64_t* hb_off, int32_t* hb_z, void* stream);

/* NEXT-2: QEq charge equilibration, PAPER.md:204-208 (§3.3
 * "QEq"; reading 33).  The charges minimise
 *   E(q) = sum_i (chi_i q_i + 1/2 eta_i q_i^2) + sum_{i<j} H_ij q_i q_j,  sum_i q_i = 0,
 * i.e. H s = -chi, H t = -1 ("two linear systems ... with a common kernel H"),
 * q = s - (sum s / sum t) t, with H_ii = eta_i and H_ij = C Tap(r_ij)
 * (r_ij^3 + gamma_ij^-3)^(-1/3) for the pairs of the current half list (the
 * shielded Coulomb kernel of the nonbonded term without charges; positions
 * and parameters of the last reax_build_lists / reax_step).
 *  - reax_qeq_bytes: scratch bytes for the current list ([dev] caller-owned,
 *    256-byte aligned); synchronises `stream`.
 *  - reax_qeq_build: computes every unique H_ij once from the half list and
 *    stores it in scratch (both row segments, sorted: deterministic).  The
 *    scratch then belongs to this list: a new build of the lists (or another
 *    scratch pointer) makes the solves return REAX_ERR_STATE.
 *  - reax_qeq_matvec: y = H x for two vectors ([dev] n fp64 each, input
 *    order); eta [host] ntypes.
 *  - reax_qeq_solve: Jacobi-preconditioned CG on both systems at once (one
 *    pass over H per iteration serves both right-hand sides), each to
 *    ||b - H x|| <= tol ||b|| (the paper's runs: tol = 1e-6) or
 *    maxiter iterations.  chi, eta [host] ntypes (eta > 0); s, t [dev] n fp64
 *    in/out: initial guesses in (zeros, or an extrapolation of earlier
 *    solutions), solutions out; q [dev] n fp64 out; iters [host]
 *    2 (iterations of the s and t systems).  REAX_ERR_CONVERGENCE if either
 *    system is not converged after maxiter.  Synchronous on `stream`;
 *    deterministic (fixed summation order everywhere). */
reax_status reax_qeq_bytes(reax_ctx* ctx, size_t* bytes, void* stream);
reax_status reax_qeq_build(reax_ctx* ctx, void* scratch, size_t scratch_bytes, void* stream);
reax_status reax_qeq_matvec(reax_ctx* ctx, const double* eta, void* scratch, size_t scratch_bytes, const double* x_s,
                            const double* x_t, double* y_s, double* y_t, void* stream);
reax_status reax_qeq_solve(reax_ctx* ctx, const double* chi, const double* eta, double tol, int32_t maxiter,
                           void* scratch, size_t scratch_bytes, double* s, double* t, double* q, int32_t* iters,
                           void* stream);

/* NEXT-4: in situ molecular species analysis of the
 * corrected bond orders of the last reax_bond_orders / reax_step
 * (§3.4 "A Tool for Molecular Species Analysis"):
 *   - atoms i, j are bonded iff BO_ij > bo_threshold[t_i * nt + t_j] (strict;
 *     bo_threshold [host] nt*nt symmetric, or NULL for the paper's default 0.3);
 *   - the molecule ID of an atom is the smallest global ID (0-based input
 *     index) of its connected component ("the smaller value of the two global
 *     IDs ... repeated until every atom has been assigned a molecule ID");
 *   - molecule IDs are sorted and renumbered 1..M: mol_id [dev] n int32, input
 *     order; *n_molecules = M;
 *   - species = molecules with the same number of atoms per element (type):
 *     species_comp [host] species_cap*nt int32 (atoms of each type),
 *     species_count [host] species_cap int64 (molecules), sorted by the
 *     composition vector ascending; *n_species = the number of species
 *     (REAX_ERR_CAPACITY, with *n_species set, if it exceeds species_cap).
 * scratch [dev] is caller-owned, >= reax_species_bytes(n, nt), 256-byte
 * aligned (REAX_ERR_CAPACITY if smaller).  Synchronous on `stream`.
 * REAX_ERR_STATE without a current bond list. */
reax_status reax_species_bytes(int64_t n, int32_t ntypes, size_t* bytes);
reax_status reax_species(reax_ctx* ctx, const double* bo_threshold, void* scratch, size_t scratch_bytes,
                         int32_t* mol_id, int64_t* n_molecules, int32_t* species_comp, int64_t* species_count,
                         int64_t species_cap, int64_t* n_species, void* stream);

/* a7-a8: Alg. 2 over the half list: tapered shielded vdW + Coulomb (N1-N6)
 * at the given charges.  q [dev] n fp64; force [dev] n*3 fp64 (overwritten,
 * input order, F = -dE/dx); energy [dev] 2 fp64 {E_vdW, E_Coul}
 * (overwritten).  pos/type/box must be those of the last reax_build_lists. */
reax_status reax_nonbonded(reax_ctx* ctx, int64_t n, const double* pos, const int32_t* type,
                           const double* q, const double box[3], const reax_params* params,
                           const reax_cutoffs* cut, double* force, double* energy, void* stream);

/* reax_build_lists + reax_bond_orders + reax_nonbonded. */
reax_status reax_step(reax_ctx* ctx, int64_t n, const double* pos, const int32_t* type,
                      const double* q, const double box[3], const reax_params* params,
                      const reax_cutoffs* cut, double* force, double* energy, void* stream);

/* reax_step with HOST buffers: pos/type/q [host], force [host] n*3,
 * energy [host] 2.  Copies in, runs the step, copies out and synchronises
 * `stream`.  Host buffers should be pinned for full copy bandwidth.  The
 * input copies run on a context-owned copy stream in the order positions,
 * types, charges; the step waits for each array only where it first needs
 * it (binning: positions; cell gather: types; nonbonded kernel: charges), so
 * the type and charge copies overlap the binning and the list build.  The
 * host buffers must stay unchanged until the call returns.  The whole
 * sequence is captured into a CUDA graph and replayed while the buffers,
 * box and parameters stay the same. */
reax_status reax_step_host(reax_ctx* ctx, int64_t n, const double* pos, const int32_t* type,
                           const double* q, const double box[3], const reax_params* params,
                           const reax_cutoffs* cut, double* force, double* energy, void* stream);

/* Asynchronous mode: no host synchronisation inside compute calls (CUDA-graph
 * capturable); device errors are collected by reax_check(). */
reax_status reax_set_async(reax_ctx* ctx, int enable);
/* Synchronise `stream` and return the first latched device error (or OK). */
reax_status reax_check(reax_ctx* ctx, void* stream);

/* Per-kernel timing with CUDA events on `stream` (off by default).
 * groups: 0 "bin" (wrap + counting sort), 1 "nbr" (k_nbr_build), 2 "bonds"
 * (bond evaluation, scan, fill, row sort + Delta'), 3 "bond_orders"
 * (k_bond_correct), 4 "nonbonded" (k_nonbonded alone), 5 "other" (work plan, charge
 * gather, force un-permute, energy reduction), 6 "bond_energy" (NEXT-1,
 * reax_bond_energy), 7 "species" (NEXT-4, reax_species), 8 "qeq" (NEXT-2,
 * reax_qeq). */
#define REAX_NKERNELS 9
reax_status reax_set_timing(reax_ctx* ctx, int enable);
/* Accumulated milliseconds and launch counts per kernel group since the last
 * reset (synchronises the last recorded events).  reset = 0: accumulate and
 * keep; 1: return and clear; 2 (peek): return the times of the currently
 * recorded events without consuming them, for CUDA-graph replays (events
 * captured in a graph are external event nodes re-recorded by each replay). */
reax_status reax_kernel_ms(reax_ctx* ctx, double ms[REAX_NKERNELS], int64_t launches[REAX_NKERNELS],
                           int reset);
/* Number of device kernels launched by the last reax_step. */
int32_t reax_launches_per_step(const reax_ctx* ctx);

/* Diagnostics: evaluates the nonbonded kernel's fp64 device math on x [dev] n:
 * out [dev] n*5 = {exp(x), ln x, x^-1/2, 1/x, x^-1/3} (the last four for x > 0,
 * else 0).  Synchronises.  Used by the tests to bound their error. */
reax_status reax_selftest_math(reax_ctx* ctx, int64_t n, const double* x, double* out,
                               const reax_params* params, const reax_cutoffs* cut, void* stream);

/* ------------------------------------------------------------------ export
 * Outside the hot path; canonical, original-index form.  Synchronise. */
reax_status reax_pair_count(reax_ctx* ctx, int64_t* n_half_pairs, int64_t* n_bond_entries,
                            void* stream);
/* All half-list pairs as (i, j) original indices, i < j, unordered rows:
 * pi/pj [dev] n_half_pairs int32 each. */
reax_status reax_export_pairs(reax_ctx* ctx, int32_t* pi, int32_t* pj, void* stream);
/* Per atom (original index): number of pairs it belongs to, and the sum
 * mod 2^64 of mix64(min, max) over them. cnt/dig [dev] n. */
reax_status reax_export_nbr_digest(reax_ctx* ctx, int64_t* cnt, uint64_t* dig, void* stream);
/* Full bond list in original order: brow [dev] n+1 int64 (CSR), bcol [dev] B
 * int32 (rows sorted by partner), mirror [dev] B int32 (entry of the reverse
 * bond), bo [dev] B*8 fp64 {BO'sigma, BO'pi, BO'pipi, BO', BO, BOsigma, BOpi,
 * BOpipi}, delta [dev] n*2 fp64 {Delta', Delta'boc}.  Any pointer may be NULL. */
reax_status reax_export_bonds(reax_ctx* ctx, int64_t* brow, int32_t* bcol, int32_t* mirror,
                              double* bo, double* delta, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* REAX_H */
