// Shared device/host definitions of libreax (B200, sm_100a).
// Product code: independent of oracle/ (no shared code, tables or constants).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rx {

// ----------------------------------------------------------------- geometry
// Atoms are counting-sorted into sub-cells of side h >= r_nonb/2 (x fastest).
// A pair within r_nonb is then at most SR = 2 sub-cells apart per axis.  Work
// is organised in home blocks of HB^3 sub-cells; a home block's "window" is
// the union of the half stencils (forward 62 offsets + own cell) of its
// sub-cells, inside a WB^3 box of sub-cells.
constexpr int SR = 2;
constexpr int HB = 2;
constexpr int WB = HB + 2 * SR;   // 6
constexpr int NWB = WB * WB * WB; // 216
constexpr int NHOME = HB * HB * HB;
constexpr int MAX_RUNS = 16;
constexpr int NWU_MAX = 136;   // used window cells (130 for HB = 2, SR = 2; checked at table build)
constexpr int NMW = (NWB + 31) / 32;  // mask words over used window cells
constexpr int NT_MAX = 16;
constexpr int NTP_MAX = NT_MAX * NT_MAX;

struct WindowTables {
  int nwu;                       // used window cells
  int wu[NWB];                   // used-list index -> window-box index (wx + WB*(wy + WB*wz))
  int widx[NWB];                 // window-box index -> used-list index, -1 if unused
  int home_k[NHOME];             // used-list index of each home sub-cell (h = hx + HB*(hy + HB*hz))
  int nrun[NHOME];               // forward runs of home sub-cell h (own cell excluded)
  int run_a[NHOME][MAX_RUNS];    // first used-list index of the run
  int run_b[NHOME][MAX_RUNS];    // last used-list index of the run (inclusive)
  int nrun1[NHOME];              // un-merged forward runs (one per (oy, oz)) of home sub-cell h
  int run1_a[NHOME][MAX_RUNS];
  int run1_b[NHOME][MAX_RUNS];
  unsigned mask[NHOME][NMW];     // bit k: used cell k is in home sub-cell h's half stencil or is h itself
};

struct Grid {
  int nc[3];      // sub-cells per axis
  int nb[3];      // home blocks per axis
  int ncell;      // nc0*nc1*nc2
  int nblock;     // nb0*nb1*nb2
  double L[3];    // box
  double h[3];    // sub-cell side
  double inv_h[3];
};

// ------------------------------------------------------------- parameters
struct NBPair {      // nonbonded constants per type pair (N2-N5)
  double D;          // sqrt(eps_i eps_j)
  double ahalf;      // alpha_ij / 2
  double Dadr;       // D alpha_ij / r_vdW,ij
  double inv_rvdw;   // 1 / r_vdW,ij, r_vdW,ij = 2 sqrt(r_vdw_i r_vdw_j)
  double gwmp;       // gamma_w,ij^(-p_vdW1)
  double g3;         // gamma_ij^(-3)
};

struct BOPair {      // bond-order constants per type pair (B1, B7)
  double lr0[3];     // log r0_sigma, log r0_pi, log r0_pipi  (r0 = (r_i + r_j)/2)
  double pa[3];      // p_bo1, p_bo3, p_bo5
  double pb[3];      // p_bo2, p_bo4, p_bo6
  double pboc3, pboc4, pboc5;
};

struct BEPair {      // bond-energy constants per type pair (NEXT-1, E1)
  double Ds, Dp, Dpp;  // De_sigma (reax_params.De), De_pi, De_pipi
  double pbe1, pbe2;
};

struct DevParams {
  int nt;
  double R, R2, rb2, bo_cut;
  double p_vdw, inv_p, invR, C;
  double p_boc1, p_boc2;
  float R2lo, R2hi;          // fp32 classification band around R^2
  float rcand2[NTP_MAX];     // fp32 bond-candidate radius^2 (conservative)
  float rcand2_max;
  double val[NT_MAX], val_boc[NT_MAX];
  alignas(16) NBPair nb[NTP_MAX];   // 16-byte aligned: the nonbonded kernel copies these with cp.async
  BOPair bo[NTP_MAX];
  alignas(16) double exp_tbl[256];       // 2^(j/256)
  alignas(16) double log_tbl[2 * 256];   // {1/c_j rounded, -log(that value)}, c_j = 1 + (j + 1/2)/256
};

// ------------------------------------------------------------------ status
enum : int {
  ST_NONFINITE_IN = 1,
  ST_TYPE = 2,
  ST_ROW_OVF = 4,
  ST_CAND_OVF = 8,
  ST_BOND_OVF = 16,
  ST_WIN_OVF = 32,
  ST_NONFINITE_OUT = 64,
  ST_RANGE = 128,           // a force contribution outside the fixed-point range
  ST_HB_OVF = 512,          // an H atom's H-bond list beyond HB_CAP entries
  ST_QEQ_UNSORTED = 1024,   // a QEq lower segment too long to sort (results stay correct, not reproducible)
};

struct Status {
  int flags;
  int max_row;      // longest half-list row seen
  int max_cand;     // most bond candidates of one atom
  int max_window;   // largest window
  long long bonds;  // full bond entries
  long long pairs;  // half-list pairs (filled by reax_pair_count)
  int pad[8];
};

// ----------------------------------------------------- workspace views
struct WS {
  int* cell_cnt;     // ncell + 1
  int* cell_start;   // ncell + 1
  int* cell_of;      // n
  int* perm;         // n   sorted -> original
  int* iperm;        // n   original -> sorted
  double4* spos;     // n   wrapped x, y, z; w = q (set by the nonbonded prep)
  float4* sloc;      // n   fp32 coordinates relative to the own sub-cell origin; w = type bits
  int* stype;        // n
  uint16_t* nbr;     // n * row_cap   half list: window slots
  int* nbr_len;      // n
  int* wpack;        // nblock * WPACK_INTS: each home block's window as the list build made it
  int2* wsinfo;      // nblock * window_cap: its slot info {sorted atom, window cell | type << 8}
  int* bc;           // n * cand_cap  bond candidates (sorted j), then kept half bonds
  int* bc_len;       // n
  double4* bc_raw;   // n * cand_cap  BO'sigma, BO'pi, BO'pipi, BO' of kept half bonds
  int* bdeg;         // n + 1
  int* brow;         // n + 1
  int* bcol;         // bond_cap  partner (sorted index)
  int* bkey;         // bond_cap  partner (original index): the row sort key
  int* bown;         // bond_cap  row owner (sorted index)
  int* bmir;         // bond_cap
  double* bo;        // 8 arrays of bond_cap: BO'sigma, BO'pi, BO'pipi, BO', BO, BOsigma, BOpi, BOpipi (entry e of array k at k * bond_cap + e)
  double2* delta;    // n
  unsigned long long* sf;    // 3n: sorted-order forces {x, y, z} per atom (one 24-byte record),
                             //     int64 fixed point (2^-35 kcal/mol/A)
  double2* erow;     // n   per-row (E_vdW, E_Coul)
  double* epart;     // energy reduction partials
  unsigned* ticket;  // last-block counter of the energy reduction
  int* ucol;         // bond_cap  unsorted full-list entries (fill order)
  int* ukey;         // bond_cap
  int* uown;         // bond_cap
  double4* uraw;     // bond_cap: first 8 bytes per entry = its candidate index (fill -> rank)
  long long* scan_tmp;  // scan partials
  long long* exp_off;   // n + 1 (export scratch)
  unsigned long long* lb_status;  // look-back scan tile status
  unsigned* lb_ticket;            // look-back scan tile ticket
  unsigned* bin_ticket;           // k_bin last-block ticket (fused cell scan)
  int* blk_pairs;    // nblock  half-list entries per home block (list build; nonbonded plan)
  int* blkrow;       // nblock  shared row counters of split home blocks
  int* units;        // NB_UNIT_SPLIT * nblock  planned nonbonded units (block | n_b << 24)
  int* nunits;       // 4       [0]: planned unit count
  unsigned long long* ilist_tot;  // 2: interaction-list totals (reax_interaction_counts)
  DevParams* prm;
  Status* st;
  double* h_pos;     // staging for reax_step_host
  int* h_type;
  double* h_q;
  double* h_force;
  double* h_energy;  // 2
  // NEXT-1 bond energy (reax_bond_energy)
  BEPair* bep;       // NTP_MAX
  double* bD;        // n   D_i = sum over the row's bonds of de/dS_i
  double4* bde;      // bond_cap per entry {de/dr|S, dBO'/dr, e, de/dS_owner}: aliases uraw (dead after the bond fill)
};

}  // namespace rx
