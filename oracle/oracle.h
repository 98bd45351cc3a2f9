/* CPU oracle — test infrastructure only (see oracle.c header).
 * Own header: shares nothing with include/reax.h or the CUDA library. */
#ifndef REAX_ORACLE_H
#define REAX_ORACLE_H
#include <stdint.h>

typedef struct {
  int32_t ntypes;
  /* per type [ntypes] */
  const double *r_sigma, *r_pi, *r_pipi, *gamma, *r_vdw, *eps, *alpha, *gamma_w, *b131, *b132,
      *b133, *val, *val_boc;
  /* per type pair [ntypes*ntypes], symmetric */
  const double *p_bo1, *p_bo2, *p_bo3, *p_bo4, *p_bo5, *p_bo6;
  double p_boc1, p_boc2, p_vdw1, coulomb_c;
} orc_params;

/* Bond-energy parameters (NEXT-1), per type pair [ntypes*ntypes], symmetric. */
typedef struct {
  const double *De_s, *De_p, *De_pp, *p_be1, *p_be2;
} orc_bond_params;

#endif
