/* nclopf_mpcc.h — mpcc_check C-ABI (Eq. 6-11).
 *
 * The reference has no code for this module (SPEC only); these are the
 * operations SPEC names, over plain arrays: index_sets, recover_mpcc_multipliers
 * and certify_strong for the vertical complementarity form 0 <= w1 ⊥ w2 >= 0,
 * plus the SCOPF's complementarity pairs (the droop / PV-PQ recourse rows
 * w1 * w2 <= 0 of csrc/host/scopf.cpp) so a solver output can be certified.
 * Host functions (not on the per-iteration path). */
#ifndef NCLOPF_MPCC_H
#define NCLOPF_MPCC_H

#include <stdint.h>

#include "nclopf_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define NCL_MPCC_PLUS_ZERO 0 /* I+0: w1 > tol_act, w2 <= tol_act */
#define NCL_MPCC_ZERO_PLUS 1 /* I0+ */
#define NCL_MPCC_ZERO_ZERO 2 /* I00: both <= tol_act */

typedef struct ncl_mpcc_cert {
  int n_p0, n_0p, n_00;       /* index-set sizes */
  double grad_residual;       /* ||grad_w L^MPCC||_inf (caller-supplied) */
  double feas_residual;       /* feasibility residual (caller-supplied) */
  double comp_residual;       /* max_i |w1_i w2_i| */
  int inactive_violations;    /* |mu1| > tol on I+0 or |mu2| > tol on I0+ */
  int sign_violations;        /* mu1 or mu2 < -tol on I00 (Eq. 11) */
  int first_violation;        /* first violating pair or -1 */
  int strong;                 /* 1: strongly stationary, 0: weak / unclassified */
} ncl_mpcc_cert;

/* index_sets(w1, w2, tol_act): cls[p] in NCL_MPCC_*; a pair with both
 * components > tol_act is BothPositive: NCL_E_INVALID, its index in
 * *both_positive (else -1) */
int ncl_mpcc_index_sets(int p, const double* w1, const double* w2, double tol_act, int8_t* cls, int* both_positive);
/* mu1 = nu1 - nu0 o w2, mu2 = nu2 - nu0 o w1 */
int ncl_mpcc_recover(int p, const double* nu0, const double* nu1, const double* nu2, const double* w1,
                     const double* w2, double* mu1, double* mu2);
/* certify_strong; cls may be NULL */
int ncl_mpcc_certify(int p, const double* w1, const double* w2, const double* mu1, const double* mu2,
                     double grad_residual, double feas_residual, double tol, double tol_act, int8_t* cls,
                     ncl_mpcc_cert* out);
/* the SCOPF's pairs (ncl_scopf_info.ncomp of them): row of w1 * w2 <= 0,
 * variable of w1, variable x and bound of w2 = side * (x - bound) */
int ncl_scopf_comp_pairs(ncl_scopf_t S, int* rows, int* w1var, int* xvar, int* side, double* bound);

#ifdef __cplusplus
}
#endif
#endif
