// mpcc_check: classification of MPCC points of the vertical
// complementarity form 0 <= w1 ⊥ w2 >= 0 (Eq. 6-11): active index
// sets, recovery of the MPCC multipliers from the NLP multipliers of the
// relaxed form (bounds w1, w2 >= 0 with nu1, nu2; bilinear rows w1 o w2 <= 0
// with nu0), and the strong-stationarity certificate of Eq. 11. Host code:
// pure functions over the solver's output, not on the per-iteration path.
#pragma once

#include <cstdint>
#include <vector>

namespace nclb::mpcc {

enum Cls : int8_t { kPlusZero = 0, kZeroPlus = 1, kZeroZero = 2 };

// index_sets: I+0 iff w1 > tol and w2 <= tol, I0+
// symmetric, both small -> I00. Returns the first index with both
// components > tol (BothPositive), or -1.
int index_sets(int p, const double* w1, const double* w2, double tol_act, int8_t* cls);

// recover_mpcc_multipliers: mu1 = nu1 - nu0 o w2,
// mu2 = nu2 - nu0 o w1 (lambda, xi pass through)
void recover(int p, const double* nu0, const double* nu1, const double* nu2, const double* w1, const double* w2,
             double* mu1, double* mu2);

struct Certificate {
  int n_p0 = 0, n_0p = 0, n_00 = 0;
  double grad_residual = 0.0;  // ||grad_w L^MPCC||_inf (the caller's, = the NLP's by the recovery identity)
  double feas_residual = 0.0;
  double comp_residual = 0.0;  // max_i |w1_i w2_i|
  int inactive_violations = 0; // |mu1| > tol on I+0, |mu2| > tol on I0+
  int sign_violations = 0;     // mu1 or mu2 < -tol on I00
  int first_violation = -1;
  bool strong = false;
};

// certify_strong
Certificate certify(int p, const double* w1, const double* w2, const double* mu1, const double* mu2,
                    double grad_residual, double feas_residual, double tol, double tol_act, int8_t* cls);

}  // namespace nclb::mpcc
