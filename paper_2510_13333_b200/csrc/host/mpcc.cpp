// mpcc_check; see mpcc.hpp.
#include "host/mpcc.hpp"

#include <algorithm>
#include <cmath>

namespace nclb::mpcc {

int index_sets(int p, const double* w1, const double* w2, double tol_act, int8_t* cls) {
  int bad = -1;
  for (int i = 0; i < p; ++i) {
    const bool a = w1[i] > tol_act, b = w2[i] > tol_act;
    if (a && b) {
      if (bad < 0) bad = i;
      cls[i] = kZeroZero;  // unclassifiable; reported through `bad`
    } else if (a) {
      cls[i] = kPlusZero;
    } else if (b) {
      cls[i] = kZeroPlus;
    } else {
      cls[i] = kZeroZero;
    }
  }
  return bad;
}

void recover(int p, const double* nu0, const double* nu1, const double* nu2, const double* w1, const double* w2,
             double* mu1, double* mu2) {
  for (int i = 0; i < p; ++i) {
    mu1[i] = nu1[i] - nu0[i] * w2[i];
    mu2[i] = nu2[i] - nu0[i] * w1[i];
  }
}

Certificate certify(int p, const double* w1, const double* w2, const double* mu1, const double* mu2,
                    double grad_residual, double feas_residual, double tol, double tol_act, int8_t* cls) {
  Certificate C;
  C.grad_residual = grad_residual;
  C.feas_residual = feas_residual;
  std::vector<int8_t> own;
  if (!cls) {
    own.resize(p);
    cls = own.data();
  }
  const int bad = index_sets(p, w1, w2, tol_act, cls);
  for (int i = 0; i < p; ++i) {
    C.comp_residual = std::max(C.comp_residual, std::fabs(w1[i] * w2[i]));
    bool viol = false;
    switch (cls[i]) {
      case kPlusZero:
        ++C.n_p0;
        if (std::fabs(mu1[i]) > tol) ++C.inactive_violations, viol = true;  // w1 > 0: its bound is inactive
        break;
      case kZeroPlus:
        ++C.n_0p;
        if (std::fabs(mu2[i]) > tol) ++C.inactive_violations, viol = true;
        break;
      default:
        ++C.n_00;
        if (mu1[i] < -tol || mu2[i] < -tol) ++C.sign_violations, viol = true;  // Eq. 11 sign rule on I00
    }
    if (viol && C.first_violation < 0) C.first_violation = i;
  }
  C.strong = bad < 0 && feas_residual <= tol && grad_residual <= tol && C.inactive_violations == 0 &&
             C.sign_violations == 0;
  return C;
}

}  // namespace nclb::mpcc
