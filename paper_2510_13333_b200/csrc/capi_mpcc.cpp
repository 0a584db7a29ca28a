// mpcc_check C-ABI (include/nclopf_mpcc.h); host code.
#include <algorithm>
#include <string>

#include "../../include/nclopf_mpcc.h"
#include "capi_internal.hpp"
#include "host/mpcc.hpp"
#include "host/scopf.hpp"

using namespace nclb;

#define API extern "C" __attribute__((visibility("default")))
#define GUARD(...)    \
  try {               \
    __VA_ARGS__;      \
  } catch (...) {     \
    return map_exc(); \
  }                   \
  return NCL_OK;

API int ncl_mpcc_index_sets(int p, const double* w1, const double* w2, double tol_act, int8_t* cls,
                            int* both_positive) {
  GUARD({
    const int bad = mpcc::index_sets(p, w1, w2, tol_act, cls);
    if (both_positive) *both_positive = bad;
    if (bad >= 0) throw Error{NCL_E_INVALID, "mpcc index_sets: BothPositive(" + std::to_string(bad) + ")"};
  });
}
API int ncl_mpcc_recover(int p, const double* nu0, const double* nu1, const double* nu2, const double* w1,
                         const double* w2, double* mu1, double* mu2) {
  GUARD(mpcc::recover(p, nu0, nu1, nu2, w1, w2, mu1, mu2));
}
API int ncl_mpcc_certify(int p, const double* w1, const double* w2, const double* mu1, const double* mu2,
                         double grad_residual, double feas_residual, double tol, double tol_act, int8_t* cls,
                         ncl_mpcc_cert* out) {
  GUARD({
    const mpcc::Certificate C = mpcc::certify(p, w1, w2, mu1, mu2, grad_residual, feas_residual, tol, tol_act, cls);
    out->n_p0 = C.n_p0;
    out->n_0p = C.n_0p;
    out->n_00 = C.n_00;
    out->grad_residual = C.grad_residual;
    out->feas_residual = C.feas_residual;
    out->comp_residual = C.comp_residual;
    out->inactive_violations = C.inactive_violations;
    out->sign_violations = C.sign_violations;
    out->first_violation = C.first_violation;
    out->strong = C.strong ? 1 : 0;
  });
}
