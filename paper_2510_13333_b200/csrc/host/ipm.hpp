// Host C++ control flow of the NCL outer loop and the interior-point inner
// loop. Written ONCE against an abstract
// backend that owns every vector: the product binds it to the B200 backend
// (csrc/capi_ipm.cpp: device-resident state, sm_100a kernels, scalars-only
// host traffic); the oracle binds the very same source to the reference CPU
// sparse_core/model_ad (oracle/ref_ipm.cpp). Branch decisions therefore
// differ only through the numbers the backends return.
#pragma once

#include <chrono>
#include <cstdint>
#include <string>
#include <vector>

#include "../../../include/nclopf_ipm.h"
#include "ipm_elem.hpp"

namespace nclb::ipm {

struct KktErr {
  double du = 0, pr = 0, dur = 0, cmu = 0, c0 = 0, ysum = 0, zsum = 0;
};
struct FactorOut {
  int status = 0;  // 0 ok, 1 zero pivot
  int npos = 0, nneg = 0, nzero = 0;
};
struct SolveOut {
  double residual = 0;
  int sweeps = 0;
  bool converged = true;
};
struct Merit {
  double theta = 0, phi = 0;
  bool valid = true;
};

// Everything vector-sized lives behind this interface. Every method returns
// only scalars (the C-ABI contract of SURVEY.md §3: w, λ, ν, J, H, K, L, D stay
// on the device). Methods are called in the order documented in ipm.cpp.
class Backend {
 public:
  virtual ~Backend() = default;
  virtual int n() const = 0;
  virtual int m() const = 0;
  virtual int num_bound_duals() const = 0;  // finite bounds on x and on inequality slacks
  // project x0, evaluate f, c, grad at x; s, r, y, duals; returns f and max|grad f|
  virtual void init_point(const Scal& S, double* f, double* gmax) = 0;
  // grad, J, H(sf, y) at x; jty = J'y
  virtual void eval_derivatives(double sf) = 0;
  virtual KktErr kkt_error(const Scal& S) = 0;
  virtual double hess_absmax() = 0;
  virtual void form_newton(const Scal& S) = 0;                   // sigx, gx, D, q, Dq
  virtual FactorOut factor(double dw, double pivot_tol) = 0;     // K assembly + LDL^T
  virtual SolveOut solve(const Scal& S, double target, int max_sweeps) = 0;  // rhs, solve, recovery
  virtual void max_steps(const Scal& S, double* apri, double* adual) = 0;
  virtual double dphi(const Scal& S) = 0;
  virtual Merit merit_current(const Scal& S) = 0;
  virtual Merit trial(const Scal& S) = 0;  // xt = x + alpha dx ...; f, c at xt
  virtual void accept(const Scal& S) = 0;
  virtual void restore() = 0;
  virtual void r_inf(double* rinf, double* dxinf, double* xinf) = 0;
  virtual double update_multipliers() = 0;  // lamN <- y on rows; returns |lamN|_inf
  virtual double objective() const = 0;  // unscaled f at x
  virtual void get_solution(double* x, double* y, double* r) = 0;
  virtual void get_bound_duals(double* zl, double* zu) = 0;  // variable-bound multipliers at x
  // newton_step() only: overwrite the primal-dual state (then f, c at x are
  // re-evaluated) and read the last step back
  virtual void set_state(const ncl_ipm_state& st) = 0;
  virtual void get_step(ncl_newton_step& out) = 0;
};

// One Newton step at a caller-given state (ncl_solver_newton_step): the
// symbolic analysis (init_point), then exactly the per-iteration sequence of
// Solver::subproblem — eval_derivatives, form_newton, factor, solve (with
// recovery) — without inertia correction.
void newton_step(Backend& be, const ncl_ipm_state& st, const ncl_options& o, ncl_newton_step& out);

class Solver {
 public:
  Solver(Backend& be, const ncl_options& o) : be_(be), o_(o) {}
  ncl_result solve();
  const std::string& trace() const { return trace_; }
  double objective_scale() const { return S_.sf; }  // sf of the scaled Lagrangian (ipm_elem.hpp)

 private:
  using clk = std::chrono::steady_clock;
  int subproblem(double tol, int outer);
  bool filter_ok(double theta, double phi) const;
  void augment_filter(double theta, double phi);
  double since(clk::time_point t0) const { return std::chrono::duration<double>(clk::now() - t0).count(); }

  Backend& be_;
  ncl_options o_;
  ncl_result res_{};
  Scal S_;
  std::vector<std::pair<double, double>> filter_;
  double theta_max_ = 0, theta_min_ = 0;
  double dw_last_ = 0;
  double last_e0_ = 0;  // scaled KKT error at the last subproblem's exit
  std::string trace_;
};

ncl_options default_options();

}  // namespace nclb::ipm
