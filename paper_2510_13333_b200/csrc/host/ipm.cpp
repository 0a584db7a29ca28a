// NCL outer loop + filter-line-search primal-dual IPM (host control flow).
//
// Outer: solve the subproblem to omega_n; if
// |r|_inf <= eta_n take the multiplier branch lamN <- y and
// tighten (eta, omega) by 10x down to (eta*, omega*), else rho <- 10 rho with
// the multipliers frozen. Optimal when |r|_inf <= eta* after a solve at
// omega*. Infeasible when rho = rho_max and |r|_inf stalls (<10% decrease over
// 3 outer iterations).
//
// Inner: per iteration
//   eval_derivatives -> kkt_error (termination / Fiacco-McCormick update)
//   -> form_newton -> [factor -> inertia check -> dw/dc escalation]*
//   -> solve (rhs, LDL^T solve + refinement, recovery) -> max_steps
//   -> filter line search (trial evaluations) -> accept.
// The tolerance test uses Ipopt's scaled error
//   E_mu = max(du / s_d, pr, |compl - mu| / s_c).
#include "ipm.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>

namespace nclb::ipm {

ncl_options default_options() {
  ncl_options o{};
  o.rho0 = 100.0;
  o.rho_growth = 10.0;
  o.rho_max = 1e12;
  o.eta_star = 1e-6;
  o.omega_star = 1e-6;
  o.eta0 = 0.1;
  o.omega0 = 0.1;
  o.lambda_max = 1e12;
  o.max_outer = 40;
  o.max_inner = 3000;
  o.mu_init = 0.1;
  o.mu_min = 1e-7;
  o.kappa_mu = 0.2;
  o.theta_mu = 1.5;
  o.kappa_eps = 10.0;
  o.tau_min = 0.99;
  o.bound_push = 1e-2;
  o.bound_frac = 1e-2;
  o.kappa_sigma = 1e10;
  o.s_max = 100.0;
  o.obj_max_grad = 100.0;
  o.gamma_theta = 1e-5;
  o.gamma_phi = 1e-8;
  o.eta_phi = 1e-8;
  o.delta = 1.0;
  o.s_theta = 1.1;
  o.s_phi = 2.3;
  o.alpha_min_frac = 0.05;
  o.max_backtrack = 40;
  o.dw_first_rel = 1e-8;
  o.dw_growth = 10.0;
  o.dw_decrease = 1.0 / 3.0;
  o.dw_max = 1e40;
  o.dc_base = 1e-8;
  o.kappa_c = 0.25;
  o.dw_reuse = 1;
  o.pivot_tol = 1e-14;
  o.refine_target = 1e-8;
  // 2, not the solve_refined default of 5: at rho >= 1e8 the condensed K is
  // too ill-conditioned for refinement to reach 1e-8 and the extra sweeps
  // (each a full solve) buy nothing (measured: 52 of 448 iterations at
  // 500x256 stalled at 5 sweeps)
  o.refine_max_sweeps = 2;
  o.mu_warm_frac = 0.1;
  o.acceptable_factor = 10.0;
  o.acceptable_iter = 15;
  o.verbose = 1;
  return o;
}

bool Solver::filter_ok(double theta, double phi) const {
  for (const auto& e : filter_)
    if (theta >= e.first && phi >= e.second) return false;
  return true;
}
void Solver::augment_filter(double theta, double phi) {
  // drop dominated entries, keep the list small
  filter_.erase(std::remove_if(filter_.begin(), filter_.end(),
                               [&](const std::pair<double, double>& e) { return e.first >= theta && e.second >= phi; }),
                filter_.end());
  filter_.emplace_back(theta, phi);
}

namespace {
double scaled_err(const KktErr& e, double sd, double sc, bool mu_part) {
  return std::max({e.du / sd, e.dur / sd, e.pr, (mu_part ? e.cmu : e.c0) / sc});
}
}  // namespace

// returns 0 converged (E_0 <= tol), 1 iteration cap, 2 regularisation
// exhausted, 3 converged on Ipopt's 'acceptable' rule only (E_0 <=
// acceptable_factor * tol for acceptable_iter consecutive iterations)
int Solver::subproblem(double tol, int outer) {
  filter_.clear();
  const int nmult = std::max(1, be_.m() + be_.num_bound_duals());
  const int nz = std::max(1, be_.num_bound_duals());
  const double inf = std::numeric_limits<double>::infinity();
  bool first = true;
  int acc_count = 0;
  for (;;) {
    auto t0 = clk::now();
    be_.eval_derivatives(S_.sf);
    res_.t_eval += since(t0);
    t0 = clk::now();
    KktErr e = be_.kkt_error(S_);
    double sd = std::max(o_.s_max, (e.ysum + e.zsum) / nmult) / o_.s_max;
    double sc = std::max(o_.s_max, e.zsum / nz) / o_.s_max;
    res_.inf_pr = e.pr;
    res_.inf_du = std::max(e.du, e.dur);
    res_.compl_ = e.c0;
    const double e0 = scaled_err(e, sd, sc, false);
    acc_count = e0 <= o_.acceptable_factor * tol ? acc_count + 1 : 0;
    if (e0 <= tol || (o_.acceptable_iter > 0 && acc_count >= o_.acceptable_iter)) {
      res_.t_other += since(t0);
      last_e0_ = e0;
      return e0 <= tol ? 0 : 3;
    }
    // monotone Fiacco-McCormick barrier update
    while (S_.mu > o_.mu_min && scaled_err(e, sd, sc, true) <= o_.kappa_eps * S_.mu) {
      S_.mu = std::max(o_.mu_min, std::min(o_.kappa_mu * S_.mu, std::pow(S_.mu, o_.theta_mu)));
      filter_.clear();
      first = true;
      e = be_.kkt_error(S_);
    }
    if (res_.inner_iters >= o_.max_inner) {
      res_.t_other += since(t0);
      return 1;
    }
    S_.tau = std::max(o_.tau_min, 1.0 - S_.mu);
    res_.t_other += since(t0);

    // ---- Newton system with inertia correction
    t0 = clk::now();
    S_.dc = 0.0;
    be_.form_newton(S_);
    // dw_reuse: when the previous iteration needed dw > 0, skip the dw = 0
    // trial and start at dw_last / 3 (one factorization saved per
    // iteration in the non-convex phase; Ipopt always tries 0 first)
    double dw = (o_.dw_reuse && dw_last_ > 0.0)
                    ? std::max(o_.dw_first_rel * std::max(1.0, be_.hess_absmax()), o_.dw_decrease * dw_last_)
                    : 0.0;
    double hnorm = -1.0;
    int tries = 0;
    for (;;) {
      const FactorOut f = be_.factor(dw, o_.pivot_tol);
      res_.factorizations++;
      tries++;
      if (f.status == 0 && f.npos == be_.n() && f.nneg == 0 && f.nzero == 0) break;
      if (f.status == 1 && S_.dc == 0.0) {
        S_.dc = o_.dc_base * std::pow(S_.mu, o_.kappa_c);
        be_.form_newton(S_);
      }
      if (hnorm < 0) hnorm = std::max(1.0, be_.hess_absmax());
      const double first_dw = o_.dw_first_rel * hnorm;
      if (dw == 0.0)
        dw = dw_last_ == 0.0 ? first_dw : std::max(first_dw, o_.dw_decrease * dw_last_);
      else
        dw *= o_.dw_growth;
      if (dw > o_.dw_max) {
        res_.t_factor += since(t0);
        return 2;
      }
    }
    dw_last_ = dw;
    res_.t_factor += since(t0);

    t0 = clk::now();
    const SolveOut so = be_.solve(S_, o_.refine_target, o_.refine_max_sweeps);
    res_.t_solve += since(t0);

    // ---- filter line search
    t0 = clk::now();
    double apri = 1.0, adual = 1.0;
    be_.max_steps(S_, &apri, &adual);
    const Merit cur = be_.merit_current(S_);
    if (first) {
      theta_max_ = 1e4 * std::max(1.0, cur.theta);
      theta_min_ = 1e-4 * std::max(1.0, cur.theta);
      first = false;
    }
    const double g = be_.dphi(S_);
    double rinf, dxinf, xinf;
    be_.r_inf(&rinf, &dxinf, &xinf);
    const bool tiny = dxinf <= 10.0 * std::numeric_limits<double>::epsilon() * (1.0 + xinf);
    double alpha = apri;
    double amin = o_.gamma_theta;
    if (g < 0.0)
      amin = std::min({o_.gamma_theta, o_.gamma_phi * cur.theta / -g,
                       o_.delta * std::pow(cur.theta, o_.s_theta) / std::pow(-g, o_.s_phi)});
    amin *= o_.alpha_min_frac;
    bool ok = false;
    int ls = 0;
    for (; ls < o_.max_backtrack; ++ls) {
      S_.alpha = alpha;
      const Merit tr = be_.trial(S_);
      if (tiny) {
        ok = tr.valid;
        if (ok) break;
      }
      if (tr.valid && tr.theta <= theta_max_) {
        const bool switching =
            g < 0.0 && alpha * std::pow(-g, o_.s_phi) > o_.delta * std::pow(cur.theta, o_.s_theta);
        if (cur.theta <= theta_min_ && switching) {
          if (tr.phi <= cur.phi + o_.eta_phi * alpha * g) {
            ok = true;  // f-type step: no filter augmentation
            break;
          }
        } else if (filter_ok(tr.theta, tr.phi) &&
                   (tr.theta <= (1.0 - o_.gamma_theta) * cur.theta || tr.phi <= cur.phi - o_.gamma_phi * cur.theta)) {
          augment_filter((1.0 - o_.gamma_theta) * cur.theta, cur.phi - o_.gamma_phi * cur.theta);
          ok = true;
          break;
        }
      }
      alpha *= 0.5;
      if (alpha < amin) break;
    }
    S_.alpha_dual = adual;
    if (ok) {
      be_.accept(S_);
    } else {
      // restoration: the subproblem is always feasible through r
      be_.restore();
      res_.restorations++;
      filter_.clear();
      first = true;
    }
    res_.inner_iters++;
    res_.t_linesearch += since(t0);
    if (o_.verbose) {
      // full precision (%.17g) so two backends' traces can be diffed to the
      // first differing bit (tools/trace_diff.py); e0 = scaled KKT error,
      // theta/phi = current merit, g = directional derivative of phi
      char buf[768];
      std::snprintf(buf, sizeof buf,
                    "{\"outer\": %d, \"iter\": %d, \"mu\": %.17g, \"rho\": %.17g, \"inf_pr\": %.17g, "
                    "\"inf_du\": %.17g, \"e0\": %.17g, \"obj\": %.17g, \"theta\": %.17g, \"phi\": %.17g, "
                    "\"g\": %.17g, \"dw\": %.17g, \"dc\": %.17g, \"alpha_pr\": %.17g, \"alpha_du\": %.17g, "
                    "\"ls\": %d, \"factorizations\": %d, \"refine_res\": %.17g, \"sweeps\": %d, \"accepted\": %d}\n",
                    outer, res_.inner_iters, S_.mu, S_.rho, e.pr, std::max(e.du, e.dur), e0, be_.objective(), cur.theta,
                    cur.phi, g, dw, S_.dc, ok ? S_.alpha : 0.0, adual, ls, tries, so.residual, so.sweeps, ok ? 1 : 0);
      trace_ += buf;
    }
    (void)inf;
  }
}

ncl_result Solver::solve() {
  res_ = ncl_result{};
  trace_.clear();
  last_e0_ = 0.0;
  const auto t_start = clk::now();
  S_ = Scal{};
  S_.mu = o_.mu_init;
  S_.rho = o_.rho0;
  S_.kappa_sigma = o_.kappa_sigma;
  S_.push = o_.bound_push;
  S_.frac = o_.bound_frac;
  double f0 = 0, gmax = 0;
  auto t0 = clk::now();
  be_.init_point(S_, &f0, &gmax);
  S_.sf = std::min(1.0, o_.obj_max_grad / std::max(gmax, 1e-300));
  res_.t_init = since(t0);
  double eta = o_.eta0, omega = o_.omega0;
  std::vector<double> rhist;
  res_.status = NCL_SOLVE_ITERATION_LIMIT;
  for (int outer = 0; outer < o_.max_outer; ++outer) {
    const double tol = std::max(omega, o_.omega_star);
    const int st = subproblem(tol, outer);
    res_.outer_iters = outer + 1;
    double rinf, dxinf, xinf;
    be_.r_inf(&rinf, &dxinf, &xinf);
    res_.r_inf = rinf;
    rhist.push_back(rinf);
    if (o_.verbose) {
      char buf[256];
      std::snprintf(buf, sizeof buf,
                    "{\"outer_summary\": %d, \"rho\": %.3e, \"r_inf\": %.6e, \"inner_iters\": %d, \"omega\": %.3e, "
                    "\"eta\": %.3e, \"obj\": %.12e, \"status\": %d}\n",
                    outer, S_.rho, rinf, res_.inner_iters, tol, eta, be_.objective(), st);
      trace_ += buf;
    }
    if (st == 2) {
      res_.status = NCL_SOLVE_REG_EXHAUSTED;
      break;
    }
    if (st == 1) {
      res_.status = NCL_SOLVE_ITERATION_LIMIT;
      break;
    }
    if (rinf <= std::max(eta, o_.eta_star)) {
      if (rinf <= o_.eta_star && tol <= o_.omega_star) {
        // optimal only when the last subproblem met omega* itself; an exit
        // on the 'acceptable' rule (E_0 <= acceptable_factor * omega*) is
        // reported as such (optimal => stationarity <= omega*)
        res_.status = st == 0 ? NCL_SOLVE_OPTIMAL : NCL_SOLVE_ACCEPTABLE;
        break;
      }
      // multiplier branch; bounded-multiplier guard
      if (be_.update_multipliers() > o_.lambda_max) res_.multiplier_warning = 1;
      eta = std::max(o_.eta_star, 0.1 * eta);
      omega = std::max(o_.omega_star, 0.1 * omega);
    } else {
      if (S_.rho >= o_.rho_max && rhist.size() >= 4 && rhist.back() > 0.9 * rhist[rhist.size() - 4]) {
        res_.status = NCL_SOLVE_INFEASIBLE;
        break;
      }
      S_.rho = std::min(o_.rho_max, o_.rho_growth * S_.rho);
    }
    // warm start: same primal-dual point, smaller barrier
    S_.mu = std::max(o_.mu_min, std::min(S_.mu > 0 ? std::max(S_.mu, o_.mu_min) : o_.mu_init,
                                         o_.mu_warm_frac * std::max(omega, o_.omega_star)));
  }
  res_.objective = be_.objective();
  res_.final_e0 = last_e0_;
  res_.rho = S_.rho;
  res_.mu = S_.mu;
  res_.t_total = since(t_start);
  return res_;
}

void newton_step(Backend& be, const ncl_ipm_state& st, const ncl_options& o, ncl_newton_step& out) {
  Scal S;
  S.mu = st.mu;
  S.rho = st.rho;
  S.sf = st.sf;
  S.kappa_sigma = o.kappa_sigma;
  S.push = o.bound_push;
  S.frac = o.bound_frac;
  double f0 = 0, gmax = 0;
  be.init_point(S, &f0, &gmax);
  be.set_state(st);
  be.eval_derivatives(S.sf);
  S.dc = st.dc;
  be.form_newton(S);
  const FactorOut f = be.factor(st.dw, o.pivot_tol);
  out.status = f.status;
  out.npos = f.npos;
  out.nneg = f.nneg;
  out.nzero = f.nzero;
  out.residual = 0;
  out.sweeps = 0;
  out.converged = 0;
  if (f.status == 0) {
    const SolveOut so = be.solve(S, o.refine_target, o.refine_max_sweeps);
    out.residual = so.residual;
    out.sweeps = so.sweeps;
    out.converged = so.converged ? 1 : 0;
    be.get_step(out);
  }
}

}  // namespace nclb::ipm
