// ORACLE — test infrastructure only (see ref_capi.cpp header for the rules).
//
// The NCL/IPM of the reference exists only as SPEC text, so
// its CPU oracle is the host control flow of the product
// (paper_2510_13333_b200/csrc/host/ipm.cpp, the single statement of the
// algorithm; SURVEY.md §7 "one host IPM/NCL implementation ... linked against
// the reference sources as the CPU oracle") bound to a CPU backend made of
// the UNMODIFIED reference sparse_core/model_ad:
//   evaluation  nclopf::ModelFunctions::eval_*        (model.cpp:134-223)
//   assembly    nclopf::SparseSym add/finalize/refill (sparse_sym.cpp:12-67)
//   ordering    nclopf::analyze / symbolic_order      (sparse_sym.cpp:139-262)
//   factor      nclopf::factorize                     (sparse_sym.cpp:268-337)
//   solve       nclopf::solve_refined                 (sparse_sym.cpp:371-401)
// and the element-wise IPM formulas of csrc/host/ipm_elem.hpp evaluated in
// plain host loops, with reductions in the GPU's fixed order.
//
// The condensed K is fed to the reference SparseSym as triplets in the
// order restated here (the product's csrc/host/kkt.hpp contract):
//   1. Hessian entries in hess_coords order,
//   2. one diagonal per variable: sigma_x,i + delta_w,
//   3. for every row r ascending, every pair a >= b of its Jacobian entries
//      (jac_coords order): (col_a, col_b) with value (D_r J_a) J_b.
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "nclopf/model.hpp"
#include "nclopf/sparse_sym.hpp"

#include "ipm.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

using namespace nclb;

class RefBackend final : public ipm::Backend {
 public:
  RefBackend(const nclopf::ModelFunctions& M, const double* xl, const double* xu, const double* x0, const double* gl,
             const double* gu, const int* perm)
      : M_(M), n_(M.num_vars()), m_(M.num_cons()), K_(M.num_vars()) {
    const int n = n_, m = m_;
    auto vx = [&](std::vector<double>& v) { v.assign(n, 0.0); return v.data(); };
    auto vr = [&](std::vector<double>& v) { v.assign(m, 0.0); return v.data(); };
    xl_.assign(xl, xl + n);
    xu_.assign(xu, xu + n);
    gl_.assign(gl, gl + m);
    gu_.assign(gu, gu + m);
    V_.n = n;
    V_.m = m;
    V_.xl = xl_.data();
    V_.xu = xu_.data();
    V_.gl = gl_.data();
    V_.gu = gu_.data();
    V_.x = vx(x_);
    std::copy(x0, x0 + n, x_.begin());
    V_.zl = vx(zl_), V_.zu = vx(zu_), V_.grad = vx(grad_), V_.jty = vx(jty_), V_.sigx = vx(sigx_);
    V_.gx = vx(gx_), V_.rhs = vx(rhs_), V_.jtdq = vx(jtdq_), V_.dx = vx(dx_), V_.dzl = vx(dzl_);
    V_.dzu = vx(dzu_), V_.xt = vx(xt_);
    V_.r = vr(r_), V_.s = vr(s_), V_.y = vr(y_), V_.vl = vr(vl_), V_.vu = vr(vu_), V_.lamN = vr(lamN_);
    V_.c = vr(c_), V_.D = vr(D_), V_.q = vr(q_), V_.dq = vr(dq_), V_.dr = vr(dr_), V_.ds = vr(ds_);
    V_.dy = vr(dy_), V_.dvl = vr(dvl_), V_.dvu = vr(dvu_), V_.jdx = vr(jdx_), V_.rt = vr(rt_), V_.st = vr(st_);
    V_.ct = vr(ct_);
    for (int i = 0; i < n; ++i) nbd_ += (xl[i] > -ipm::kBig) + (xu[i] < ipm::kBig);
    for (int i = 0; i < m; ++i)
      if (gl[i] != gu[i]) nbd_ += (gl[i] > -ipm::kBig) + (gu[i] < ipm::kBig);
    jac_.assign(M.jac_coords().size(), 0.0);
    hess_.assign(M.hess_coords().size(), 0.0);
    if (perm) perm_.assign(perm, perm + n);
    // K triplet coordinates (fixed order, see header)
    const auto& hc = M.hess_coords();
    const auto& jc = M.jac_coords();
    for (const auto& e : hc) trow_.push_back(e.first), tcol_.push_back(e.second);
    for (int i = 0; i < n; ++i) trow_.push_back(i), tcol_.push_back(i);
    rp_.assign(m + 1, 0);
    for (const auto& e : jc) rp_[e.first + 1]++;
    for (int r = 0; r < m; ++r) rp_[r + 1] += rp_[r];
    for (int r = 0; r < m; ++r)
      for (int64_t a = rp_[r]; a < rp_[r + 1]; ++a)
        for (int64_t b = rp_[r]; b <= a; ++b) trow_.push_back(jc[a].second), tcol_.push_back(jc[b].second);
    tval_.assign(trow_.size(), 0.0);
  }
  int n() const override { return n_; }
  int m() const override { return m_; }
  int num_bound_duals() const override { return static_cast<int>(nbd_); }

  void init_point(const ipm::Scal& S, double* f, double* gmax) override {
    for (int i = 0; i < n_; ++i) ipm::init_x(V_, i, S);
    fcur_ = M_.eval_objective(x_);
    M_.eval_grad_objective(x_, grad_);
    M_.eval_constraints(x_, c_);
    double g = 0.0;
    for (double v : grad_) g = std::fmax(g, std::fabs(v));
    for (int i = 0; i < m_; ++i) ipm::init_row(V_, i, S);
    *f = fcur_;
    *gmax = g;
    // first assembly fixes the pattern, then the one-time symbolic analysis
    for (size_t k = 0; k < trow_.size(); ++k) K_.add(trow_[k], tcol_[k], 0.0);
    K_.finalize();
    symb_ = perm_.empty() ? nclopf::analyze(K_) : nclopf::analyze(K_, perm_);
  }
  void eval_derivatives(double sf) override {
    M_.eval_grad_objective(x_, grad_);
    M_.eval_jacobian(x_, jac_);
    M_.eval_hessian_lag(x_, sf, y_, hess_);
    M_.jac_trans_times(jac_, y_, jty_);
  }
  ipm::KktErr kkt_error(const ipm::Scal& S) override {
    double a[8];
    ipm::reduce_host<ipm::RedKkt>(V_, S, a);
    ipm::KktErr e;
    e.du = a[0], e.pr = a[1], e.dur = a[2], e.cmu = a[3], e.c0 = a[4], e.ysum = a[5], e.zsum = a[6];
    return e;
  }
  double hess_absmax() override {
    double h = 0.0;
    for (double v : hess_) h = std::fmax(h, std::fabs(v));
    return h;
  }
  void form_newton(const ipm::Scal& S) override {
    for (int i = 0; i < n_; ++i) ipm::newton_x(V_, i, S);
    for (int i = 0; i < m_; ++i) ipm::newton_row(V_, i, S);
  }
  ipm::FactorOut factor(double dw, double pivot_tol) override {
    const int64_t nh = static_cast<int64_t>(hess_.size());
    int64_t k = 0;
    for (; k < nh; ++k) tval_[k] = hess_[k];
    for (int i = 0; i < n_; ++i, ++k) tval_[k] = sigx_[i] + dw;
    const auto& jc = M_.jac_coords();
    (void)jc;
    for (int r = 0; r < m_; ++r)
      for (int64_t a = rp_[r]; a < rp_[r + 1]; ++a)
        for (int64_t b = rp_[r]; b <= a; ++b) tval_[k++] = (D_[r] * jac_[a]) * jac_[b];
    K_.begin_refill();
    for (size_t t = 0; t < trow_.size(); ++t) K_.add(trow_[t], tcol_[t], tval_[t]);
    K_.refill();
    F_ = nclopf::factorize(K_, symb_, pivot_tol);
    ipm::FactorOut o;
    o.status = F_.ok() ? 0 : 1;
    o.npos = F_.inertia.n_pos;
    o.nneg = F_.inertia.n_neg;
    o.nzero = F_.inertia.n_zero;
    return o;
  }
  ipm::SolveOut solve(const ipm::Scal& S, double target, int max_sweeps) override {
    M_.jac_trans_times(jac_, dq_, jtdq_);
    for (int i = 0; i < n_; ++i) ipm::rhs_x(V_, i);
    const nclopf::RefinedSolve rs = nclopf::solve_refined(F_, K_, rhs_, target, max_sweeps);
    std::copy(rs.x.begin(), rs.x.end(), dx_.begin());
    M_.jac_times(jac_, dx_, jdx_);
    for (int i = 0; i < n_; ++i) ipm::recover_x(V_, i, S);
    for (int i = 0; i < m_; ++i) ipm::recover_row(V_, i, S);
    ipm::SolveOut o;
    o.residual = rs.residual;
    o.sweeps = rs.sweeps;
    o.converged = rs.converged;
    return o;
  }
  void max_steps(const ipm::Scal& S, double* apri, double* adual) override {
    double a[8];
    ipm::reduce_host<ipm::RedFtb>(V_, S, a);
    *apri = std::fmin(1.0, a[0]);
    *adual = std::fmin(1.0, a[1]);
  }
  double dphi(const ipm::Scal& S) override {
    double a[8];
    ipm::reduce_host<ipm::RedDphi>(V_, S, a);
    return a[0];
  }
  ipm::Merit merit_current(const ipm::Scal& S) override {
    ipm::Vecs W = V_;
    W.xt = V_.x;
    W.rt = V_.r;
    W.st = V_.s;
    W.ct = V_.c;
    double a[8];
    ipm::reduce_host<ipm::RedMerit>(W, S, a);
    return merit(S, fcur_, a);
  }
  ipm::Merit trial(const ipm::Scal& S) override {
    for (int i = 0; i < n_; ++i) ipm::trial_x(V_, i, S);
    for (int i = 0; i < m_; ++i) ipm::trial_row(V_, i, S);
    ftrial_ = M_.eval_objective(xt_);
    M_.eval_constraints(xt_, ct_);
    double a[8];
    ipm::reduce_host<ipm::RedMerit>(V_, S, a);
    return merit(S, ftrial_, a);
  }
  void accept(const ipm::Scal& S) override {
    for (int i = 0; i < n_; ++i) ipm::accept_x(V_, i, S);
    for (int i = 0; i < m_; ++i) ipm::accept_row(V_, i, S);
    fcur_ = ftrial_;
  }
  void restore() override {
    for (int i = 0; i < m_; ++i) ipm::restore_row(V_, i);
  }
  void r_inf(double* rinf, double* dxinf, double* xinf) override {
    double a[8];
    ipm::reduce_host<ipm::RedRinf>(V_, ipm::Scal{}, a);
    *rinf = a[0];
    *dxinf = a[1];
    *xinf = a[2];
  }
  double update_multipliers() override {
    double a = 0.0;
    for (int i = 0; i < m_; ++i) {
      ipm::update_multiplier_row(V_, i);
      a = std::fmax(a, std::fabs(lamN_[i]));
    }
    return a;
  }
  double objective() const override { return fcur_; }
  void set_state(const ncl_ipm_state& st) override {
    std::copy(st.x, st.x + n_, x_.begin()), std::copy(st.zl, st.zl + n_, zl_.begin());
    std::copy(st.zu, st.zu + n_, zu_.begin());
    std::copy(st.r, st.r + m_, r_.begin()), std::copy(st.s, st.s + m_, s_.begin());
    std::copy(st.y, st.y + m_, y_.begin()), std::copy(st.vl, st.vl + m_, vl_.begin());
    std::copy(st.vu, st.vu + m_, vu_.begin()), std::copy(st.lamN, st.lamN + m_, lamN_.begin());
    fcur_ = M_.eval_objective(x_);
    M_.eval_constraints(x_, c_);
  }
  void get_step(ncl_newton_step& o) override {
    auto dn = [](double* h, const std::vector<double>& v) {
      if (h) std::copy(v.begin(), v.end(), h);
    };
    dn(o.dx, dx_), dn(o.dzl, dzl_), dn(o.dzu, dzu_), dn(o.dr, dr_), dn(o.ds, ds_), dn(o.dy, dy_);
    dn(o.dvl, dvl_), dn(o.dvu, dvu_);
  }
  void get_bound_duals(double* zl, double* zu) override {
    if (zl) std::copy(zl_.begin(), zl_.end(), zl);
    if (zu) std::copy(zu_.begin(), zu_.end(), zu);
  }
  void get_solution(double* x, double* y, double* r) override {
    if (x) std::copy(x_.begin(), x_.end(), x);
    if (y) std::copy(y_.begin(), y_.end(), y);
    if (r) std::copy(r_.begin(), r_.end(), r);
  }

 private:
  static ipm::Merit merit(const ipm::Scal& S, double f, const double* a) {
    ipm::Merit mr;
    mr.theta = a[0];
    mr.phi = S.sf * f + a[1] + S.mu * a[2];
    mr.valid = a[3] == 0.0 && std::isfinite(mr.phi) && std::isfinite(mr.theta);
    return mr;
  }

  const nclopf::ModelFunctions& M_;
  int n_, m_;
  int64_t nbd_ = 0;
  ipm::Vecs V_;
  std::vector<double> xl_, xu_, gl_, gu_;
  std::vector<double> x_, zl_, zu_, grad_, jty_, sigx_, gx_, rhs_, jtdq_, dx_, dzl_, dzu_, xt_;
  std::vector<double> r_, s_, y_, vl_, vu_, lamN_, c_, D_, q_, dq_, dr_, ds_, dy_, dvl_, dvu_, jdx_, rt_, st_, ct_;
  std::vector<double> jac_, hess_;
  std::vector<int> trow_, tcol_, perm_;
  std::vector<int64_t> rp_;
  std::vector<double> tval_;
  nclopf::SparseSym K_;
  nclopf::SymbolicFactor symb_;
  nclopf::Factorization F_;
  double fcur_ = 0, ftrial_ = 0;
};

thread_local std::string g_ipm_err;

}  // namespace

REF_API const char* ref_ipm_last_error() { return g_ipm_err.c_str(); }

REF_API void ref_ipm_default_options(ncl_options* o) { *o = ipm::default_options(); }

// ncl_solve on the reference CPU backend. perm: optional precomputed
// symbolic_order permutation of the K pattern (NULL = run the reference's).
REF_API int ref_ncl_solve(void* model, const double* xl, const double* xu, const double* x0, const double* gl,
                          const double* gu, const int* perm, const ncl_options* opt, ncl_result* res, double* x_out,
                          double* y_out, double* r_out, char* trace, int64_t cap, int64_t* len) {
  try {
    const auto& M = *static_cast<const nclopf::ModelFunctions*>(model);
    RefBackend be(M, xl, xu, x0, gl, gu, perm);
    const ncl_options o = opt ? *opt : ipm::default_options();
    ipm::Solver sol(be, o);
    *res = sol.solve();
    be.get_solution(x_out, y_out, r_out);
    const std::string& t = sol.trace();
    if (len) *len = static_cast<int64_t>(t.size());
    if (trace && cap > 0) {
      const int64_t k = std::min<int64_t>(cap - 1, static_cast<int64_t>(t.size()));
      std::memcpy(trace, t.data(), k);
      trace[k] = 0;
    }
    return 0;
  } catch (const std::exception& e) {
    g_ipm_err = e.what();
    return -5;
  }
}

// one Newton step at a caller-given state (ncl_solver_newton_step on the
// reference CPU backend)
REF_API int ref_newton_step(void* model, const double* xl, const double* xu, const double* x0, const double* gl,
                            const double* gu, const ncl_ipm_state* st, const ncl_options* opt, ncl_newton_step* out) {
  try {
    const auto& M = *static_cast<const nclopf::ModelFunctions*>(model);
    RefBackend be(M, xl, xu, x0, gl, gu, nullptr);
    const ncl_options o = opt ? *opt : ipm::default_options();
    ipm::newton_step(be, *st, o, *out);
    return 0;
  } catch (const std::exception& e) {
    g_ipm_err = e.what();
    return -5;
  }
}
