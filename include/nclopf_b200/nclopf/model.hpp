// Drop-in façade for /root/reference/proj/include/nclopf/model.hpp over the
// B200 library's C-ABI: ModelBuilder / ModelFunctions / fd_check with the
// reference's names, signatures and exceptions; every evaluation runs on the
// GPU (host spans, synchronous — the reference's semantics). Terms cross the
// boundary one call each so misuse throws at the call site as in
// model.cpp:53-74.
#pragma once

#include <memory>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "nclopf/expr.hpp"
#include "nclopf/sparse_sym.hpp"

namespace nclopf {

/// model.hpp:16-20
struct Instance {
  std::vector<int> vars;
  std::vector<double> params;
  int row = -1;
};

class ModelBuilder;

/// model.hpp:29-71
class ModelFunctions {
 public:
  int num_vars() const { return n_; }
  int num_cons() const { return m_; }

  double eval_objective(std::span<const double> w) const {
    need(w.size(), n_);
    double out = 0.0;
    detail::check(ncl_model_eval_objective(h_.get(), w.data(), &out, NCL_HOST));
    return out;
  }
  void eval_grad_objective(std::span<const double> w, std::span<double> grad) const {
    need(w.size(), n_);
    need(grad.size(), n_);
    detail::check(ncl_model_eval_grad_objective(h_.get(), w.data(), grad.data(), NCL_HOST));
  }
  void eval_constraints(std::span<const double> w, std::span<double> c) const {
    need(w.size(), n_);
    need(c.size(), m_);
    detail::check(ncl_model_eval_constraints(h_.get(), w.data(), c.data(), NCL_HOST));
  }
  const std::vector<std::pair<int, int>>& jac_coords() const { return jac_; }
  void eval_jacobian(std::span<const double> w, std::span<double> vals) const {
    need(w.size(), n_);
    need(vals.size(), jac_.size());
    detail::check(ncl_model_eval_jacobian(h_.get(), w.data(), vals.data(), NCL_HOST));
  }
  const std::vector<std::pair<int, int>>& hess_coords() const { return hess_; }
  void eval_hessian_lag(std::span<const double> w, double sigma, std::span<const double> lam,
                        std::span<double> vals) const {
    need(w.size(), n_);
    need(lam.size(), m_);
    need(vals.size(), hess_.size());
    detail::check(ncl_model_eval_hessian_lag(h_.get(), w.data(), sigma, lam.data(), vals.data(), NCL_HOST));
  }
  SparseSym hessian_lag(std::span<const double> w, double sigma, std::span<const double> lam) const {
    need(w.size(), n_);
    need(lam.size(), m_);
    ncl_sym_t out = nullptr;
    detail::check(ncl_model_hessian_lag(h_.get(), w.data(), sigma, lam.data(), &out));
    return SparseSym(out);
  }
  void jac_times(std::span<const double> jac_vals, std::span<const double> v, std::span<double> out) const {
    need(jac_vals.size(), jac_.size());
    need(v.size(), n_);
    need(out.size(), m_);
    detail::check(ncl_model_jac_times(h_.get(), jac_vals.data(), v.data(), out.data(), NCL_HOST));
  }
  void jac_trans_times(std::span<const double> jac_vals, std::span<const double> y, std::span<double> out) const {
    need(jac_vals.size(), jac_.size());
    need(y.size(), m_);
    need(out.size(), n_);
    detail::check(ncl_model_jac_trans_times(h_.get(), jac_vals.data(), y.data(), out.data(), NCL_HOST));
  }

  ncl_model_t handle() const { return h_.get(); }

 private:
  friend class ModelBuilder;
  static void need(size_t have, size_t want) {
    if (have != want) throw std::invalid_argument("ModelFunctions: span size mismatch");
  }
  void load(ncl_model_t h) {
    h_.reset(h, ncl_model_destroy);
    int64_t nj = 0, nh = 0;
    detail::check(ncl_model_sizes(h, &n_, &m_, &nj, &nh));
    std::vector<int> r(nj), c(nj);
    detail::check(ncl_model_jac_coords(h, r.data(), c.data()));
    for (int64_t k = 0; k < nj; ++k) jac_.emplace_back(r[k], c[k]);
    r.resize(nh);
    c.resize(nh);
    detail::check(ncl_model_hess_coords(h, r.data(), c.data()));
    for (int64_t k = 0; k < nh; ++k) hess_.emplace_back(r[k], c[k]);
  }
  std::shared_ptr<ncl_model> h_;
  int n_ = 0, m_ = 0;
  std::vector<std::pair<int, int>> jac_, hess_;
};

/// model.hpp:74-97
class ModelBuilder {
 public:
  explicit ModelBuilder(int num_vars) {
    ncl_builder_t b = nullptr;
    detail::check(ncl_builder_create(num_vars, &b));
    h_.reset(b, ncl_builder_destroy);
  }
  int num_vars() const { return ncl_builder_num_vars(h_.get()); }
  int num_rows() const { return ncl_builder_num_rows(h_.get()); }

  int add_template(ExpressionTemplate t) {
    const auto prog = t.expr().program();
    int id = -1;
    detail::check(ncl_builder_add_template(h_.get(), static_cast<int>(prog.size()), prog.data(), t.num_var_slots(),
                                           t.name().c_str(), &id));
    return id;
  }
  int add_rows(int count) {
    int first = 0;
    detail::check(ncl_builder_add_rows(h_.get(), count, &first));
    return first;
  }
  void add_objective_term(int tmpl_id, std::vector<int> vars, std::vector<double> params = {}) {
    detail::check(ncl_builder_add_objective_terms(h_.get(), tmpl_id, 1, static_cast<int>(vars.size()), vars.data(),
                                                  static_cast<int>(params.size()), params.data()));
  }
  void add_constraint_term(int tmpl_id, int row, std::vector<int> vars, std::vector<double> params = {}) {
    detail::check(ncl_builder_add_constraint_terms(h_.get(), tmpl_id, 1, &row, static_cast<int>(vars.size()),
                                                   vars.data(), static_cast<int>(params.size()), params.data()));
  }
  ModelFunctions build() && {
    ncl_model_t m = nullptr;
    detail::check(ncl_builder_build(h_.get(), &m));
    ModelFunctions f;
    f.load(m);
    return f;
  }

 private:
  std::shared_ptr<ncl_builder> h_;
};

/// model.hpp:99-109
struct FdReport {
  double grad_err = 0.0;
  double jac_err = 0.0;
  double hess_err = 0.0;
  bool pass = false;
};

inline FdReport fd_check(const ModelFunctions& m, std::span<const double> w, unsigned seed, double tol = 1e-6) {
  double errs[3] = {0, 0, 0};
  int pass = 0;
  detail::check(ncl_fd_check(m.handle(), w.data(), seed, tol, errs, &pass));
  return FdReport{errs[0], errs[1], errs[2], pass != 0};
}

}  // namespace nclopf
