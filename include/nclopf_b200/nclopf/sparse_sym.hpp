// Drop-in façade for /root/reference/proj/include/nclopf/sparse_sym.hpp over
// the B200 library's C-ABI (include/nclopf_b200.h): same namespace, names,
// signatures and exception types, numerics on the GPU. Header-only; link
// libnclopf_b200.so. Differences from the reference, all in ownership:
// SparseSym is move-only (its triplets and values live in the library), and
// SymbolicFactor / Factorization keep the library handles alive through
// shared_ptr members next to the reference's public fields.
#pragma once

#include <cstdint>
#include <limits>
#include <memory>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "nclopf/expr.hpp"
#include "nclopf_b200.h"

namespace nclopf {

namespace detail {
/// return code -> the reference's exception (nclopf_expr_program.h)
inline void check(int rc) {
  if (rc == NCL_OK) return;
  const std::string msg = ncl_last_error();
  if (rc == NCL_E_INVALID) throw std::invalid_argument(msg);
  if (rc == NCL_E_LOGIC) throw std::logic_error(msg);
  if (rc == NCL_E_DOMAIN) throw DomainError(msg);
  throw std::runtime_error(msg);
}
}  // namespace detail

/// sparse_sym.hpp:20-66
class SparseSym {
 public:
  explicit SparseSym(int n) { detail::check(ncl_sym_create(n, &h_)); }
  explicit SparseSym(ncl_sym_t adopt) : h_(adopt) {}
  SparseSym(SparseSym&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  SparseSym& operator=(SparseSym&& o) noexcept {
    std::swap(h_, o.h_);
    return *this;
  }
  SparseSym(const SparseSym&) = delete;
  SparseSym& operator=(const SparseSym&) = delete;
  ~SparseSym() {
    if (h_) ncl_sym_destroy(h_);
  }

  int dim() const { return ncl_sym_dim(h_); }
  bool finalized() const { return ncl_sym_finalized(h_) != 0; }

  void add(int row, int col, double value) { detail::check(ncl_sym_add(h_, 1, &row, &col, &value)); }
  void finalize() { detail::check(ncl_sym_finalize(h_)); }
  void begin_refill() { detail::check(ncl_sym_begin_refill(h_)); }
  void refill() { detail::check(ncl_sym_refill(h_)); }

  int nnz() const { return ncl_sym_nnz(h_); }
  const std::vector<int>& col_ptr() const { return fetch(), cp_; }
  const std::vector<int>& row_ind() const { return fetch(), ri_; }
  const std::vector<double>& values() const { return fetch(), v_; }

  double max_abs_diag() const { return scalar(ncl_sym_max_abs_diag); }
  double norm_inf() const { return scalar(ncl_sym_norm_inf); }
  double frobenius_norm() const { return scalar(ncl_sym_frobenius_norm); }

  void multiply(std::span<const double> x, std::span<double> y) const {
    if (static_cast<int>(x.size()) != dim() || static_cast<int>(y.size()) != dim())
      throw std::invalid_argument("SparseSym::multiply: size mismatch");
    detail::check(ncl_sym_multiply(h_, x.data(), y.data(), NCL_HOST));
  }
  bool same_pattern(const SparseSym& other) const { return ncl_sym_same_pattern(h_, other.h_) == 1; }
  void write_matrix_market(std::ostream& os) const {
    int64_t len = 0;
    detail::check(ncl_sym_write_matrix_market(h_, nullptr, 0, &len));
    std::string buf(static_cast<size_t>(len) + 1, '\0');
    detail::check(ncl_sym_write_matrix_market(h_, buf.data(), len + 1, &len));
    os.write(buf.data(), len);
  }

  ncl_sym_t handle() const { return h_; }

 private:
  void fetch() const {
    if (!finalized()) {
      cp_.assign(1, 0);
      ri_.clear();
      v_.clear();
      return;
    }
    cp_.resize(dim() + 1);
    ri_.resize(nnz());
    v_.resize(nnz());
    detail::check(ncl_sym_get_csc(h_, cp_.data(), ri_.data(), v_.data()));
  }
  double scalar(int (*f)(ncl_sym_t, double*)) const {
    double out = 0.0;
    detail::check(f(h_, &out));
    return out;
  }
  ncl_sym_t h_ = nullptr;
  mutable std::vector<int> cp_, ri_;
  mutable std::vector<double> v_;
};

/// sparse_sym.hpp:68-70
inline std::vector<int> symbolic_order(const SparseSym& pattern) {
  std::vector<int> perm(pattern.dim());
  detail::check(ncl_symbolic_order(pattern.handle(), perm.data()));
  return perm;
}

/// sparse_sym.hpp:74-85 (+ the library handle the numeric factorization uses)
struct SymbolicFactor {
  int n = 0;
  std::vector<int> perm;
  std::vector<int> iperm;
  std::vector<int> parent;
  std::vector<int> up_colptr, up_rowind;
  std::vector<int> entry_map;
  std::vector<int> l_colcount;
  std::int64_t l_nnz = 0;
  std::shared_ptr<ncl_symb> handle;  // ncl_symb_t
};

namespace detail {
inline SymbolicFactor analyze(const SparseSym& M, const int* perm) {
  ncl_symb_t h = nullptr;
  check(ncl_analyze(M.handle(), perm, &h));
  SymbolicFactor S;
  S.handle.reset(h, ncl_symb_destroy);
  ncl_symb_info info{};
  check(ncl_symb_info_get(h, &info));
  S.n = info.n;
  S.l_nnz = info.l_nnz;
  const int nz = M.nnz();
  S.perm.resize(S.n);
  S.iperm.resize(S.n);
  S.parent.resize(S.n);
  S.up_colptr.resize(S.n + 1);
  S.up_rowind.resize(nz);
  S.entry_map.resize(nz);
  S.l_colcount.resize(S.n);
  check(ncl_symb_get(h, S.perm.data(), S.iperm.data(), S.parent.data(), S.up_colptr.data(), S.up_rowind.data(),
                     S.entry_map.data(), S.l_colcount.data()));
  return S;
}
}  // namespace detail

/// sparse_sym.hpp:87-88
inline SymbolicFactor analyze(const SparseSym& M) { return detail::analyze(M, nullptr); }
inline SymbolicFactor analyze(const SparseSym& M, std::vector<int> perm) {
  if (static_cast<int>(perm.size()) != M.dim()) throw std::invalid_argument("analyze: bad permutation");
  return detail::analyze(M, perm.data());
}

enum class FactorizeStatus : std::uint8_t { ok, zero_pivot };

struct Inertia {
  int n_pos = 0, n_neg = 0, n_zero = 0;
  bool operator==(const Inertia&) const = default;
};

/// sparse_sym.hpp:97-121
class Factorization {
 public:
  FactorizeStatus status = FactorizeStatus::ok;
  int zero_pivot_index = -1;
  Inertia inertia;

  bool ok() const { return status == FactorizeStatus::ok; }

  void solve_in_place(std::span<double> x) const {
    if (!h_) throw std::logic_error("Factorization::solve: no factor");
    if (static_cast<int>(x.size()) != symb_->n) throw std::invalid_argument("Factorization::solve: size mismatch");
    detail::check(ncl_fact_solve(h_.get(), x.data(), NCL_HOST));
  }
  std::vector<double> solve(std::span<const double> b) const {
    std::vector<double> x(b.begin(), b.end());
    solve_in_place(x);
    return x;
  }
  const std::vector<double>& diagonal() const { return d_; }
  const SymbolicFactor* symbolic() const { return symb_; }
  ncl_fact_t handle() const { return h_.get(); }

 private:
  friend Factorization factorize(const SparseSym&, const SymbolicFactor&, double);
  friend Factorization factorize(const SparseSym&, double);
  void finish() {
    int st = 0, zp = -1;
    detail::check(ncl_fact_status(h_.get(), &st, &zp, &inertia.n_pos, &inertia.n_neg, &inertia.n_zero));
    status = st == 0 ? FactorizeStatus::ok : FactorizeStatus::zero_pivot;
    zero_pivot_index = zp;
    d_.resize(symb_->n);
    detail::check(ncl_fact_diagonal(h_.get(), d_.data()));
  }
  const SymbolicFactor* symb_ = nullptr;
  std::shared_ptr<const SymbolicFactor> owned_symb_;
  std::shared_ptr<ncl_fact> h_;
  std::vector<double> d_;
};

/// sparse_sym.hpp:123-126
inline Factorization factorize(const SparseSym& M, const SymbolicFactor& symb, double pivot_tol = 1e-12) {
  Factorization F;
  ncl_fact_t h = nullptr;
  detail::check(ncl_factorize(M.handle(), symb.handle.get(), pivot_tol, &h));
  F.h_.reset(h, ncl_fact_destroy);
  F.symb_ = &symb;
  F.finish();
  return F;
}
inline Factorization factorize(const SparseSym& M, double pivot_tol = 1e-12) {
  auto owned = std::make_shared<const SymbolicFactor>(analyze(M));
  Factorization F = factorize(M, *owned, pivot_tol);
  F.owned_symb_ = owned;
  return F;
}

/// sparse_sym.hpp:128-139
struct RefinedSolve {
  std::vector<double> x;
  double residual = std::numeric_limits<double>::infinity();
  int sweeps = 0;
  bool converged = false;
};

inline RefinedSolve solve_refined(const Factorization& F, const SparseSym& M, std::span<const double> b,
                                  double target = 1e-8, int max_sweeps = 5) {
  if (static_cast<int>(b.size()) != M.dim()) throw std::invalid_argument("solve_refined: size mismatch");
  RefinedSolve r;
  r.x.resize(b.size());
  int sw = 0, cv = 0;
  detail::check(ncl_solve_refined(F.handle(), M.handle(), b.data(), target, max_sweeps, r.x.data(), NCL_HOST,
                                  &r.residual, &sw, &cv));
  r.sweeps = sw;
  r.converged = cv != 0;
  return r;
}

}  // namespace nclopf
