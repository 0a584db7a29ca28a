// ORACLE — test infrastructure only. Never linked into, loaded by, or called
// from the product library (paper_2510_13333_b200). Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
// arm may load oracle/_ref/libnclopf_ref.so, and only as the checker or the
// timed CPU reference arm.
//
// What this is: a thin extern "C" shim over the UNMODIFIED reference sources
// /root/reference/proj/src/{sparse_sym,expr,model}.cpp, compiled in place by
// oracle/Makefile into oracle/_ref/. Every entry point forwards to the
// reference function named in its comment; no arithmetic happens here except
// marshalling.  Exceptions are mapped to the same integer codes the product
// C-ABI uses (include/nclopf_b200.h: NCL_E_*).
//
// Test-only L access: the reference keeps L private
// (proj/include/nclopf/sparse_sym.hpp:119-120); like the survey probe we
// expose it via `#define private public` in THIS translation unit only, after
// all standard headers are included.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>
#include <map>
#include <set>
#include <algorithm>
#include <iosfwd>
#include <limits>

#define private public
#include "nclopf/sparse_sym.hpp"
#include "nclopf/expr.hpp"
#include "nclopf/model.hpp"
#undef private

#include "../include/nclopf_expr_program.h"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {
thread_local std::string g_err;

int map_exc() {
  try {
    throw;
  } catch (const nclopf::DomainError& e) {
    g_err = e.what();
    return NCL_E_DOMAIN;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return NCL_E_INVALID;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return NCL_E_LOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NCL_E_INTERNAL;
  }
}

#define GUARD(...)       \
  try {                  \
    __VA_ARGS__;         \
  } catch (...) {        \
    return map_exc();    \
  }                      \
  return NCL_OK;

nclopf::Expr build_expr(int nn, const ncl_expr_node* nodes) {
  // Replays the node list through the reference's smart constructors
  // (proj/src/expr.cpp:38-93) so folding is identical to hand-built Exprs.
  std::vector<nclopf::Expr> e(nn);
  for (int k = 0; k < nn; ++k) {
    const ncl_expr_node& n = nodes[k];
    switch (n.op) {
      case NCL_OP_CONST: e[k] = nclopf::Expr::constant(n.value); break;
      case NCL_OP_VAR: e[k] = nclopf::Expr::var(n.slot); break;
      case NCL_OP_PARAM: e[k] = nclopf::Expr::param(n.slot); break;
      case NCL_OP_ADD: e[k] = e[n.a] + e[n.b]; break;
      case NCL_OP_SUB: e[k] = e[n.a] - e[n.b]; break;
      case NCL_OP_MUL: e[k] = e[n.a] * e[n.b]; break;
      case NCL_OP_DIV: e[k] = e[n.a] / e[n.b]; break;
      case NCL_OP_POW: e[k] = pow(e[n.a], n.value); break;
      case NCL_OP_NEG: e[k] = -e[n.a]; break;
      case NCL_OP_SIN: e[k] = sin(e[n.a]); break;
      case NCL_OP_COS: e[k] = cos(e[n.a]); break;
      default: throw std::invalid_argument("expr program: bad op");
    }
  }
  return e[nn - 1];
}
}  // namespace

REF_API const char* ref_last_error() { return g_err.c_str(); }

// ---------------- SparseSym (proj/src/sparse_sym.cpp:12-131) ----------------
REF_API void* ref_sym_new(int n) { return new nclopf::SparseSym(n); }
REF_API void ref_sym_free(void* h) { delete static_cast<nclopf::SparseSym*>(h); }
REF_API int ref_sym_add_many(void* h, int64_t nt, const int* r, const int* c, const double* v) {
  auto* M = static_cast<nclopf::SparseSym*>(h);
  GUARD(for (int64_t k = 0; k < nt; ++k) M->add(r[k], c[k], v[k]));
}
REF_API int ref_sym_finalize(void* h) { GUARD(static_cast<nclopf::SparseSym*>(h)->finalize()); }
REF_API int ref_sym_begin_refill(void* h) { GUARD(static_cast<nclopf::SparseSym*>(h)->begin_refill()); }
REF_API int ref_sym_refill(void* h) { GUARD(static_cast<nclopf::SparseSym*>(h)->refill()); }
REF_API int ref_sym_dim(void* h) { return static_cast<nclopf::SparseSym*>(h)->dim(); }
REF_API int ref_sym_nnz(void* h) { return static_cast<nclopf::SparseSym*>(h)->nnz(); }
REF_API void ref_sym_get_csc(void* h, int* colptr, int* rowind, double* vals) {
  auto* M = static_cast<nclopf::SparseSym*>(h);
  if (colptr) std::memcpy(colptr, M->col_ptr().data(), sizeof(int) * M->col_ptr().size());
  if (rowind) std::memcpy(rowind, M->row_ind().data(), sizeof(int) * M->row_ind().size());
  if (vals) std::memcpy(vals, M->values().data(), sizeof(double) * M->values().size());
}
REF_API double ref_sym_max_abs_diag(void* h) { return static_cast<nclopf::SparseSym*>(h)->max_abs_diag(); }
REF_API double ref_sym_norm_inf(void* h) { return static_cast<nclopf::SparseSym*>(h)->norm_inf(); }
REF_API double ref_sym_frobenius(void* h) { return static_cast<nclopf::SparseSym*>(h)->frobenius_norm(); }
REF_API int ref_sym_multiply(void* h, const double* x, double* y) {
  auto* M = static_cast<nclopf::SparseSym*>(h);
  const int n = M->dim();
  GUARD(M->multiply(std::span<const double>(x, n), std::span<double>(y, n)));
}
REF_API int ref_sym_write_mm(void* h, char* buf, int64_t cap, int64_t* len) {
  std::ostringstream os;
  GUARD({
    static_cast<nclopf::SparseSym*>(h)->write_matrix_market(os);
    const std::string s = os.str();
    *len = static_cast<int64_t>(s.size());
    if (buf && cap > 0) std::memcpy(buf, s.data(), std::min<int64_t>(cap, *len));
  });
}

// ---------------- symbolic_order / analyze (proj/src/sparse_sym.cpp:139-262) ----
REF_API int ref_symbolic_order(void* h, int* perm) {
  GUARD({
    auto p = nclopf::symbolic_order(*static_cast<nclopf::SparseSym*>(h));
    std::memcpy(perm, p.data(), sizeof(int) * p.size());
  });
}
REF_API int ref_analyze(void* h, const int* perm, void** out) {
  auto* M = static_cast<nclopf::SparseSym*>(h);
  GUARD({
    nclopf::SymbolicFactor S =
        perm ? nclopf::analyze(*M, std::vector<int>(perm, perm + M->dim())) : nclopf::analyze(*M);
    *out = new nclopf::SymbolicFactor(std::move(S));
  });
}
REF_API void ref_symb_free(void* s) { delete static_cast<nclopf::SymbolicFactor*>(s); }
REF_API int64_t ref_symb_lnnz(void* s) { return static_cast<nclopf::SymbolicFactor*>(s)->l_nnz; }
REF_API void ref_symb_get(void* s, int* perm, int* iperm, int* parent, int* up_colptr,
                          int* up_rowind, int* entry_map, int* l_colcount) {
  auto* S = static_cast<nclopf::SymbolicFactor*>(s);
  auto cp = [](int* dst, const std::vector<int>& v) {
    if (dst) std::memcpy(dst, v.data(), sizeof(int) * v.size());
  };
  cp(perm, S->perm);
  cp(iperm, S->iperm);
  cp(parent, S->parent);
  cp(up_colptr, S->up_colptr);
  cp(up_rowind, S->up_rowind);
  cp(entry_map, S->entry_map);
  cp(l_colcount, S->l_colcount);
}

// ---------------- factorize / solve (proj/src/sparse_sym.cpp:268-401) --------
REF_API int ref_factorize(void* h, void* s, double pivot_tol, void** out) {
  auto* M = static_cast<nclopf::SparseSym*>(h);
  GUARD({
    if (s)
      *out = new nclopf::Factorization(
          nclopf::factorize(*M, *static_cast<nclopf::SymbolicFactor*>(s), pivot_tol));
    else
      *out = new nclopf::Factorization(nclopf::factorize(*M, pivot_tol));
  });
}
REF_API void ref_fact_free(void* f) { delete static_cast<nclopf::Factorization*>(f); }
REF_API int ref_fact_status(void* f, int* zero_pivot_index, int* npos, int* nneg, int* nzero) {
  auto* F = static_cast<nclopf::Factorization*>(f);
  *zero_pivot_index = F->zero_pivot_index;
  *npos = F->inertia.n_pos;
  *nneg = F->inertia.n_neg;
  *nzero = F->inertia.n_zero;
  return F->ok() ? 0 : 1;
}
REF_API void ref_fact_diag(void* f, double* d) {
  auto* F = static_cast<nclopf::Factorization*>(f);
  std::memcpy(d, F->diagonal().data(), sizeof(double) * F->diagonal().size());
}
// test-only: L in CSC over permuted indices (lp_/li_/lx_, sparse_sym.hpp:119-120)
REF_API void ref_fact_get_L(void* f, int* lp, int* li, double* lx) {
  auto* F = static_cast<nclopf::Factorization*>(f);
  if (lp) std::memcpy(lp, F->lp_.data(), sizeof(int) * F->lp_.size());
  if (li) std::memcpy(li, F->li_.data(), sizeof(int) * F->li_.size());
  if (lx) std::memcpy(lx, F->lx_.data(), sizeof(double) * F->lx_.size());
}
REF_API int ref_fact_solve_in_place(void* f, double* x, int n) {
  GUARD(static_cast<nclopf::Factorization*>(f)->solve_in_place(std::span<double>(x, n)));
}
REF_API int ref_solve_refined(void* f, void* h, const double* b, double target, int max_sweeps,
                              double* x, double* residual, int* sweeps, int* converged) {
  auto* F = static_cast<nclopf::Factorization*>(f);
  auto* M = static_cast<nclopf::SparseSym*>(h);
  GUARD({
    auto R = nclopf::solve_refined(*F, *M, std::span<const double>(b, M->dim()), target, max_sweeps);
    std::memcpy(x, R.x.data(), sizeof(double) * R.x.size());
    *residual = R.residual;
    *sweeps = R.sweeps;
    *converged = R.converged ? 1 : 0;
  });
}

// ---------------- model_ad (proj/src/model.cpp, proj/src/expr.cpp) ----------
REF_API void* ref_mb_new(int nvars) { return new nclopf::ModelBuilder(nvars); }
REF_API void ref_mb_free(void* b) { delete static_cast<nclopf::ModelBuilder*>(b); }
REF_API int ref_mb_add_template(void* b, int nn, const ncl_expr_node* nodes, int nslots,
                                const char* name, int* id) {
  GUARD({
    nclopf::ExpressionTemplate t(build_expr(nn, nodes), nslots, name ? name : "");
    *id = static_cast<nclopf::ModelBuilder*>(b)->add_template(std::move(t));
  });
}
REF_API int ref_mb_add_rows(void* b, int count) { return static_cast<nclopf::ModelBuilder*>(b)->add_rows(count); }
REF_API int ref_mb_add_terms(void* b, int tid, int objective, int64_t count, int nv, const int* vars,
                             int np, const double* params, const int* rows) {
  auto* B = static_cast<nclopf::ModelBuilder*>(b);
  GUARD({
    for (int64_t k = 0; k < count; ++k) {
      std::vector<int> v(vars + k * nv, vars + (k + 1) * nv);
      std::vector<double> p;
      if (np > 0) p.assign(params + k * np, params + (k + 1) * np);
      if (objective)
        B->add_objective_term(tid, std::move(v), std::move(p));
      else
        B->add_constraint_term(tid, rows[k], std::move(v), std::move(p));
    }
  });
}
REF_API int ref_mb_build(void* b, void** out) {
  auto* B = static_cast<nclopf::ModelBuilder*>(b);
  GUARD(*out = new nclopf::ModelFunctions(std::move(*B).build()));
}
REF_API void ref_mf_free(void* m) { delete static_cast<nclopf::ModelFunctions*>(m); }
REF_API void ref_mf_sizes(void* m, int* n, int* mm, int64_t* nnzj, int64_t* nnzh) {
  auto* M = static_cast<nclopf::ModelFunctions*>(m);
  *n = M->num_vars();
  *mm = M->num_cons();
  *nnzj = static_cast<int64_t>(M->jac_coords().size());
  *nnzh = static_cast<int64_t>(M->hess_coords().size());
}
REF_API void ref_mf_jac_coords(void* m, int* rows, int* cols) {
  const auto& jc = static_cast<nclopf::ModelFunctions*>(m)->jac_coords();
  for (size_t k = 0; k < jc.size(); ++k) rows[k] = jc[k].first, cols[k] = jc[k].second;
}
REF_API void ref_mf_hess_coords(void* m, int* rows, int* cols) {
  const auto& hc = static_cast<nclopf::ModelFunctions*>(m)->hess_coords();
  for (size_t k = 0; k < hc.size(); ++k) rows[k] = hc[k].first, cols[k] = hc[k].second;
}
REF_API int ref_mf_eval_objective(void* m, const double* w, double* out) {
  auto* M = static_cast<nclopf::ModelFunctions*>(m);
  GUARD(*out = M->eval_objective(std::span<const double>(w, M->num_vars())));
}
REF_API int ref_mf_eval_grad(void* m, const double* w, double* g) {
  auto* M = static_cast<nclopf::ModelFunctions*>(m);
  const int n = M->num_vars();
  GUARD(M->eval_grad_objective(std::span<const double>(w, n), std::span<double>(g, n)));
}
REF_API int ref_mf_eval_cons(void* m, const double* w, double* c) {
  auto* M = static_cast<nclopf::ModelFunctions*>(m);
  GUARD(M->eval_constraints(std::span<const double>(w, M->num_vars()),
                            std::span<double>(c, M->num_cons())));
}
REF_API int ref_mf_eval_jac(void* m, const double* w, double* vals) {
  auto* M = static_cast<nclopf::ModelFunctions*>(m);
  GUARD(M->eval_jacobian(std::span<const double>(w, M->num_vars()),
                         std::span<double>(vals, M->jac_coords().size())));
}
REF_API int ref_mf_eval_hess(void* m, const double* w, double sigma, const double* lam, double* vals) {
  auto* M = static_cast<nclopf::ModelFunctions*>(m);
  GUARD(M->eval_hessian_lag(std::span<const double>(w, M->num_vars()), sigma,
                            std::span<const double>(lam, M->num_cons()),
                            std::span<double>(vals, M->hess_coords().size())));
}
REF_API int ref_mf_jac_times(void* m, const double* jv, const double* v, double* out) {
  auto* M = static_cast<nclopf::ModelFunctions*>(m);
  GUARD(M->jac_times(std::span<const double>(jv, M->jac_coords().size()),
                     std::span<const double>(v, M->num_vars()), std::span<double>(out, M->num_cons())));
}
REF_API int ref_mf_jac_trans_times(void* m, const double* jv, const double* y, double* out) {
  auto* M = static_cast<nclopf::ModelFunctions*>(m);
  GUARD(M->jac_trans_times(std::span<const double>(jv, M->jac_coords().size()),
                           std::span<const double>(y, M->num_cons()),
                           std::span<double>(out, M->num_vars())));
}
REF_API int ref_mf_fd_check(void* m, const double* w, unsigned seed, double tol, double* errs, int* pass) {
  auto* M = static_cast<nclopf::ModelFunctions*>(m);
  GUARD({
    auto r = nclopf::fd_check(*M, std::span<const double>(w, M->num_vars()), seed, tol);
    errs[0] = r.grad_err;
    errs[1] = r.jac_err;
    errs[2] = r.hess_err;
    *pass = r.pass ? 1 : 0;
  });
}
