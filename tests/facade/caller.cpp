// A caller written against the REFERENCE API (/root/reference/proj/include/
// nclopf/{expr,model,sparse_sym}.hpp) and nothing else. tests/test_facade.py
// compiles this one source twice — against the reference headers + sources
// (oracle/_ref/facade_caller_ref) and against the B200 façade
// (include/nclopf_b200/nclopf/*.hpp + libnclopf_b200.so) — and compares the
// two outputs: the drop-in claim of INTEGRATION.md, checked by a compiler.
#include <cmath>
#include <cstdio>
#include <sstream>
#include <stdexcept>
#include <vector>

#include "nclopf/expr.hpp"
#include "nclopf/model.hpp"
#include "nclopf/sparse_sym.hpp"

using namespace nclopf;

static void vec(const char* k, const std::vector<double>& v) {
  std::printf("\"%s\": [", k);
  for (size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? ", " : "", v[i]);
  std::printf("],\n");
}
static void ivec(const char* k, const std::vector<int>& v) {
  std::printf("\"%s\": [", k);
  for (size_t i = 0; i < v.size(); ++i) std::printf("%s%d", i ? ", " : "", v[i]);
  std::printf("],\n");
}

int main() {
  // --- a 3-bus AC power-flow toy: variables v0..v2, t0..t2, p0, p1 --------
  const int nb = 3, nv = 2 * nb + 2;
  auto V = [](int i) { return i; };
  auto T = [nb](int i) { return nb + i; };
  ModelBuilder B(nv);
  // objective: c2 p^2 + c1 p (params c2, c1)
  const Expr p = Expr::var(0);
  const int cost = B.add_template(ExpressionTemplate(Expr::param(0) * pow(p, 2.0) + Expr::param(1) * p, 1, "cost"));
  // branch flow into bus i: vi vj (g cos(ti - tj) + b sin(ti - tj)) - g vi^2
  const Expr vi = Expr::var(0), vj = Expr::var(1), ti = Expr::var(2), tj = Expr::var(3);
  const Expr g = Expr::param(0), b = Expr::param(1);
  const int flow = B.add_template(
      ExpressionTemplate(vi * vj * (g * cos(ti - tj) + b * sin(ti - tj)) - g * pow(vi, 2.0), 4, "flow"));
  const int inj = B.add_template(ExpressionTemplate(-Expr::var(0), 1, "injection"));
  const int load = B.add_template(ExpressionTemplate(Expr::param(0) / Expr::var(0) + Expr::var(0), 1, "load"));
  const int r0 = B.add_rows(nb);
  const double gl[3] = {4.0, 3.0, 5.0}, bl[3] = {-12.0, -9.0, -15.0};
  const int fr[3] = {0, 1, 0}, to[3] = {1, 2, 2};
  for (int l = 0; l < 3; ++l) {
    B.add_constraint_term(flow, r0 + fr[l], {V(fr[l]), V(to[l]), T(fr[l]), T(to[l])}, {gl[l], bl[l]});
    B.add_constraint_term(flow, r0 + to[l], {V(to[l]), V(fr[l]), T(to[l]), T(fr[l])}, {gl[l], bl[l]});
  }
  B.add_constraint_term(inj, r0 + 0, {2 * nb});
  B.add_constraint_term(inj, r0 + 1, {2 * nb + 1});
  for (int i = 0; i < nb; ++i) B.add_constraint_term(load, r0 + i, {V(i)}, {0.3 + 0.1 * i});
  B.add_objective_term(cost, {2 * nb}, {0.11, 5.0});
  B.add_objective_term(cost, {2 * nb + 1}, {0.085, 1.2});
  // misuse is reported with the reference's exception types
  int caught = 0;
  try {
    B.add_objective_term(flow, {0, 1, 2, 3}, {1.0, 1.0});
  } catch (const std::logic_error&) {
    caught |= 1;
  }
  try {
    B.add_constraint_term(inj, 99, {0});
  } catch (const std::invalid_argument&) {
    caught |= 2;
  }
  ModelFunctions M = std::move(B).build();

  std::vector<double> w = {1.02, 0.98, 1.01, 0.0, -0.05, -0.03, 0.9, 0.7};
  std::vector<double> lam = {0.7, -0.4, 1.3};
  std::printf("{\n\"n\": %d, \"m\": %d, \"nnzj\": %zu, \"nnzh\": %zu, \"caught\": %d,\n", M.num_vars(), M.num_cons(),
              M.jac_coords().size(), M.hess_coords().size(), caught);
  std::printf("\"obj\": %.17g,\n", M.eval_objective(w));
  std::vector<double> grad(nv), c(nb), jac(M.jac_coords().size()), hess(M.hess_coords().size());
  M.eval_grad_objective(w, grad);
  M.eval_constraints(w, c);
  M.eval_jacobian(w, jac);
  M.eval_hessian_lag(w, 1.5, lam, hess);
  vec("grad", grad);
  vec("cons", c);
  vec("jac", jac);
  vec("hess", hess);
  std::vector<int> jr, jc, hr, hc;
  for (auto [r, cc] : M.jac_coords()) jr.push_back(r), jc.push_back(cc);
  for (auto [r, cc] : M.hess_coords()) hr.push_back(r), hc.push_back(cc);
  ivec("jac_rows", jr);
  ivec("jac_cols", jc);
  ivec("hess_rows", hr);
  ivec("hess_cols", hc);
  std::vector<double> jv(nb), jty(nv), ones(nv, 1.0);
  M.jac_times(jac, ones, jv);
  M.jac_trans_times(jac, lam, jty);
  vec("jv", jv);
  vec("jty", jty);
  const FdReport fd = fd_check(M, w, 7u);
  std::printf("\"fd_pass\": %d,\n", fd.pass ? 1 : 0);

  // --- condensed Newton matrix H + I + 10 J^T J through SparseSym ----------
  SparseSym K(nv);
  const auto& hco = M.hess_coords();
  for (size_t k = 0; k < hco.size(); ++k) K.add(hco[k].first, hco[k].second, hess[k]);
  for (int i = 0; i < nv; ++i) K.add(i, i, 1.0 + 0.25 * i);
  const auto& jco = M.jac_coords();
  for (size_t a = 0; a < jco.size(); ++a)
    for (size_t bb = 0; bb <= a; ++bb)
      if (jco[a].first == jco[bb].first) {
        const int i = jco[a].second, j = jco[bb].second;
        K.add(std::max(i, j), std::min(i, j), 10.0 * jac[a] * jac[bb]);
      }
  K.finalize();
  try {
    K.finalize();
  } catch (const std::logic_error&) {
    caught |= 4;
  }
  try {
    K.add(0, 1, 1.0);  // upper triangle
  } catch (const std::invalid_argument&) {
    caught |= 8;
  }
  std::printf("\"caught_after_finalize\": %d, \"nnzK\": %d,\n", caught, K.nnz());
  std::printf("\"max_abs_diag\": %.17g, \"norm_inf\": %.17g, \"frobenius\": %.17g,\n", K.max_abs_diag(),
              K.norm_inf(), K.frobenius_norm());
  std::vector<double> Kx(nv);
  K.multiply(ones, Kx);
  vec("K_times_ones", Kx);
  ivec("col_ptr", K.col_ptr());
  ivec("row_ind", K.row_ind());
  vec("values", K.values());
  std::ostringstream mm;
  K.write_matrix_market(mm);
  std::printf("\"mm_bytes\": %zu,\n", mm.str().size());
  const std::vector<int> perm = symbolic_order(K);
  ivec("perm", perm);
  const SymbolicFactor S = analyze(K);
  ivec("parent", S.parent);
  ivec("l_colcount", S.l_colcount);
  ivec("entry_map", S.entry_map);
  std::printf("\"l_nnz\": %lld,\n", static_cast<long long>(S.l_nnz));
  const Factorization F = factorize(K, S);
  std::printf("\"status_ok\": %d, \"zpi\": %d, \"inertia\": [%d, %d, %d],\n", F.ok() ? 1 : 0, F.zero_pivot_index,
              F.inertia.n_pos, F.inertia.n_neg, F.inertia.n_zero);
  vec("D", F.diagonal());
  std::vector<double> rhs(nv);
  for (int i = 0; i < nv; ++i) rhs[i] = std::sin(1.0 + i);
  vec("x", F.solve(rhs));
  const RefinedSolve R = solve_refined(F, K, rhs);
  vec("x_refined", R.x);
  std::printf("\"refined_converged\": %d, \"refined_sweeps\": %d,\n", R.converged ? 1 : 0, R.sweeps);
  const Factorization F2 = factorize(K);  // owning overload
  std::printf("\"owning_same_perm\": %d,\n", F2.symbolic()->perm == S.perm ? 1 : 0);

  // --- an indefinite KKT (saddle point) and a zero pivot -------------------
  SparseSym Q(3);
  Q.add(0, 0, 2.0);
  Q.add(1, 1, 3.0);
  Q.add(2, 0, 1.0);
  Q.add(2, 1, 1.0);
  Q.add(2, 2, -1e-8);
  Q.finalize();
  const Factorization FQ = factorize(Q);
  std::printf("\"kkt_inertia\": [%d, %d, %d],\n", FQ.inertia.n_pos, FQ.inertia.n_neg, FQ.inertia.n_zero);
  SparseSym Z(3);
  Z.add(0, 0, 1.0);
  Z.add(1, 0, 1.0);
  Z.add(1, 1, 1.0);
  Z.add(2, 2, 4.0);
  Z.finalize();
  const Factorization FZ = factorize(Z);
  std::printf("\"zero_pivot_status\": %d, \"zero_pivot_index\": %d\n}\n",
              FZ.status == FactorizeStatus::zero_pivot ? 1 : 0, FZ.zero_pivot_index);
  return 0;
}
