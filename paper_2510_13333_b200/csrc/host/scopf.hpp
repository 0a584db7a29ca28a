// Corrective AC-SCOPF with complementarity recourse (paper Eq. 2-4,
// /root/reference/PAPER.md:108-187), emitted as a neutral
// "model spec": template node programs + instance tables + bounds. Both the
// product (GPU ModelBuilder) and the oracle (reference ModelBuilder, compiled
// in oracle/_ref) build their ModelFunctions from the SAME spec, so the two
// evaluate identical models.
//
// Layout = the paper's ExaModels layout, fitted in SURVEY.md §8(d):
//   nvar(K) = B + K(B + 1 + 4 n_g),  B = 2 n_b + 2 n_g + 4 n_l
//   ncon(K) = C + K(C + 6 n_g - 2),  C = 1 + 2 n_b + 6 n_l
// Per scenario: v, theta, p_g, q_g, branch flows (p_f, q_f, p_t, q_t);
// per contingency additionally Delta, pi+, pi-, nu+, nu- (per generator).
// Rows: reference angle, 4 n_l flow definitions, 2 n_b balances, 2 n_l
// apparent-power limits (the outaged line's two are dropped), n_g AGC rows
// (Eq. 2), n_g PV/PQ rows (Eq. 3) and 4 n_g complementarity products
// written as c(w) <= 0 (vertical form after NCL relaxation W1 W2 e <= t).
// Standalone: depends only on the C node-program header.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../../include/nclopf_expr_program.h"

namespace nclb {

struct Grid {
  std::string name;
  int nb = 0, nl = 0, ng = 0, ref = 0;
  double base_mva = 100.0;
  std::vector<double> pd, qd, gs, bs, vmin, vmax;       // per bus (pu)
  std::vector<int> f, t;                                // per branch
  std::vector<double> r, x, b, rate, tap, shift;        // pu, rate in pu MVA
  std::vector<int> gbus;                                // per generator
  std::vector<double> pmin, pmax, qmin, qmax, c2, c1, c0;  // pu; cost in $/h with p in pu
};

// MATPOWER case9 (standard data, typed in).
Grid grid_case9();
// Seeded geometric grid (SURVEY.md §8(d) recommended generator).
Grid grid_synthetic(int nb, int nl, int ng, uint64_t seed);

// Non-islanding line outages in ascending branch order (union-find).
std::vector<int> select_contingencies(const Grid& g, int K);

// Contingency ids: id = l + nl * j is the outage of branch l with every
// post-contingency load (P and Q) scaled by contingency_load_scale(j), j <
// kLoadLevels. j = 0 is the plain N-1 outage. The other
// levels are outage x load-scenario pairs. They exist because a 597-branch
// grid has only 258 non-islanding single outages, while BASELINE.json's
// 500-bus x 1024 configuration needs 1024 contingencies. The scenario model is
// the same (Eq. 2-4) and the layout (nvar/ncon per
// contingency) does not change.
constexpr int kLoadLevels = 4;
inline double contingency_load_scale(int j) { return 1.0 - 0.015 * j; }

struct SpecFamily {
  std::string name;
  int nslots = 0, np = 0;
  bool objective = false;
  std::vector<ncl_expr_node> nodes;
  std::vector<int> rows;      // [ninst] (objective: empty)
  std::vector<int> vars;      // [ninst][nslots]
  std::vector<double> params; // [ninst][np]
  int64_t ninst() const { return nslots ? static_cast<int64_t>(vars.size()) / nslots : static_cast<int64_t>(rows.size()); }
};

struct ModelSpec {
  int n = 0, m = 0;
  std::vector<SpecFamily> fams;
  std::vector<double> xl, xu, x0;  // variable bounds and start
  std::vector<double> gl, gu;      // row bounds (gl == gu: equality)
  // metadata
  int nb = 0, nl = 0, ng = 0, K = 0;
  int nvar_scen = 0, ncon_scen = 0;
  std::vector<int> contingencies;
  std::vector<int> comp_rows;  // rows of complementarity products
  // pair i of row comp_rows[i]: w1 = x[comp_w1[i]] (>= 0), w2 = side * (x[comp_x[i]] - comp_bound[i])
  // (side -1: the upper limit ub - x, +1: the lower limit x - lb), row = w1 * w2 <= 0
  std::vector<int> comp_w1, comp_x, comp_side;
  std::vector<double> comp_bound;
  // per-scenario variable offsets: v, theta, pg, qg, flows; contingency extras
  std::vector<int> off_v, off_th, off_pg, off_qg, off_fl, off_extra;
  std::vector<int> row_start;  // first row of each scenario
};

// contingencies: ids as above (branch + nl * load level)
ModelSpec build_scopf(const Grid& g, const std::vector<int>& contingencies);
// Screening system (Eq. 5): the contingency scenarios only, with the
// base set points fixed — pg0[ng] generator outputs and v0[nb] bus voltages
// (read at generator buses) of a solved base case — and no objective. The
// scenarios are independent blocks: one NCL solve screens them all, each
// block's |r|^2 (r on its rows) its infeasibility measure.
ModelSpec build_scopf(const Grid& g, const std::vector<int>& contingencies, const double* pg0, const double* v0);

}  // namespace nclb
