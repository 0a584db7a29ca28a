#include "scopf.hpp"

#include <algorithm>
#include <cmath>
#include <complex>
#include <limits>
#include <numeric>
#include <stdexcept>

namespace nclb {

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

// splitmix64: portable, seed-stable stream (same numbers on every compiler)
struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double uniform() { return (next() >> 11) * (1.0 / 9007199254740992.0); }
  double uniform(double a, double b) { return a + (b - a) * uniform(); }
};

struct NB {  // node-program builder
  std::vector<ncl_expr_node> n;
  int push(int op, int a, int b, int slot, double v) {
    n.push_back(ncl_expr_node{op, a, b, slot, v});
    return static_cast<int>(n.size()) - 1;
  }
  int c(double v) { return push(NCL_OP_CONST, -1, -1, -1, v); }
  int var(int s) { return push(NCL_OP_VAR, -1, -1, s, 0.0); }
  int par(int s) { return push(NCL_OP_PARAM, -1, -1, s, 0.0); }
  int add(int a, int b) { return push(NCL_OP_ADD, a, b, -1, 0.0); }
  int sub(int a, int b) { return push(NCL_OP_SUB, a, b, -1, 0.0); }
  int mul(int a, int b) { return push(NCL_OP_MUL, a, b, -1, 0.0); }
  int neg(int a) { return push(NCL_OP_NEG, a, -1, -1, 0.0); }
  int sin_(int a) { return push(NCL_OP_SIN, a, -1, -1, 0.0); }
  int cos_(int a) { return push(NCL_OP_COS, a, -1, -1, 0.0); }
};

struct UF {
  std::vector<int> p;
  explicit UF(int n) : p(n) { std::iota(p.begin(), p.end(), 0); }
  int find(int x) {
    while (p[x] != x) x = p[x] = p[p[x]];
    return x;
  }
  bool unite(int a, int b) {
    a = find(a);
    b = find(b);
    if (a == b) return false;
    p[a] = b;
    return true;
  }
};

struct BranchY {
  double gff, bff, gft, bft, gtf, btf, gtt, btt;
};
BranchY branch_y(const Grid& g, int l) {
  using cd = std::complex<double>;
  const cd ys = 1.0 / cd(g.r[l], g.x[l]);
  const double tau = g.tap[l] == 0.0 ? 1.0 : g.tap[l];
  const cd t = std::polar(tau, g.shift[l] * M_PI / 180.0);
  const cd ych(0.0, g.b[l] / 2.0);
  const cd yff = (ys + ych) / (tau * tau);
  const cd ytt = ys + ych;
  const cd yft = -ys / std::conj(t);
  const cd ytf = -ys / t;
  return {yff.real(), yff.imag(), yft.real(), yft.imag(), ytf.real(), ytf.imag(), ytt.real(), ytt.imag()};
}

// DC power flow angles with generation proportional to pmax (CG on the
// reduced Laplacian), optionally with branch `out` removed. Deterministic.
std::vector<double> dc_angles(const Grid& g, int out = -1, const std::vector<double>* warm = nullptr) {
  const int n = g.nb;
  std::vector<double> P(n, 0.0);
  double pd = 0, pm = 0;
  for (int i = 0; i < n; ++i) pd += g.pd[i];
  for (int k = 0; k < g.ng; ++k) pm += g.pmax[k];
  for (int k = 0; k < g.ng; ++k) P[g.gbus[k]] += g.pmax[k] * pd / pm;
  for (int i = 0; i < n; ++i) P[i] -= g.pd[i];
  auto apply = [&](const std::vector<double>& th, std::vector<double>& y) {
    std::fill(y.begin(), y.end(), 0.0);
    for (int l = 0; l < g.nl; ++l) {
      if (l == out) continue;
      const double w = 1.0 / g.x[l];
      const double d = th[g.f[l]] - th[g.t[l]];
      y[g.f[l]] += w * d;
      y[g.t[l]] -= w * d;
    }
    y[g.ref] = th[g.ref];  // pin the reference angle
  };
  std::vector<double> th(n, 0.0), r(P), p, Ap(n);
  r[g.ref] = 0.0;
  double pp = 0;
  for (double v : r) pp += v * v;
  if (warm) {  // start from the base-case angles: the outage perturbs them locally
    th = *warm;
    apply(th, Ap);
    for (int i = 0; i < n; ++i) r[i] = (i == g.ref ? 0.0 : P[i]) - Ap[i];
    r[g.ref] = -th[g.ref];
  }
  p = r;
  double rr = 0;
  for (double v : r) rr += v * v;
  const double stop = std::max(1e-24, 1e-24 * pp);
  for (int it = 0; it < 20 * n && rr > stop; ++it) {
    apply(p, Ap);
    double pAp = 0;
    for (int i = 0; i < n; ++i) pAp += p[i] * Ap[i];
    const double a = rr / pAp;
    double rr2 = 0;
    for (int i = 0; i < n; ++i) {
      th[i] += a * p[i];
      r[i] -= a * Ap[i];
      rr2 += r[i] * r[i];
    }
    const double beta = rr2 / rr;
    rr = rr2;
    for (int i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
  }
  return th;
}

}  // namespace

Grid grid_case9() {
  Grid g;
  g.name = "case9";
  g.nb = 9;
  g.nl = 9;
  g.ng = 3;
  g.ref = 0;
  g.base_mva = 100.0;
  const double B = g.base_mva;
  g.pd = {0, 0, 0, 0, 90 / B, 0, 100 / B, 0, 125 / B};
  g.qd = {0, 0, 0, 0, 30 / B, 0, 35 / B, 0, 50 / B};
  g.gs.assign(9, 0.0);
  g.bs.assign(9, 0.0);
  g.vmin.assign(9, 0.9);
  g.vmax.assign(9, 1.1);
  const int F[9] = {1, 4, 5, 3, 6, 7, 8, 8, 9}, T[9] = {4, 5, 6, 6, 7, 8, 2, 9, 4};
  const double R[9] = {0, 0.017, 0.039, 0, 0.0119, 0.0085, 0, 0.032, 0.01};
  const double X[9] = {0.0576, 0.092, 0.17, 0.0586, 0.1008, 0.072, 0.0625, 0.161, 0.085};
  const double Bc[9] = {0, 0.158, 0.358, 0, 0.209, 0.149, 0, 0.306, 0.176};
  const double RATE[9] = {250, 250, 150, 300, 150, 250, 250, 250, 250};
  for (int l = 0; l < 9; ++l) {
    g.f.push_back(F[l] - 1);
    g.t.push_back(T[l] - 1);
    g.r.push_back(R[l]);
    g.x.push_back(X[l]);
    g.b.push_back(Bc[l]);
    g.rate.push_back(RATE[l] / B);
    g.tap.push_back(1.0);
    g.shift.push_back(0.0);
  }
  g.gbus = {0, 1, 2};
  g.pmin = {10 / B, 10 / B, 10 / B};
  g.pmax = {250 / B, 300 / B, 270 / B};
  g.qmin = {-300 / B, -300 / B, -300 / B};
  g.qmax = {300 / B, 300 / B, 300 / B};
  // gencost (MW based) -> p in pu
  const double c2[3] = {0.11, 0.085, 0.1225}, c1[3] = {5, 1.2, 1}, c0[3] = {150, 600, 335};
  for (int k = 0; k < 3; ++k) {
    g.c2.push_back(c2[k] * B * B);
    g.c1.push_back(c1[k] * B);
    g.c0.push_back(c0[k]);
  }
  return g;
}

Grid grid_synthetic(int nb, int nl, int ng, uint64_t seed) {
  if (nb < 2 || nl < nb - 1 || ng < 1 || ng > nb) throw std::invalid_argument("grid_synthetic: bad sizes");
  Grid g;
  g.name = "synthetic_" + std::to_string(nb) + "_" + std::to_string(nl) + "_" + std::to_string(ng);
  g.nb = nb;
  g.ng = ng;
  Rng rng(seed);
  std::vector<double> px(nb), py(nb);
  for (int i = 0; i < nb; ++i) {
    px[i] = rng.uniform();
    py[i] = rng.uniform();
  }
  auto dist = [&](int i, int j) { return std::hypot(px[i] - px[j], py[i] - py[j]); };
  // Euclidean MST (Prim, O(n^2))
  std::vector<std::pair<int, int>> edges;
  {
    std::vector<double> best(nb, kInf);
    std::vector<int> from(nb, -1);
    std::vector<char> in(nb, 0);
    best[0] = 0;
    for (int it = 0; it < nb; ++it) {
      int u = -1;
      for (int i = 0; i < nb; ++i)
        if (!in[i] && (u < 0 || best[i] < best[u])) u = i;
      if (u < 0) break;
      in[u] = 1;
      if (from[u] >= 0) edges.emplace_back(std::min(u, from[u]), std::max(u, from[u]));
      for (int i = 0; i < nb; ++i)
        if (!in[i] && dist(u, i) < best[i]) {
          best[i] = dist(u, i);
          from[i] = u;
        }
    }
  }
  // leaf-pairing chords: an MST leaf's only line is a bridge (its outage
  // islands the bus). Pair leaves greedily by distance so each chord closes a
  // short cycle through both; ACTIVSg-size grids then admit >= 256
  // non-islanding line outages like the real cases do.
  {
    std::vector<int> deg0(nb, 0);
    for (const auto& e : edges) deg0[e.first]++, deg0[e.second]++;
    std::vector<int> leaves;
    for (int i = 0; i < nb; ++i)
      if (deg0[i] == 1) leaves.push_back(i);
    std::vector<std::pair<double, std::pair<int, int>>> lp;
    for (size_t a = 0; a < leaves.size(); ++a)
      for (size_t b = a + 1; b < leaves.size(); ++b)
        lp.push_back({dist(leaves[a], leaves[b]), {leaves[a], leaves[b]}});
    std::sort(lp.begin(), lp.end());
    std::vector<char> used(nb, 0);
    const int budget = (nl - static_cast<int>(edges.size())) * 3 / 4;
    int added = 0;
    for (const auto& c : lp) {
      if (added >= budget) break;
      const int u = c.second.first, v = c.second.second;
      if (used[u] || used[v]) continue;
      used[u] = used[v] = 1;
      edges.emplace_back(u, v);
      ++added;
    }
  }
  // nearest-neighbour chords (8-NN candidates, shortest first)
  {
    std::vector<std::pair<double, std::pair<int, int>>> cand;
    std::vector<int> idx(nb);
    for (int i = 0; i < nb; ++i) {
      std::iota(idx.begin(), idx.end(), 0);
      const int k = std::min(9, nb);
      std::partial_sort(idx.begin(), idx.begin() + k, idx.end(), [&](int a, int b) {
        const double da = dist(i, a), db = dist(i, b);
        return da != db ? da < db : a < b;
      });
      for (int q = 0; q < k; ++q)
        if (idx[q] != i) cand.push_back({dist(i, idx[q]), {std::min(i, idx[q]), std::max(i, idx[q])}});
    }
    std::sort(cand.begin(), cand.end());
    std::vector<std::pair<int, int>> have(edges.begin(), edges.end());
    std::sort(have.begin(), have.end());
    for (const auto& c : cand) {
      if (static_cast<int>(edges.size()) >= nl) break;
      if (std::binary_search(have.begin(), have.end(), c.second)) continue;
      edges.push_back(c.second);
      have.insert(std::lower_bound(have.begin(), have.end(), c.second), c.second);
    }
  }
  g.nl = static_cast<int>(edges.size());
  for (const auto& e : edges) {
    const double d = dist(e.first, e.second);
    const double x = 0.01 + 0.3 * d;
    g.f.push_back(e.first);
    g.t.push_back(e.second);
    g.x.push_back(x);
    g.r.push_back(x / 8.0);
    g.b.push_back(0.02 * d);
    g.tap.push_back(1.0);
    g.shift.push_back(0.0);
  }
  g.pd.assign(nb, 0.0);
  g.qd.assign(nb, 0.0);
  for (int i = 0; i < nb; ++i)
    if (rng.uniform() < 0.8) {
      // ~0.19 pu mean per bus: ACTIVSg500 carries ~7.75 GW on 500 buses; the
      // survey's U(0.2, 1.0) loads 3x heavier and leaves N-1 reactive
      // balances infeasible at |v| in [0.94, 1.06].
      g.pd[i] = rng.uniform(0.05, 0.33);
      g.qd[i] = 0.3 * g.pd[i];
    }
  g.gs.assign(nb, 0.0);
  // switched-shunt compensation of the load's reactive demand (like the
  // ACTIVSg cases' shunts): without it reactive power cannot reach load
  // pockets far from the 56 generator buses inside |v| in [0.94, 1.06]
  g.bs.assign(nb, 0.0);
  for (int i = 0; i < nb; ++i) g.bs[i] = g.qd[i];
  g.vmin.assign(nb, 0.94);
  g.vmax.assign(nb, 1.06);
  // generators on the highest-degree buses
  std::vector<int> deg(nb, 0);
  for (int l = 0; l < g.nl; ++l) deg[g.f[l]]++, deg[g.t[l]]++;
  std::vector<int> order(nb);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return deg[a] > deg[b]; });
  double pdsum = 0;
  for (double v : g.pd) pdsum += v;
  std::vector<double> wgt(ng);
  double wsum = 0;
  for (int k = 0; k < ng; ++k) wsum += (wgt[k] = rng.uniform(0.5, 1.5));
  for (int k = 0; k < ng; ++k) {
    g.gbus.push_back(order[k]);
    const double pmax = 1.6 * pdsum * wgt[k] / wsum;
    g.pmin.push_back(0.0);
    g.pmax.push_back(pmax);
    g.qmin.push_back(-0.3 * pmax);
    g.qmax.push_back(0.5 * pmax);
    g.c2.push_back(rng.uniform(0.01, 0.1) * g.base_mva * g.base_mva);
    g.c1.push_back(rng.uniform(10.0, 40.0) * g.base_mva);
    g.c0.push_back(0.0);
  }
  g.ref = g.gbus[std::max_element(g.pmax.begin(), g.pmax.end()) - g.pmax.begin()];
  // Ratings: 1.2 x the largest |DC flow| over the base case and every
  // non-islanding single-branch outage, + 0.25 pu headroom for reactive flow.
  // (SURVEY.md §8(d)'s "1.5 x base DC flow + 0.1" leaves N-1 AC-infeasible
  // instances — the NCL penalty then diverges; this keeps every selectable
  // contingency feasible while the limits still bind near the N-1 maxima.)
  // Independent of K, so every config of one grid shares the same network.
  std::vector<double> fmax(g.nl, 0.0);
  auto absorb = [&](const std::vector<double>& th, int out) {
    for (int l = 0; l < g.nl; ++l)
      if (l != out) fmax[l] = std::max(fmax[l], std::abs((th[g.f[l]] - th[g.t[l]]) / g.x[l]));
  };
  const std::vector<double> th0 = dc_angles(g);
  absorb(th0, -1);
  // the first 600 non-islanding outages cover every config's contingency set
  for (int l : select_contingencies(g, std::min(g.nl, 600))) absorb(dc_angles(g, l, &th0), l);
  g.rate.resize(g.nl);
  for (int l = 0; l < g.nl; ++l) g.rate[l] = 1.2 * fmax[l] + 0.25;
  return g;
}

std::vector<int> select_contingencies(const Grid& g, int K) {
  std::vector<int> out;
  for (int l = 0; l < g.nl && static_cast<int>(out.size()) < K; ++l) {
    UF uf(g.nb);
    int comps = g.nb;
    for (int e = 0; e < g.nl; ++e)
      if (e != l && uf.unite(g.f[e], g.t[e])) comps--;
    if (comps == 1) out.push_back(l);
  }
  return out;
}

ModelSpec build_scopf(const Grid& g, const std::vector<int>& cont) { return build_scopf(g, cont, nullptr, nullptr); }

ModelSpec build_scopf(const Grid& g, const std::vector<int>& cont, const double* pg0, const double* v0) {
  // screening mode (pg0, v0 given, SPEC.md:264-271 / PAPER.md Eq. 5): no base
  // scenario; every contingency scenario with the base set points fixed as
  // constants (moved to the row bounds of its AGC and PV/PQ rows) and no
  // objective — a feasibility system per contingency, all of them side by
  // side in one problem
  const bool screen = pg0 != nullptr;
  ModelSpec S;
  const int nb = g.nb, nl = g.nl, ng = g.ng, K = static_cast<int>(cont.size());
  S.nb = nb;
  S.nl = nl;
  S.ng = ng;
  S.K = K;
  S.contingencies = cont;
  const int B = 2 * nb + 2 * ng + 4 * nl;
  S.nvar_scen = B;
  S.ncon_scen = 1 + 2 * nb + 6 * nl;

  // ---- templates
  enum { T_FP, T_FQ, T_PLUS, T_MINUS, T_SHUNT, T_SQ2, T_AGC, T_PVPQ, T_COMPU, T_COMPL, T_COST, T_AGCS, T_PVPQS, T_N };
  S.fams.resize(T_N);
  auto def = [&](int id, const char* name, int nslots, int np, bool obj, NB& nbld) {
    S.fams[id].name = name;
    S.fams[id].nslots = nslots;
    S.fams[id].np = np;
    S.fams[id].objective = obj;
    S.fams[id].nodes = nbld.n;
  };
  {
    // p - (gii vi^2 + vi vj (gij cos(ti-tj) + bij sin(ti-tj)))
    NB e;
    int p = e.var(0), vi = e.var(1), vj = e.var(2), ti = e.var(3), tj = e.var(4);
    int gii = e.par(0), gij = e.par(1), bij = e.par(2);
    int d = e.sub(ti, tj);
    int inner = e.add(e.mul(gij, e.cos_(d)), e.mul(bij, e.sin_(d)));
    int flow = e.add(e.mul(gii, e.mul(vi, vi)), e.mul(e.mul(vi, vj), inner));
    e.sub(p, flow);
    def(T_FP, "branch_flow_p", 5, 3, false, e);
  }
  {
    // q - (-bii vi^2 + vi vj (gij sin(ti-tj) - bij cos(ti-tj)))
    NB e;
    int q = e.var(0), vi = e.var(1), vj = e.var(2), ti = e.var(3), tj = e.var(4);
    int bii = e.par(0), gij = e.par(1), bij = e.par(2);
    int d = e.sub(ti, tj);
    int inner = e.sub(e.mul(gij, e.sin_(d)), e.mul(bij, e.cos_(d)));
    int flow = e.add(e.neg(e.mul(bii, e.mul(vi, vi))), e.mul(e.mul(vi, vj), inner));
    e.sub(q, flow);
    def(T_FQ, "branch_flow_q", 5, 3, false, e);
  }
  {
    NB e;
    e.var(0);
    def(T_PLUS, "plus", 1, 0, false, e);
  }
  {
    NB e;
    e.neg(e.var(0));
    def(T_MINUS, "minus", 1, 0, false, e);
  }
  {
    NB e;
    int v = e.var(0);
    e.mul(e.par(0), e.mul(v, v));
    def(T_SHUNT, "bus_shunt", 1, 1, false, e);
  }
  {
    NB e;
    int a = e.var(0), b = e.var(1);
    e.add(e.mul(a, a), e.mul(b, b));
    def(T_SQ2, "apparent_power_sq", 2, 0, false, e);
  }
  {
    // pi+ - pi- - p_k + p_0 + alpha Delta   (Eq. 2, first row)
    NB e;
    int pp = e.var(0), pm = e.var(1), pk = e.var(2), p0 = e.var(3), dl = e.var(4);
    e.add(e.add(e.sub(e.sub(pp, pm), pk), p0), e.mul(e.par(0), dl));
    def(T_AGC, "agc_droop", 5, 1, false, e);
  }
  {
    // nu+ - nu- - v_k + v_0   (Eq. 3, first row)
    NB e;
    int np_ = e.var(0), nm = e.var(1), vk = e.var(2), v0 = e.var(3);
    e.add(e.sub(e.sub(np_, nm), vk), v0);
    def(T_PVPQ, "pvpq_switch", 4, 0, false, e);
  }
  {
    // mult * (ub - x) <= 0
    NB e;
    int m = e.var(0), x = e.var(1);
    e.mul(m, e.sub(e.par(0), x));
    def(T_COMPU, "comp_upper", 2, 1, false, e);
  }
  {
    // mult * (x - lb) <= 0
    NB e;
    int m = e.var(0), x = e.var(1);
    e.mul(m, e.sub(x, e.par(0)));
    def(T_COMPL, "comp_lower", 2, 1, false, e);
  }
  {
    // screening: pi+ - pi- - p_k + alpha Delta (= -p_0, a row constant)
    NB e;
    int pp = e.var(0), pm = e.var(1), pk = e.var(2), dl = e.var(3);
    e.add(e.sub(e.sub(pp, pm), pk), e.mul(e.par(0), dl));
    def(T_AGCS, "agc_droop_fixed_base", 4, 1, false, e);
  }
  {
    // screening: nu+ - nu- - v_k (= -v_0)
    NB e;
    int np_ = e.var(0), nm = e.var(1), vk = e.var(2);
    e.sub(e.sub(np_, nm), vk);
    def(T_PVPQS, "pvpq_switch_fixed_base", 3, 0, false, e);
  }
  {
    // c2 p^2 + c1 p + c0
    NB e;
    int p = e.var(0);
    e.add(e.add(e.mul(e.par(0), e.mul(p, p)), e.mul(e.par(1), p)), e.par(2));
    def(T_COST, "generation_cost", 1, 3, true, e);
  }
  auto term = [&](int fam, int row, std::initializer_list<int> vars, std::initializer_list<double> params) {
    SpecFamily& f = S.fams[fam];
    if (!f.objective) f.rows.push_back(row);
    f.vars.insert(f.vars.end(), vars.begin(), vars.end());
    f.params.insert(f.params.end(), params.begin(), params.end());
  };

  // ---- variables
  const int nvar = (screen ? 0 : B) + K * (B + 1 + 4 * ng);
  S.n = nvar;
  S.xl.assign(nvar, -kInf);
  S.xu.assign(nvar, kInf);
  S.x0.assign(nvar, 0.0);
  std::vector<BranchY> Y(nl);
  for (int l = 0; l < nl; ++l) Y[l] = branch_y(g, l);
  int off = 0, row = 0;
  std::vector<double> gl, gu;
  auto newrow = [&](double lo, double hi) {
    gl.push_back(lo);
    gu.push_back(hi);
    return row++;
  };
  for (int s = screen ? 1 : 0; s <= K; ++s) {
    // contingency id = outaged branch + nl * load level (contingency_load_scale)
    if (s > 0 && (cont[s - 1] < 0 || cont[s - 1] / nl >= kLoadLevels))
      throw std::invalid_argument("build_scopf: contingency id out of range");
    const int out = s == 0 ? -1 : cont[s - 1] % nl;
    const double lsc = s == 0 ? 1.0 : contingency_load_scale(cont[s - 1] / nl);
    const int ov = off, oth = ov + nb, opg = oth + nb, oqg = opg + ng, ofl = oqg + ng;
    const int oex = ofl + 4 * nl;
    off = oex + (s == 0 ? 0 : 1 + 4 * ng);
    S.off_v.push_back(ov);
    S.off_th.push_back(oth);
    S.off_pg.push_back(opg);
    S.off_qg.push_back(oqg);
    S.off_fl.push_back(ofl);
    S.off_extra.push_back(s == 0 ? -1 : oex);
    S.row_start.push_back(row);
    for (int i = 0; i < nb; ++i) {
      // post-contingency states use the emergency band (+-0.04 pu wider);
      // SPEC.md:298 leaves the bound set on v^k open
      const double em = s == 0 ? 0.0 : 0.04;
      S.xl[ov + i] = g.vmin[i] - em;
      S.xu[ov + i] = g.vmax[i] + em;
      S.x0[ov + i] = std::min(std::max(1.0, g.vmin[i]), g.vmax[i]);
    }
    for (int k = 0; k < ng; ++k) {
      S.xl[opg + k] = g.pmin[k];
      S.xu[opg + k] = g.pmax[k];
      S.x0[opg + k] = 0.5 * (g.pmin[k] + g.pmax[k]);
      S.xl[oqg + k] = g.qmin[k];
      S.xu[oqg + k] = g.qmax[k];
      S.x0[oqg + k] = 0.5 * (g.qmin[k] + g.qmax[k]);
    }
    auto pf = [&](int l) { return ofl + l; };
    auto qf = [&](int l) { return ofl + nl + l; };
    auto pt = [&](int l) { return ofl + 2 * nl + l; };
    auto qt = [&](int l) { return ofl + 3 * nl + l; };
    // reference angle
    term(T_PLUS, newrow(0.0, 0.0), {oth + g.ref}, {});
    // flow definitions
    for (int l = 0; l < nl; ++l) {
      const int vf = ov + g.f[l], vt = ov + g.t[l], tf = oth + g.f[l], tt = oth + g.t[l];
      if (l == out) {
        term(T_PLUS, newrow(0.0, 0.0), {pf(l)}, {});
        term(T_PLUS, newrow(0.0, 0.0), {qf(l)}, {});
        term(T_PLUS, newrow(0.0, 0.0), {pt(l)}, {});
        term(T_PLUS, newrow(0.0, 0.0), {qt(l)}, {});
        continue;
      }
      const BranchY& y = Y[l];
      term(T_FP, newrow(0.0, 0.0), {pf(l), vf, vt, tf, tt}, {y.gff, y.gft, y.bft});
      term(T_FQ, newrow(0.0, 0.0), {qf(l), vf, vt, tf, tt}, {y.bff, y.gft, y.bft});
      term(T_FP, newrow(0.0, 0.0), {pt(l), vt, vf, tt, tf}, {y.gtt, y.gtf, y.btf});
      term(T_FQ, newrow(0.0, 0.0), {qt(l), vt, vf, tt, tf}, {y.btt, y.gtf, y.btf});
      const double v0f = S.x0[vf], v0t = S.x0[vt];
      S.x0[pf(l)] = y.gff * v0f * v0f + v0f * v0t * y.gft;
      S.x0[qf(l)] = -y.bff * v0f * v0f - v0f * v0t * y.bft;
      S.x0[pt(l)] = y.gtt * v0t * v0t + v0f * v0t * y.gtf;
      S.x0[qt(l)] = -y.btt * v0t * v0t - v0f * v0t * y.btf;
    }
    // bus balances: sum p_g - sum flows - Gs v^2 = Pd ; sum q_g - sum flows + Bs v^2 = Qd
    std::vector<std::vector<int>> gens_at(nb), from_at(nb), to_at(nb);
    for (int k = 0; k < ng; ++k) gens_at[g.gbus[k]].push_back(k);
    for (int l = 0; l < nl; ++l)
      if (l != out) {
        from_at[g.f[l]].push_back(l);
        to_at[g.t[l]].push_back(l);
      }
    for (int i = 0; i < nb; ++i) {
      const int rp = newrow(lsc * g.pd[i], lsc * g.pd[i]);
      for (int k : gens_at[i]) term(T_PLUS, rp, {opg + k}, {});
      for (int l : from_at[i]) term(T_MINUS, rp, {pf(l)}, {});
      for (int l : to_at[i]) term(T_MINUS, rp, {pt(l)}, {});
      if (g.gs[i] != 0.0) term(T_SHUNT, rp, {ov + i}, {-g.gs[i]});
    }
    for (int i = 0; i < nb; ++i) {
      const int rq = newrow(lsc * g.qd[i], lsc * g.qd[i]);
      for (int k : gens_at[i]) term(T_PLUS, rq, {oqg + k}, {});
      for (int l : from_at[i]) term(T_MINUS, rq, {qf(l)}, {});
      for (int l : to_at[i]) term(T_MINUS, rq, {qt(l)}, {});
      if (g.bs[i] != 0.0) term(T_SHUNT, rq, {ov + i}, {g.bs[i]});
    }
    // apparent-power limits at both ends
    for (int l = 0; l < nl; ++l) {
      if (l == out) continue;
      const double r2 = g.rate[l] * g.rate[l];
      term(T_SQ2, newrow(-kInf, r2), {pf(l), qf(l)}, {});
      term(T_SQ2, newrow(-kInf, r2), {pt(l), qt(l)}, {});
    }
    if (s == 0) continue;
    // recourse: Delta, pi+, pi-, nu+, nu-
    const int odl = oex, opp = oex + 1, opm = opp + ng, onp = opm + ng, onm = onp + ng;
    double psum = 0;
    for (int k = 0; k < ng; ++k) psum += g.pmax[k];
    for (int k = 0; k < ng; ++k) {
      S.xl[opp + k] = S.xl[opm + k] = S.xl[onp + k] = S.xl[onm + k] = 0.0;
    }
    for (int k = 0; k < ng; ++k) {
      if (screen)
        term(T_AGCS, newrow(-pg0[k], -pg0[k]), {opp + k, opm + k, opg + k, odl}, {g.pmax[k] / psum});
      else
        term(T_AGC, newrow(0.0, 0.0), {opp + k, opm + k, opg + k, S.off_pg[0] + k, odl}, {g.pmax[k] / psum});
    }
    for (int k = 0; k < ng; ++k) {
      const int vb = g.gbus[k];
      if (screen) term(T_PVPQS, newrow(-v0[vb], -v0[vb]), {onp + k, onm + k, ov + vb}, {});
      else term(T_PVPQ, newrow(0.0, 0.0), {onp + k, onm + k, ov + vb, S.off_v[0] + vb}, {});
    }
    auto pair = [&](int tmpl, int w1, int x, double bound) {
      const int r = newrow(-kInf, 0.0);
      term(tmpl, r, {w1, x}, {bound});
      S.comp_rows.push_back(r);
      S.comp_w1.push_back(w1);
      S.comp_x.push_back(x);
      S.comp_side.push_back(tmpl == T_COMPU ? -1 : 1);
      S.comp_bound.push_back(bound);
    };
    for (int k = 0; k < ng; ++k) {
      pair(T_COMPU, opm + k, opg + k, g.pmax[k]);
      pair(T_COMPL, opp + k, opg + k, g.pmin[k]);
      pair(T_COMPU, onm + k, oqg + k, g.qmax[k]);
      pair(T_COMPL, onp + k, oqg + k, g.qmin[k]);
    }
  }
  // objective: base-case generation cost (none in screening mode)
  if (!screen)
    for (int k = 0; k < ng; ++k) term(T_COST, -1, {S.off_pg[0] + k}, {g.c2[k], g.c1[k], g.c0[k]});
  S.m = row;
  S.gl = std::move(gl);
  S.gu = std::move(gu);
  if (off != nvar) throw std::logic_error("build_scopf: layout mismatch");
  return S;
}

}  // namespace nclb
