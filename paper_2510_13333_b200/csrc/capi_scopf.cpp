// C-ABI for the SCOPF problem generator (host setup code).
#include <cstring>
#include <algorithm>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>
#include <stdexcept>
#include <string>

#include "../../include/nclopf_b200.h"
#include "capi_internal.hpp"
#include "../../include/nclopf_matpower.h"
#include "host/matpower.hpp"
#include "host/scopf.hpp"
#include "host/sparse.hpp"

using namespace nclb;

#define API extern "C" __attribute__((visibility("default")))
#define GUARD(...)    \
  try {               \
    __VA_ARGS__;      \
  } catch (...) {     \
    return map_exc(); \
  }                   \
  return NCL_OK;

namespace {
// grid generation (N-1 DC ratings) is deterministic and the costliest part of
// instance creation; keep the last few grids
Grid cached_synthetic(int nb, int nl, int ng, uint64_t seed) {
  static std::mutex mu;
  static std::vector<std::pair<std::tuple<int, int, int, uint64_t>, Grid>> cache;
  const auto key = std::make_tuple(nb, nl, ng, seed);
  {
    std::lock_guard<std::mutex> lk(mu);
    for (const auto& e : cache)
      if (e.first == key) return e.second;
  }
  Grid g = grid_synthetic(nb, nl, ng, seed);
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() >= 4) cache.erase(cache.begin());
  cache.emplace_back(key, g);
  return g;
}
}  // namespace

struct ncl_scopf {
  Grid grid;
  ModelSpec spec;
};

namespace {
void finish_scopf(ncl_scopf* s, int K, const int* branch_ids) {
  std::vector<int> cont;
  if (branch_ids) {
    const auto ok = select_contingencies(s->grid, s->grid.nl);  // non-islanding set
    for (int k = 0; k < K; ++k) {
      const int id = branch_ids[k];  // branch + nl * load level (host/scopf.hpp)
      if (id < 0 || id / s->grid.nl >= kLoadLevels || !std::binary_search(ok.begin(), ok.end(), id % s->grid.nl))
        throw Error{NCL_E_INVALID, "scopf: contingency islands the network or is out of range"};
      cont.push_back(id);
    }
  } else {
    cont = select_contingencies(s->grid, K);
  }
  if (static_cast<int>(cont.size()) < K)
    throw Error{NCL_E_INVALID, "scopf: fewer non-islanding contingencies than requested"};
  s->spec = build_scopf(s->grid, cont);
}
}  // namespace

API int ncl_scopf_create_list(int grid, int nb, int nl, int ng, uint64_t seed, int K, const int* branch_ids,
                              ncl_scopf_t* out) {
  GUARD({
    auto s = std::make_unique<ncl_scopf>();
    try {
      s->grid = grid == 0 ? grid_case9() : cached_synthetic(nb, nl, ng, seed);
    } catch (const std::invalid_argument& e) {
      throw Error{NCL_E_INVALID, e.what()};
    }
    finish_scopf(s.get(), K, branch_ids);
    *out = s.release();
  });
}
API int ncl_scopf_create(int grid, int nb, int nl, int ng, uint64_t seed, int K, ncl_scopf_t* out) {
  return ncl_scopf_create_list(grid, nb, nl, ng, seed, K, nullptr, out);
}
API void ncl_scopf_destroy(ncl_scopf_t S) { delete S; }
API int ncl_scopf_get_info(ncl_scopf_t S, ncl_scopf_info* info) {
  GUARD({
    const ModelSpec& p = S->spec;
    info->n = p.n;
    info->m = p.m;
    info->nfam = static_cast<int>(p.fams.size());
    info->K = p.K;
    info->nb = p.nb;
    info->nl = p.nl;
    info->ng = p.ng;
    info->ncomp = static_cast<int>(p.comp_rows.size());
    info->nvar_scen = p.nvar_scen;
    info->ncon_scen = p.ncon_scen;
  });
}
API int ncl_scopf_family_info(ncl_scopf_t S, int f, char* name, int* nnodes, int* nslots, int* np, int* objective,
                              int64_t* ninst) {
  GUARD({
    if (f < 0 || f >= static_cast<int>(S->spec.fams.size())) throw Error{NCL_E_INVALID, "scopf: bad family"};
    const SpecFamily& F = S->spec.fams[f];
    if (name) {
      std::strncpy(name, F.name.c_str(), 63);
      name[63] = 0;
    }
    *nnodes = static_cast<int>(F.nodes.size());
    *nslots = F.nslots;
    *np = F.np;
    *objective = F.objective ? 1 : 0;
    *ninst = F.ninst();
  });
}
API int ncl_scopf_family_data(ncl_scopf_t S, int f, ncl_expr_node* nodes, int* rows, int* vars, double* params) {
  GUARD({
    const SpecFamily& F = S->spec.fams.at(f);
    if (nodes) std::memcpy(nodes, F.nodes.data(), F.nodes.size() * sizeof(ncl_expr_node));
    if (rows && !F.rows.empty()) std::memcpy(rows, F.rows.data(), F.rows.size() * sizeof(int));
    if (vars && !F.vars.empty()) std::memcpy(vars, F.vars.data(), F.vars.size() * sizeof(int));
    if (params && !F.params.empty()) std::memcpy(params, F.params.data(), F.params.size() * sizeof(double));
  });
}
API int ncl_scopf_bounds(ncl_scopf_t S, double* xl, double* xu, double* x0, double* gl, double* gu) {
  GUARD({
    const ModelSpec& p = S->spec;
    auto cp = [](double* d, const std::vector<double>& v) {
      if (d && !v.empty()) std::memcpy(d, v.data(), v.size() * sizeof(double));
    };
    cp(xl, p.xl);
    cp(xu, p.xu);
    cp(x0, p.x0);
    cp(gl, p.gl);
    cp(gu, p.gu);
  });
}
API int ncl_scopf_contingencies(ncl_scopf_t S, int* ids) {
  GUARD(if (!S->spec.contingencies.empty()) std::memcpy(ids, S->spec.contingencies.data(),
                                                         S->spec.contingencies.size() * sizeof(int)));
}
API int ncl_scopf_var_groups(ncl_scopf_t S, int* groups) {
  GUARD({
    const ModelSpec& p = S->spec;
    const int ns = static_cast<int>(p.off_v.size());
    for (int s = 0; s < ns; ++s) {
      const int b = p.off_v[s], e = s + 1 < ns ? p.off_v[s + 1] : p.n;
      for (int i = b; i < e; ++i) groups[i] = s;
    }
  });
}
API int ncl_scopf_candidates(ncl_scopf_t S, int* ids, int* count) {
  GUARD({
    const auto all = select_contingencies(S->grid, S->grid.nl);
    *count = static_cast<int>(all.size());
    if (ids && !all.empty()) std::memcpy(ids, all.data(), all.size() * sizeof(int));
  });
}
API int ncl_scopf_build_model(ncl_scopf_t S, ncl_model_t* out) {
  GUARD({
    const ModelSpec& p = S->spec;
    ncl_builder_t B = nullptr;
    int rc = ncl_builder_create(p.n, &B);
    if (rc != NCL_OK) return rc;
    std::unique_ptr<ncl_builder, void (*)(ncl_builder_t)> guard(B, ncl_builder_destroy);
    int first = 0;
    if ((rc = ncl_builder_add_rows(B, p.m, &first)) != NCL_OK) return rc;
    for (const SpecFamily& F : p.fams) {
      int tid = 0;
      if ((rc = ncl_builder_add_template(B, static_cast<int>(F.nodes.size()), F.nodes.data(), F.nslots,
                                         F.name.c_str(), &tid)) != NCL_OK)
        return rc;
      const int64_t cnt = F.ninst();
      if (cnt == 0) continue;
      rc = F.objective ? ncl_builder_add_objective_terms(B, tid, cnt, F.nslots, F.vars.data(), F.np, F.params.data())
                       : ncl_builder_add_constraint_terms(B, tid, cnt, F.rows.data(), F.nslots, F.vars.data(), F.np,
                                                          F.params.data());
      if (rc != NCL_OK) return rc;
    }
    if ((rc = ncl_builder_build(B, out)) != NCL_OK) return rc;
  });
}

API int ncl_scopf_comp_pairs(ncl_scopf_t S, int* rows, int* w1var, int* xvar, int* side, double* bound) {
  GUARD({
    const ModelSpec& p = S->spec;
    auto cp = [](auto* dst, const auto& v) {
      if (dst) std::copy(v.begin(), v.end(), dst);
    };
    cp(rows, p.comp_rows);
    cp(w1var, p.comp_w1);
    cp(xvar, p.comp_x);
    cp(side, p.comp_side);
    cp(bound, p.comp_bound);
  });
}

// ---- matpower_io (include/nclopf_matpower.h) -------------------------------
struct ncl_network {
  matpower::PowerNetwork net;
};
namespace {
template <class F>
void rethrow_invalid(F&& f) {
  try {
    f();
  } catch (const std::invalid_argument& e) {  // ParseError / ValidationError
    throw Error{NCL_E_INVALID, e.what()};
  }
}
void text_out(const std::string& t, char* buf, int64_t cap, int64_t* len) {
  *len = static_cast<int64_t>(t.size());
  if (buf && cap > 0) {
    const int64_t k = std::min<int64_t>(cap - 1, *len);
    std::memcpy(buf, t.data(), k);
    buf[k] = 0;
  }
}
}  // namespace
API int ncl_matpower_parse(const char* text, ncl_network_t* out) {
  GUARD({
    auto n = std::make_unique<ncl_network>();
    rethrow_invalid([&] { n->net = matpower::parse_case(text); });
    *out = n.release();
  });
}
API void ncl_network_destroy(ncl_network_t N) { delete N; }
API int ncl_network_info_get(ncl_network_t N, ncl_network_info* info) {
  GUARD({
    const auto& n = N->net;
    info->base_mva = n.base_mva;
    info->nbus = static_cast<int>(n.bus.size());
    info->nbranch = static_cast<int>(n.branch.size());
    info->ngen = static_cast<int>(n.gen.size());
    info->ref = n.ref;
    info->nbranch_in = 0;
    for (const auto& e : n.branch) info->nbranch_in += e.status;
    info->ngen_in = 0;
    for (const auto& g : n.gen) info->ngen_in += g.status;
  });
}
API int ncl_network_buses(ncl_network_t N, int* id, int* type, double* pd, double* qd, double* vmin, double* vmax) {
  GUARD({
    const auto& b = N->net.bus;
    for (size_t i = 0; i < b.size(); ++i) {
      if (id) id[i] = b[i].id;
      if (type) type[i] = b[i].type;
      if (pd) pd[i] = b[i].pd;
      if (qd) qd[i] = b[i].qd;
      if (vmin) vmin[i] = b[i].vmin;
      if (vmax) vmax[i] = b[i].vmax;
    }
  });
}
API int ncl_network_branch_admittances(ncl_network_t N, double* y) {
  GUARD({
    std::vector<matpower::TwoPort> v;
    rethrow_invalid([&] { v = matpower::branch_admittances(N->net); });
    for (size_t l = 0; l < v.size(); ++l) {
      const std::complex<double> a[4] = {v[l].yff, v[l].yft, v[l].ytf, v[l].ytt};
      for (int k = 0; k < 4; ++k) {
        y[8 * l + 2 * k] = a[k].real();
        y[8 * l + 2 * k + 1] = a[k].imag();
      }
    }
  });
}
API int ncl_network_serialize(ncl_network_t N, char* buf, int64_t cap, int64_t* len) {
  GUARD(text_out(matpower::serialize(N->net), buf, cap, len));
}
API int ncl_network_json(ncl_network_t N, char* buf, int64_t cap, int64_t* len) {
  GUARD(text_out(matpower::to_json(N->net), buf, cap, len));
}
API int ncl_scopf_create_network(ncl_network_t N, int K, const int* branch_ids, ncl_scopf_t* out) {
  GUARD({
    auto s = std::make_unique<ncl_scopf>();
    s->grid = matpower::to_grid(N->net);
    finish_scopf(s.get(), K, branch_ids);
    *out = s.release();
  });
}

// ---- screening (Eq. 5) ----------------------------
API int ncl_scopf_create_screening(ncl_scopf_t base, const double* pg0, const double* v0, int K, const int* ids,
                                   ncl_scopf_t* out) {
  GUARD({
    if (!pg0 || !v0 || K < 1) throw Error{NCL_E_INVALID, "screening: base set points and K >= 1 contingencies"};
    auto s = std::make_unique<ncl_scopf>();
    s->grid = base->grid;
    std::vector<int> cont;
    const auto ok = select_contingencies(s->grid, s->grid.nl);
    for (int k = 0; k < K; ++k) {
      const int id = ids ? ids[k] : (k < static_cast<int>(ok.size()) ? ok[k] : -1);
      if (id < 0 || id / s->grid.nl >= kLoadLevels || !std::binary_search(ok.begin(), ok.end(), id % s->grid.nl))
        throw Error{NCL_E_INVALID, "screening: contingency islands the network or is out of range"};
      cont.push_back(id);
    }
    try {
      s->spec = build_scopf(s->grid, cont, pg0, v0);
    } catch (const std::invalid_argument& e) {
      throw Error{NCL_E_INVALID, e.what()};
    }
    *out = s.release();
  });
}
