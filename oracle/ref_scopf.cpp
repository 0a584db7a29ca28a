// ORACLE — test infrastructure only (see ref_capi.cpp header for the rules).
//
// Lets bench.py's `--impl reference` arm build its input WITHOUT the product
// library (libnclopf_b200.so): the SCOPF instance generator
// (paper_2510_13333_b200/csrc/host/scopf.cpp, plain host C++ that only emits
// node programs, instance tables and bounds) is compiled into this oracle,
// the model goes through the reference's own ModelBuilder
// (proj/src/model.cpp:75-128, via ref_mb_* in ref_capi.cpp), and the
// condensed KKT matrix through the reference SparseSym add/finalize
// (proj/src/sparse_sym.cpp:12-37) in the triplet order of ref_ipm.cpp's
// RefBackend::factor (the product's csrc/host/kkt.hpp contract).
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "nclopf/model.hpp"
#include "nclopf/sparse_sym.hpp"

#include "../include/nclopf_expr_program.h"
#include "scopf.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

// ref_capi.cpp (same shared object)
extern "C" {
const char* ref_last_error();
void* ref_mb_new(int nvars);
void ref_mb_free(void* b);
int ref_mb_add_template(void* b, int nn, const ncl_expr_node* nodes, int nslots, const char* name, int* id);
int ref_mb_add_rows(void* b, int count);
int ref_mb_add_terms(void* b, int tid, int objective, int64_t count, int nv, const int* vars, int np,
                     const double* params, const int* rows);
int ref_mb_build(void* b, void** out);
}

namespace {
thread_local std::string g_err2;
struct RefScopf {
  nclb::ModelSpec spec;
};
}  // namespace

REF_API const char* ref_scopf_last_error() { return g_err2.c_str(); }

// grid: 0 = MATPOWER case9, 1 = synthetic (nb, nl, ng, seed); ids: K
// contingency ids (branch + nl * load level, csrc/host/scopf.hpp) or NULL for
// the first K non-islanding outages.
REF_API int ref_scopf_new(int grid, int nb, int nl, int ng, uint64_t seed, int K, const int* ids, void** out,
                          int* n, int* m) {
  try {
    auto s = std::make_unique<RefScopf>();
    const nclb::Grid g = grid == 0 ? nclb::grid_case9() : nclb::grid_synthetic(nb, nl, ng, seed);
    std::vector<int> cont = ids ? std::vector<int>(ids, ids + K) : nclb::select_contingencies(g, K);
    if (static_cast<int>(cont.size()) < K) throw std::invalid_argument("fewer contingencies than requested");
    s->spec = nclb::build_scopf(g, cont);
    *n = s->spec.n;
    *m = s->spec.m;
    *out = s.release();
    return 0;
  } catch (const std::exception& e) {
    g_err2 = e.what();
    return 1;
  }
}
REF_API void ref_scopf_free(void* h) { delete static_cast<RefScopf*>(h); }

REF_API void ref_scopf_bounds(void* h, double* xl, double* xu, double* x0, double* gl, double* gu) {
  const auto& S = static_cast<RefScopf*>(h)->spec;
  std::memcpy(xl, S.xl.data(), S.n * sizeof(double));
  std::memcpy(xu, S.xu.data(), S.n * sizeof(double));
  std::memcpy(x0, S.x0.data(), S.n * sizeof(double));
  std::memcpy(gl, S.gl.data(), S.m * sizeof(double));
  std::memcpy(gu, S.gu.data(), S.m * sizeof(double));
}

// The reference ModelFunctions of the instance (free with ref_mf_free).
REF_API int ref_scopf_model(void* h, void** mf) {
  const auto& S = static_cast<RefScopf*>(h)->spec;
  void* b = ref_mb_new(S.n);
  int rc = 0;
  if (S.m) ref_mb_add_rows(b, S.m);
  for (const auto& F : S.fams) {
    int tid = 0;
    if ((rc = ref_mb_add_template(b, static_cast<int>(F.nodes.size()), F.nodes.data(), F.nslots, F.name.c_str(),
                                  &tid)))
      break;
    const int64_t cnt = F.ninst();
    if (cnt == 0) continue;
    if ((rc = ref_mb_add_terms(b, tid, F.objective ? 1 : 0, cnt, F.nslots, F.vars.data(), F.np,
                               F.np ? F.params.data() : nullptr, F.objective ? nullptr : F.rows.data())))
      break;
  }
  if (!rc) rc = ref_mb_build(b, mf);
  if (rc) g_err2 = ref_last_error();
  ref_mb_free(b);
  return rc;
}

// Condensed K = H + diag(sig + dw) + J' diag(D) J through the reference
// SparseSym: triplets (1) Hessian in hess_coords order, (2) one diagonal per
// variable, (3) per row r ascending, every pair a >= b of its Jacobian
// entries, value (D_r J_a) J_b. Returns a finalized nclopf::SparseSym*.
REF_API int ref_condensed_kkt(void* mf, const double* hess, const double* jac, const double* sig, double dw,
                              const double* D, void** out) {
  try {
    const auto* M = static_cast<const nclopf::ModelFunctions*>(mf);
    const int n = M->num_vars(), m = M->num_cons();
    const auto& hc = M->hess_coords();
    const auto& jc = M->jac_coords();
    auto K = std::make_unique<nclopf::SparseSym>(n);
    for (std::size_t k = 0; k < hc.size(); ++k) K->add(hc[k].first, hc[k].second, hess[k]);
    for (int i = 0; i < n; ++i) K->add(i, i, sig[i] + dw);
    std::vector<int64_t> rp(m + 1, 0);
    for (const auto& e : jc) rp[e.first + 1]++;
    for (int r = 0; r < m; ++r) rp[r + 1] += rp[r];
    for (int r = 0; r < m; ++r)
      for (int64_t a = rp[r]; a < rp[r + 1]; ++a)
        for (int64_t b = rp[r]; b <= a; ++b) K->add(jc[a].second, jc[b].second, (D[r] * jac[a]) * jac[b]);
    K->finalize();
    *out = K.release();
    return 0;
  } catch (const std::exception& e) {
    g_err2 = e.what();
    return 1;
  }
}
