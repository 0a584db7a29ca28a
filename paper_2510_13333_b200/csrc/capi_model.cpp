// C-ABI for model_ad (ModelBuilder / ModelFunctions / fd_check).
// Host: template differentiation, index maps (csrc/host/model.cpp).
// Device: every evaluation (csrc/cuda/eval.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "../../include/nclopf_b200.h"
#include "capi_internal.hpp"
#include "cuda/dev.hpp"
#include "cuda/eval.hpp"
#include "host/model.hpp"
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

struct ncl_builder {
  HostBuilder b;
  explicit ncl_builder(int n) : b(n) {}
};

struct DevFamBufs {
  DevBuf<int> vars, rows, hess_hi, hess_lo;
  DevBuf<double> params;
  DevBuf<Instr> prog[PK_N];
  DevBuf<int> outs[PK_N];
};

struct ncl_model {
  BuiltModel B;
  bool dev_ready = false;
  std::vector<DevFamBufs> fb;
  DevBuf<DevFam> fams;
  DevBuf<double> contrib;
  DevBuf<unsigned long long> err;
  DevBuf<int64_t> c_ptr, j_ptr, h_ptr, g_ptr, o_ptr, jr_ptr, jt_ptr;
  DevBuf<int> c_idx, j_idx, h_idx, g_idx, o_idx, jcol, jrow, jt_idx;
  DevBuf<double> w_tmp, lam_tmp, out_tmp, v_tmp;
  DevModel dm;
};

namespace {
template <class T>
std::vector<int> to_i32(const std::vector<T>& v) {
  std::vector<int> o(v.size());
  for (size_t i = 0; i < v.size(); ++i) {
    if (v[i] > static_cast<T>(INT32_MAX)) throw Error{NCL_E_INVALID, "model too large for int32 gather indices"};
    o[i] = static_cast<int>(v[i]);
  }
  return o;
}

void upload_model(ncl_model* M) {
  if (M->dev_ready) return;
  ensure_init();
  BuiltModel& B = M->B;
  const int nf = static_cast<int>(B.f.size());
  M->fb.resize(nf);
  std::vector<DevFam> hf(nf);
  int64_t blocks = 0;
  int maxr[PK_N] = {0, 0, 0, 0};
  for (int i = 0; i < nf; ++i) {
    auto& F = B.f[i];
    auto& D = M->fb[i];
    D.vars.upload(F.vars);
    D.params.upload(F.params);
    D.rows.upload(F.rows);
    D.hess_hi.upload(F.hess_hi);
    D.hess_lo.upload(F.hess_lo);
    DevFam& d = hf[i];
    d.ninst = F.ninst;
    d.block0 = blocks;
    blocks += (F.ninst + 255) / 256;
    d.base = F.base;
    d.nv = F.nv;
    d.np = F.np;
    d.G = F.G;
    d.H = F.H;
    d.obj = F.objective ? 1 : 0;
    d.vars = D.vars.p;
    d.params = D.params.p;
    d.rows = D.rows.p;
    d.hess_hi = D.hess_hi.p;
    d.hess_lo = D.hess_lo.p;
    for (int k = 0; k < PK_N; ++k) {
      D.prog[k].upload(encode(F.prog[k]));
      D.outs[k].upload(F.prog[k].out);
      d.prog[k] = D.prog[k].p;
      d.outs[k] = D.outs[k].p;
      d.plen[k] = static_cast<int>(F.prog[k].code.size());
      if (F.ninst > 0) maxr[k] = std::max(maxr[k], F.nregs[k]);
    }
  }
  for (int k = 0; k < PK_N; ++k)
    if (maxr[k] > 256) throw Error{NCL_E_INVALID, "template needs more than 256 live registers on the GPU"};
  if (blocks > INT32_MAX) throw Error{NCL_E_INVALID, "too many instances"};
  M->fams.alloc(std::max(1, nf));
  if (nf) ck(cudaMemcpyAsync(M->fams.p, hf.data(), nf * sizeof(DevFam), cudaMemcpyHostToDevice, g_stream), "H2D");
  M->contrib.alloc(std::max<int64_t>(1, B.ncontrib));
  M->err.alloc(1);
  ck(cudaMemsetAsync(M->err.p, 0xff, sizeof(unsigned long long), g_stream), "memset");
  M->c_ptr.upload(B.c_ptr);
  M->j_ptr.upload(B.j_ptr);
  M->h_ptr.upload(B.h_ptr);
  M->g_ptr.upload(B.g_ptr);
  M->o_ptr.upload(B.o_ptr);
  M->c_idx.upload(to_i32(B.c_idx));
  M->j_idx.upload(to_i32(B.j_idx));
  M->h_idx.upload(to_i32(B.h_idx));
  M->g_idx.upload(to_i32(B.g_idx));
  M->o_idx.upload(to_i32(B.o_idx));
  M->jr_ptr.upload(B.jr_ptr);
  M->jt_ptr.upload(B.jt_ptr);
  M->jcol.upload(B.jcol);
  M->jrow.upload(B.jrow);
  M->jt_idx.upload(B.jt_idx);
  M->w_tmp.alloc(std::max(1, B.n));
  M->v_tmp.alloc(std::max(1, B.n));
  M->lam_tmp.alloc(std::max(1, B.m));
  M->out_tmp.alloc(std::max<int64_t>({1, static_cast<int64_t>(B.n), static_cast<int64_t>(B.m),
                                      static_cast<int64_t>(B.jac_coords.size()),
                                      static_cast<int64_t>(B.hess_coords.size())}));
  M->dm.fams = M->fams.p;
  M->dm.nfam = nf;
  M->dm.nblocks = static_cast<int>(blocks);
  for (int k = 0; k < PK_N; ++k) M->dm.maxregs[k] = maxr[k];
  M->dm.contrib = M->contrib.p;
  M->dm.err = M->err.p;
  ck(cudaStreamSynchronize(g_stream), "upload model");
  M->dev_ready = true;
}

const char* domain_msg(int code) {
  switch (code) {
    case 1: return "division by ~0";
    case 2: return "fractional power of negative base";
    default: return "negative power of zero";
  }
}

void check_domain_sync(ncl_model* M) {
  unsigned long long h = ~0ull;
  ck(cudaMemcpyAsync(&h, M->err.p, sizeof(h), cudaMemcpyDeviceToHost, g_stream), "D2H");
  ck(cudaStreamSynchronize(g_stream), "sync");
  if (h != ~0ull) {
    ck(cudaMemsetAsync(M->err.p, 0xff, sizeof(unsigned long long), g_stream), "memset");
    const int fam = static_cast<int>(h >> 40);
    const long long inst = static_cast<long long>((h >> 2) & ((1ull << 38) - 1));
    throw Error{NCL_E_DOMAIN, std::string(domain_msg(static_cast<int>(h & 3))) + " in template " +
                                  M->B.fams[fam].tmpl.name + " instance " + std::to_string(inst)};
  }
}

// Host-path helper: upload inputs, run, download `nout` doubles.
struct HostCall {
  ncl_model* M;
  const double* w;  // device pointer of w
  explicit HostCall(ncl_model* m, const double* hw) : M(m) {
    upload_model(M);
    if (M->B.n > 0)
      ck(cudaMemcpyAsync(M->w_tmp.p, hw, M->B.n * sizeof(double), cudaMemcpyHostToDevice, g_stream), "H2D");
    w = M->w_tmp.p;
  }
  void fetch(double* out, int64_t nout) {
    if (nout > 0) ck(cudaMemcpyAsync(out, M->out_tmp.p, nout * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
    check_domain_sync(M);
  }
};

void eval_into(ncl_model* M, int kind, const double* w, double sigma, const double* lam, double* out) {
  const BuiltModel& B = M->B;
  dev_eval(M->dm, kind == 4 ? PK_V : (kind == 5 ? PK_G : kind), w, sigma, lam, g_stream);
  switch (kind) {
    case 0:  // constraints
      dev_gather64(B.m, M->c_ptr.p, M->c_idx.p, M->contrib.p, out, g_stream);
      break;
    case 1:  // jacobian
      dev_gather64(static_cast<int64_t>(B.jac_coords.size()), M->j_ptr.p, M->j_idx.p, M->contrib.p, out, g_stream);
      break;
    case 2:  // hessian
      dev_gather64(static_cast<int64_t>(B.hess_coords.size()), M->h_ptr.p, M->h_idx.p, M->contrib.p, out, g_stream);
      break;
    case 4:  // objective
      dev_gather64(1, M->o_ptr.p, M->o_idx.p, M->contrib.p, out, g_stream);
      break;
    case 5:  // gradient
      dev_gather64(B.n, M->g_ptr.p, M->g_idx.p, M->contrib.p, out, g_stream);
      break;
  }
  check_launch("eval");
}

int run_eval(ncl_model_t M, int kind, const double* w, double sigma, const double* lam, double* out, int where,
             int64_t nout) {
  GUARD({
    if (where == NCL_DEVICE) {
      upload_model(M);
      eval_into(M, kind, w, sigma, lam, out);
      return NCL_OK;
    }
    HostCall hc(M, w);
    const double* dlam = nullptr;
    if (lam) {
      if (M->B.m > 0)
        ck(cudaMemcpyAsync(M->lam_tmp.p, lam, M->B.m * sizeof(double), cudaMemcpyHostToDevice, g_stream), "H2D");
      dlam = M->lam_tmp.p;
    }
    eval_into(M, kind, hc.w, sigma, dlam, M->out_tmp.p);
    hc.fetch(out, nout);
  });
}
}  // namespace

API int ncl_builder_create(int num_vars, ncl_builder_t* out) {
  GUARD({
    if (num_vars < 0) throw Error{NCL_E_INVALID, "ModelBuilder: negative variable count"};
    *out = new ncl_builder(num_vars);
  });
}
API void ncl_builder_destroy(ncl_builder_t B) { delete B; }
API int ncl_builder_num_vars(ncl_builder_t B) { return B->b.num_vars(); }
API int ncl_builder_num_rows(ncl_builder_t B) { return B->b.num_rows(); }
API int ncl_builder_add_template(ncl_builder_t B, int nnodes, const ncl_expr_node* nodes, int nslots,
                                 const char* name, int* id) {
  GUARD({
    Template t(build_from_program(nnodes, nodes), nslots, name ? name : "");
    *id = B->b.add_template(std::move(t));
  });
}
API int ncl_builder_add_rows(ncl_builder_t B, int count, int* first) { GUARD(*first = B->b.add_rows(count)); }
API int ncl_builder_add_objective_terms(ncl_builder_t B, int tid, int64_t count, int nv, const int* vars, int np,
                                        const double* params) {
  GUARD(B->b.add_terms(tid, true, count, nullptr, nv, vars, np, params));
}
API int ncl_builder_add_constraint_terms(ncl_builder_t B, int tid, int64_t count, const int* rows, int nv,
                                         const int* vars, int np, const double* params) {
  GUARD(B->b.add_terms(tid, false, count, rows, nv, vars, np, params));
}
API int ncl_builder_build(ncl_builder_t B, ncl_model_t* out) {
  GUARD({
    auto m = std::make_unique<ncl_model>();
    m->B = B->b.build();
    B->b = HostBuilder(B->b.num_vars());
    *out = m.release();
  });
}
API void ncl_model_destroy(ncl_model_t M) { delete M; }
API int ncl_model_sizes(ncl_model_t M, int* n, int* m, int64_t* nj, int64_t* nh) {
  GUARD({
    *n = M->B.n;
    *m = M->B.m;
    *nj = static_cast<int64_t>(M->B.jac_coords.size());
    *nh = static_cast<int64_t>(M->B.hess_coords.size());
  });
}
API int ncl_model_jac_coords(ncl_model_t M, int* rows, int* cols) {
  GUARD(for (size_t k = 0; k < M->B.jac_coords.size(); ++k) rows[k] = M->B.jac_coords[k].first,
        cols[k] = M->B.jac_coords[k].second);
}
API int ncl_model_hess_coords(ncl_model_t M, int* rows, int* cols) {
  GUARD(for (size_t k = 0; k < M->B.hess_coords.size(); ++k) rows[k] = M->B.hess_coords[k].first,
        cols[k] = M->B.hess_coords[k].second);
}
API int ncl_model_eval_objective(ncl_model_t M, const double* w, double* out, int where) {
  return run_eval(M, 4, w, 0.0, nullptr, out, where, 1);
}
API int ncl_model_eval_grad_objective(ncl_model_t M, const double* w, double* g, int where) {
  return run_eval(M, 5, w, 0.0, nullptr, g, where, M->B.n);
}
API int ncl_model_eval_constraints(ncl_model_t M, const double* w, double* c, int where) {
  return run_eval(M, 0, w, 0.0, nullptr, c, where, M->B.m);
}
API int ncl_model_eval_jacobian(ncl_model_t M, const double* w, double* vals, int where) {
  return run_eval(M, 1, w, 0.0, nullptr, vals, where, static_cast<int64_t>(M->B.jac_coords.size()));
}
API int ncl_model_eval_hessian_lag(ncl_model_t M, const double* w, double sigma, const double* lam, double* vals,
                                   int where) {
  return run_eval(M, 2, w, sigma, lam, vals, where, static_cast<int64_t>(M->B.hess_coords.size()));
}
API int ncl_model_hessian_lag(ncl_model_t M, const double* w, double sigma, const double* lam, ncl_sym_t* out) {
  GUARD({
    const auto& hc = M->B.hess_coords;
    std::vector<double> vals(hc.size());
    int rc = ncl_model_eval_hessian_lag(M, w, sigma, lam, vals.data(), NCL_HOST);
    if (rc != NCL_OK) return rc;
    std::vector<int> r(hc.size()), c(hc.size());
    for (size_t k = 0; k < hc.size(); ++k) r[k] = hc[k].first, c[k] = hc[k].second;
    ncl_sym_t H = nullptr;
    if ((rc = ncl_sym_create(M->B.n, &H)) != NCL_OK) return rc;
    if ((rc = ncl_sym_add(H, static_cast<int64_t>(hc.size()), r.data(), c.data(), vals.data())) != NCL_OK ||
        (rc = ncl_sym_finalize(H)) != NCL_OK) {
      ncl_sym_destroy(H);
      return rc;
    }
    *out = H;
  });
}
API int ncl_model_jac_times(ncl_model_t M, const double* jv, const double* v, double* out, int where) {
  GUARD({
    upload_model(M);
    const int64_t nj = static_cast<int64_t>(M->B.jac_coords.size());
    if (where == NCL_DEVICE) {
      dev_csr_mv(M->B.m, M->jr_ptr.p, nullptr, M->jcol.p, jv, v, out, g_stream);
      check_launch("jac_times");
      return NCL_OK;
    }
    DevBuf<double> dj;
    dj.alloc(nj);
    if (nj) ck(cudaMemcpyAsync(dj.p, jv, nj * sizeof(double), cudaMemcpyHostToDevice, g_stream), "H2D");
    if (M->B.n) ck(cudaMemcpyAsync(M->v_tmp.p, v, M->B.n * sizeof(double), cudaMemcpyHostToDevice, g_stream), "H2D");
    dev_csr_mv(M->B.m, M->jr_ptr.p, nullptr, M->jcol.p, dj.p, M->v_tmp.p, M->out_tmp.p, g_stream);
    check_launch("jac_times");
    if (M->B.m) ck(cudaMemcpyAsync(out, M->out_tmp.p, M->B.m * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
    ck(cudaStreamSynchronize(g_stream), "sync");
  });
}
API int ncl_model_jac_trans_times(ncl_model_t M, const double* jv, const double* y, double* out, int where) {
  GUARD({
    upload_model(M);
    const int64_t nj = static_cast<int64_t>(M->B.jac_coords.size());
    if (where == NCL_DEVICE) {
      dev_csr_mv(M->B.n, M->jt_ptr.p, M->jt_idx.p, M->jrow.p, jv, y, out, g_stream);
      check_launch("jac_trans_times");
      return NCL_OK;
    }
    DevBuf<double> dj;
    dj.alloc(nj);
    if (nj) ck(cudaMemcpyAsync(dj.p, jv, nj * sizeof(double), cudaMemcpyHostToDevice, g_stream), "H2D");
    if (M->B.m) ck(cudaMemcpyAsync(M->lam_tmp.p, y, M->B.m * sizeof(double), cudaMemcpyHostToDevice, g_stream), "H2D");
    dev_csr_mv(M->B.n, M->jt_ptr.p, M->jt_idx.p, M->jrow.p, dj.p, M->lam_tmp.p, M->out_tmp.p, g_stream);
    check_launch("jac_trans_times");
    if (M->B.n) ck(cudaMemcpyAsync(out, M->out_tmp.p, M->B.n * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
    ck(cudaStreamSynchronize(g_stream), "sync");
  });
}
API int ncl_model_eval_all_device(ncl_model_t M, const double* w, double sigma, const double* lam, double* obj,
                                  double* grad, double* c, double* jac, double* hess) {
  GUARD({
    upload_model(M);
    const BuiltModel& B = M->B;
    dev_eval(M->dm, PK_VGH, w, sigma, lam, g_stream);
    if (obj) dev_gather64(1, M->o_ptr.p, M->o_idx.p, M->contrib.p, obj, g_stream);
    if (grad) dev_gather64(B.n, M->g_ptr.p, M->g_idx.p, M->contrib.p, grad, g_stream);
    if (c) dev_gather64(B.m, M->c_ptr.p, M->c_idx.p, M->contrib.p, c, g_stream);
    if (jac) dev_gather64(static_cast<int64_t>(B.jac_coords.size()), M->j_ptr.p, M->j_idx.p, M->contrib.p, jac, g_stream);
    if (hess) dev_gather64(static_cast<int64_t>(B.hess_coords.size()), M->h_ptr.p, M->h_idx.p, M->contrib.p, hess, g_stream);
    check_launch("eval_all");
  });
}
API int ncl_model_eval_values_device(ncl_model_t M, const double* w, double* obj, double* c) {
  GUARD({
    upload_model(M);
    const BuiltModel& B = M->B;
    dev_eval(M->dm, PK_V, w, 1.0, nullptr, g_stream);
    if (obj) dev_gather64(1, M->o_ptr.p, M->o_idx.p, M->contrib.p, obj, g_stream);
    if (c) dev_gather64(B.m, M->c_ptr.p, M->c_idx.p, M->contrib.p, c, g_stream);
    check_launch("eval_values");
  });
}
API int ncl_model_check_domain(ncl_model_t M) { GUARD(upload_model(M); check_domain_sync(M)); }

// fd_check (model.cpp:229-315): same RNG stream and probe arithmetic; the
// evaluations run on the GPU.
API int ncl_fd_check(ncl_model_t M, const double* w, unsigned seed, double tol, double* errs, int* pass) {
  GUARD({
    const int n = M->B.n, mm = M->B.m;
    const size_t nj = M->B.jac_coords.size(), nh = M->B.hess_coords.size();
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> unit(-1.0, 1.0);
    double winf = 0.0;
    for (int i = 0; i < n; ++i) winf = std::max(winf, std::abs(w[i]));
    const double h = 1e-6 * std::max(1.0, winf);
    std::vector<double> dir(n), wp(w, w + n), wm(w, w + n), lam(mm);
    for (auto& l : lam) l = unit(rng);
    std::vector<double> grad(n), jl(nj), hv(n), cp(mm), cm(mm), hvals(nh);
    std::vector<double> gl_p(n), gl_m(n), jp(nj), jm(nj), jd(mm);
    auto rel = [](double err, double ref) { return err / std::max(1.0, ref); };
    auto chk = [](int rc) {
      if (rc != NCL_OK) throw Error{rc, g_err};
    };
    double ge = 0, je = 0, he = 0;
    const auto& jc = M->B.jac_coords;
    const auto& hc = M->B.hess_coords;
    for (int probe = 0; probe < 4; ++probe) {
      double dn = 0.0;
      for (int i = 0; i < n; ++i) {
        dir[i] = unit(rng);
        dn += dir[i] * dir[i];
      }
      dn = std::sqrt(dn);
      for (int i = 0; i < n; ++i) {
        dir[i] /= dn;
        wp[i] = w[i] + h * dir[i];
        wm[i] = w[i] - h * dir[i];
      }
      chk(ncl_model_eval_grad_objective(M, w, grad.data(), NCL_HOST));
      double gd = 0.0, gref = 0.0;
      for (int i = 0; i < n; ++i) {
        gd += grad[i] * dir[i];
        gref = std::max(gref, std::abs(grad[i]));
      }
      double fp = 0, fm = 0;
      chk(ncl_model_eval_objective(M, wp.data(), &fp, NCL_HOST));
      chk(ncl_model_eval_objective(M, wm.data(), &fm, NCL_HOST));
      const double fd_g = (fp - fm) / (2.0 * h);
      ge = std::max(ge, rel(std::abs(gd - fd_g), std::max(gref, std::abs(fd_g))));
      chk(ncl_model_eval_jacobian(M, w, jl.data(), NCL_HOST));
      chk(ncl_model_jac_times(M, jl.data(), dir.data(), jd.data(), NCL_HOST));
      chk(ncl_model_eval_constraints(M, wp.data(), cp.data(), NCL_HOST));
      chk(ncl_model_eval_constraints(M, wm.data(), cm.data(), NCL_HOST));
      double jerr = 0.0, jref = 0.0;
      for (int r = 0; r < mm; ++r) {
        const double fd = (cp[r] - cm[r]) / (2.0 * h);
        jerr = std::max(jerr, std::abs(jd[r] - fd));
        jref = std::max({jref, std::abs(jd[r]), std::abs(fd)});
      }
      je = std::max(je, rel(jerr, jref));
      chk(ncl_model_eval_hessian_lag(M, w, 1.0, lam.data(), hvals.data(), NCL_HOST));
      std::fill(hv.begin(), hv.end(), 0.0);
      for (size_t k = 0; k < nh; ++k) {
        hv[hc[k].first] += hvals[k] * dir[hc[k].second];
        if (hc[k].first != hc[k].second) hv[hc[k].second] += hvals[k] * dir[hc[k].first];
      }
      auto grad_lag = [&](const std::vector<double>& x, std::vector<double>& out, std::vector<double>& jb) {
        chk(ncl_model_eval_grad_objective(M, x.data(), out.data(), NCL_HOST));
        chk(ncl_model_eval_jacobian(M, x.data(), jb.data(), NCL_HOST));
        for (size_t k = 0; k < nj; ++k) out[jc[k].second] += jb[k] * lam[jc[k].first];
      };
      grad_lag(wp, gl_p, jp);
      grad_lag(wm, gl_m, jm);
      double herr = 0.0, href = 0.0;
      for (int i = 0; i < n; ++i) {
        const double fd = (gl_p[i] - gl_m[i]) / (2.0 * h);
        herr = std::max(herr, std::abs(hv[i] - fd));
        href = std::max({href, std::abs(hv[i]), std::abs(fd)});
      }
      he = std::max(he, rel(herr, href));
    }
    errs[0] = ge;
    errs[1] = je;
    errs[2] = he;
    *pass = (ge <= tol && je <= tol && he <= tol) ? 1 : 0;
  });
}

API int ncl_kkt_create_for_model(ncl_model_t M, ncl_kkt_t* out) {
  GUARD({
    const auto& hc = M->B.hess_coords;
    const auto& jc = M->B.jac_coords;
    std::vector<int> hr(hc.size()), hcl(hc.size()), jr(jc.size()), jcl(jc.size());
    for (size_t k = 0; k < hc.size(); ++k) hr[k] = hc[k].first, hcl[k] = hc[k].second;
    for (size_t k = 0; k < jc.size(); ++k) jr[k] = jc[k].first, jcl[k] = jc[k].second;
    const int rc = ncl_kkt_create(M->B.n, M->B.m, static_cast<int64_t>(hc.size()), hr.data(), hcl.data(),
                                  static_cast<int64_t>(jc.size()), jr.data(), jcl.data(), out);
    if (rc != NCL_OK) return rc;
  });
}
