// C-ABI of the NCL + IPM solve on the B200 backend (nclopf_ipm.h).
//
// GpuBackend keeps every vector of the iteration in HBM and drives the hot
// path through the library's own device entry points: K1 evaluation
// (ncl_model_eval_*_device), K2 assembly (ncl_kkt_assemble), K3/K4
// factor + refined solve (ncl_refactorize, ncl_solve_refined), K5 J/J' products
// (ncl_model_jac_*times) and the K7 vector kernels (csrc/cuda/ipm.cu). The
// host sees scalars only: one pinned D2H of <= 8 doubles per reduction.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../include/nclopf_ipm.h"
#include "capi_internal.hpp"
#include "cuda/ipm_dev.hpp"
#include "host/ipm.hpp"

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

void chk(int rc) {
  if (rc != NCL_OK) throw Error{rc, g_err};
}

class GpuBackend final : public ipm::Backend {
 public:
  GpuBackend(ncl_model_t M, const double* xl, const double* xu, const double* x0, const double* gl,
             const double* gu)
      : M_(M) {
    ensure_init();
    int n = 0, m = 0;
    int64_t nj = 0, nh = 0;
    chk(ncl_model_sizes(M, &n, &m, &nj, &nh));
    n_ = n;
    m_ = m;
    nnzj_ = nj;
    nnzh_ = nh;
    nbd_ = 0;
    for (int i = 0; i < n; ++i) nbd_ += (xl[i] > -ipm::kBig) + (xu[i] < ipm::kBig);
    for (int i = 0; i < m; ++i)
      if (gl[i] != gu[i]) nbd_ += (gl[i] > -ipm::kBig) + (gu[i] < ipm::kBig);
    const int64_t NX = 15, NR = 21;
    slab_.alloc(NX * n + NR * m + nj + nh + 16);
    ck(cudaMemsetAsync(slab_.p, 0, slab_.n * sizeof(double), g_stream), "memset");
    double* p = slab_.p;
    auto take = [&](int64_t cnt) {
      double* q = p;
      p += cnt;
      return q;
    };
    V_.n = n;
    V_.m = m;
    double* dxl = take(n);
    double* dxu = take(n);
    V_.xl = dxl;
    V_.xu = dxu;
    V_.x = take(n), V_.zl = take(n), V_.zu = take(n), V_.grad = take(n), V_.jty = take(n);
    V_.sigx = take(n), V_.gx = take(n), V_.rhs = take(n), V_.jtdq = take(n);
    V_.dx = take(n), V_.dzl = take(n), V_.dzu = take(n), V_.xt = take(n);
    double* dgl = take(m);
    double* dgu = take(m);
    V_.gl = dgl;
    V_.gu = dgu;
    V_.r = take(m), V_.s = take(m), V_.y = take(m), V_.vl = take(m), V_.vu = take(m), V_.lamN = take(m);
    V_.c = take(m), V_.D = take(m), V_.q = take(m), V_.dq = take(m);
    V_.dr = take(m), V_.ds = take(m), V_.dy = take(m), V_.dvl = take(m), V_.dvu = take(m), V_.jdx = take(m);
    V_.rt = take(m), V_.st = take(m), V_.ct = take(m);
    jac_ = take(nj);
    hess_ = take(nh);
    dsc_ = take(16);  // [0] f(x) [1] f(xt) [2..9] reduction outputs
    part_.alloc(static_cast<int64_t>(ipm::kRedBlocks) * 8 + 1);  // + completion ticket
    ck(cudaMemsetAsync(part_.p, 0, part_.n * sizeof(double), g_stream), "memset");
    auto up = [&](double* d, const double* h, int64_t cnt) {
      if (cnt) ck(cudaMemcpyAsync(d, h, cnt * sizeof(double), cudaMemcpyHostToDevice, g_stream), "H2D");
    };
    up(dxl, xl, n);
    up(dxu, xu, n);
    up(V_.x, x0, n);
    up(dgl, gl, m);
    up(dgu, gu, m);
    ck(cudaMallocHost(reinterpret_cast<void**>(&hsc_), 16 * sizeof(double)), "cudaMallocHost");
    ck(cudaStreamSynchronize(g_stream), "sync");
    chk(ncl_kkt_create_for_model(M, &kkt_));
    K_ = ncl_kkt_matrix(kkt_);
  }
  ~GpuBackend() override {
    if (F_) ncl_fact_destroy(F_);
    if (S_) ncl_symb_destroy(S_);
    if (kkt_) ncl_kkt_destroy(kkt_);
    if (hsc_) cudaFreeHost(hsc_);
    if (tm_[3] > 0)
      std::fprintf(stderr, "[ipm] %d refactorizations: assembly %.3f ms + factor %.3f ms on the device, %.3f ms host wall per call\n",
                   static_cast<int>(tm_[3]), tm_[0] / tm_[3], tm_[1] / tm_[3], tm_[2] / tm_[3]);
  }
  int n() const override { return n_; }
  int m() const override { return m_; }
  int num_bound_duals() const override { return static_cast<int>(nbd_); }

  void init_point(const ipm::Scal& S, double* f, double* gmax) override {
    dev_ipm_elem(IE_INIT_X, V_, S, g_stream);
    chk(ncl_model_eval_all_device(M_, V_.x, 1.0, V_.y, dsc_, V_.grad, V_.c, jac_, hess_));
    ck(cudaMemsetAsync(dsc_ + 2, 0, sizeof(double), g_stream), "memset");
    dev_absmax(V_.grad, n_, dsc_ + 2, g_stream);
    dev_ipm_elem(IE_INIT_ROW, V_, S, g_stream);
    fetch(0, 3);
    chk(ncl_model_check_domain(M_));
    fcur_ = hsc_[0];
    *f = hsc_[0];
    *gmax = hsc_[2];
    // one-time symbolic analysis of the fixed K pattern (exact MD, etree,
    // supernodes) — values are irrelevant to it. The KKT assembly's device
    // maps (host-built, then uploaded) are independent of it: a second host
    // thread prepares them meanwhile (same device; its error, if any, is
    // reported after the analysis)
    int dev = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    int prc = NCL_OK;
    std::string perr;
    std::thread prep([&] {
      if (cudaSetDevice(dev) != cudaSuccess) {
        prc = NCL_E_CUDA;
        perr = "kkt: cudaSetDevice failed in the preparation thread";
        return;
      }
      prc = kkt_prepare_device(kkt_);
      if (prc != NCL_OK) perr = g_err;
    });
    const int arc = ncl_analyze(K_, nullptr, &S_);
    prep.join();
    chk(arc);
    if (prc != NCL_OK) throw Error{prc, perr};
    // the symbolic factor's device copy is setup too (t_init), not the first
    // factorization's cost
    chk(symb_prepare_device(S_));
  }
  void eval_derivatives(double sf) override {
    chk(ncl_model_eval_all_device(M_, V_.x, sf, V_.y, nullptr, V_.grad, nullptr, jac_, hess_));
    chk(ncl_model_jac_trans_times(M_, jac_, V_.y, V_.jty, NCL_DEVICE));
    // complete here so the host timer charges evaluation to t_eval rather
    // than to whichever phase synchronises next
    ck(cudaStreamSynchronize(g_stream), "sync");
  }
  ipm::KktErr kkt_error(const ipm::Scal& S) override {
    reduce(IR_KKT, S, 7);
    ipm::KktErr e;
    e.du = hsc_[2];
    e.pr = hsc_[3];
    e.dur = hsc_[4];
    e.cmu = hsc_[5];
    e.c0 = hsc_[6];
    e.ysum = hsc_[7];
    e.zsum = hsc_[8];
    return e;
  }
  double hess_absmax() override {
    ck(cudaMemsetAsync(dsc_ + 2, 0, sizeof(double), g_stream), "memset");
    dev_absmax(hess_, nnzh_, dsc_ + 2, g_stream);
    fetch(2, 1);
    return hsc_[2];
  }
  void form_newton(const ipm::Scal& S) override { dev_ipm_elem(IE_NEWTON, V_, S, g_stream); }
  ipm::FactorOut factor(double dw, double pivot_tol) override {
    // NCL_IPM_TIMING=1: device time of assembly / factorization per call vs
    // the host's wall time of the call (printed at exit; debug only)
    static const bool timing = std::getenv("NCL_IPM_TIMING") != nullptr;
    const auto h0 = std::chrono::steady_clock::now();
    if (timing) {
      if (!ev_[0]) for (auto& e : ev_) cudaEventCreate(&e);
      cudaEventRecord(ev_[0], g_stream);
    }
    chk(ncl_kkt_assemble(kkt_, hess_, jac_, V_.sigx, dw, V_.D, NCL_DEVICE));
    if (timing) cudaEventRecord(ev_[1], g_stream);
    const bool first = !F_;
    if (!F_) chk(ncl_factorize(K_, S_, pivot_tol, &F_));
    else chk(ncl_refactorize(F_, K_, pivot_tol));
    if (timing) cudaEventRecord(ev_[2], g_stream);
    ipm::FactorOut o;
    int zp = -1;
    chk(ncl_fact_status(F_, &o.status, &zp, &o.npos, &o.nneg, &o.nzero));
    if (timing && !first) {
      float a = 0, f = 0;
      cudaEventElapsedTime(&a, ev_[0], ev_[1]);
      cudaEventElapsedTime(&f, ev_[1], ev_[2]);
      tm_[0] += a, tm_[1] += f;
      tm_[2] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
      tm_[3] += 1;
    }
    if (timing && first)
      std::fprintf(stderr, "[ipm] first factorization (allocation + upload): %.3f ms\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
    return o;
  }
  ipm::SolveOut solve(const ipm::Scal& S, double target, int max_sweeps) override {
    chk(ncl_model_jac_trans_times(M_, jac_, V_.dq, V_.jtdq, NCL_DEVICE));
    dev_ipm_elem(IE_RHS_X, V_, S, g_stream);
    ipm::SolveOut o;
    int sw = 0, cv = 0;
    chk(ncl_solve_refined(F_, K_, V_.rhs, target, max_sweeps, V_.dx, NCL_DEVICE, &o.residual, &sw, &cv));
    o.sweeps = sw;
    o.converged = cv != 0;
    chk(ncl_model_jac_times(M_, jac_, V_.dx, V_.jdx, NCL_DEVICE));
    dev_ipm_elem(IE_RECOVER, V_, S, g_stream);
    return o;
  }
  void max_steps(const ipm::Scal& S, double* apri, double* adual) override {
    reduce(IR_FTB, S, 2);
    *apri = std::min(1.0, hsc_[2]);
    *adual = std::min(1.0, hsc_[3]);
  }
  double dphi(const ipm::Scal& S) override {
    reduce(IR_DPHI, S, 1);
    return hsc_[2];
  }
  ipm::Merit merit_current(const ipm::Scal& S) override {
    ipm::Vecs W = V_;
    W.xt = V_.x;
    W.rt = V_.r;
    W.st = V_.s;
    W.ct = V_.c;
    dev_ipm_reduce(IR_MERIT, W, S, part_.p, dsc_ + 2, g_stream);
    fetch(2, 4);
    return merit(S, fcur_);
  }
  ipm::Merit trial(const ipm::Scal& S) override {
    dev_ipm_elem(IE_TRIAL, V_, S, g_stream);
    chk(ncl_model_eval_values_device(M_, V_.xt, dsc_ + 1, V_.ct));
    dev_ipm_reduce(IR_MERIT, V_, S, part_.p, dsc_ + 2, g_stream);
    fetch(1, 5);
    ftrial_ = hsc_[1];
    return merit(S, ftrial_);
  }
  void accept(const ipm::Scal& S) override {
    dev_ipm_elem(IE_ACCEPT, V_, S, g_stream);
    fcur_ = ftrial_;
  }
  void restore() override { dev_ipm_elem(IE_RESTORE_ROW, V_, ipm::Scal{}, g_stream); }
  void r_inf(double* rinf, double* dxinf, double* xinf) override {
    reduce(IR_RINF, ipm::Scal{}, 3);
    *rinf = hsc_[2];
    *dxinf = hsc_[3];
    *xinf = hsc_[4];
  }
  double update_multipliers() override {
    dev_ipm_elem(IE_UPDATE_MULT, V_, ipm::Scal{}, g_stream);
    ck(cudaMemsetAsync(dsc_ + 2, 0, sizeof(double), g_stream), "memset");
    dev_absmax(V_.lamN, m_, dsc_ + 2, g_stream);
    fetch(2, 1);
    return hsc_[2];
  }
  double objective() const override { return fcur_; }
  void set_state(const ncl_ipm_state& st) override {
    auto up = [&](double* d, const double* h, int64_t cnt) {
      if (cnt) ck(cudaMemcpyAsync(d, h, cnt * sizeof(double), cudaMemcpyHostToDevice, g_stream), "H2D");
    };
    up(V_.x, st.x, n_), up(V_.zl, st.zl, n_), up(V_.zu, st.zu, n_);
    up(V_.r, st.r, m_), up(V_.s, st.s, m_), up(V_.y, st.y, m_), up(V_.vl, st.vl, m_), up(V_.vu, st.vu, m_);
    up(V_.lamN, st.lamN, m_);
    chk(ncl_model_eval_values_device(M_, V_.x, dsc_, V_.c));
    fetch(0, 1);
    fcur_ = hsc_[0];
  }
  void get_step(ncl_newton_step& o) override {
    auto dn = [&](double* h, const double* d, int64_t cnt) {
      if (h && cnt) ck(cudaMemcpyAsync(h, d, cnt * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
    };
    dn(o.dx, V_.dx, n_), dn(o.dzl, V_.dzl, n_), dn(o.dzu, V_.dzu, n_);
    dn(o.dr, V_.dr, m_), dn(o.ds, V_.ds, m_), dn(o.dy, V_.dy, m_), dn(o.dvl, V_.dvl, m_), dn(o.dvu, V_.dvu, m_);
    ck(cudaStreamSynchronize(g_stream), "sync");
  }
  void get_bound_duals(double* zl, double* zu) override {
    if (zl && n_) ck(cudaMemcpyAsync(zl, V_.zl, n_ * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
    if (zu && n_) ck(cudaMemcpyAsync(zu, V_.zu, n_ * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
    ck(cudaStreamSynchronize(g_stream), "sync");
  }
  void get_solution(double* x, double* y, double* r) override {
    auto dn = [&](double* h, const double* d, int64_t cnt) {
      if (h && cnt) ck(cudaMemcpyAsync(h, d, cnt * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
    };
    dn(x, V_.x, n_);
    dn(y, V_.y, m_);
    dn(r, V_.r, m_);
    ck(cudaStreamSynchronize(g_stream), "sync");
  }

 private:
  ipm::Merit merit(const ipm::Scal& S, double f) const {
    ipm::Merit mr;
    mr.theta = hsc_[2];
    mr.phi = S.sf * f + hsc_[3] + S.mu * hsc_[4];
    mr.valid = hsc_[5] == 0.0 && std::isfinite(mr.phi) && std::isfinite(mr.theta);
    return mr;
  }
  void reduce(int which, const ipm::Scal& S, int nv) {
    dev_ipm_reduce(which, V_, S, part_.p, dsc_ + 2, g_stream);
    fetch(2, nv);
  }
  void fetch(int off, int cnt) {
    ck(cudaMemcpyAsync(hsc_ + off, dsc_ + off, cnt * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
    ck(cudaStreamSynchronize(g_stream), "sync");
  }

  cudaEvent_t ev_[3] = {};
  double tm_[4] = {0, 0, 0, 0};
  ncl_model_t M_;
  int n_ = 0, m_ = 0;
  int64_t nnzj_ = 0, nnzh_ = 0, nbd_ = 0;
  DevBuf<double> slab_, part_;
  ipm::Vecs V_;
  double *jac_ = nullptr, *hess_ = nullptr, *dsc_ = nullptr, *hsc_ = nullptr;
  double fcur_ = 0, ftrial_ = 0;
  ncl_kkt_t kkt_ = nullptr;
  ncl_sym_t K_ = nullptr;
  ncl_symb_t S_ = nullptr;
  ncl_fact_t F_ = nullptr;
};

}  // namespace

struct ncl_solver {
  std::unique_ptr<GpuBackend> be;
  std::string trace;
  ncl_result last{};
  double sf = 1.0;  // objective scale of the last solve
};

API int ncl_options_default(ncl_options* o) { GUARD(*o = ipm::default_options()); }

API int ncl_solver_create(ncl_model_t M, const double* xl, const double* xu, const double* x0, const double* gl,
                          const double* gu, ncl_solver_t* out) {
  GUARD({
    auto s = std::make_unique<ncl_solver>();
    s->be = std::make_unique<GpuBackend>(M, xl, xu, x0, gl, gu);
    *out = s.release();
  });
}
API void ncl_solver_destroy(ncl_solver_t S) { delete S; }
API int ncl_solver_solve(ncl_solver_t S, const ncl_options* opt, ncl_result* res) {
  GUARD({
    const ncl_options o = opt ? *opt : ipm::default_options();
    ipm::Solver sol(*S->be, o);
    S->last = sol.solve();
    S->trace = sol.trace();
    S->sf = sol.objective_scale();
    *res = S->last;
  });
}
API int ncl_solver_newton_step(ncl_solver_t S, const ncl_ipm_state* st, const ncl_options* opt,
                               ncl_newton_step* out) {
  GUARD({
    const ncl_options o = opt ? *opt : ipm::default_options();
    ipm::newton_step(*S->be, *st, o, *out);
  });
}
API int ncl_solver_solution(ncl_solver_t S, double* x, double* y, double* r) { GUARD(S->be->get_solution(x, y, r)); }
API int ncl_solver_bound_duals(ncl_solver_t S, double* zl, double* zu, double* sf) {
  GUARD({
    S->be->get_bound_duals(zl, zu);
    if (sf) *sf = S->sf;
  });
}
API int ncl_solver_trace(ncl_solver_t S, char* buf, int64_t cap, int64_t* len) {
  GUARD({
    *len = static_cast<int64_t>(S->trace.size());
    if (buf && cap > 0) {
      const int64_t k = std::min<int64_t>(cap - 1, *len);
      std::memcpy(buf, S->trace.data(), k);
      buf[k] = 0;
    }
  });
}
