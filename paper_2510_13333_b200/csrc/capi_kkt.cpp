// C-ABI for the condensed Newton matrix (K2 assembly).
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <vector>

#include "capi_internal.hpp"
#include "host/kkt.hpp"

using namespace nclb;

#define API extern "C" __attribute__((visibility("default")))
#define GUARD(...)    \
  try {               \
    __VA_ARGS__;      \
  } catch (...) {     \
    return map_exc(); \
  }                   \
  return NCL_OK;

struct ncl_kkt {
  KktMap map;
  std::unique_ptr<ncl_sym> K;
  bool dev_ready = false;
  DevBuf<int> slot_h, slot_diag, jterm;
  DevBuf<int64_t> jptr;
  DevBuf<double> h, j, s, d;  // host-path staging
  // compact form (dev_kkt_assemble_compact): term starts (uint32), terms as
  // J position + uint8 partner offset, J-entry rows, diagonal-slot bitmask +
  // per-word rank; unused (compact = false) when a term's offset exceeds 255
  bool compact = false;
  DevBuf<uint32_t> tp;
  DevBuf<int> ta, jrow, dgrank;
  DevBuf<uint8_t> td;
  DevBuf<uint64_t> dgmask;
};

namespace {
void kkt_upload(ncl_kkt* k) {
  if (k->dev_ready) return;
  static const bool timing = std::getenv("NCL_ANALYZE_TIMING") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  ensure_dev(k->K.get(), "kkt");
  k->slot_h.upload(k->map.slot_h);
  // compact form (csrc/host/kkt.hpp); the per-slot gather form only when a
  // Jacobian row is too long for the byte offsets or the term count
  // overflows 32 bits
  const KktMap& M = k->map;
  const int64_t nnz = static_cast<int64_t>(M.slot_h.size()), nt = M.jptr.empty() ? 0 : M.jptr.back();
  const bool ok = M.compact && nt < (int64_t(1) << 32) && M.nnzj < (int64_t(1) << 31);
  if (!ok) {
    KktMap& W = k->map;
    if (W.jterm.empty()) {  // rebuild the triples from the compact terms
      W.jterm.resize(3 * nt);
      for (int64_t t = 0; t < nt; ++t) {
        W.jterm[3 * t] = W.jrow[W.ta[t]];
        W.jterm[3 * t + 1] = W.ta[t];
        W.jterm[3 * t + 2] = W.ta[t] - W.td[t];
      }
    }
    k->slot_diag.upload(W.slot_diag);
    k->jptr.upload(W.jptr);
    k->jterm.upload(W.jterm);
  } else {
    std::vector<uint32_t> tp(nnz + 1);
    for (int64_t s = 0; s <= nnz; ++s) tp[s] = static_cast<uint32_t>(M.jptr[s]);
    std::vector<uint64_t> dgmask((nnz + 63) / 64 + 1, 0);
    std::vector<int> dgrank(dgmask.size(), 0);
    // diagonal slots carry variables 0, 1, 2, ... in slot order (one per column, its first slot)
    int next = 0;
    for (int64_t s = 0; s < nnz; ++s)
      if (M.slot_diag[s] >= 0) {
        if (M.slot_diag[s] != next++) throw Error{NCL_E_INTERNAL, "kkt: diagonal slots out of order"};
        dgmask[s >> 6] |= 1ull << (s & 63);
      }
    for (size_t w = 1; w < dgmask.size(); ++w) dgrank[w] = dgrank[w - 1] + __builtin_popcountll(dgmask[w - 1]);
    k->tp.upload(tp);
    k->ta.upload(M.ta);
    k->td.upload(M.td);
    k->jrow.upload(M.jrow);
    k->dgmask.upload(dgmask);
    k->dgrank.upload(dgrank);
  }
  k->compact = ok;
  k->dev_ready = true;
  if (timing)
    std::fprintf(stderr, "[kkt] device maps      %.3f s\n",
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
}
void assemble(ncl_kkt* K, const double* hess, const double* jac, const double* sigx, double dw, const double* D,
              double* out) {
  const int64_t nnz = K->K->pat.nnz();
  if (K->compact)
    dev_kkt_assemble_compact(nnz, K->slot_h.p, K->dgmask.p, K->dgrank.p, K->tp.p, K->ta.p, K->td.p, K->jrow.p, hess,
                             jac, sigx, dw, D, out, g_stream);
  else
    dev_kkt_assemble(nnz, K->slot_h.p, K->slot_diag.p, K->jptr.p, K->jterm.p, hess, jac, sigx, dw, D, out, g_stream);
}
}  // namespace

namespace nclb {
int kkt_prepare_device(ncl_kkt* K) {
  try {
    kkt_upload(K);
  } catch (...) {
    return map_exc();
  }
  return NCL_OK;
}
}  // namespace nclb

API int ncl_kkt_create(int n, int m, int64_t nnzh, const int* hr, const int* hcl, int64_t nnzj, const int* jr,
                       const int* jcl, ncl_kkt_t* out) {
  GUARD({
    std::vector<std::pair<int, int>> hc(nnzh), jc(nnzj);
    for (int64_t k = 0; k < nnzh; ++k) hc[k] = {hr[k], hcl[k]};
    for (int64_t k = 0; k < nnzj; ++k) {
      jc[k] = {jr[k], jcl[k]};
      if (k > 0 && jc[k] < jc[k - 1]) throw Error{NCL_E_INVALID, "kkt: jacobian coordinates must be row-sorted"};
    }
    auto k = std::make_unique<ncl_kkt>();
    k->K = std::make_unique<ncl_sym>(n);
    k->map = build_kkt(n, m, hc, jc, k->K->pat);
    k->K->hash = pattern_hash(k->K->pat.col_ptr(), k->K->pat.row_ind());
    *out = k.release();
  });
}
API void ncl_kkt_destroy(ncl_kkt_t K) { delete K; }
API ncl_sym_t ncl_kkt_matrix(ncl_kkt_t K) { return K->K.get(); }
API int64_t ncl_kkt_num_triplets(ncl_kkt_t K) { return static_cast<int64_t>(K->map.trow.size()); }
API int ncl_kkt_triplets(ncl_kkt_t K, int* rows, int* cols) {
  GUARD({
    std::copy(K->map.trow.begin(), K->map.trow.end(), rows);
    std::copy(K->map.tcol.begin(), K->map.tcol.end(), cols);
  });
}
API int ncl_kkt_assemble(ncl_kkt_t K, const double* hess, const double* jac, const double* sigx, double dw,
                         const double* D, int where) {
  GUARD({
    kkt_upload(K);
    const KktMap& m = K->map;
    if (where == NCL_DEVICE) {
      assemble(K, hess, jac, sigx, dw, D, K->K->vals.p);
      check_launch("kkt_assemble");
      return NCL_OK;
    }
    auto put = [](DevBuf<double>& b, const double* src, int64_t n) {
      b.alloc(n);
      if (n > 0) ck(cudaMemcpyAsync(b.p, src, n * sizeof(double), cudaMemcpyHostToDevice, g_stream), "H2D");
    };
    put(K->h, hess, m.nnzh);
    put(K->j, jac, m.nnzj);
    put(K->s, sigx, m.n);
    put(K->d, D, m.m);
    assemble(K, K->h.p, K->j.p, K->s.p, dw, K->d.p, K->K->vals.p);
    check_launch("kkt_assemble");
    ck(cudaStreamSynchronize(g_stream), "sync");
  });
}
