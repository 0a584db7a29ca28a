#include "kkt.hpp"

#include <algorithm>

namespace nclb {

KktMap build_kkt(int n, int m, const std::vector<std::pair<int, int>>& hc,
                 const std::vector<std::pair<int, int>>& jc, SymPattern& P) {
  KktMap K;
  K.n = n;
  K.m = m;
  K.nnzh = static_cast<int64_t>(hc.size());
  K.nnzj = static_cast<int64_t>(jc.size());
  // row ranges of the (row-sorted) Jacobian
  std::vector<int64_t> rp(m + 1, 0);
  for (const auto& e : jc) rp[e.first + 1]++;
  for (int r = 0; r < m; ++r) rp[r + 1] += rp[r];
  int64_t njt = 0;
  for (int r = 0; r < m; ++r) {
    const int64_t d = rp[r + 1] - rp[r];
    njt += d * (d + 1) / 2;
  }
  const int64_t nt = K.nnzh + n + njt;
  K.trow.reserve(nt);
  K.tcol.reserve(nt);
  for (const auto& e : hc) K.trow.push_back(e.first), K.tcol.push_back(e.second);
  for (int i = 0; i < n; ++i) K.trow.push_back(i), K.tcol.push_back(i);
  std::vector<int> terms;
  terms.reserve(3 * njt);
  for (int r = 0; r < m; ++r)
    for (int64_t a = rp[r]; a < rp[r + 1]; ++a)
      for (int64_t b = rp[r]; b <= a; ++b) {
        K.trow.push_back(jc[a].second);  // columns ascending inside a row: col[a] >= col[b]
        K.tcol.push_back(jc[b].second);
        terms.push_back(r);
        terms.push_back(static_cast<int>(a));
        terms.push_back(static_cast<int>(b));
      }
  P.add_pattern(K.trow, K.tcol);
  P.finalize();
  const int nnz = P.nnz();
  const auto& slot = P.trip_slot();
  K.slot_h.assign(nnz, -1);
  K.slot_diag.assign(nnz, -1);
  K.jptr.assign(nnz + 1, 0);
  for (int64_t k = K.nnzh + n; k < nt; ++k) K.jptr[slot[k] + 1]++;
  for (int s = 0; s < nnz; ++s) K.jptr[s + 1] += K.jptr[s];
  K.jterm.resize(3 * njt);
  std::vector<int64_t> fp(K.jptr.begin(), K.jptr.end() - 1);
  for (int64_t k = 0; k < nt; ++k) {
    const int s = slot[k];
    if (k < K.nnzh) {
      K.slot_h[s] = static_cast<int>(k);
    } else if (k < K.nnzh + n) {
      K.slot_diag[s] = static_cast<int>(k - K.nnzh);
    } else {
      const int64_t t = k - K.nnzh - n;
      const int64_t q = fp[s]++;
      K.jterm[3 * q] = terms[3 * t];
      K.jterm[3 * q + 1] = terms[3 * t + 1];
      K.jterm[3 * q + 2] = terms[3 * t + 2];
    }
  }
  return K;
}

}  // namespace nclb
