#include "kkt.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace nclb {

KktMap build_kkt(int n, int m, const std::vector<std::pair<int, int>>& hc,
                 const std::vector<std::pair<int, int>>& jc, SymPattern& P) {
  static const bool timing = std::getenv("NCL_ANALYZE_TIMING") != nullptr;
  auto t = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[kkt] %-16s %.3f s\n", what, std::chrono::duration<double>(now - t).count());
    t = now;
  };
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
  K.jrow.resize(K.nnzj);
  for (int r = 0; r < m; ++r) {
    if (rp[r + 1] - rp[r] > 256) K.compact = false;  // a - b would not fit a byte
    for (int64_t a = rp[r]; a < rp[r + 1]; ++a) {
      K.jrow[a] = r;
      for (int64_t b = rp[r]; b <= a; ++b) {
        K.trow.push_back(jc[a].second);  // columns ascending inside a row: col[a] >= col[b]
        K.tcol.push_back(jc[b].second);
      }
    }
  }
  lap("triplets");
  P.add_pattern(K.trow, K.tcol);
  lap("add_pattern");
  P.finalize();
  lap("finalize");
  const int nnz = P.nnz();
  const auto& slot = P.trip_slot();
  K.slot_h.assign(nnz, -1);
  K.slot_diag.assign(nnz, -1);
  K.jptr.assign(nnz + 1, 0);
  for (int64_t k = K.nnzh + n; k < nt; ++k) K.jptr[slot[k] + 1]++;
  for (int s = 0; s < nnz; ++s) K.jptr[s + 1] += K.jptr[s];
  for (int64_t k = 0; k < K.nnzh; ++k) K.slot_h[slot[k]] = static_cast<int>(k);
  for (int64_t k = K.nnzh; k < K.nnzh + n; ++k) K.slot_diag[slot[k]] = static_cast<int>(k - K.nnzh);
  // terms in triplet order (rows ascending, a ascending, b <= a) dealt to
  // their slots: inside a slot they stay in triplet order (the refill's
  // summation order)
  std::vector<int64_t> fp(K.jptr.begin(), K.jptr.end() - 1);
  if (K.compact) {
    K.ta.resize(njt);
    K.td.resize(njt);
  } else {
    K.jterm.resize(3 * njt);
  }
  int64_t k = K.nnzh + n;
  for (int r = 0; r < m; ++r)
    for (int64_t a = rp[r]; a < rp[r + 1]; ++a)
      for (int64_t b = rp[r]; b <= a; ++b, ++k) {
        const int64_t q = fp[slot[k]]++;
        if (K.compact) {
          K.ta[q] = static_cast<int>(a);
          K.td[q] = static_cast<uint8_t>(a - b);
        } else {
          K.jterm[3 * q] = r;
          K.jterm[3 * q + 1] = static_cast<int>(a);
          K.jterm[3 * q + 2] = static_cast<int>(b);
        }
      }
  lap("slot maps");
  return K;
}

}  // namespace nclb
