// Host symbolic layer. See sparse.hpp for the contract; every function below
// names the reference routine whose semantics it reproduces.
#include "sparse.hpp"

#include "../limits.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <atomic>
#include <thread>
#include <queue>

#include "../../../include/nclopf_expr_program.h"

namespace nclb {

static inline void fail(int code, const char* msg) { throw Error{code, msg}; }

// Host threads for the independent per-column / per-front passes of the
// analysis (outputs are position-addressed, so the result does not depend on
// the thread count). NCL_HOST_THREADS overrides (1 = sequential).
static int host_threads() {
  static const int n = [] {
    const char* e = std::getenv("NCL_HOST_THREADS");
    const int hw = static_cast<int>(std::thread::hardware_concurrency());
    return std::max(1, e ? std::atoi(e) : std::min(8, hw > 0 ? hw : 1));
  }();
  return n;
}
// fn(t, begin, end) over [0, n) split into contiguous per-thread ranges
template <class F>
static void parallel_ranges(int64_t n, int64_t min_per_thread, F fn) {
  const int nt = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(host_threads(), n / std::max<int64_t>(1, min_per_thread))));
  if (nt <= 1) {
    fn(0, int64_t(0), n);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) th.emplace_back([&, t] { fn(t, n * t / nt, n * (t + 1) / nt); });
  for (auto& x : th) x.join();
}
// fn(i) for the items of `order`, claimed dynamically (costly items first)
template <class F>
static void parallel_items(const std::vector<int>& order, F fn) {
  const int nt = std::min<int>(host_threads(), static_cast<int>(order.size()));
  if (nt <= 1) {
    for (int i : order) fn(i);
    return;
  }
  std::atomic<size_t> next{0};
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&] {
      for (size_t k; (k = next.fetch_add(1)) < order.size();) fn(order[k]);
    });
  for (auto& x : th) x.join();
}

// --- SparseSym::add (sparse_sym.cpp:12-26) ---------------------------------
void SymPattern::add(int row, int col, double value) {
  if (row < col) fail(NCL_E_INVALID, "SparseSym::add: row < col (store lower triangle)");
  if (col < 0 || row >= n_) fail(NCL_E_INVALID, "SparseSym::add: index out of range");
  if (!finalized_) {
    ensure_tvals();
    trows_.push_back(row);
    tcols_.push_back(col);
    tvals_.push_back(value);
    return;
  }
  // refill mode: coordinates must replay the original assembly order
  if (cursor_ >= static_cast<int64_t>(trows_.size()) || trows_[cursor_] != row || tcols_[cursor_] != col)
    fail(NCL_E_LOGIC, "SparseSym::add: refill coordinates do not match original assembly");
  ensure_tvals();
  tvals_[cursor_] = value;
  ++cursor_;
}

void SymPattern::add_pattern(const std::vector<int>& rows, const std::vector<int>& cols) {
  if (finalized_) fail(NCL_E_LOGIC, "SparseSym::add: pattern already finalized");
  for (size_t k = 0; k < rows.size(); ++k) {
    if (rows[k] < cols[k]) fail(NCL_E_INVALID, "SparseSym::add: row < col (store lower triangle)");
    if (cols[k] < 0 || rows[k] >= n_) fail(NCL_E_INVALID, "SparseSym::add: index out of range");
  }
  ensure_tvals();  // earlier explicit values keep their positions; these are implicit zeros
  trows_.insert(trows_.end(), rows.begin(), rows.end());
  tcols_.insert(tcols_.end(), cols.begin(), cols.end());
}

// --- SparseSym::finalize (sparse_sym.cpp:28-56) -----------------------------
// Stable (col,row) ordering realised as a stable counting sort on col
// followed by a stable sort on row inside each column; identical order to the
// reference's std::stable_sort with the same comparator.
void SymPattern::finalize() {
  if (finalized_) fail(NCL_E_LOGIC, "SparseSym::finalize: already finalized");
  const int64_t nt = static_cast<int64_t>(trows_.size());
  // LSD radix order: a stable counting sort by row, then a stable counting
  // sort by column — the (col, row) order with ties in insertion order, i.e.
  // exactly the reference's std::stable_sort result, in O(nt).
  std::vector<int> by_row(nt), order(nt);
  {
    std::vector<int64_t> rs(n_ + 1, 0);
    for (int64_t k = 0; k < nt; ++k) rs[trows_[k] + 1]++;
    for (int r = 0; r < n_; ++r) rs[r + 1] += rs[r];
    for (int64_t k = 0; k < nt; ++k) by_row[rs[trows_[k]]++] = static_cast<int>(k);
  }
  {
    std::vector<int64_t> cs(n_ + 1, 0);
    for (int64_t k = 0; k < nt; ++k) cs[tcols_[k] + 1]++;
    for (int c = 0; c < n_; ++c) cs[c + 1] += cs[c];
    for (int64_t q = 0; q < nt; ++q) {
      const int k = by_row[q];
      order[cs[tcols_[k]]++] = k;
    }
  }
  colptr_.assign(n_ + 1, 0);
  rowind_.clear();
  rowind_.reserve(nt);
  trip_slot_.assign(nt, -1);
  int prev_row = -1, prev_col = -1;
  for (int64_t s = 0; s < nt; ++s) {
    const int k = order[s];
    if (trows_[k] != prev_row || tcols_[k] != prev_col) {
      rowind_.push_back(trows_[k]);
      colptr_[tcols_[k] + 1]++;
      prev_row = trows_[k];
      prev_col = tcols_[k];
    }
    trip_slot_[k] = static_cast<int>(rowind_.size()) - 1;
  }
  for (int c = 0; c < n_; ++c) colptr_[c + 1] += colptr_[c];
  finalized_ = true;
  refill();
}

void SymPattern::begin_refill() {
  if (!finalized_) fail(NCL_E_LOGIC, "SparseSym::begin_refill: not finalized");
  cursor_ = 0;
}

// --- SparseSym::refill (sparse_sym.cpp:63-67): host copy of the merge, used
// only to keep the reference-compatible host accessor values() coherent. The
// hot-path refill is the GPU gather in csrc/cuda/assemble.cu.
void SymPattern::refill() {
  if (!finalized_) fail(NCL_E_LOGIC, "SparseSym::refill: not finalized");
  vals_.assign(rowind_.size(), 0.0);
  // triplets past tvals_.size() are implicit zeros (add_pattern): nothing to add
  for (size_t k = 0; k < tvals_.size(); ++k) vals_[trip_slot_[k]] += tvals_[k];
}

void SymPattern::slot_trip_csr(std::vector<int>& ptr, std::vector<int>& idx) const {
  const int nz = nnz();
  ptr.assign(nz + 1, 0);
  for (int s : trip_slot_) ptr[s + 1]++;
  for (int s = 0; s < nz; ++s) ptr[s + 1] += ptr[s];
  idx.resize(trip_slot_.size());
  std::vector<int> fillp(ptr.begin(), ptr.end() - 1);
  for (size_t k = 0; k < trip_slot_.size(); ++k) idx[fillp[trip_slot_[k]]++] = static_cast<int>(k);
}

// --- symbolic_order (sparse_sym.cpp:139-191) --------------------------------
// Same rule: repeatedly eliminate the node with the lexicographically smallest
// (current degree, original index); its neighbours become a clique. The
// reference keeps a std::set of (degree,node); we keep a bucket queue of
// per-degree min-heaps with lazy invalidation (a popped entry is live iff the
// node is alive and its current degree still equals the entry's degree). Adjacency lists stay sorted; the clique merge is the same
// (adj[u] \ {v}) ∪ (clique \ {u}).
std::vector<int> symbolic_order(int n, const std::vector<int>& cp, const std::vector<int>& ri) {
  std::vector<int> cnt(n + 1, 0);
  for (int c = 0; c < n; ++c)
    for (int p = cp[c]; p < cp[c + 1]; ++p) {
      const int r = ri[p];
      if (r != c) {
        cnt[r]++;
        cnt[c]++;
      }
    }
  std::vector<std::vector<int>> adj(n);
  for (int i = 0; i < n; ++i) adj[i].reserve(cnt[i]);
  for (int c = 0; c < n; ++c)
    for (int p = cp[c]; p < cp[c + 1]; ++p) {
      const int r = ri[p];
      if (r != c) {
        adj[r].push_back(c);
        adj[c].push_back(r);
      }
    }
  for (auto& a : adj) {
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
  }
  static const bool md_timing = std::getenv("NCL_SN_TIMING") != nullptr;
  const auto md_t0 = std::chrono::steady_clock::now();

  // Bucket queue: one min-heap of node ids per degree. Popping the smallest
  // node of the smallest non-empty degree yields exactly the (degree, node)
  // lexicographic sequence of one global heap (stale entries included), i.e.
  // the reference std::set's begin() sequence.
  //
  // Degrees below kSmallDeg (where nearly all eliminations happen) use exact
  // buckets instead: a three-level bitmap per degree over the node ids, a
  // node sits in the bucket of its current degree only (moved on every
  // degree change, so these buckets hold no stale entries), and the
  // smallest id is three find-first-set steps away.
  std::vector<std::vector<int>> bucket(n + 1);
  int dmin = n + 1;
  constexpr int kSmallDeg = 64;
  const int64_t w0 = (static_cast<int64_t>(n) + 63) / 64, w1 = (w0 + 63) / 64, w2 = (w1 + 63) / 64;
  std::vector<uint64_t> b0(kSmallDeg * w0, 0), b1(kSmallDeg * w1, 0), b2(kSmallDeg * w2, 0);
  std::vector<int> bcount(kSmallDeg, 0), inbm(n, -1);  // bitmap bucket of a node (its degree) or -1
  auto bm_insert = [&](int d, int v) {
    uint64_t* l0 = b0.data() + d * w0;
    uint64_t* l1 = b1.data() + d * w1;
    uint64_t* l2 = b2.data() + d * w2;
    l0[v >> 6] |= 1ull << (v & 63);
    l1[v >> 12] |= 1ull << ((v >> 6) & 63);
    l2[v >> 18] |= 1ull << ((v >> 12) & 63);
    bcount[d]++;
    inbm[v] = d;
  };
  auto bm_erase = [&](int d, int v) {
    uint64_t* l0 = b0.data() + d * w0;
    uint64_t* l1 = b1.data() + d * w1;
    uint64_t* l2 = b2.data() + d * w2;
    if ((l0[v >> 6] &= ~(1ull << (v & 63))) == 0)
      if ((l1[v >> 12] &= ~(1ull << ((v >> 6) & 63))) == 0) l2[v >> 18] &= ~(1ull << ((v >> 12) & 63));
    bcount[d]--;
    inbm[v] = -1;
  };
  auto bm_min = [&](int d) {
    const uint64_t* l0 = b0.data() + d * w0;
    const uint64_t* l1 = b1.data() + d * w1;
    const uint64_t* l2 = b2.data() + d * w2;
    int64_t i2 = 0;
    while (l2[i2] == 0) ++i2;
    const int64_t i1 = i2 * 64 + __builtin_ctzll(l2[i2]);
    const int64_t i0 = i1 * 64 + __builtin_ctzll(l1[i1]);
    return static_cast<int>(i0 * 64 + __builtin_ctzll(l0[i0]));
  };
  // (re)file node v under degree d (its old small-degree bucket, if any, is left)
  auto push = [&](int d, int v) {
    if (inbm[v] >= 0) bm_erase(inbm[v], v);
    if (d < kSmallDeg) {
      bm_insert(d, v);
    } else {
      auto& b = bucket[d];
      b.push_back(v);
      std::push_heap(b.begin(), b.end(), std::greater<int>());
    }
    if (d < dmin) dmin = d;
  };
  for (int i = 0; i < n; ++i) push(static_cast<int>(adj[i].size()), i);
  std::vector<char> dead(n, 0);
  std::vector<int> perm;
  perm.reserve(n);
  // Hybrid adjacency: sorted vectors, switched to a bitmap once a node's
  // degree exceeds kBig (the SCOPF's base-case nodes touch every
  // contingency: a vector merge would cost O(degree) per neighbouring
  // elimination, the bitmap costs O(|clique|)). Only the SET of neighbours is
  // observable (degrees and clique membership), so the representation does
  // not change the ordering.
  constexpr int kBig = 256;
  const int64_t nwords = (static_cast<int64_t>(n) + 63) / 64;
  std::vector<int> bmap(n, -1), bdeg(n, 0);  // bitmap slot per node, degree in bitmap mode
  std::vector<std::vector<uint64_t>> pool;
  std::vector<int> free_slots;
  auto degree = [&](int u) { return bmap[u] >= 0 ? bdeg[u] : static_cast<int>(adj[u].size()); };
  auto to_bitmap = [&](int u) {
    int slot;
    if (!free_slots.empty()) {
      slot = free_slots.back();
      free_slots.pop_back();
    } else {
      slot = static_cast<int>(pool.size());
      pool.emplace_back(nwords, 0ull);
    }
    auto& bm = pool[slot];
    for (int x : adj[u]) bm[x >> 6] |= 1ull << (x & 63);
    bdeg[u] = static_cast<int>(adj[u].size());
    bmap[u] = slot;
    std::vector<int>().swap(adj[u]);
  };
  std::vector<int> clique;
  std::vector<int> mark(n, 0);
  int stamp_id = 0;
  for (;;) {
    while (dmin < kSmallDeg && bcount[dmin] == 0) ++dmin;
    if (dmin >= kSmallDeg)
      while (dmin <= n && bucket[dmin].empty()) ++dmin;
    if (dmin > n) break;
    int v;
    if (dmin < kSmallDeg) {
      v = bm_min(dmin);
      bm_erase(dmin, v);
    } else {
      auto& bk = bucket[dmin];
      std::pop_heap(bk.begin(), bk.end(), std::greater<int>());
      v = bk.back();
      bk.pop_back();
      if (dead[v] || dmin != degree(v) || inbm[v] >= 0) continue;  // stale heap entry
    }
    perm.push_back(v);
    dead[v] = 1;
    if (bmap[v] >= 0) {  // enumerate the bitmap ascending, release it
      auto& bm = pool[bmap[v]];
      clique.clear();
      clique.reserve(bdeg[v]);
      for (int64_t wd = 0; wd < nwords; ++wd) {
        uint64_t bits = bm[wd];
        while (bits) {
          const int t = __builtin_ctzll(bits);
          clique.push_back(static_cast<int>(wd * 64 + t));
          bits &= bits - 1;
        }
        bm[wd] = 0;
      }
      free_slots.push_back(bmap[v]);
      bmap[v] = -1;
    } else {
      clique.swap(adj[v]);
    }
    for (int u : clique) {
      const int old = degree(u);
      if (bmap[u] >= 0) {
        auto& bm = pool[bmap[u]];
        int d = bdeg[u];
        for (int x : clique)
          if (x != u) {
            uint64_t& wd = bm[x >> 6];
            const uint64_t bit = 1ull << (x & 63);
            if (!(wd & bit)) wd |= bit, ++d;
          }
        uint64_t& wv = bm[v >> 6];
        const uint64_t bv = 1ull << (v & 63);
        if (wv & bv) wv &= ~bv, --d;
        bdeg[u] = d;
      } else {
        // (adj[u] \ {v}) ∪ (clique \ {u}) with a stamp array instead of a
        // sorted merge: adjacency lists are unordered sets (only the set is
        // observable — degrees and clique membership — so the elimination
        // order is unchanged)
        std::vector<int>& au = adj[u];
        ++stamp_id;
        size_t pv = au.size();
        for (size_t i = 0; i < au.size(); ++i) {
          const int x = au[i];
          mark[x] = stamp_id;
          if (x == v) pv = i;
        }
        if (pv < au.size()) {
          au[pv] = au.back();
          au.pop_back();
        }
        mark[u] = stamp_id;
        mark[v] = stamp_id;
        for (int x : clique)
          if (mark[x] != stamp_id) au.push_back(x);
        if (static_cast<int>(au.size()) > kBig) to_bitmap(u);
      }
      if (degree(u) != old) push(degree(u), u);
    }
    clique.clear();
    std::vector<int>().swap(clique);
  }
  if (md_timing)
    std::fprintf(stderr, "[order] elimination loop %.3f s\n",
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - md_t0).count());
  return perm;
}

// --- analyze(M, perm) (sparse_sym.cpp:198-260) ------------------------------
SymbolicCore analyze_core(int n, const std::vector<int>& cp, const std::vector<int>& ri,
                          std::vector<int> perm) {
  if (static_cast<int>(perm.size()) != n) fail(NCL_E_INVALID, "analyze: bad permutation");
  SymbolicCore S;
  S.n = n;
  S.perm = std::move(perm);
  S.iperm.assign(n, -1);
  for (int k = 0; k < n; ++k) {
    if (S.perm[k] < 0 || S.perm[k] >= n || S.iperm[S.perm[k]] != -1)
      fail(NCL_E_INVALID, "analyze: permutation is not a bijection");
    S.iperm[S.perm[k]] = k;
  }
  // Permuted upper CSC: (i,j) lower -> column max(pi,pj), row min(pi,pj),
  // columns ascending, rows ascending inside a column (keys are unique).
  const int nnz = cp[n];
  S.up_colptr.assign(n + 1, 0);
  S.up_rowind.resize(nnz);
  S.entry_map.resize(nnz);
  for (int c = 0; c < n; ++c)
    for (int p = cp[c]; p < cp[c + 1]; ++p) {
      const int pi = S.iperm[ri[p]], pj = S.iperm[c];
      S.up_colptr[std::max(pi, pj) + 1]++;
    }
  for (int c = 0; c < n; ++c) S.up_colptr[c + 1] += S.up_colptr[c];
  {
    std::vector<int> fillp(S.up_colptr.begin(), S.up_colptr.end() - 1);
    std::vector<int> src(nnz);
    for (int c = 0; c < n; ++c)
      for (int p = cp[c]; p < cp[c + 1]; ++p) {
        const int pi = S.iperm[ri[p]], pj = S.iperm[c];
        const int col = std::max(pi, pj);
        const int q = fillp[col]++;
        S.up_rowind[q] = std::min(pi, pj);
        src[q] = p;
      }
    std::vector<std::pair<int, int>> tmp;
    for (int c = 0; c < n; ++c) {
      const int b = S.up_colptr[c], e = S.up_colptr[c + 1];
      if (e - b > 1) {
        tmp.clear();
        for (int q = b; q < e; ++q) tmp.emplace_back(S.up_rowind[q], src[q]);
        std::sort(tmp.begin(), tmp.end());
        for (int q = b; q < e; ++q) {
          S.up_rowind[q] = tmp[q - b].first;
          src[q] = tmp[q - b].second;
        }
      }
    }
    for (int q = 0; q < nnz; ++q) S.entry_map[src[q]] = q;
  }
  // Elimination tree + column counts via row subtrees (flag marking).
  S.parent.assign(n, -1);
  S.l_colcount.assign(n, 0);
  std::vector<int> flag(n, -1);
  for (int k = 0; k < n; ++k) {
    flag[k] = k;
    for (int p = S.up_colptr[k]; p < S.up_colptr[k + 1]; ++p) {
      int i = S.up_rowind[p];
      while (i < k && flag[i] != k) {
        if (S.parent[i] == -1) S.parent[i] = k;
        S.l_colcount[i]++;
        flag[i] = k;
        i = S.parent[i];
      }
    }
  }
  S.l_nnz = 0;
  for (int c = 0; c < n; ++c) S.l_nnz += S.l_colcount[c];
  return S;
}

// --- supernodal schedule (product-only) -------------------------------------
// True column structure of L (reference layout): row k of L is the etree reach
// of A's row k (the same row-subtree walk as the colcounts above,
// sparse_sym.cpp:241-258); transposed into columns with rows ascending.
void true_L_structure(const SymbolicCore& S, std::vector<int64_t>& lp, std::vector<int>& li) {
  const int n = S.n;
  lp.assign(n + 1, 0);
  for (int j = 0; j < n; ++j) lp[j + 1] = lp[j] + S.l_colcount[j];
  li.resize(lp[n]);
  std::vector<int64_t> fp(lp.begin(), lp.end() - 1);
  std::vector<int> flag(n, -1);
  for (int k = 0; k < n; ++k) {
    flag[k] = k;
    for (int p = S.up_colptr[k]; p < S.up_colptr[k + 1]; ++p) {
      int i = S.up_rowind[p];
      while (i < k && flag[i] != k) {
        li[fp[i]++] = k;  // k ascending: rows sorted inside every column
        flag[i] = k;
        i = S.parent[i];
      }
    }
  }
}

Supernodal build_supernodes(const SymbolicCore& S, const std::vector<int>& cp,
                            const std::vector<int>& ri, int relax) {
  constexpr int64_t kSmemFront = kCtaFront;  // csrc/limits.hpp
  // child entries one CTA assembles comfortably; beyond, the front is assembled
  // by a multi-CTA gather (NCL_HEAVY_GATHER overrides: tests drive that path)
  static const char* heavy_env = std::getenv("NCL_HEAVY_GATHER");
  const int64_t kHeavyGather = heavy_env ? std::atoll(heavy_env) : 400000;
  const int n = S.n;
  Supernodal Z;
  static const bool timing = std::getenv("NCL_ANALYZE_TIMING") != nullptr && std::getenv("NCL_SN_TIMING") != nullptr;
  auto tl = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[supernodes] %-14s %.3f s\n", what, std::chrono::duration<double>(now - tl).count());
    tl = now;
  };
  // 1a. fundamental partition: j+1 joins j's supernode iff parent[j]==j+1 and
  //     colcount[j]==colcount[j+1]+1 (nested structure, identical rows).
  std::vector<int> fund{0};
  for (int j = 0; j + 1 < n; ++j) {
    const bool join = S.parent[j] == j + 1 && S.l_colcount[j] == S.l_colcount[j + 1] + 1;
    if (!join) fund.push_back(j + 1);
  }
  if (n > 0) fund.push_back(n);
  else fund.assign(1, 0);
  // 1b. relaxed amalgamation (CHOLMOD-style thresholds): a run of fundamental
  //     supernodes is merged into the next one when that one is its etree
  //     parent AND is adjacent in the (fixed, reference) column order, and the
  //     explicit zeros introduced stay small. Structurally-zero entries of a
  //     merged panel stay exactly 0.0 through the factorization, so D, the
  //     solution and the true-structure entries of L are unaffected up to
  //     summation order; perm/etree/colcounts are untouched.
  Z.sn_first.push_back(0);
  if (n > 0) {
    const int nf = static_cast<int>(fund.size()) - 1;
    auto true_nnz = [&](int a, int b) {  // columns [a, b)
      int64_t t = 0;
      for (int j = a; j < b; ++j) t += S.l_colcount[j] + 1;
      return t;
    };
    int g0 = 0;                                  // first column of the open group
    int64_t gtrue = true_nnz(fund[0], fund[1]);  // true entries of the group
    for (int t = 0; t + 1 < nf; ++t) {
      const int l = fund[t + 1];                 // group ends at l
      const int W = l - g0;
      bool merge = false;
      if (relax && S.parent[l - 1] == l) {       // next fundamental sn is the parent, adjacent
        const int wp = fund[t + 2] - l;
        const int64_t nrp = S.l_colcount[l] + 1;  // rows of the parent panel (incl. its columns)
        const int64_t Wm = W + wp;
        const int64_t nrm = W + nrp;
        const int64_t dense = Wm * nrm - Wm * (Wm - 1) / 2;
        const int64_t tru = gtrue + true_nnz(l, fund[t + 2]);
        const double z = dense > 0 ? static_cast<double>(dense - tru) / static_cast<double>(dense) : 0.0;
        merge = Wm <= 256 && (Wm <= 4 || (Wm <= 16 && z < 0.8) || (Wm <= 48 && z < 0.1) || z < 0.05);
        if (merge) gtrue = tru;
      }
      if (!merge) {
        Z.sn_first.push_back(l);
        g0 = l;
        gtrue = true_nnz(l, fund[t + 2]);
      }
    }
    Z.sn_first.push_back(n);
  }
  Z.nsn = static_cast<int>(Z.sn_first.size()) - 1;
  const int nsn = Z.nsn;
  Z.sn_of_col.assign(n, -1);
  for (int s = 0; s < nsn; ++s)
    for (int j = Z.sn_first[s]; j < Z.sn_first[s + 1]; ++j) Z.sn_of_col[j] = s;
  Z.sn_parent.assign(nsn, -1);
  for (int s = 0; s < nsn; ++s) {
    const int last = Z.sn_first[s + 1] - 1;
    if (S.parent[last] >= 0) Z.sn_parent[s] = Z.sn_of_col[S.parent[last]];
  }
  // children CSR (ascending child index = ascending columns)
  Z.cptr.assign(nsn + 1, 0);
  for (int s = 0; s < nsn; ++s)
    if (Z.sn_parent[s] >= 0) Z.cptr[Z.sn_parent[s] + 1]++;
  for (int s = 0; s < nsn; ++s) Z.cptr[s + 1] += Z.cptr[s];
  Z.child.resize(Z.cptr[nsn]);
  {
    std::vector<int> fp(Z.cptr.begin(), Z.cptr.end() - 1);
    for (int s = 0; s < nsn; ++s)
      if (Z.sn_parent[s] >= 0) Z.child[fp[Z.sn_parent[s]]++] = s;
  }
  lap("partition");
  // 2. lower structure of A (permuted): column j holds rows i>j.
  std::vector<int> lcp(n + 1, 0), lri;
  for (int c = 0; c < n; ++c)
    for (int p = S.up_colptr[c]; p < S.up_colptr[c + 1]; ++p)
      if (S.up_rowind[p] < c) lcp[S.up_rowind[p] + 1]++;
  for (int j = 0; j < n; ++j) lcp[j + 1] += lcp[j];
  lri.resize(lcp[n]);
  {
    std::vector<int> fp(lcp.begin(), lcp.end() - 1);
    for (int c = 0; c < n; ++c)
      for (int p = S.up_colptr[c]; p < S.up_colptr[c + 1]; ++p)
        if (S.up_rowind[p] < c) lri[fp[S.up_rowind[p]]++] = c;
  }
  lap("lower A");
  // 3. row structures R_s = cols(s) ∪ (A rows ∪ children's rows below s),
  //    children before parents.
  Z.sn_rptr.assign(nsn + 1, 0);
  std::vector<std::vector<int>> R(nsn);
  std::vector<int> mark(n, -1), buf;
  for (int s = 0; s < nsn; ++s) {
    const int f = Z.sn_first[s], l = Z.sn_first[s + 1];
    buf.clear();
    for (int j = f; j < l; ++j)
      for (int p = lcp[j]; p < lcp[j + 1]; ++p) {
        const int r = lri[p];
        if (r >= l && mark[r] != s) {
          mark[r] = s;
          buf.push_back(r);
        }
      }
    for (int q = Z.cptr[s]; q < Z.cptr[s + 1]; ++q)
      for (int r : R[Z.child[q]])
        if (r >= l && mark[r] != s) {
          mark[r] = s;
          buf.push_back(r);
        }
    std::sort(buf.begin(), buf.end());
    R[s].reserve(l - f + buf.size());
    for (int j = f; j < l; ++j) R[s].push_back(j);
    R[s].insert(R[s].end(), buf.begin(), buf.end());
  }
  lap("row structures");
  // structure check against the reference column counts: exact for
  // fundamental columns, a superset inside amalgamated panels
  for (int s = 0; s < nsn; ++s) {
    const int f = Z.sn_first[s], l = Z.sn_first[s + 1];
    const int nr = static_cast<int>(R[s].size());
    for (int j = f; j < l; ++j) {
      const int have = nr - (j - f) - 1;
      if (relax ? have < S.l_colcount[j] : have != S.l_colcount[j])
        fail(NCL_E_INTERNAL, "supernode structure disagrees with l_colcount");
    }
  }
  for (int s = 0; s < nsn; ++s) Z.sn_rptr[s + 1] = Z.sn_rptr[s] + static_cast<int64_t>(R[s].size());
  Z.rows.resize(Z.sn_rptr[nsn]);
  for (int s = 0; s < nsn; ++s) std::copy(R[s].begin(), R[s].end(), Z.rows.begin() + Z.sn_rptr[s]);
  // panels (nr x w, column-major) and contribution blocks (m2 x m2, m2 = nr - w)
  Z.sn_loff.assign(nsn + 1, 0);
  Z.cb_off.assign(nsn + 1, 0);
  for (int s = 0; s < nsn; ++s) {
    const int64_t w = Z.sn_first[s + 1] - Z.sn_first[s];
    const int64_t nr = static_cast<int64_t>(R[s].size());
    Z.sn_loff[s + 1] = Z.sn_loff[s] + w * nr;
    Z.cb_off[s + 1] = Z.cb_off[s] + (nr - w) * (nr - w + 1) / 2;  // packed lower, column-major
    Z.max_w = std::max<int>(Z.max_w, static_cast<int>(w));
    Z.max_nr = std::max<int>(Z.max_nr, static_cast<int>(nr));
  }
  Z.l_storage = Z.sn_loff[nsn];
  Z.cb_storage = Z.cb_off[nsn];
  lap("offsets");
  // 4. relative positions of every child row below the child's columns in
  //    its parent's row list (extend-add maps of the multifrontal scheme)
  Z.relp.assign(Z.rows.size(), -1);
  for (int c = 0; c < nsn; ++c) {
    const int p = Z.sn_parent[c];
    if (p < 0) continue;
    const int wc = Z.sn_first[c + 1] - Z.sn_first[c];
    const auto& Rp = R[p];
    size_t q = 0;
    for (size_t k = wc; k < R[c].size(); ++k) {
      const int r = R[c][k];
      while (Rp[q] < r) ++q;  // both ascending
      if (Rp[q] != r) fail(NCL_E_INTERNAL, "child row missing from parent structure");
      Z.relp[Z.sn_rptr[c] + k] = static_cast<int>(q);
    }
  }
  lap("relp");
  // 5. heights and ticket order (leaves first)
  Z.height.assign(nsn, 0);
  for (int s = 0; s < nsn; ++s)
    if (Z.sn_parent[s] >= 0) Z.height[Z.sn_parent[s]] = std::max(Z.height[Z.sn_parent[s]], Z.height[s] + 1);
  Z.max_height = 0;
  for (int s = 0; s < nsn; ++s) Z.max_height = std::max(Z.max_height, Z.height[s]);
  Z.order.resize(nsn);
  std::vector<int> hc(Z.max_height + 2, 0);
  for (int s = 0; s < nsn; ++s) hc[Z.height[s] + 1]++;
  for (int h = 0; h <= Z.max_height; ++h) hc[h + 1] += hc[h];
  {
    std::vector<int> fp(hc.begin(), hc.end() - 1);
    for (int s = 0; s < nsn; ++s) Z.order[fp[Z.height[s]]++] = s;
  }
  // phase split: the narrow top of the tree (at most kTopTasks supernodes)
  // runs with a whole CTA per supernode, everything below with a warp each.
  static const char* top_env = std::getenv("NCL_TOP_TASKS");  // tuning experiments only
  // measured (r02, 500x256): 8192 (h >= 11 on the CTA path) 1.69 ms, 6144 (h >= 12) 1.64, 4096 (h >= 13) 1.69, 2048 2.27
  const int kTopTasks = top_env ? std::atoi(top_env) : 6144;
  Z.nsplit = nsn;
  for (int h = Z.max_height; h >= 0; --h) {
    if (nsn - hc[h] > kTopTasks) break;
    Z.nsplit = hc[h];
  }
  Z.nleaf = hc[1] - hc[0];
  lap("heights");
  // 6. A -> panel map, diagonal positions
  const int nnz = cp[n];
  Z.amap.resize(nnz);
  std::vector<int> asn(nnz);  // target supernode of every A entry
  Z.diag_pos.clear();
  {
    std::vector<std::vector<int>> dpos(host_threads());
    parallel_ranges(n, 4096, [&](int t, int64_t c0, int64_t c1) {
      for (int c = static_cast<int>(c0); c < c1; ++c)
        for (int p = cp[c]; p < cp[c + 1]; ++p) {
          const int r = ri[p];
          if (r == c) dpos[t].push_back(p);
          const int pi = S.iperm[r], pj = S.iperm[c];
          const int lo = std::min(pi, pj), hi = std::max(pi, pj);
          const int s = Z.sn_of_col[lo];
          const int f = Z.sn_first[s];
          const int* rb = Z.rows.data() + Z.sn_rptr[s];
          const int nr = static_cast<int>(Z.sn_rptr[s + 1] - Z.sn_rptr[s]);
          const int pos = static_cast<int>(std::lower_bound(rb, rb + nr, hi) - rb);
          Z.amap[p] = Z.sn_loff[s] + static_cast<int64_t>(lo - f) * nr + pos;
          asn[p] = s;
        }
    });
    for (auto& v : dpos) Z.diag_pos.insert(Z.diag_pos.end(), v.begin(), v.end());  // column order
  }
  lap("A map");
  // 6b. A entries grouped by target supernode (source slot, offset in panel)
  {
    Z.a_ptr.assign(nsn + 1, 0);
    for (size_t e = 0; e < Z.amap.size(); ++e) Z.a_ptr[asn[e] + 1]++;
    for (int sn = 0; sn < nsn; ++sn) Z.a_ptr[sn + 1] += Z.a_ptr[sn];
    Z.a_src.resize(Z.amap.size());
    Z.a_off.resize(Z.amap.size());
    std::vector<int64_t> fp(Z.a_ptr.begin(), Z.a_ptr.end() - 1);
    for (size_t e = 0; e < Z.amap.size(); ++e) {
      const int sn = asn[e];
      const int64_t q = fp[sn]++;
      Z.a_src[q] = static_cast<int>(e);
      Z.a_off[q] = static_cast<int>(Z.amap[e] - Z.sn_loff[sn]);
    }
  }
  lap("A groups");
  // 7. gather maps of the CTA-part fronts (order >= nsplit): for every front entry that receives anything,
  //    its sources in assembly order — the A value (encoded ~slot) first, then
  //    the children's packed CB entries in ascending child order — so the
  //    assembly is one independent gather-sum per entry (no per-child
  //    barriers; same summation order as the scatter/extend-add path).
  {
    Z.gm_ptr.assign(nsn + 1, 0);
    std::vector<uint8_t> want(nsn, 0);
    for (int t = Z.nsplit; t < nsn; ++t) {
      const int sn = Z.order[t];
      want[sn] = 1;
    }
    // counting sort by destination over the packed lower front (the only
    // entries that receive anything); two passes over the fronts (sizes,
    // then the fill at prefix-summed offsets), each front independent, so
    // both run on host threads with the sequential result
    std::vector<int> wl;
    for (int sn = 0; sn < nsn; ++sn)
      if (want[sn]) wl.push_back(sn);
    std::vector<int64_t> cost(nsn, 0);
    for (int sn : wl) {
      int64_t c = Z.a_ptr[sn + 1] - Z.a_ptr[sn];
      for (int q = Z.cptr[sn]; q < Z.cptr[sn + 1]; ++q) {
        const int ch = Z.child[q];
        const int64_t m2c = (Z.sn_rptr[ch + 1] - Z.sn_rptr[ch]) - (Z.sn_first[ch + 1] - Z.sn_first[ch]);
        c += m2c * (m2c + 1) / 2;
      }
      const int64_t nr = Z.sn_rptr[sn + 1] - Z.sn_rptr[sn];
      cost[sn] = c + nr * (nr + 1) / 2;
    }
    std::vector<int> byc = wl;
    std::stable_sort(byc.begin(), byc.end(), [&](int x, int y) { return cost[x] > cost[y]; });
    // per front: the count of sources landing on every packed entry
    auto count = [&](int sn, std::vector<int64_t>& cnt) {
      const int nr = static_cast<int>(Z.sn_rptr[sn + 1] - Z.sn_rptr[sn]);
      const size_t np = static_cast<size_t>(nr) * (nr + 1) / 2;
      auto pk = [nr](int rj, int ri) { return static_cast<size_t>(rj) * nr - static_cast<size_t>(rj) * (rj + 1) / 2 + ri; };
      cnt.assign(np + 1, 0);
      for (int64_t q = Z.a_ptr[sn]; q < Z.a_ptr[sn + 1]; ++q) {
        const int d = Z.a_off[q];
        cnt[pk(d / nr, d % nr) + 1]++;
      }
      for (int q = Z.cptr[sn]; q < Z.cptr[sn + 1]; ++q) {
        const int c = Z.child[q];
        const int wc = Z.sn_first[c + 1] - Z.sn_first[c];
        const int m2c = static_cast<int>(Z.sn_rptr[c + 1] - Z.sn_rptr[c]) - wc;
        const int* rel = Z.relp.data() + Z.sn_rptr[c] + wc;
        for (int j = 0; j < m2c; ++j)
          for (int i = j; i < m2c; ++i) cnt[pk(rel[j], rel[i]) + 1]++;
      }
    };
    std::vector<int64_t> nsrc(nsn, 0), ndst(nsn, 0);
    parallel_items(byc, [&](int sn) {
      thread_local std::vector<int64_t> cnt;
      count(sn, cnt);
      int64_t a = 0, b = 0;
      for (size_t d = 1; d < cnt.size(); ++d) a += cnt[d], b += cnt[d] != 0;
      nsrc[sn] = a;
      ndst[sn] = b;
    });
    std::vector<int64_t> sbase(nsn, 0);
    int64_t ts = 0;
    for (int sn = 0; sn < nsn; ++sn) {
      sbase[sn] = ts;
      ts += nsrc[sn];
      Z.gm_ptr[sn + 1] = Z.gm_ptr[sn] + ndst[sn];
    }
    Z.gsrc.assign(ts, 0);
    Z.gdst.assign(Z.gm_ptr[nsn], 0);
    Z.gsp.assign(Z.gm_ptr[nsn] + 1, 0);
    parallel_items(byc, [&](int sn) {
      thread_local std::vector<int64_t> cnt, fill;
      count(sn, cnt);
      const int nr = static_cast<int>(Z.sn_rptr[sn + 1] - Z.sn_rptr[sn]);
      const size_t np = static_cast<size_t>(nr) * (nr + 1) / 2;
      auto pk = [nr](int rj, int ri) { return static_cast<size_t>(rj) * nr - static_cast<size_t>(rj) * (rj + 1) / 2 + ri; };
      // CSR over the entries that receive something, in front (column-major) order
      const int64_t base = sbase[sn];
      fill.resize(np);
      int64_t run = 0;
      for (size_t d = 0; d < np; ++d) {
        fill[d] = run;
        run += cnt[d + 1];
      }
      for (int64_t q = Z.a_ptr[sn]; q < Z.a_ptr[sn + 1]; ++q) {
        const int d = Z.a_off[q];
        Z.gsrc[base + fill[pk(d / nr, d % nr)]++] = ~static_cast<int64_t>(Z.a_src[q]);
      }
      for (int q = Z.cptr[sn]; q < Z.cptr[sn + 1]; ++q) {
        const int c = Z.child[q];
        const int wc = Z.sn_first[c + 1] - Z.sn_first[c];
        const int m2c = static_cast<int>(Z.sn_rptr[c + 1] - Z.sn_rptr[c]) - wc;
        const int* rel = Z.relp.data() + Z.sn_rptr[c] + wc;
        for (int j = 0; j < m2c; ++j) {
          const int64_t colb = Z.cb_off[c] + static_cast<int64_t>(j) * m2c - static_cast<int64_t>(j) * (j + 1) / 2;
          for (int i = j; i < m2c; ++i) Z.gsrc[base + fill[pk(rel[j], rel[i])]++] = colb + i;
        }
      }
      // destination: packed lower offset for fronts that fit the CTA path
      // (shared-memory and one-CTA large fronts), full column-major
      // rj * nr + ri for the wider ones (blocked DMMA path)
      int64_t at = base, e = Z.gm_ptr[sn];
      for (int rj = 0; rj < nr; ++rj)
        for (int ri = rj; ri < nr; ++ri) {
          const size_t d = pk(rj, ri);
          if (cnt[d + 1]) {
            Z.gdst[e] = nr <= kSmemFront ? static_cast<int>(d) : rj * nr + ri;
            Z.gsp[e++] = at;
            at += cnt[d + 1];
          }
        }
    });
    Z.gsp[Z.gm_ptr[nsn]] = static_cast<int64_t>(Z.gsrc.size());
  lap("gather maps");
    // forward-solve gather map of the same fronts: row r of s sums its
    // children's contribution-vector entries (global CV index) in child order
    Z.cv_ptr.assign(nsn + 1, 0);
    Z.cvsp.clear();
    Z.cvsrc.clear();
    std::vector<std::vector<int64_t>> rowsrc;
    for (int sn = 0; sn < nsn; ++sn) {
      if (!want[sn]) {
        Z.cv_ptr[sn + 1] = Z.cv_ptr[sn];
        continue;
      }
      const int nr = static_cast<int>(Z.sn_rptr[sn + 1] - Z.sn_rptr[sn]);
      rowsrc.assign(nr, {});
      for (int q = Z.cptr[sn]; q < Z.cptr[sn + 1]; ++q) {
        const int c = Z.child[q];
        const int wc = Z.sn_first[c + 1] - Z.sn_first[c];
        const int m2c = static_cast<int>(Z.sn_rptr[c + 1] - Z.sn_rptr[c]) - wc;
        for (int k = 0; k < m2c; ++k)
          rowsrc[Z.relp[Z.sn_rptr[c] + wc + k]].push_back(Z.sn_rptr[c] + wc + k);
      }
      for (int r = 0; r < nr; ++r) {
        Z.cvsp.push_back(static_cast<int64_t>(Z.cvsrc.size()));
        Z.cvsrc.insert(Z.cvsrc.end(), rowsrc[r].begin(), rowsrc[r].end());
      }
      Z.cv_ptr[sn + 1] = Z.cv_ptr[sn] + nr;
    }
    Z.cvsp.push_back(static_cast<int64_t>(Z.cvsrc.size()));
    // large-front path: fronts beyond the 200 KB shared-memory cap, and fronts
    // whose assembly gathers too many child entries for one CTA (e.g. the
    // separator root under every contingency subtree)
    lap("cv maps");
    Z.big.assign(nsn, 0);
    for (int sn = 0; sn < nsn; ++sn) {
      if (!want[sn]) continue;
      const int64_t nsrc = Z.gsp[Z.gm_ptr[sn + 1]] - Z.gsp[Z.gm_ptr[sn]];
      if (Z.sn_rptr[sn + 1] - Z.sn_rptr[sn] > kSmemFront || nsrc > kHeavyGather) Z.big[sn] = 1;
    }
  }
  double fl = 0.0;
  for (int j = 0; j < n; ++j) {
    const double c = S.l_colcount[j];
    fl += c * c + 2.0 * c;
  }
  Z.flops = fl;
  return Z;
}

}  // namespace nclb
