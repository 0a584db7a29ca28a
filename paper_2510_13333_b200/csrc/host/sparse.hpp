// Host-side sparse pattern container and one-time symbolic analysis.
//
// Clean-room re-implementation of the reference sparse_core *semantics*
// (/root/reference/proj/include/nclopf/sparse_sym.hpp:20-88,
//  /root/reference/proj/src/sparse_sym.cpp:12-262): the pattern, the
// duplicate map, the ordering, the etree and the column counts must be
// bit-identical to the reference, because the north_star requires the
// symbolic analysis to match exactly. All numeric work on values happens on
// the GPU (csrc/cuda); this file never touches per-iteration values except
// for the reference-compatible host accessors.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace nclb {

struct Error {
  int code;  // NCL_E_* (include/nclopf_expr_program.h)
  std::string msg;
};

// SparseSym pattern: lower-triangle COO -> CSC with deterministic duplicate
// summation. Mirrors SparseSym::add/finalize/begin_refill/refill
// (sparse_sym.cpp:12-67).
class SymPattern {
 public:
  explicit SymPattern(int n) : n_(n) {}
  int dim() const { return n_; }
  bool finalized() const { return finalized_; }

  // throws Error{NCL_E_INVALID|NCL_E_LOGIC}
  void add(int row, int col, double value);
  // bulk add() of zero-valued triplets before finalize (same checks)
  void add_pattern(const std::vector<int>& rows, const std::vector<int>& cols);
  void finalize();
  void begin_refill();
  void refill();  // host-side merge of recorded triplets (reference refill semantics)

  int nnz() const { return static_cast<int>(rowind_.size()); }
  const std::vector<int>& col_ptr() const { return colptr_; }
  const std::vector<int>& row_ind() const { return rowind_; }
  const std::vector<double>& values() const { return vals_; }
  std::vector<double>& values_mut() { return vals_; }
  // triplet k -> value slot (the refill map, sparse_sym.cpp:41-51)
  const std::vector<int>& trip_slot() const { return trip_slot_; }
  int64_t num_trips() const { return static_cast<int64_t>(trows_.size()); }
  const std::vector<int>& trip_rows() const { return trows_; }
  const std::vector<int>& trip_cols() const { return tcols_; }
  // triplet values; triplets added by add_pattern carry an implicit 0.0
  // that is materialised only when a value is asked for
  const std::vector<double>& trip_vals() const {
    ensure_tvals();
    return tvals_;
  }
  // CSR over value slots listing triplet indices in triplet order; the GPU
  // refill gathers with it so sums happen in the reference order (:66).
  void slot_trip_csr(std::vector<int>& ptr, std::vector<int>& idx) const;
  bool in_refill() const { return finalized_; }
  int64_t refill_cursor() const { return cursor_; }

 private:
  int n_;
  bool finalized_ = false;
  std::vector<int> trows_, tcols_;
  mutable std::vector<double> tvals_;  // may be shorter than trows_: the rest are 0.0
  void ensure_tvals() const {
    if (tvals_.size() < trows_.size()) tvals_.resize(trows_.size(), 0.0);
  }
  std::vector<int> trip_slot_;
  std::vector<int> colptr_, rowind_;
  std::vector<double> vals_;
  int64_t cursor_ = 0;
};

// Exact minimum degree, (degree, index)-lexicographic, explicit clique fill.
// Bit-identical to symbolic_order (sparse_sym.cpp:139-191).
std::vector<int> symbolic_order(int n, const std::vector<int>& colptr, const std::vector<int>& rowind);

// Reference-compatible SymbolicFactor fields (sparse_sym.hpp:74-85).
struct SymbolicCore {
  int n = 0;
  std::vector<int> perm, iperm, parent;
  std::vector<int> up_colptr, up_rowind, entry_map;
  std::vector<int> l_colcount;
  int64_t l_nnz = 0;
};

// analyze(M, perm) (sparse_sym.cpp:198-260). Throws Error on a bad perm.
SymbolicCore analyze_core(int n, const std::vector<int>& colptr, const std::vector<int>& rowind,
                          std::vector<int> perm);

// ---------------------------------------------------------------------------
// Supernodal schedule consumed by the GPU factor/solve kernels (product-only;
// does not alter perm/etree/fill).
// ---------------------------------------------------------------------------
struct Supernodal {
  int nsn = 0;
  std::vector<int> sn_first;   // [nsn+1] first column (permuted index) of each supernode
  std::vector<int> sn_of_col;  // [n]
  std::vector<int> sn_parent;  // [nsn] parent supernode or -1
  std::vector<int64_t> sn_rptr;  // [nsn+1] offsets into rows
  std::vector<int> rows;         // row structure R_s (permuted, ascending; starts with the s columns)
  std::vector<int> relp;         // [rows] position of a child row (k >= w) in the parent's R
  std::vector<int64_t> sn_loff;  // [nsn+1] offsets of dense column-major panels (nr x w)
  std::vector<int64_t> cb_off;   // [nsn+1] offsets of packed-lower contribution blocks (m2 (m2+1)/2)
  int64_t l_storage = 0, cb_storage = 0;
  // children lists (supernode etree)
  std::vector<int> cptr, child;
  // ticket order (leaves first by height), heights, phase split, leaf count
  std::vector<int> order;
  std::vector<int> height;
  int max_height = 0, nsplit = 0, nleaf = 0;
  // A -> panel offsets for every entry of the source lower CSC
  std::vector<int64_t> amap;
  // diagonal entry positions of the source CSC (for max|diag|)
  std::vector<int> diag_pos;
  // gather maps of the CTA-part shared-memory fronts (see build_supernodes §7):
  // supernode s owns front entries gdst[gm_ptr[s] .. gm_ptr[s+1]); entry k sums
  // gsrc[gsp[k] .. gsp[k+1]) (~slot = A value, else a global CB index)
  std::vector<int64_t> gm_ptr, gsp, gsrc;
  std::vector<int> gdst;
  // forward-solve gather of the same fronts: rows [cv_ptr[s], cv_ptr[s+1]) of
  // s, row k sums cvsrc[cvsp[k] .. cvsp[k+1]) (global CV indices)
  std::vector<int64_t> cv_ptr, cvsp, cvsrc;
  std::vector<uint8_t> big;  // [nsn] large-front path (multi-CTA gather + blocked DMMA factor)
  // A entries grouped by supernode: [a_ptr[s], a_ptr[s+1]) -> source value slot, offset in the panel
  std::vector<int64_t> a_ptr;
  std::vector<int> a_src, a_off;
  int max_w = 0, max_nr = 0;
  double flops = 0.0;  // sum_j (c_j^2 + 2 c_j) over reference column counts
};

// relax = 1: CHOLMOD-style relaxed amalgamation of adjacent parent/child
// supernodes (does not change perm, etree or the reference fill pattern).
Supernodal build_supernodes(const SymbolicCore& S, const std::vector<int>& colptr,
                            const std::vector<int>& rowind, int relax = 1);

// True column structure of L in the reference layout (lp[n+1], li[l_nnz]).
void true_L_structure(const SymbolicCore& S, std::vector<int64_t>& lp, std::vector<int>& li);

}  // namespace nclb
