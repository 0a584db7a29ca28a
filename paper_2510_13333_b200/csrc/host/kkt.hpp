// Condensed Newton matrix of the NCL subproblem (paper Eq. 16 with the
// (Δλ) block eliminated; north_star step (2)):
//
//     K = H + Σ_x + δ_w I + Jᵀ D J,   D = (C + δ_c I)⁻¹,
//     C = diag(ρ⁻¹ + [row i inequality] Σ_s,i⁻¹)
//
// assembled as a SparseSym in a FIXED triplet order:
//   1. the Lagrangian-Hessian entries in hess_coords order,
//   2. one diagonal entry per variable (Σ_x,i + δ_w),
//   3. for every constraint row r (ascending) and every pair a>=b of its
//      Jacobian entries (jac_coords order): D_r J_ra J_rb.
// SparseSym::refill (sparse_sym.cpp:63-67) sums duplicates in triplet order;
// the GPU assembly kernel reproduces that order per slot, so the CPU oracle
// (reference SparseSym fed the same triplets) and the GPU build bit-identical K.
#pragma once

#include <cstdint>
#include <vector>

#include "sparse.hpp"

namespace nclb {

struct KktMap {
  int n = 0, m = 0;
  int64_t nnzh = 0, nnzj = 0;
  // triplet coordinates in assembly order (for the oracle / host façade)
  std::vector<int> trow, tcol;
  // per K slot: Hessian entry index or -1; diagonal flag; JᵀDJ terms
  std::vector<int> slot_h;
  std::vector<int> slot_diag;   // variable index if the slot is a diagonal, else -1
  std::vector<int64_t> jptr;    // [nnzK+1] term range of each slot (triplet order inside)
  // the terms D_r J_a J_b of every slot, a >= b in the same Jacobian row r:
  // ta = a, td = a - b (uint8: a row has <= 256 entries, else `compact` is
  // false and jterm holds (r, a, b) triples instead), jrow = row of each
  // Jacobian entry
  bool compact = true;
  std::vector<int> ta, jrow;
  std::vector<uint8_t> td;
  std::vector<int> jterm;
};

// Builds the triplet order and finalizes `pattern` (a fresh SymPattern of
// dimension n) with it; fills the per-slot gather structure.
KktMap build_kkt(int n, int m, const std::vector<std::pair<int, int>>& hess_coords,
                 const std::vector<std::pair<int, int>>& jac_coords, SymPattern& pattern);

}  // namespace nclb
