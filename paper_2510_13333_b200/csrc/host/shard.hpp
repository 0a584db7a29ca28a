// Contingency sharding of the multifrontal factorization.
//
// The KKT of the SCOPF is block-arrowhead: the reference's own exact-MD
// ordering puts every contingency's variables in etree subtrees that hang
// below a small top separator. Each supernode gets a
// group label from its subtree: a single contingency k, base-case only, or
// mixed. Contingencies are dealt to ranks in contiguous blocks; a supernode
// whose subtree is one contingency is OWNED by that contingency's rank; base-
// only and mixed subtrees are SHARED (computed redundantly by every rank).
//
//   phase A (local):  owned supernodes + shared supernodes whose subtree holds
//                     no contingency column (the base-only subtrees)
//   exchange:         CBs of owned supernodes whose parent is shared
//                     ("boundary" children) — one all-gather
//   phase B:          the remaining shared supernodes (the separator)
//
// Every supernode is computed from identical inputs whichever rank computes
// it, and the extend-add order is the fixed child order, so L, D and the
// solution are bitwise identical for every number of ranks.
#pragma once

#include <cstdint>
#include <vector>

#include "sparse.hpp"

namespace nclb {

struct ShardPlan {
  int world = 1, rank = 0, ngroups = 1;
  std::vector<int> owner;             // per supernode: owning rank, -1 = shared
  std::vector<int> listA, listB;      // this rank's tasks, leaves-first height order
  int nleafA = 0, nleafB = 0;         // leaf tasks at the head of each list
  int splitA = 0, splitB = 0;         // index where CTA-per-task starts in each list
  // boundary supernodes (all ranks), ascending id; their CBs / CVs cross ranks
  std::vector<int> boundary, bowner;
  std::vector<int64_t> cb_pack_off, cv_pack_off;  // offset inside the owner's chunk
  int64_t cb_chunk = 0, cv_chunk = 0;              // max packed doubles over ranks
  std::vector<uint8_t> col_report;    // per pivot position: this rank reports D / x for it
  int64_t owned_supernodes = 0, shared_supernodes = 0;
};

// var_group[i] = group of ORIGINAL variable i: 0 = base case, 1..ngroups-1 =
// contingency. Contingency g goes to rank ((g-1) * world) / (ngroups-1).
ShardPlan build_shard_plan(const Supernodal& Z, const SymbolicCore& S, const std::vector<int>& var_group,
                           int ngroups, int world, int rank);

}  // namespace nclb
