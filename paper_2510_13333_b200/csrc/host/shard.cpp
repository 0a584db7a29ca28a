#include "shard.hpp"

#include <algorithm>
#include <stdexcept>

#include "../../../include/nclopf_expr_program.h"

namespace nclb {

namespace {
constexpr int kMixed = -2;

// index in `list` (height-sorted) where the CTA-per-task part starts: the
// GLOBAL split height of the unsharded schedule, so every supernode is
// processed by the same team kind — hence the same arithmetic — for every
// number of ranks (bitwise G-independence)
int split_of(const std::vector<int>& list, const std::vector<int>& height, int hsplit) {
  int i = 0;
  while (i < static_cast<int>(list.size()) && height[list[i]] < hsplit) ++i;
  return i;
}
int leaves_of(const std::vector<int>& list, const std::vector<int>& height) {
  int i = 0;
  while (i < static_cast<int>(list.size()) && height[list[i]] == 0) ++i;
  return i;
}
}  // namespace

ShardPlan build_shard_plan(const Supernodal& Z, const SymbolicCore& S, const std::vector<int>& var_group,
                           int ngroups, int world, int rank) {
  if (world < 1 || rank < 0 || rank >= world) throw Error{NCL_E_INVALID, "shard: bad rank/world"};
  if (static_cast<int>(var_group.size()) != S.n) throw Error{NCL_E_INVALID, "shard: var_group size != n"};
  ShardPlan P;
  P.world = world;
  P.rank = rank;
  P.ngroups = ngroups;
  const int nsn = Z.nsn;
  const int ncont = std::max(1, ngroups - 1);
  auto rank_of = [&](int g) { return static_cast<int>((static_cast<int64_t>(g - 1) * world) / ncont); };
  // subtree group label (children precede parents in index order)
  std::vector<int> sg(nsn, -1);  // -1 = not yet set
  std::vector<uint8_t> anyc(nsn, 0);
  for (int s = 0; s < nsn; ++s) {
    int g = sg[s];
    for (int j = Z.sn_first[s]; j < Z.sn_first[s + 1]; ++j) {
      const int gj = var_group[S.perm[j]];
      if (gj < 0 || gj >= ngroups) throw Error{NCL_E_INVALID, "shard: group id out of range"};
      if (gj > 0) anyc[s] = 1;
      g = (g == -1 || g == gj) ? gj : kMixed;
    }
    sg[s] = g;
    const int p = Z.sn_parent[s];
    if (p >= 0) {
      sg[p] = (sg[p] == -1 || sg[p] == g) ? g : kMixed;
      anyc[p] |= anyc[s];
    }
  }
  P.owner.assign(nsn, -1);
  for (int s = 0; s < nsn; ++s)
    if (sg[s] >= 1) P.owner[s] = rank_of(sg[s]);
  for (int t = 0; t < nsn; ++t) {  // Z.order: leaves first by height
    const int s = Z.order[t];
    if (P.owner[s] == rank || (P.owner[s] < 0 && !anyc[s])) P.listA.push_back(s);
    else if (P.owner[s] < 0) P.listB.push_back(s);
    if (P.owner[s] >= 0) P.owned_supernodes += P.owner[s] == rank;
    else P.shared_supernodes++;
  }
  P.nleafA = leaves_of(P.listA, Z.height);
  P.nleafB = leaves_of(P.listB, Z.height);
  const int hsplit = Z.nsplit < nsn ? Z.height[Z.order[Z.nsplit]] : Z.max_height + 1;
  P.splitA = split_of(P.listA, Z.height, hsplit);
  P.splitB = split_of(P.listB, Z.height, hsplit);
  // boundary children and packing offsets per owning rank
  std::vector<int64_t> cbfill(world, 0), cvfill(world, 0);
  for (int s = 0; s < nsn; ++s) {
    const int p = Z.sn_parent[s];
    if (P.owner[s] < 0 || p < 0 || P.owner[p] >= 0) continue;
    const int q = P.owner[s];
    const int64_t w = Z.sn_first[s + 1] - Z.sn_first[s];
    const int64_t m2 = (Z.sn_rptr[s + 1] - Z.sn_rptr[s]) - w;
    P.boundary.push_back(s);
    P.bowner.push_back(q);
    P.cb_pack_off.push_back(cbfill[q]);
    P.cv_pack_off.push_back(cvfill[q]);
    cbfill[q] += m2 * (m2 + 1) / 2;
    cvfill[q] += m2;
  }
  for (int q = 0; q < world; ++q) {
    P.cb_chunk = std::max(P.cb_chunk, cbfill[q]);
    P.cv_chunk = std::max(P.cv_chunk, cvfill[q]);
  }
  P.col_report.assign(S.n, 0);
  for (int s = 0; s < nsn; ++s) {
    const bool mine = P.owner[s] == rank || (P.owner[s] < 0 && rank == 0);
    if (mine)
      for (int j = Z.sn_first[s]; j < Z.sn_first[s + 1]; ++j) P.col_report[j] = 1;
  }
  return P;
}

}  // namespace nclb
