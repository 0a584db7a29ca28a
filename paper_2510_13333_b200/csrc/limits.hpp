// Front-size cutoffs shared by the host schedule builder (csrc/host/sparse.cpp,
// csrc/capi.cpp) and the kernels (csrc/cuda/ldlt.cu): the gather maps store
// packed-lower destinations exactly for the fronts the CTA shared-memory path
// takes, so both sides must agree on one number.
#pragma once

namespace nclb {

// nr cap of the CTA shared-memory front (packed lower: 160 * 161 / 2 * 8 B =
// 100.6 KB, two CTAs per SM); larger fronts take the blocked DMMA path
constexpr int kCtaFront = 160;
static_assert(kCtaFront * (kCtaFront + 1) / 2 * 8 <= 113 * 1024, "two CTA fronts must fit one SM's shared memory");

// Register-resident fronts (csrc/capi.cpp build_batches, ldlt.cu
// reg_factor_kernel): front shapes (rows nr, pivots w) compiled as
// specialisations, R lanes per front (lane r owns rows r, r + R, ...), the
// front in registers (<= 46 doubles per lane).
constexpr int kRegShapes[][3] = {{5, 2, 1}, {6, 1, 1}, {7, 1, 1}, {8, 1, 1}, {8, 2, 1},
                                 {9, 1, 1}, {10, 1, 1}, {10, 2, 1}};
// measured (r02): adding (11..14, 1..4) with four lanes per front moved 31 k
// supernodes out of the subtree groups (warp phase 375 -> 301 us) but grew
// the register phase 226 -> 345 us and the forward register solve 89 -> 155
// us (195 registers): a net loss
constexpr int kNumRegShapes = sizeof(kRegShapes) / sizeof(kRegShapes[0]);
// shapes [0, kRegTier1) run first as their own closed forest in a kernel
// compiled for them alone (small register footprint, high occupancy); the
// rest in a second kernel whose fronts may also have tier-1 children
constexpr int kRegTier1 = kNumRegShapes;  // measured best: one kernel for all shapes

}  // namespace nclb
