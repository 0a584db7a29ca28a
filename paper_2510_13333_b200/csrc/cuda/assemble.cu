// K2 assembly primitives: deterministic gather-sum of contributions into
// value slots in a precomputed order.
//
// Replaces SparseSym::refill (/root/reference/proj/src/sparse_sym.cpp:63-67),
// which accumulates vals_[trip_slot_[k]] += trips_[k].val in triplet order.
// The GPU version inverts trip_slot_ once (CSR: slot -> triplet indices in
// ascending k) and lets one thread sum each slot sequentially in that order,
// so every value is bit-identical to the reference (no FMA, same
// association), with no atomics.
#include <cuda_runtime.h>

#include <cstdint>

#include "dev.hpp"

namespace nclb {

__global__ void gather_sum_kernel(int64_t nslots, const int* __restrict__ ptr, const int* __restrict__ idx,
                                  const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots; s += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int p = ptr[s]; p < ptr[s + 1]; ++p) acc = __dadd_rn(acc, src[idx[p]]);
    dst[s] = acc;
  }
}

void dev_gather_sum(int64_t nslots, const int* ptr, const int* idx, const double* src, double* dst,
                    cudaStream_t st) {
  if (nslots <= 0) return;
  int64_t g = (nslots + 255) / 256;
  const int cap = dev_num_sms() * 8;
  if (g > cap) g = cap;
  g_kernel_launches += 1;
  gather_sum_kernel<<<static_cast<int>(g), 256, 0, st>>>(nslots, ptr, idx, src, dst);
}

}  // namespace nclb
