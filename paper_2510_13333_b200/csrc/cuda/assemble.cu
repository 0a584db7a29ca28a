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

// Condensed KKT K = H + Σ_x + δ_w I + Jᵀ D J (csrc/host/kkt.hpp): one thread
// per K slot, contributions summed in the SparseSym triplet order (Hessian
// entry, diagonal entry, then (r,a,b) products row by row), no FMA.
__global__ void kkt_assemble_kernel(int64_t nnz, const int* __restrict__ slot_h, const int* __restrict__ slot_diag,
                                    const int64_t* __restrict__ jptr, const int* __restrict__ jterm,
                                    const double* __restrict__ H, const double* __restrict__ J,
                                    const double* __restrict__ sigx, double dw, const double* __restrict__ D,
                                    double* __restrict__ K) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nnz; s += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    const int h = slot_h[s];
    if (h >= 0) acc = __dadd_rn(acc, H[h]);
    const int d = slot_diag[s];
    if (d >= 0) acc = __dadd_rn(acc, __dadd_rn(sigx[d], dw));
    for (int64_t p = jptr[s]; p < jptr[s + 1]; ++p) {
      const int r = jterm[3 * p], a = jterm[3 * p + 1], b = jterm[3 * p + 2];
      acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(D[r], J[a]), J[b]));
    }
    K[s] = acc;
  }
}

void dev_kkt_assemble(int64_t nnz, const int* slot_h, const int* slot_diag, const int64_t* jptr, const int* jterm,
                      const double* H, const double* J, const double* sigx, double dw, const double* D, double* K,
                      cudaStream_t st) {
  if (nnz <= 0) return;
  int64_t g = (nnz + 255) / 256;
  const int cap = dev_num_sms() * 8;
  if (g > cap) g = cap;
  g_kernel_launches += 1;
  kkt_assemble_kernel<<<static_cast<int>(g), 256, 0, st>>>(nnz, slot_h, slot_diag, jptr, jterm, H, J, sigx, dw, D, K);
}

}  // namespace nclb
