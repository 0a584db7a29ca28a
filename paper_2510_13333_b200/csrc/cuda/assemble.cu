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

// K2, compact form: the same sums, bitwise (same operands, same order, no
// FMA), with a third of the index traffic and coalesced loads. A warp owns 32
// consecutive K slots; their JᵀDJ terms are contiguous in slot order, so the
// warp streams them 32 at a time (term = J position a (int32) + the offset
// of its partner b = a - delta (uint8); D's row from jrow[a]), every lane
// forms one product D_r J_a J_b into a shared-memory window, and each lane
// then adds its own slot's products in triplet order after its Hessian and
// diagonal contributions. The diagonal variable of a slot is the rank of the
// slot among the diagonal slots (one per column, the column's first slot):
// a bitmask + per-word prefix instead of an index per slot.
constexpr int kAsmWin = 256;  // products per warp window (doubles of shared memory)
__global__ void __launch_bounds__(256) kkt_assemble_compact(int64_t nnz, const int* __restrict__ slot_h,
                                                            const uint64_t* __restrict__ dgmask,
                                                            const int* __restrict__ dgrank,
                                                            const uint32_t* __restrict__ tp,
                                                            const int* __restrict__ ta,
                                                            const uint8_t* __restrict__ td,
                                                            const int* __restrict__ jrow,
                                                            const double* __restrict__ H, const double* __restrict__ J,
                                                            const double* __restrict__ sigx, double dw,
                                                            const double* __restrict__ D, double* __restrict__ K) {
  __shared__ double win[8][kAsmWin];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* pw = win[w];
  const int64_t ngrp = (nnz + 31) / 32;
  for (int64_t g = blockIdx.x * 8ll + w; g < ngrp; g += static_cast<int64_t>(gridDim.x) * 8) {
    const int64_t s = g * 32 + lane;
    const bool live = s < nnz;
    const int64_t se = min(g * 32 + 32, nnz);
    const uint32_t T0 = __ldg(tp + g * 32), T1 = __ldg(tp + se);
    const uint32_t t0 = live ? __ldg(tp + s) : T1, t1 = live ? __ldg(tp + s + 1) : T1;
    double acc = 0.0;
    if (live) {
      const int h = __ldg(slot_h + s);
      if (h >= 0) acc = __dadd_rn(acc, __ldg(H + h));
      const uint64_t m = __ldg(dgmask + (s >> 6));
      if ((m >> (s & 63)) & 1ull) {
        const int c = __ldg(dgrank + (s >> 6)) + __popcll(m & ((1ull << (s & 63)) - 1ull));
        acc = __dadd_rn(acc, __dadd_rn(__ldg(sigx + c), dw));
      }
    }
    for (uint32_t W0 = T0; W0 < T1; W0 += kAsmWin) {
      const uint32_t W1 = min(T1, W0 + kAsmWin);
      for (uint32_t t = W0 + lane; t < W1; t += 32) {
        const int a = __ldg(ta + t), b = a - static_cast<int>(__ldg(td + t));
        pw[t - W0] = __dmul_rn(__dmul_rn(__ldg(D + __ldg(jrow + a)), __ldg(J + a)), __ldg(J + b));
      }
      __syncwarp();
      const uint32_t lo = max(t0, W0), hi = min(t1, W1);
      for (uint32_t t = lo; t < hi; ++t) acc = __dadd_rn(acc, pw[t - W0]);
      __syncwarp();
    }
    if (live) K[s] = acc;
  }
}

void dev_kkt_assemble_compact(int64_t nnz, const int* slot_h, const uint64_t* dgmask, const int* dgrank,
                              const uint32_t* tp, const int* ta, const uint8_t* td, const int* jrow, const double* H,
                              const double* J, const double* sigx, double dw, const double* D, double* K,
                              cudaStream_t st) {
  if (nnz <= 0) return;
  const int64_t ngrp = (nnz + 31) / 32;
  int64_t g = (ngrp + 7) / 8;
  const int cap = dev_num_sms() * 8;
  if (g > cap) g = cap;
  g_kernel_launches += 1;
  kkt_assemble_compact<<<static_cast<int>(g), 256, 0, st>>>(nnz, slot_h, dgmask, dgrank, tp, ta, td, jrow, H, J, sigx,
                                                           dw, D, K);
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
