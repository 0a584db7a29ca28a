// Boundary exchange of the sharded multifrontal factorization / solve
// (csrc/host/shard.hpp): pack the contribution blocks (or forward-solve
// contribution vectors) of this rank's boundary supernodes into one send
// chunk; after the all-gather, copy every other rank's boundary blocks into
// place and publish their completion flags so the separator tasks can start.
// Pure copies: the exchange never changes a bit.
#include <cuda_runtime.h>

#include <algorithm>

#include "dev.hpp"

namespace nclb {

namespace {

__device__ __forceinline__ int64_t blk_size(const DevSymb& S, int s, int cv) {
  const int w = __ldg(S.sn_first + s + 1) - __ldg(S.sn_first + s);
  const int64_t m2 = (__ldg(S.sn_rptr + s + 1) - __ldg(S.sn_rptr + s)) - w;
  return cv ? m2 : m2 * (m2 + 1) / 2;
}
__device__ __forceinline__ int64_t blk_off(const DevSymb& S, int s, int cv) {
  if (!cv) return __ldg(S.cb_off + s);
  const int w = __ldg(S.sn_first + s + 1) - __ldg(S.sn_first + s);
  return __ldg(S.sn_rptr + s) + w;  // CV rows below the supernode's columns
}

__global__ void pack_kernel(DevSymb S, const double* __restrict__ src, const int* __restrict__ bids,
                            const int* __restrict__ bowner, const int64_t* __restrict__ off, int nb, int rank, int cv,
                            double* __restrict__ send) {
  for (int k = blockIdx.x; k < nb; k += gridDim.x) {
    if (__ldg(bowner + k) != rank) continue;
    const int s = __ldg(bids + k);
    const int64_t n = blk_size(S, s, cv), o = blk_off(S, s, cv), d = __ldg(off + k);
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) send[d + i] = __ldcg(src + o + i);
  }
}

__global__ void unpack_kernel(DevSymb S, double* __restrict__ dst, const int* __restrict__ bids,
                              const int* __restrict__ bowner, const int64_t* __restrict__ off, int nb, int rank,
                              int cv, const double* __restrict__ recv, int64_t chunk, int* flags, int epoch) {
  for (int k = blockIdx.x; k < nb; k += gridDim.x) {
    const int q = __ldg(bowner + k);
    if (q == rank) continue;
    const int s = __ldg(bids + k);
    const int64_t n = blk_size(S, s, cv), o = blk_off(S, s, cv), d = q * chunk + __ldg(off + k);
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[o + i] = recv[d + i];
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      flags[s] = epoch;
    }
  }
}

__global__ void zero_idx_kernel(double* __restrict__ x, const int* __restrict__ idx, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[__ldg(idx + i)] = 0.0;
}

}  // namespace

void dev_zero_indexed(double* x, const int* idx, int64_t n, cudaStream_t st) {
  if (n == 0) return;
  g_kernel_launches += 1;
  const int64_t b = std::min<int64_t>((n + 255) / 256, 1184);
  zero_idx_kernel<<<static_cast<int>(b), 256, 0, st>>>(x, idx, n);
}

void dev_shard_pack(const DevSymb& S, const double* src, const int* bids, const int* bowner, const int64_t* pack_off,
                    int nb, int rank, int cv, double* send, cudaStream_t st) {
  if (nb == 0) return;
  g_kernel_launches += 1;
  pack_kernel<<<std::min(nb, 1184), 256, 0, st>>>(S, src, bids, bowner, pack_off, nb, rank, cv, send);
}

void dev_shard_unpack(const DevSymb& S, double* dst, const int* bids, const int* bowner, const int64_t* pack_off,
                      int nb, int rank, int cv, const double* recv, int64_t chunk, int* flags, int epoch,
                      cudaStream_t st) {
  if (nb == 0) return;
  g_kernel_launches += 1;
  unpack_kernel<<<std::min(nb, 1184), 256, 0, st>>>(S, dst, bids, bowner, pack_off, nb, rank, cv, recv, chunk, flags,
                                                    epoch);
}

}  // namespace nclb
