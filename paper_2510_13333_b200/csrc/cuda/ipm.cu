// K7: IPM vector kernels (north_star step (4)): Newton right-hand side and
// diagonal terms, direction recovery, fraction-to-boundary, trial points,
// merit / KKT-error reductions. The per-element arithmetic is the shared
// source csrc/host/ipm_elem.hpp (compiled here with --fmad=false so it rounds
// exactly like the CPU oracle built with -ffp-contract=off); reductions run
// with the fixed grid kRedBlocks x kRedThreads and a fixed tree (one launch:
// warp-shuffle block trees, the last block folds the block partials), which
// reduce_host() reproduces on the CPU.
#include <cuda_runtime.h>

#include "../host/ipm_elem.hpp"
#include "dev.hpp"
#include "ipm_dev.hpp"

namespace nclb {

namespace {

using namespace nclb::ipm;

__global__ void __launch_bounds__(256) elem_kernel(int op, Vecs V, Scal S) {
  const int64_t n = V.n, m = V.m;
  int64_t N;
  switch (op) {
    case IE_INIT_X:
    case IE_RHS_X:
      N = n;
      break;
    case IE_INIT_ROW:
    case IE_RESTORE_ROW:
    case IE_UPDATE_MULT:
      N = m;
      break;
    default:
      N = n + m;
  }
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < N;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const bool xp = j < n;
    const int i = static_cast<int>(xp ? j : j - n);
    switch (op) {
      case IE_INIT_X: init_x(V, static_cast<int>(j), S); break;
      case IE_INIT_ROW: init_row(V, static_cast<int>(j), S); break;
      case IE_NEWTON:
        if (xp) newton_x(V, i, S);
        else newton_row(V, i, S);
        break;
      case IE_RHS_X: rhs_x(V, static_cast<int>(j)); break;
      case IE_RECOVER:
        if (xp) recover_x(V, i, S);
        else recover_row(V, i, S);
        break;
      case IE_TRIAL:
        if (xp) trial_x(V, i, S);
        else trial_row(V, i, S);
        break;
      case IE_ACCEPT:
        if (xp) accept_x(V, i, S);
        else accept_row(V, i, S);
        break;
      case IE_RESTORE_ROW: restore_row(V, static_cast<int>(j)); break;
      case IE_UPDATE_MULT: update_multiplier_row(V, static_cast<int>(j)); break;
    }
  }
}

// Block-local halving tree over kRedThreads values per accumulator: pairs
// (t, t+h) for h = T/2..1 — shared memory while h >= 32, warp shuffles below
// (the same pairs, so the same result as the all-shared tree).
template <int NV>
__device__ __forceinline__ void block_tree(double (&a)[NV], double* sh, const int (&kind)[NV]) {
  const int t = threadIdx.x;
#pragma unroll
  for (int k = 0; k < NV; ++k) sh[t * NV + k] = a[k];
  __syncthreads();
  for (int h = kRedThreads / 2; h >= 32; h >>= 1) {
    if (t < h)
#pragma unroll
      for (int k = 0; k < NV; ++k) sh[t * NV + k] = comb(kind[k], sh[t * NV + k], sh[(t + h) * NV + k]);
    __syncthreads();
  }
  if (t < 32) {
#pragma unroll
    for (int k = 0; k < NV; ++k) a[k] = sh[t * NV + k];
#pragma unroll
    for (int h = 16; h > 0; h >>= 1)
#pragma unroll
      for (int k = 0; k < NV; ++k) a[k] = comb(kind[k], a[k], __shfl_down_sync(0xffffffffu, a[k], h));
  }
}

// One launch per reduction: every block reduces its grid-stride slice, the
// last block to finish (atomic ticket) folds the kRedBlocks partials with a
// fixed tree and writes out[0..NV). The ticket lives after the partials and
// is reset by the last block, so back-to-back launches on one stream reuse it.
template <class R>
__global__ void __launch_bounds__(kRedThreads) reduce_kernel(Vecs V, Scal S, double* __restrict__ part,
                                                             double* __restrict__ out) {
  constexpr int NV = R::NV;
  static_assert(kRedBlocks > kRedThreads && kRedBlocks <= 2 * kRedThreads, "final fold assumes T < B <= 2T");
  __shared__ double sh[kRedThreads * NV];
  __shared__ bool last;
  int kind[NV];
  double a[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) kind[k] = R::kind(k), a[k] = comb_init(kind[k]);
  const int64_t N = static_cast<int64_t>(V.n) + V.m;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * kRedThreads + threadIdx.x; j < N;
       j += static_cast<int64_t>(kRedBlocks) * kRedThreads)
    R::elem(V, j, S, a);
  block_tree<NV>(a, sh, kind);
  unsigned int* ticket = reinterpret_cast<unsigned int*>(part + kRedBlocks * 8);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) part[blockIdx.x * NV + k] = a[k];
    __threadfence();
    last = atomicAdd(ticket, 1u) == kRedBlocks - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int t = threadIdx.x;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double p0 = __ldcg(part + t * NV + k);
    a[k] = t + kRedThreads < kRedBlocks ? comb(kind[k], p0, __ldcg(part + (t + kRedThreads) * NV + k)) : p0;
  }
  __syncthreads();  // sh is reused
  block_tree<NV>(a, sh, kind);
  if (t == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) out[k] = a[k];
    *ticket = 0u;
  }
}

template <class R>
void launch_reduce(const Vecs& V, const Scal& S, double* part, double* out, cudaStream_t st) {
  reduce_kernel<R><<<kRedBlocks, kRedThreads, 0, st>>>(V, S, part, out);
  g_kernel_launches += 1;
}

}  // namespace

void dev_ipm_elem(int op, const Vecs& V, const Scal& S, cudaStream_t st) {
  int64_t N = static_cast<int64_t>(V.n) + V.m;
  if (N == 0) return;
  int64_t blocks = (N + 255) / 256;
  const int64_t cap = static_cast<int64_t>(dev_num_sms()) * 8;
  if (blocks > cap) blocks = cap;
  elem_kernel<<<static_cast<int>(blocks), 256, 0, st>>>(op, V, S);
  g_kernel_launches += 1;
}

void dev_ipm_reduce(int which, const Vecs& V, const Scal& S, double* part, double* out, cudaStream_t st) {
  switch (which) {
    case IR_KKT: launch_reduce<RedKkt>(V, S, part, out, st); break;
    case IR_FTB: launch_reduce<RedFtb>(V, S, part, out, st); break;
    case IR_MERIT: launch_reduce<RedMerit>(V, S, part, out, st); break;
    case IR_DPHI: launch_reduce<RedDphi>(V, S, part, out, st); break;
    case IR_RINF: launch_reduce<RedRinf>(V, S, part, out, st); break;
  }
}

}  // namespace nclb
