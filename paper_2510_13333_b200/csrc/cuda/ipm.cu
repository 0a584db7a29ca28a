// K7: IPM vector kernels (north_star step (4)): Newton right-hand side and
// diagonal terms, direction recovery, fraction-to-boundary, trial points,
// merit / KKT-error reductions. The per-element arithmetic is the shared
// source csrc/host/ipm_elem.hpp (compiled here with --fmad=false so it rounds
// exactly like the CPU oracle built with -ffp-contract=off); reductions run
// with the fixed grid kRedBlocks x kRedThreads and a fixed tree, which
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

template <class R>
__global__ void __launch_bounds__(kRedThreads) reduce_kernel(Vecs V, Scal S, double* __restrict__ part) {
  constexpr int NV = R::NV;
  __shared__ double sh[kRedThreads * NV];
  double a[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) a[k] = comb_init(R::kind(k));
  const int64_t N = static_cast<int64_t>(V.n) + V.m;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * kRedThreads + threadIdx.x; j < N;
       j += static_cast<int64_t>(kRedBlocks) * kRedThreads)
    R::elem(V, j, S, a);
#pragma unroll
  for (int k = 0; k < NV; ++k) sh[threadIdx.x * NV + k] = a[k];
  __syncthreads();
  for (int h = kRedThreads / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h)
#pragma unroll
      for (int k = 0; k < NV; ++k)
        sh[threadIdx.x * NV + k] = comb(R::kind(k), sh[threadIdx.x * NV + k], sh[(threadIdx.x + h) * NV + k]);
    __syncthreads();
  }
  if (threadIdx.x < NV) part[blockIdx.x * NV + threadIdx.x] = sh[threadIdx.x];
}

template <class R>
__global__ void reduce_final_kernel(const double* __restrict__ part, double* __restrict__ out) {
  constexpr int NV = R::NV;
  const int k = threadIdx.x;
  if (k >= NV) return;
  double acc = comb_init(R::kind(k));
  for (int b = 0; b < kRedBlocks; ++b) acc = comb(R::kind(k), acc, part[b * NV + k]);
  out[k] = acc;
}

template <class R>
void launch_reduce(const Vecs& V, const Scal& S, double* part, double* out, cudaStream_t st) {
  reduce_kernel<R><<<kRedBlocks, kRedThreads, 0, st>>>(V, S, part);
  reduce_final_kernel<R><<<1, 32, 0, st>>>(part, out);
  g_kernel_launches += 2;
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
