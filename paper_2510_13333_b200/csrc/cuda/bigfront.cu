// Large fronts (nr > kCtaFront, the separator of the 2000-bus grids): the
// front is assembled into a dense column-major scratch buffer by a multi-CTA
// kernel, factored with a blocked right-looking LDLᵀ — one CTA factors each
// 32-column panel, the trailing Schur update F22 -= L21 (D L21)ᵀ runs on the
// FP64 tensor cores (warp-level DMMA, mma.sync.m8n8k4.f64: tcgen05 has no f64
// kind on sm_100a) over 64x64 tiles of the lower triangle — and written back
// to the supernode's panel and contribution block.
//
// Determinism: every front entry is owned by exactly one CTA in every kernel,
// children are added in ascending child order, and the DMMA k-order is fixed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "dev.hpp"

namespace nclb {

namespace {

constexpr int kBs = 32;      // panel width
constexpr int kTile = 64;    // DMMA tile (64 x 64 per CTA, 4 warps x 32 x 32)
constexpr unsigned kFullMask = 0xffffffffu;

struct BigArgs {
  DevSymb S;
  int s, f, w, nr, m2;
  double* F;        // scratch front, nr x nr column-major
  double* Wb;       // scratch W = L21 * D for the current panel (nr x kBs)
  double* L;        // panels
  double* CB;       // contribution blocks
  double* D;
  const double* kvals;
  const double* thresh;
  int* zp;
};

// --- assembly: one thread per front entry that receives anything, summing
// its sources (A value, then children's CB entries in ascending child order)
// from the gather map — spread over the whole GPU
__global__ void __launch_bounds__(256) bf_gather(BigArgs a, int64_t g0, int64_t g1) {
  const DevSymb& S = a.S;
  for (int64_t k = g0 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < g1;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t q = __ldg(S.gsp + k);
    const int64_t q1 = __ldg(S.gsp + k + 1);
    double acc = 0.0;
    for (; q + 4 <= q1; q += 4) {
      const int64_t s0 = __ldg(S.gsrc + q), s1 = __ldg(S.gsrc + q + 1), s2 = __ldg(S.gsrc + q + 2),
                    s3 = __ldg(S.gsrc + q + 3);
      const double v0 = s0 < 0 ? __ldg(a.kvals + ~s0) : __ldcg(a.CB + s0);
      const double v1 = s1 < 0 ? __ldg(a.kvals + ~s1) : __ldcg(a.CB + s1);
      const double v2 = s2 < 0 ? __ldg(a.kvals + ~s2) : __ldcg(a.CB + s2);
      const double v3 = s3 < 0 ? __ldg(a.kvals + ~s3) : __ldcg(a.CB + s3);
      acc += v0;
      acc += v1;
      acc += v2;
      acc += v3;
    }
    for (; q < q1; ++q) {
      const int64_t src = __ldg(S.gsrc + q);
      acc += src < 0 ? __ldg(a.kvals + ~src) : __ldcg(a.CB + src);
    }
    a.F[__ldg(S.gdst + k)] = acc;
  }
}

// --- panel: unblocked LDLᵀ of columns [k0, k1) over rows [k0, nr) (one CTA)
// staged in shared memory (rows k0..nr of the kBs panel columns), warps own
// columns c2 and lanes rows in the rank-1 updates; then W(:, c-k0) =
// L(:, c) * d_c for the rows below the panel.
__global__ void __launch_bounds__(256) bf_panel(BigArgs a, int k0, int k1) {
  extern __shared__ double Ps[];  // (nr - k0) x kBs, column-major, ld = nr - k0
  const int nr = a.nr, ld = nr - k0, kw = k1 - k0;
  const double thresh = __ldcg(a.thresh);
  double* F = a.F;
  for (int e = threadIdx.x; e < ld * kw; e += blockDim.x) {
    const int c = e / ld, i = e % ld;
    Ps[e] = F[static_cast<int64_t>(k0 + c) * nr + k0 + i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = 0; c < kw; ++c) {
    double* Pc = Ps + c * ld;
    const double d = Pc[c];
    if (threadIdx.x == 0) {
      a.D[a.f + k0 + c] = d;
      if (fabs(d) <= thresh) atomicMin(a.zp, a.f + k0 + c);
    }
    for (int i = c + 1 + threadIdx.x; i < ld; i += blockDim.x) Pc[i] = Pc[i] / d;
    __syncthreads();
    for (int c2 = c + 1 + warp; c2 < kw; c2 += 8) {
      const double dl = d * Pc[c2];
      double* P2 = Ps + c2 * ld;
      for (int i = c2 + lane; i < ld; i += 32) P2[i] -= Pc[i] * dl;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < ld * kw; e += blockDim.x) {
    const int c = e / ld, i = e % ld;
    F[static_cast<int64_t>(k0 + c) * nr + k0 + i] = Ps[e];
    const int gi = k0 + i;
    a.Wb[static_cast<int64_t>(c) * nr + gi] = gi >= k1 ? Ps[e] * Ps[c * ld + c] : 0.0;
  }
  for (int e = threadIdx.x; e < kw * k0; e += blockDim.x) {  // rows above the panel: W = 0
    const int c = e / k0, i = e % k0;
    a.Wb[static_cast<int64_t>(c) * nr + i] = 0.0;
  }
}

// --- panel: unblocked LDLᵀ of columns [k0, k1) over rows [k0, nr) (one CTA),
// then W(:, c-k0) = L(:, c) * d_c for the rows below the panel.
__global__ void __launch_bounds__(256) bf_panel_global(BigArgs a, int k0, int k1) {
  const int nr = a.nr;
  const double thresh = __ldcg(a.thresh);
  double* F = a.F;
  for (int c = k0; c < k1; ++c) {
    double* Fc = F + static_cast<int64_t>(c) * nr;
    const double d = Fc[c];
    if (threadIdx.x == 0) {
      a.D[a.f + c] = d;
      if (fabs(d) <= thresh) atomicMin(a.zp, a.f + c);
    }
    for (int i = c + 1 + threadIdx.x; i < nr; i += blockDim.x) Fc[i] = Fc[i] / d;
    __syncthreads();
    const int rem = k1 - c - 1;
    for (int64_t e = threadIdx.x; e < static_cast<int64_t>(rem) * nr; e += blockDim.x) {
      const int c2 = c + 1 + static_cast<int>(e / nr), i = static_cast<int>(e % nr);
      if (i >= c2) F[static_cast<int64_t>(c2) * nr + i] -= Fc[i] * (d * Fc[c2]);
    }
    __syncthreads();
  }
  for (int64_t e = threadIdx.x; e < static_cast<int64_t>(k1 - k0) * nr; e += blockDim.x) {
    const int c = k0 + static_cast<int>(e / nr), i = static_cast<int>(e % nr);
    const double* Fc = F + static_cast<int64_t>(c) * nr;
    a.Wb[static_cast<int64_t>(c - k0) * nr + i] = i >= k1 ? Fc[i] * Fc[c] : 0.0;
  }
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double av, double bv) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(av), "d"(bv));
}

// --- trailing update on the tensor cores: for the lower triangle of
// [k1, nr)^2, F(i, j) -= sum_{c in [k0,k1)} L(i, c) W(j, c). Grid: one CTA per
// 64x64 tile (ti >= tj), 4 warps of 32x32, k = kBs in steps of 4.
__global__ void __launch_bounds__(128) bf_syrk_dmma(BigArgs a, int k0, int k1, int ntiles) {
  __shared__ double As[kBs][kTile + 1];
  __shared__ double Bs[kBs][kTile + 1];
  const int nr = a.nr;
  // tile index -> (ti, tj), ti >= tj
  int t = blockIdx.x, ti = 0;
  while (t > ti) t -= ++ti;
  const int tj = t;
  const int i0 = k1 + ti * kTile, j0 = k1 + tj * kTile;
  const int kw = k1 - k0;
  for (int e = threadIdx.x; e < kBs * kTile; e += blockDim.x) {
    const int c = e / kTile, r = e % kTile;
    const bool okc = c < kw;
    const int gi = i0 + r, gj = j0 + r;
    As[c][r] = okc && gi < nr ? a.F[static_cast<int64_t>(k0 + c) * nr + gi] : 0.0;
    Bs[c][r] = okc && gj < nr ? a.Wb[static_cast<int64_t>(c) * nr + gj] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wi = (warp >> 1) * 32, wj = (warp & 1) * 32;
  const int g = lane >> 2, tg = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < kBs; kk += 4) {
    double av[4], bv[4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) av[mi] = As[kk + tg][wi + mi * 8 + g];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) bv[ni] = Bs[kk + tg][wj + ni * 8 + g];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], av[mi], bv[ni]);
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gi = i0 + wi + mi * 8 + g, gj = j0 + wj + ni * 8 + 2 * tg + h;
        if (gi < nr && gj < nr && gi >= gj) a.F[static_cast<int64_t>(gj) * nr + gi] -= acc[mi][ni][h];
      }
}

__global__ void __launch_bounds__(256) bf_writeout(BigArgs a, int* flags, int epoch) {
  const int nr = a.nr, w = a.w, m2 = a.m2;
  double* P = a.L + __ldg(a.S.sn_loff + a.s);
  double* C = a.CB + __ldg(a.S.cb_off + a.s);
  const int64_t np = static_cast<int64_t>(w) * nr, nc = static_cast<int64_t>(m2) * m2;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < np + nc;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (e < np) {
      P[e] = a.F[e];
    } else {
      const int64_t k = e - np;
      const int i = static_cast<int>(k % m2), j = static_cast<int>(k / m2);
      if (i >= j) C[cb_col(j, m2) + i] = a.F[static_cast<int64_t>(w + j) * nr + (w + i)];
    }
  }
}

__global__ void bf_publish(int* flags, int s, int epoch) {
  __threadfence();
  flags[s] = epoch;
}

}  // namespace

// Factor one large supernode (all launches on st, in order). F / Wb: scratch
// of nr*nr and nr*kBs doubles.
void dev_factor_big(const DevSymb& S, DevFactor& Fa, const double* kvals, int s, int f, int w, int nr, int64_t g0,
                    int64_t g1, double* F, double* Wb, cudaStream_t st) {
  BigArgs a{S, s, f, w, nr, nr - w, F, Wb, Fa.L, Fa.CB, Fa.D, kvals, Fa.scal, Fa.istat};
  cudaMemsetAsync(F, 0, static_cast<size_t>(nr) * nr * sizeof(double), st);
  const int64_t ne = g1 - g0;
  if (ne > 0) {
    bf_gather<<<static_cast<int>(std::min<int64_t>((ne + 255) / 256, 4 * 148)), 256, 0, st>>>(a, g0, g1);
    g_kernel_launches += 1;
  }
  // panel width: 32 columns while a panel fits 220 KB of shared memory,
  // narrower for very tall fronts (a function of nr only: deterministic)
  int pw = kBs;
  while (pw > 8 && static_cast<int64_t>(nr) * pw * 8 > 220 * 1024) pw /= 2;
  for (int k0 = 0; k0 < w; k0 += pw) {
    const int k1 = std::min(w, k0 + pw);
    const int psmem = (nr - k0) * (k1 - k0) * static_cast<int>(sizeof(double));
    if (psmem <= 220 * 1024) {
      if (psmem > 48 * 1024) cudaFuncSetAttribute(bf_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, psmem);
      bf_panel<<<1, 256, psmem, st>>>(a, k0, k1);
    } else {
      bf_panel_global<<<1, 256, 0, st>>>(a, k0, k1);  // panels taller than shared memory
    }
    const int rest = nr - k1;
    g_kernel_launches += 1;
    if (rest > 0) {
      const int nt = (rest + kTile - 1) / kTile;
      const int ntiles = nt * (nt + 1) / 2;
      bf_syrk_dmma<<<ntiles, 128, 0, st>>>(a, k0, k1, ntiles);
      g_kernel_launches += 1;
    }
  }
  const int64_t tot = static_cast<int64_t>(w) * nr + static_cast<int64_t>(nr - w) * (nr - w);
  bf_writeout<<<static_cast<int>(std::min<int64_t>((tot + 255) / 256, 2048)), 256, 0, st>>>(a, S.flags, S.epoch);
  bf_publish<<<1, 1, 0, st>>>(S.flags, s, S.epoch);
  g_kernel_launches += 2;
}

int big_front_panel() { return kBs; }

}  // namespace nclb
