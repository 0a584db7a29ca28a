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
constexpr int kColBlk = 32;  // assembly: target columns per CTA
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

// --- assembly: CTA b owns target columns [b*kColBlk, (b+1)*kColBlk) -------
__global__ void __launch_bounds__(256) bf_assemble(BigArgs a) {
  const DevSymb& S = a.S;
  const int nr = a.nr;
  const int c0 = blockIdx.x * kColBlk, c1 = min(nr, c0 + kColBlk);
  for (int64_t e = threadIdx.x; e < static_cast<int64_t>(c1 - c0) * nr; e += blockDim.x)
    a.F[static_cast<int64_t>(c0) * nr + e] = 0.0;
  __syncthreads();
  const int64_t a0 = __ldg(S.aptr + a.s), a1 = __ldg(S.aptr + a.s + 1);
  for (int64_t e = a0 + threadIdx.x; e < a1; e += blockDim.x) {
    const int off = __ldg(S.aoff + e);  // c * nr + r (panel layout == front layout for c < w)
    const int c = off / nr;
    if (c >= c0 && c < c1) a.F[off] = __ldg(a.kvals + __ldg(S.asrc + e));
  }
  __syncthreads();
  for (int q = __ldg(S.cptr + a.s); q < __ldg(S.cptr + a.s + 1); ++q) {
    const int ch = __ldg(S.child + q);
    const int wc = __ldg(S.sn_first + ch + 1) - __ldg(S.sn_first + ch);
    const int64_t rbc = __ldg(S.sn_rptr + ch);
    const int m2c = static_cast<int>(__ldg(S.sn_rptr + ch + 1) - rbc) - wc;
    const int* rel = S.relp + rbc + wc;
    const double* Cc = a.CB + __ldg(S.cb_off + ch);
    // child columns j with rel[j] in [c0, c1): a contiguous range (rel ascending)
    int lo = 0, hi = m2c;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(rel + mid) < c0) lo = mid + 1;
      else hi = mid;
    }
    int j1 = lo, hi2 = m2c;
    while (j1 < hi2) {
      const int mid = (j1 + hi2) >> 1;
      if (__ldg(rel + mid) < c1) j1 = mid + 1;
      else hi2 = mid;
    }
    for (int j = lo; j < j1; ++j) {
      const int rj = __ldg(rel + j);
      double* Fj = a.F + static_cast<int64_t>(rj) * nr;
      const double* Cj = Cc + cb_col(j, m2c);
      for (int i = j + threadIdx.x; i < m2c; i += blockDim.x) Fj[__ldg(rel + i)] += __ldcg(Cj + i);
    }
    __syncthreads();
  }
}

// --- panel: unblocked LDLᵀ of columns [k0, k1) over rows [k0, nr) (one CTA),
// then W(:, c-k0) = L(:, c) * d_c for the rows below the panel.
__global__ void __launch_bounds__(256) bf_panel(BigArgs a, int k0, int k1) {
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
void dev_factor_big(const DevSymb& S, DevFactor& Fa, const double* kvals, int s, int f, int w, int nr, double* F,
                    double* Wb, cudaStream_t st) {
  BigArgs a{S, s, f, w, nr, nr - w, F, Wb, Fa.L, Fa.CB, Fa.D, kvals, Fa.scal, Fa.istat};
  const int ncb = (nr + kColBlk - 1) / kColBlk;
  bf_assemble<<<ncb, 256, 0, st>>>(a);
  g_kernel_launches += 1;
  for (int k0 = 0; k0 < w; k0 += kBs) {
    const int k1 = std::min(w, k0 + kBs);
    bf_panel<<<1, 256, 0, st>>>(a, k0, k1);
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
