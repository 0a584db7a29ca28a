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
#include <cstdlib>
#include <cstdint>

#include "dev.hpp"

namespace nclb {

namespace {

constexpr int kBs = 32;      // panel width
constexpr int kTile = 64;    // DMMA tile (64 x 64 per CTA, 4 warps x 32 x 32)
constexpr unsigned kFullMask = 0xffffffffu;

struct BigArgs {
  DevSymb S;
  const BigDesc* d;   // the batch's fronts
  double* Fs;         // scratch fronts (BigDesc::foff)
  double* Ws;         // scratch W (BigDesc::woff)
  double* L;          // panels
  double* CB;         // contribution blocks
  double* D;
  const double* kvals;
  const double* thresh;
  int* zp;
};

// --- assembly: front blockIdx.y; a group of b.gsz lanes per front entry that
// receives anything: lane r sums sources r, r + gsz, ... (A value first, then
// the children's CB entries in ascending child order), the group combines its
// partial sums by a fixed xor butterfly (gsz = 1: the plain sequential sum).
// The per-front gsz is fixed by the symbolic analysis: deterministic.
__global__ void __launch_bounds__(256) bf_gather(BigArgs a) {
  const BigDesc b = a.d[blockIdx.y];
  const DevSymb& S = a.S;
  double* F = a.Fs + b.foff;
  const int G = b.gsz, lane = threadIdx.x & 31;
  const int per_warp = 32 / G;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (int64_t base = b.g0 + gw * per_warp; base < b.g1; base += nwarps * per_warp) {  // warp-uniform trip count
    const int64_t k = base + lane / G;
    const int r = lane % G;
    double acc = 0.0;
    if (k < b.g1) {
      int64_t q = __ldg(S.gsp + k) + r;
      const int64_t q1 = __ldg(S.gsp + k + 1);
      for (; q + 3 * G < q1; q += 4 * G) {
        const int64_t s0 = __ldg(S.gsrc + q), s1 = __ldg(S.gsrc + q + G), s2 = __ldg(S.gsrc + q + 2 * G),
                      s3 = __ldg(S.gsrc + q + 3 * G);
        const double v0 = s0 < 0 ? __ldg(a.kvals + ~s0) : __ldcg(a.CB + s0);
        const double v1 = s1 < 0 ? __ldg(a.kvals + ~s1) : __ldcg(a.CB + s1);
        const double v2 = s2 < 0 ? __ldg(a.kvals + ~s2) : __ldcg(a.CB + s2);
        const double v3 = s3 < 0 ? __ldg(a.kvals + ~s3) : __ldcg(a.CB + s3);
        acc += v0;
        acc += v1;
        acc += v2;
        acc += v3;
      }
      for (; q < q1; q += G) {
        const int64_t src = __ldg(S.gsrc + q);
        acc += src < 0 ? __ldg(a.kvals + ~src) : __ldcg(a.CB + src);
      }
    }
    for (int o = G >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(kFullMask, acc, o);
    if (k < b.g1 && r == 0) F[__ldg(S.gdst + k)] = acc;
  }
}

// --- panel step: front blockIdx.x factors its panel `step` (columns
// [k0, k1), rows [k0, nr)) staged in shared memory: warps own columns c2,
// lanes rows in the rank-1 updates; then W(:, c-k0) = L(:, c) d_c below it.
__global__ void __launch_bounds__(256) bf_panel(BigArgs a, int step) {
  extern __shared__ double Ps[];
  const BigDesc b = a.d[blockIdx.x];
  if (step >= b.npan) return;
  const int nr = b.nr, k0 = step * b.pw, k1 = min(b.w, k0 + b.pw);
  const int ld = nr - k0, kw = k1 - k0;
  const double thresh = __ldcg(a.thresh);
  double* F = a.Fs + b.foff;
  double* W = a.Ws + b.woff;
  for (int e = threadIdx.x; e < ld * kw; e += blockDim.x) {
    const int c = e / ld, i = e % ld;
    Ps[e] = F[static_cast<int64_t>(k0 + c) * nr + k0 + i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = 0; c < kw; ++c) {
    double* Pc = Ps + c * ld;
    const double dd = Pc[c];
    if (threadIdx.x == 0) {
      a.D[b.f + k0 + c] = dd;
      if (fabs(dd) <= thresh) atomicMin(a.zp, b.f + k0 + c);
    }
    const double rd = 1.0 / dd;  // one division per column; the column scales by multiplies
    for (int i = c + 1 + threadIdx.x; i < ld; i += blockDim.x) Pc[i] *= rd;
    __syncthreads();
    for (int c2 = c + 1 + warp; c2 < kw; c2 += 8) {
      const double dl = dd * Pc[c2];
      double* P2 = Ps + c2 * ld;
      for (int i = c2 + lane; i < ld; i += 32) P2[i] -= Pc[i] * dl;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < ld * kw; e += blockDim.x) {
    const int c = e / ld, i = e % ld;
    F[static_cast<int64_t>(k0 + c) * nr + k0 + i] = Ps[e];
    const int gi = k0 + i;
    W[static_cast<int64_t>(c) * nr + gi] = gi >= k1 ? Ps[e] * Ps[c * ld + c] : 0.0;
  }
  for (int e = threadIdx.x; e < kw * k0; e += blockDim.x) {  // rows above the panel: W = 0
    const int c = e / k0, i = e % k0;
    W[static_cast<int64_t>(c) * nr + i] = 0.0;
  }
}

// --- panel step split in two (the single-CTA bf_panel above was bound by its
// column-by-column shared-memory updates over the whole tall panel):
// bf_diag: one warp per front factors the kw x kw diagonal block of panel
// `step` in registers (lane i = row k0 + i, pivots broadcast by shuffles) and
// leaves 1 / d_c on W's diagonal and d_c L(c2, c) below it (W's rows
// [k0, k1) are otherwise unused); bf_rows: every row below the block is
// independent given those — one thread per row, rows spread over many CTAs —
// L(i, c) = x_c / d_c as x_c (1 / d_c), x_c2 -= L(i, c) (d_c L(c2, c)), and
// W(i, c) = L(i, c) d_c for the trailing update. Per row and per column the
// operations and their order are bf_panel's.
__global__ void __launch_bounds__(32) bf_diag(BigArgs a, int step) {
  const BigDesc b = a.d[blockIdx.x];
  if (step >= b.npan) return;
  const int nr = b.nr, k0 = step * b.pw, k1 = min(b.w, k0 + b.pw), kw = k1 - k0;
  const int lane = threadIdx.x;
  double* F = a.Fs + b.foff;
  double* W = a.Ws + b.woff;
  const double thresh = __ldcg(a.thresh);
  double x[kBs];
#pragma unroll
  for (int c = 0; c < kBs; ++c)
    x[c] = (c < kw && c <= lane && lane < kw) ? F[static_cast<int64_t>(k0 + c) * nr + k0 + lane] : 0.0;
#pragma unroll
  for (int c = 0; c < kBs; ++c) {
    if (c < kw) {
      const double d = __shfl_sync(kFullMask, x[c], c);
      const double rd = __drcp_rn(d);  // correctly rounded: = 1.0 / d
      if (lane == 0) {
        a.D[b.f + k0 + c] = d;
        if (fabs(d) <= thresh) atomicMin(a.zp, b.f + k0 + c);
      }
      if (lane > c && lane < kw) x[c] *= rd;
      const double dlo = d * x[c];  // lane c2: d_c L(c2, c)
      if (lane == c) W[static_cast<int64_t>(c) * nr + k0 + c] = rd;
      if (lane > c && lane < kw) W[static_cast<int64_t>(c) * nr + k0 + lane] = dlo;
#pragma unroll
      for (int c2 = c + 1; c2 < kBs; ++c2) {
        if (c2 < kw) {
          const double dl = __shfl_sync(kFullMask, dlo, c2);
          if (lane >= c2 && lane < kw) x[c2] -= x[c] * dl;
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kBs; ++c)
    if (c < kw && c <= lane && lane < kw) F[static_cast<int64_t>(k0 + c) * nr + k0 + lane] = x[c];
}

__global__ void __launch_bounds__(256) bf_rows(BigArgs a, int step) {
  __shared__ double s_dl[kBs][kBs + 1];  // [c][c2]: d_c L(c2, c); [c][c]: 1 / d_c
  __shared__ double s_d[kBs];
  const BigDesc b = a.d[blockIdx.y];
  if (step >= b.npan) return;
  const int nr = b.nr, k0 = step * b.pw, k1 = min(b.w, k0 + b.pw), kw = k1 - k0;
  const int i0 = k1 + blockIdx.x * blockDim.x;
  if (i0 >= nr) return;
  double* F = a.Fs + b.foff;
  double* W = a.Ws + b.woff;
  for (int e = threadIdx.x; e < kw * kw; e += blockDim.x) {
    const int c = e / kw, c2 = e % kw;
    if (c2 >= c) s_dl[c][c2] = W[static_cast<int64_t>(c) * nr + k0 + c2];
  }
  for (int c = threadIdx.x; c < kw; c += blockDim.x) s_d[c] = F[static_cast<int64_t>(k0 + c) * nr + k0 + c];
  __syncthreads();
  const int i = i0 + threadIdx.x;
  if (i >= nr) return;
  double x[kBs];
#pragma unroll
  for (int c = 0; c < kBs; ++c) x[c] = c < kw ? F[static_cast<int64_t>(k0 + c) * nr + i] : 0.0;
#pragma unroll
  for (int c = 0; c < kBs; ++c) {
    if (c < kw) {
      x[c] *= s_dl[c][c];
#pragma unroll
      for (int c2 = c + 1; c2 < kBs; ++c2)
        if (c2 < kw) x[c2] -= x[c] * s_dl[c][c2];
    }
  }
#pragma unroll
  for (int c = 0; c < kBs; ++c)
    if (c < kw) {
      F[static_cast<int64_t>(k0 + c) * nr + i] = x[c];
      W[static_cast<int64_t>(c) * nr + i] = x[c] * s_d[c];
    }
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double av, double bv) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(av), "d"(bv));
}

// --- trailing update of panel `step` on the tensor cores: front blockIdx.y,
// 64x64 tile blockIdx.x of the lower triangle of [k1, nr)^2:
// F(i, j) -= sum_{c in panel} L(i, c) W(j, c); 4 warps of 32x32, DMMA k = 4.
__global__ void __launch_bounds__(128) bf_syrk_dmma(BigArgs a, int step) {
  __shared__ double As[kBs][kTile + 1];
  __shared__ double Bs[kBs][kTile + 1];
  const BigDesc b = a.d[blockIdx.y];
  if (step >= b.npan) return;
  const int nr = b.nr, k0 = step * b.pw, k1 = min(b.w, k0 + b.pw);
  const int rest = nr - k1;
  if (rest <= 0) return;
  const int nt = (rest + kTile - 1) / kTile;
  if (static_cast<int>(blockIdx.x) >= nt * (nt + 1) / 2) return;
  int t = blockIdx.x, ti = 0;  // tile index -> (ti, tj), ti >= tj
  while (t > ti) t -= ++ti;
  const int tj = t;
  const int i0 = k1 + ti * kTile, j0 = k1 + tj * kTile;
  const int kw = k1 - k0;
  const double* F = a.Fs + b.foff;
  const double* W = a.Ws + b.woff;
  for (int e = threadIdx.x; e < kBs * kTile; e += blockDim.x) {
    const int c = e / kTile, r = e % kTile;
    const bool okc = c < kw;
    const int gi = i0 + r, gj = j0 + r;
    As[c][r] = okc && gi < nr ? F[static_cast<int64_t>(k0 + c) * nr + gi] : 0.0;
    Bs[c][r] = okc && gj < nr ? W[static_cast<int64_t>(c) * nr + gj] : 0.0;
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
  double* Fw = a.Fs + b.foff;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gi = i0 + wi + mi * 8 + g, gj = j0 + wj + ni * 8 + 2 * tg + h;
        if (gi < nr && gj < nr && gi >= gj) Fw[static_cast<int64_t>(gj) * nr + gi] -= acc[mi][ni][h];
      }
}

// --- write-back: front blockIdx.y, panel (w columns) to L, lower CB
__global__ void __launch_bounds__(256) bf_writeout(BigArgs a) {
  const BigDesc b = a.d[blockIdx.y];
  if (b.npan == 0) return;  // written by its CTA (dev_big_cta)
  const int nr = b.nr, w = b.w, m2 = nr - w;
  const double* F = a.Fs + b.foff;
  double* P = a.L + __ldg(a.S.sn_loff + b.s);
  double* C = a.CB + __ldg(a.S.cb_off + b.s);
  const int64_t np = static_cast<int64_t>(w) * nr, nc = static_cast<int64_t>(m2) * m2;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < np + nc;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (e < np) {
      P[e] = F[e];
    } else {
      const int64_t k = e - np;
      const int i = static_cast<int>(k % m2), j = static_cast<int>(k / m2);
      if (i >= j) C[cb_col(j, m2) + i] = F[static_cast<int64_t>(w + j) * nr + (w + i)];
    }
  }
}

__global__ void bf_publish(const BigDesc* d, int nf, int* flags, int epoch) {
  __threadfence();
  for (int k = threadIdx.x; k < nf; k += blockDim.x) flags[d[k].s] = epoch;
}

}  // namespace

// Factor all large fronts of one segment as a batch: one launch per phase
// (assembly, each panel step, its DMMA trailing update, write-back), each
// front on its own grid row. Per front the arithmetic equals processing it
// alone.
void dev_factor_big_batch(const DevSymb& S, DevFactor& Fa, const double* kvals, const std::vector<BigDesc>& h,
                          const BigDesc* d, cudaStream_t st) {
  const int nf = static_cast<int>(h.size());
  if (nf == 0) return;
  BigArgs a{S, d, Fa.bigF, Fa.bigW, Fa.L, Fa.CB, Fa.D, kvals, Fa.scal, Fa.istat};
  int64_t fsz = 0, emax = 0, wmax = 0;
  int steps = 0, ncta = 0;
  for (const BigDesc& b : h) {
    fsz = std::max(fsz, b.foff + static_cast<int64_t>(b.nr) * b.nr);
    emax = std::max(emax, (b.g1 - b.g0) * b.gsz);
    ncta += b.npan == 0;
    wmax = std::max<int64_t>(wmax, static_cast<int64_t>(b.w) * b.nr + static_cast<int64_t>(b.nr - b.w) * (b.nr - b.w));
    steps = std::max(steps, b.npan);
  }
  cudaMemsetAsync(Fa.bigF, 0, fsz * sizeof(double), st);
  if (emax > 0) {
    bf_gather<<<dim3(static_cast<unsigned>(std::min<int64_t>((emax + 255) / 256, 1024)), nf), 256, 0, st>>>(a);
    g_kernel_launches += 1;
  }
  static int smem_set = 0;
  if (!smem_set) {
    cudaFuncSetAttribute(bf_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    smem_set = 1;
  }
  if (ncta > 0) dev_big_cta(S, Fa, d, nf, st);
  for (int k = 0; k < steps; ++k) {
    int psmem = 0, tiles = 0;
    for (const BigDesc& b : h) {
      if (k >= b.npan) continue;
      const int k0 = k * b.pw, k1 = std::min(b.w, k0 + b.pw);
      psmem = std::max(psmem, (b.nr - k0) * (k1 - k0) * static_cast<int>(sizeof(double)));
      const int nt = (b.nr - k1 + kTile - 1) / kTile;
      tiles = std::max(tiles, nt * (nt + 1) / 2);
    }
    static const bool one_cta = std::getenv("NCL_BF_PANEL") != nullptr;  // A/B: the single-CTA panel step
    if (one_cta) {
      bf_panel<<<nf, 256, psmem, st>>>(a, k);
      g_kernel_launches += 1;
    } else {
      int rows = 0;
      for (const BigDesc& b : h)
        if (k < b.npan) rows = std::max(rows, b.nr - std::min(b.w, k * b.pw + b.pw));
      bf_diag<<<nf, 32, 0, st>>>(a, k);
      if (rows > 0) bf_rows<<<dim3((rows + 255) / 256, nf), 256, 0, st>>>(a, k);
      g_kernel_launches += 1 + (rows > 0);
    }
    if (tiles > 0) {
      bf_syrk_dmma<<<dim3(tiles, nf), 128, 0, st>>>(a, k);
      g_kernel_launches += 1;
    }
  }
  if (steps > 0)
    bf_writeout<<<dim3(static_cast<unsigned>(std::min<int64_t>((wmax + 255) / 256, 512)), nf), 256, 0, st>>>(a);
  bf_publish<<<1, 256, 0, st>>>(d, nf, S.flags, S.epoch);
  g_kernel_launches += (steps > 0) + 1;
}

int big_front_panel() { return kBs; }

}  // namespace nclb
