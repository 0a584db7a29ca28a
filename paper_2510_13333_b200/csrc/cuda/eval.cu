// K1 evaluation: value / gradient / Lagrangian-Hessian entries of every
// template instance, SIMD over instances.
//
// Replaces ModelFunctions::eval_* (/root/reference/proj/src/model.cpp:134-223)
// whose inner loop is one scalar Tape::eval per (instance, entry)
// (/root/reference/proj/src/expr.cpp:168-220). Here one thread evaluates one
// instance of a family with ONE CSE-compiled register program covering all
// requested entries; the instruction stream is warp-uniform (every thread of
// a block belongs to the same family), instance tables are SoA so the slot
// index loads are coalesced, and results go to a contribution buffer in SoA
// order. A second pass gathers contributions into c / J / H / ∇φ in exactly
// the reference's accumulation order (family, instance, entry) with
// round-to-nearest adds, so outputs match the reference bit for bit except
// where sin/cos/pow differ by an ulp between CUDA and glibc.
#include <cuda_runtime.h>

#include <cstdint>

#include "dev.hpp"
#include "eval.hpp"

namespace nclb {

namespace {

__device__ __forceinline__ void report(unsigned long long* err, int fam, int64_t inst, int code) {
  const unsigned long long v =
      (static_cast<unsigned long long>(fam) << 40) | (static_cast<unsigned long long>(inst) << 2) | code;
  atomicMin(err, v);
}

template <int MAXR>
__global__ void __launch_bounds__(256) eval_kernel(const DevFam* __restrict__ fams, int nfam, int kind,
                                                   const double* __restrict__ w, double sigma,
                                                   const double* __restrict__ lam, double* __restrict__ contrib,
                                                   unsigned long long* err) {
  // family of this block (block ranges are contiguous per family)
  int f = 0;
  while (f + 1 < nfam && fams[f + 1].block0 <= blockIdx.x) ++f;
  const DevFam& F = fams[f];
  const int64_t inst = (static_cast<int64_t>(blockIdx.x) - F.block0) * blockDim.x + threadIdx.x;
  if (inst >= F.ninst) return;
  const int64_t ni = F.ninst;
  const Instr* __restrict__ prog = F.prog[kind];
  const int plen = F.plen[kind];
  double hw = 1.0;  // Hessian weight: sigma (objective) or lambda_row
  if (kind == PK_H || kind == PK_VGH) {
    hw = F.obj ? sigma : __ldg(lam + F.rows[inst]);
    if (hw == 0.0 && kind == PK_H) {
      // model.cpp:187-190 skips weight-0 instances: their entries add nothing
      for (int h = 0; h < F.H; ++h) contrib[F.base + (1 + F.G + h) * ni + inst] = 0.0;
      return;
    }
  }
  double r[MAXR];
  for (int i = 0; i < plen; ++i) {
    const long long w0 = __ldg(reinterpret_cast<const long long*>(prog + i));
    const double val = __ldg(reinterpret_cast<const double*>(prog + i) + 1);
    const int op = static_cast<int>(w0 & 0xff);
    const int dst = static_cast<int16_t>((w0 >> 16) & 0xffff);
    const int a = static_cast<int16_t>((w0 >> 32) & 0xffff);
    const int b = static_cast<int16_t>((w0 >> 48) & 0xffff);
    const int slot = a;
    double x;
    switch (op) {
      case 0: x = val; break;                                        // constant
      case 1: x = __ldg(w + __ldg(F.vars + slot * ni + inst)); break;  // var
      case 2: x = __ldg(F.params + slot * ni + inst); break;           // param
      case 3: x = __dadd_rn(r[a], r[b]); break;
      case 4: x = __dsub_rn(r[a], r[b]); break;
      case 5: x = __dmul_rn(r[a], r[b]); break;
      case 6: {
        const double den = r[b];
        if (fabs(den) < 1e-300) report(err, f, inst, 1);  // expr.cpp:194-198
        x = __ddiv_rn(r[a], den);
        break;
      }
      case 7: {
        const double base = r[a];
        if (base < 0.0 && val != floor(val)) report(err, f, inst, 2);  // expr.cpp:200-206
        if (base == 0.0 && val < 0.0) report(err, f, inst, 3);
        x = (val == 2.0) ? __dmul_rn(base, base) : pow(base, val);
        break;
      }
      case 8: x = -r[a]; break;
      case 9: x = sin(r[a]); break;
      case 10: x = cos(r[a]); break;
      default: x = 0.0; break;
    }
    r[dst] = x;
  }
  const int* __restrict__ outs = F.outs[kind];
  if (kind == PK_V) {
    contrib[F.base + inst] = r[__ldg(outs)];
  } else if (kind == PK_G) {
    for (int g = 0; g < F.G; ++g) contrib[F.base + (1 + g) * ni + inst] = r[__ldg(outs + g)];
  } else {
    int o = 0;
    if (kind == PK_VGH) {
      contrib[F.base + inst] = r[__ldg(outs)];
      for (int g = 0; g < F.G; ++g) contrib[F.base + (1 + g) * ni + inst] = r[__ldg(outs + 1 + g)];
      o = 1 + F.G;
    }
    for (int h = 0; h < F.H; ++h) {
      double v = 0.0;
      if (hw != 0.0) {
        const int hi = __ldg(F.hess_hi + h), lo = __ldg(F.hess_lo + h);
        const bool alias = hi != lo && __ldg(F.vars + hi * ni + inst) == __ldg(F.vars + lo * ni + inst);
        const double mult = alias ? 2.0 : 1.0;  // model.cpp:121-123
        v = __dmul_rn(__dmul_rn(hw, mult), r[__ldg(outs + o + h)]);
      }
      contrib[F.base + (1 + F.G + h) * ni + inst] = v;
    }
  }
}

__global__ void gather_sum64(int64_t nslots, const int64_t* __restrict__ ptr, const int* __restrict__ idx,
                             const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots; s += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t p = ptr[s]; p < ptr[s + 1]; ++p) acc = __dadd_rn(acc, src[idx[p]]);
    dst[s] = acc;
  }
}

// out[r] = sum_k vals[k] * v[col[k]] over a CSR (k order), no FMA
__global__ void csr_mv(int64_t nrows, const int64_t* __restrict__ ptr, const int* __restrict__ kidx,
                       const int* __restrict__ xi, const double* __restrict__ vals, const double* __restrict__ x,
                       double* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t p = ptr[r]; p < ptr[r + 1]; ++p) {
      const int k = kidx ? kidx[p] : static_cast<int>(p);
      acc = __dadd_rn(acc, __dmul_rn(vals[k], x[xi[k]]));
    }
    out[r] = acc;
  }
}

int grid_cap(int64_t n) {
  int64_t g = (n + 255) / 256;
  const int cap = dev_num_sms() * 8;
  if (g > cap) g = cap;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

void dev_eval(const DevModel& M, int kind, const double* w, double sigma, const double* lam, cudaStream_t st) {
  if (M.nblocks <= 0) return;
  const int maxr = M.maxregs[kind];
  g_kernel_launches += 1;
  if (maxr <= 32)
    eval_kernel<32><<<M.nblocks, 256, 0, st>>>(M.fams, M.nfam, kind, w, sigma, lam, M.contrib, M.err);
  else if (maxr <= 64)
    eval_kernel<64><<<M.nblocks, 256, 0, st>>>(M.fams, M.nfam, kind, w, sigma, lam, M.contrib, M.err);
  else if (maxr <= 128)
    eval_kernel<128><<<M.nblocks, 256, 0, st>>>(M.fams, M.nfam, kind, w, sigma, lam, M.contrib, M.err);
  else
    eval_kernel<256><<<M.nblocks, 256, 0, st>>>(M.fams, M.nfam, kind, w, sigma, lam, M.contrib, M.err);
}

void dev_gather64(int64_t nslots, const int64_t* ptr, const int* idx, const double* src, double* dst,
                  cudaStream_t st) {
  if (nslots <= 0) return;
  g_kernel_launches += 1;
  gather_sum64<<<grid_cap(nslots), 256, 0, st>>>(nslots, ptr, idx, src, dst);
}

void dev_csr_mv(int64_t nrows, const int64_t* ptr, const int* kidx, const int* xi, const double* vals,
                const double* x, double* out, cudaStream_t st) {
  if (nrows <= 0) return;
  g_kernel_launches += 1;
  csr_mv<<<grid_cap(nrows), 256, 0, st>>>(nrows, ptr, kidx, xi, vals, x, out);
}

}  // namespace nclb
