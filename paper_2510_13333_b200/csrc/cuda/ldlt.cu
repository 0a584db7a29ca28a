// K3 numeric LDLᵀ, K4 triangular solves, K5 SpMV / residual, K6 norms.
//
// Replaces the reference's sequential up-looking factorization
// (/root/reference/proj/src/sparse_sym.cpp:268-337), solve_in_place (:346-363)
// and SparseSym::multiply/max_abs_diag/norm_inf (:69-115).
//
// Factorization: MULTIFRONTAL supernodal LDLᵀ with 1x1 pivots in the fixed
// symbolic order (no pivoting; the NCL regularisation keeps K quasi-definite,
// PAPER.md:431-433). Every supernode assembles its front from its own A
// entries and its children's contribution blocks only (extend-add in
// ascending child order: deterministic run to run), factors its
// pivot columns and leaves its Schur complement for its parent. One
// persistent launch per team size: warps for the wide bottom of the
// elimination tree, CTAs for the narrow top; dependencies are epoch flags
// (release/acquire at gpu scope) on the children, tickets are issued in
// leaves-first height order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <utility>
#include <vector>
#include <cstdlib>

#include "dev.hpp"

namespace nclb {

namespace {

// resident CTAs per SM the warp-part and small-CTA factor kernels are
// compiled for (register budget 65536 / (128 x MINB)); measured (r02, same
// box, step ms): 6/6 1.603, 5/6 1.614, 4/6 1.646 (no spills, 16 warps/SM),
// 6/5 1.608, 6/4 1.607 — occupancy beats the spill-free register budgets
#ifndef NCL_FK32_MINB
#define NCL_FK32_MINB 6
#endif
// the warp solve kernels' (fwd/bwd_kernel<32>) resident 128-thread CTAs per
// SM; shared memory (4 warps x kSolWarp doubles = 17 KB) allows up to 13
#ifndef NCL_SK32_MINB
#define NCL_SK32_MINB 8
#endif
#ifndef NCL_FK128_MINB
#define NCL_FK128_MINB 6
#endif
constexpr unsigned kFull = 0xffffffffu;
constexpr int kWarpFront = 32;    // nr cap of the warp smem path
// kCtaFront (nr cap of the CTA smem path) lives in csrc/limits.hpp

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Programmatic dependent launch: a persistent kernel lets the next one in the
// stream launch once every CTA has claimed one of its last tasks (or run out
// of tasks), so the next phase's CTAs take over SMs as this phase drains.
// The next phase synchronises through the completion flags only (it never
// executes griddepcontrol.wait), which is why only phases whose every task
// waits on its dependencies' flags are launched this way.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void wait_flag(const int* f, int epoch) {
  while (ld_acquire(f) != epoch) __nanosleep(32);
}


// x / d with a zero numerator short-circuited (kept for reference; the
// factor and solve chains now multiply by the correctly rounded reciprocal
// __drcp_rn(d) — 60 cycles once per pivot instead of a 113-cycle division per
// element on the dependency chain, and no slow path on zero numerators):
// the FP64 division's fast path rejects x == 0 (exponent check) and CALLs
// the slow-path subroutine, and fronts are full of structural zeros. Divides
// 1 / d instead (the operand is laundered through asm so the compiler cannot
// fold the select back into the division) and returns +0 (instead of a
// signed zero). Branch-free.
__device__ __forceinline__ double divz(double x, double d) {
  const bool z = x == 0.0;
  double xs = z ? 1.0 : x;
  asm("mov.b64 %0, %0;" : "+d"(xs));  // opaque: keeps x == 0 off the division's slow path
  const double q = xs / d;  // branch-free: the lanes stay converged
  return z ? 0.0 : q;
}

// FP64 tensor-core MMA (warp-wide, m8n8k4, row.col): {c0, c1} += A(g, tg) B(tg, g)
// per lane g = lane / 4, tg = lane % 4 (tcgen05 has no f64 kind on sm_100a)
__device__ __forceinline__ void dmma(double& c0, double& c1, double av, double bv) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(av), "d"(bv));
}

template <typename T>
__device__ __forceinline__ void prefetch_l2d(const T* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  // non-negative doubles order like their bit patterns
  atomicMax(reinterpret_cast<unsigned long long*>(addr), static_cast<unsigned long long>(__double_as_longlong(v)));
}

// ---------------------------------------------------------------------------
// Multifrontal numeric LDLᵀ (K3). Tasks are supernodes in leaves-first
// height order (Z.order). Supernode s with panel P (nr x w, column-major,
// the L storage) and contribution block CB_s ((nr-w)^2, column-major):
//   1. wait for the children's epoch flags,
//   2. P := A entries (scatter), CB_s := 0,
//   3. extend-add every child's CB into (P | CB_s) through the relative row
//      map, children in ascending index order (deterministic sums),
//   4. dense right-looking LDLᵀ of the w pivot columns of P,
//   5. CB_s -= L21 D L21ᵀ (lower triangle),
//   6. publish (fence + release flag).
// Team = one warp (NT = 32) for the wide bottom of the tree, one CTA
// (NT = 256) for the narrow top (tickets >= Z.nsplit), two launches.
// ---------------------------------------------------------------------------
constexpr int kLeafChunk = 2;  // dependency-free tasks (whole subtrees) per claim

template <int NT>
__device__ __forceinline__ void team_sync() {
  if constexpr (NT == 32) __syncwarp();
  else __syncthreads();
}

// Task claiming: warps claim individually (leaves in chunks of kLeafChunk),
// CTAs claim one task at a time. Tickets are handed out in order, so the
// minimum outstanding task always has its dependencies finished or held by a
// running team: no deadlock even when not every team is resident.
template <int NT>
struct Claim {
  int cur = 0, end = 0;
  __device__ __forceinline__ int next(int* ticket, int t0, int t1, int nleaf, int tid, int* sh) {
    if constexpr (NT == 32) {
      if (cur < end) return cur++;
      int t = 0;
      if (tid == 0) t = atomicAdd(ticket, 1);
      t = __shfl_sync(kFull, t, 0);
      const int nl = max(0, min(nleaf, t1) - t0);  // leaves inside this phase
      const int nchunks = (nl + kLeafChunk - 1) / kLeafChunk;
      if (t < nchunks) {
        cur = t0 + t * kLeafChunk;
        end = min(t0 + nl, cur + kLeafChunk);
        return cur++;
      }
      const int k = t0 + nl + (t - nchunks);
      return k < t1 ? k : -1;
    } else {
      __syncthreads();
      if (tid == 0) *sh = atomicAdd(ticket, 1);
      __syncthreads();
      const int k = t0 + *sh;
      return k < t1 ? k : -1;
    }
  }
};

struct FactorArgs {
  DevSymb S;
  double* L;
  double* CB;
  double* D;
  const double* kvals;
  const double* thresh;
  int* zp;
  int* flags;
  int* ticket;
  int epoch;
  int t0, t1;          // ticket range of this launch (indices into tasks)
  const int* tasks;    // supernode ids: tasks are ranges tptr[t]..tptr[t+1] (postorder subtrees)
  const int* tptr;     // task -> node range
  const int* prog;     // group programs (tasks < nleaf)
  const int64_t* gpo;
  int nleaf;           // dependency-free tasks at the head
  int skip_big;        // leave nr > kCtaFront to the blocked DMMA path
  unsigned long long* trace;  // optional (NCL_TASK_TRACE): globaltimer start/end per task
};

template <int NT>
__device__ __forceinline__ void factor_task(const FactorArgs& a, int s, int tid, double thresh,
                                            bool wait_children = true, bool publish = true) {
  const DevSymb& S = a.S;
  if (wait_children)  // one thread per child: the polls overlap instead of chaining
    for (int q = __ldg(S.cptr + s) + tid; q < __ldg(S.cptr + s + 1); q += NT) wait_flag(a.flags + __ldg(S.child + q), a.epoch);
  team_sync<NT>();
  const int f = __ldg(S.sn_first + s);
  const int w = __ldg(S.sn_first + s + 1) - f;
  const int64_t rb = __ldg(S.sn_rptr + s);
  const int nr = static_cast<int>(__ldg(S.sn_rptr + s + 1) - rb);
  const int m2 = nr - w;
  double* P = a.L + __ldg(S.sn_loff + s);
  double* C = a.CB + __ldg(S.cb_off + s);
  // 2. clear, scatter A (each panel entry holds at most one A entry)
  for (int i = tid; i < w * nr; i += NT) P[i] = 0.0;
  for (int i = tid; i < m2 * (m2 + 1) / 2; i += NT) C[i] = 0.0;
  team_sync<NT>();
  for (int64_t e = __ldg(S.aptr + s) + tid; e < __ldg(S.aptr + s + 1); e += NT)
    P[__ldg(S.aoff + e)] = __ldg(a.kvals + __ldg(S.asrc + e));
  team_sync<NT>();
  // 3. extend-add the children's contribution blocks
  for (int q = __ldg(S.cptr + s); q < __ldg(S.cptr + s + 1); ++q) {
    const int c = __ldg(S.child + q);
    const int fc = __ldg(S.sn_first + c);
    const int wc = __ldg(S.sn_first + c + 1) - fc;
    const int64_t rbc = __ldg(S.sn_rptr + c);
    const int m2c = static_cast<int>(__ldg(S.sn_rptr + c + 1) - rbc) - wc;
    const int* rel = S.relp + rbc + wc;
    const double* Cc = a.CB + __ldg(S.cb_off + c);
    for (int j = 0; j < m2c; ++j) {
      const int rj = __ldg(rel + j);
      for (int i = j + tid; i < m2c; i += NT) {
        const int ri = __ldg(rel + i);
        const double v = __ldcg(Cc + cb_col(j, m2c) + i);
        if (rj < w) P[static_cast<int64_t>(rj) * nr + ri] += v;
        else C[cb_col(rj - w, m2) + (ri - w)] += v;
      }
    }
    team_sync<NT>();
  }
  // 4. dense LDLᵀ of the w pivot columns: blocked right-looking, 8-column
  //    panels factored column by column, then one rank-8 update of the later
  //    pivot columns (lanes over rows, no index division)
  constexpr int kPb4 = 8;
  for (int c0 = 0; c0 < w; c0 += kPb4) {
    const int c1 = min(w, c0 + kPb4);
    for (int c = c0; c < c1; ++c) {
      double* Pc = P + static_cast<int64_t>(c) * nr;
      const double dc = Pc[c];
      if (tid == 0) {
        a.D[f + c] = dc;
        if (fabs(dc) <= thresh) atomicMin(a.zp, f + c);
      }
      const double rdc = __drcp_rn(dc);  // one reciprocal per pivot; the column scales by multiplies
      for (int i = c + 1 + tid; i < nr; i += NT) Pc[i] *= rdc;
      team_sync<NT>();
      for (int c2 = c + 1; c2 < c1; ++c2) {
        const double dl = dc * Pc[c2];
        double* P2 = P + static_cast<int64_t>(c2) * nr;
        for (int i = c2 + tid; i < nr; i += NT) P2[i] -= Pc[i] * dl;
      }
      team_sync<NT>();
    }
    const int kb = c1 - c0;
    for (int j = c1; j < w; ++j) {
      double dlj[kPb4];
#pragma unroll
      for (int k = 0; k < kPb4; ++k)
        dlj[k] = k < kb ? P[static_cast<int64_t>(c0 + k) * nr + (c0 + k)] * P[static_cast<int64_t>(c0 + k) * nr + j]
                        : 0.0;
      double* Pj = P + static_cast<int64_t>(j) * nr;
      for (int i = j + tid; i < nr; i += NT) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < kPb4; ++k)
          if (k < kb) acc += P[static_cast<int64_t>(c0 + k) * nr + i] * dlj[k];
        Pj[i] -= acc;
      }
    }
    team_sync<NT>();
  }
  // 5. Schur update of the contribution block: C -= L21 D L21ᵀ (lower)
  constexpr int kRows = 4;  // warp path: lane-held rows (m2 <= 128)
  bool done5 = false;
  if constexpr (NT == 32) {
   if (m2 <= 32 * kRows) {
    done5 = true;
    // 4-column chunks of L21 in registers (lane owns rows lane + 32 r);
    // L(w+j, c) d_c broadcast by shuffles; one CB pass per chunk
    const int lane = tid;
    for (int c0 = 0; c0 < w; c0 += 4) {
      const int kb = min(4, w - c0);
      double dd[4], Lr[kRows][4];
#pragma unroll
      for (int k = 0; k < 4; ++k) dd[k] = k < kb ? P[static_cast<int64_t>(c0 + k) * nr + (c0 + k)] : 0.0;
#pragma unroll
      for (int r = 0; r < kRows; ++r)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int i = lane + 32 * r;
          Lr[r][k] = (i < m2 && k < kb) ? P[static_cast<int64_t>(c0 + k) * nr + w + i] : 0.0;
        }
      for (int j = 0; j < m2; ++j) {
        const int rj = j >> 5, lj = j & 31;
        double dl[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          double v = 0.0;
#pragma unroll
          for (int r = 0; r < kRows; ++r) v = r == rj ? Lr[r][k] : v;
          dl[k] = dd[k] * __shfl_sync(kFull, v, lj);
        }
        double* Cj = C + cb_col(j, m2);
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          const int i = lane + 32 * r;
          if (i >= j && i < m2) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) acc += Lr[r][k] * dl[k];
            Cj[i] -= acc;
          }
        }
      }
      __syncwarp();
    }
   }
  }
  if (!done5) {
    for (int e = tid; e < m2 * m2; e += NT) {
      const int i = e % m2, j = e / m2;
      if (i < j) continue;
      double acc = 0.0;
      for (int c = 0; c < w; ++c) {
        const double* Pc = P + static_cast<int64_t>(c) * nr;
        acc += Pc[w + i] * (Pc[c] * Pc[w + j]);
      }
      C[cb_col(j, m2) + i] -= acc;
    }
  }
  team_sync<NT>();
  if (tid == 0 && publish) {
    __threadfence();
    st_release(a.flags + s, a.epoch);
  }
}

// Front held entirely in shared memory (nr <= cap): one global read of the
// A entries and children's CBs, factor + Schur update fused into one
// right-looking sweep over the w pivot columns in smem, one write of the
// panel and the lower CB. The warp version (nr <= 32) keeps lane i on row i
// and broadcasts L(c2, c) with shuffles.
// sum of gather entry k's sources in list order; loads issued 4 at a time
__device__ __forceinline__ double gather_sum(const DevSymb& S, const double* __restrict__ kvals,
                                             const double* __restrict__ CB, int64_t k) {
  int64_t q = __ldg(S.gsp + k);
  const int64_t q1 = __ldg(S.gsp + k + 1);
  double acc = 0.0;
  for (; q + 4 <= q1; q += 4) {
    const int64_t s0 = __ldg(S.gsrc + q), s1 = __ldg(S.gsrc + q + 1), s2 = __ldg(S.gsrc + q + 2),
                  s3 = __ldg(S.gsrc + q + 3);
    const double v0 = s0 < 0 ? __ldg(kvals + ~s0) : __ldcg(CB + s0);
    const double v1 = s1 < 0 ? __ldg(kvals + ~s1) : __ldcg(CB + s1);
    const double v2 = s2 < 0 ? __ldg(kvals + ~s2) : __ldcg(CB + s2);
    const double v3 = s3 < 0 ? __ldg(kvals + ~s3) : __ldcg(CB + s3);
    acc += v0;
    acc += v1;
    acc += v2;
    acc += v3;
  }
  for (; q < q1; ++q) {
    const int64_t src = __ldg(S.gsrc + q);
    acc += src < 0 ? __ldg(kvals + ~src) : __ldcg(CB + src);
  }
  return acc;
}

// Gather-sums of entries [g0, g1) into F, four entries per thread at a time
// so the dependent load chains (gsp -> gsrc -> CB) of different entries
// overlap; each entry still sums its sources strictly in list order.
template <int NT>
__device__ __forceinline__ void gather4(const DevSymb& S, const double* __restrict__ kvals,
                                        const double* __restrict__ CB, int64_t g0, int64_t g1, int tid, double* F,
                                        int nr) {
  constexpr int kU = NT == 128 ? 4 : 8;  // front entries in flight per thread (register budget)
  constexpr int kC = 2;                  // sources per entry in flight
  for (int64_t kb = g0 + tid; kb < g1; kb += kU * NT) {
    int64_t q[kU], q1[kU];
    double acc[kU];
    int cmax = 0;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t k = kb + u * NT;
      q[u] = k < g1 ? __ldg(S.gsp + k) : 0;
      q1[u] = k < g1 ? __ldg(S.gsp + k + 1) : 0;
      acc[u] = 0.0;
      cmax = max(cmax, static_cast<int>(q1[u] - q[u]));
    }
    for (int c = 0; c < cmax; c += kC) {  // kC sources per entry in flight (same summation order)
      int64_t sv[kC][kU];
#pragma unroll
      for (int r = 0; r < kC; ++r)
#pragma unroll
        for (int u = 0; u < kU; ++u) sv[r][u] = q[u] + c + r < q1[u] ? __ldg(S.gsrc + q[u] + c + r) : 0;
      double vv[kC][kU];
#pragma unroll
      for (int r = 0; r < kC; ++r)
#pragma unroll
        for (int u = 0; u < kU; ++u)
          vv[r][u] = q[u] + c + r < q1[u] ? (sv[r][u] < 0 ? __ldg(kvals + ~sv[r][u]) : __ldcg(CB + sv[r][u])) : 0.0;
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int r = 0; r < kC; ++r)
          if (q[u] + c + r < q1[u]) acc[u] += vv[r][u];
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t k = kb + u * NT;
      if (k < g1) {
        F[__ldg(S.gdst + k)] = acc[u];  // packed lower position (host-encoded for nr <= kCtaFront)
      }
    }
  }
}

#ifdef NCL_DENSE_PROF  // tools/front_bench.cu: per-phase clocks of cta_dense (thread 0)
__device__ long long g_dense_prof[8];
#define DPROF_T0 long long dp_t = clock64();
#define DPROF(k)                                  \
  if (tid == 0) {                                 \
    const long long dp_n = clock64();             \
    g_dense_prof[k] += dp_n - dp_t;               \
    dp_t = dp_n;                                  \
  }
#else
#define DPROF_T0
#define DPROF(k)
#endif

// Dense LDLᵀ of an assembled front in shared memory (packed lower, column c
// at cb_col(c, nr)): factors its w pivot columns, writes the panel (nr x w,
// column-major) to P and the Schur complement (packed lower m2 x m2) to C.
template <int NT>
__device__ __forceinline__ void cta_dense(double* F, int nr, int w, int f, double thresh, double* D, int* zp,
                                          double* P, double* C, int tid) {
  const int m2 = nr - w;
  DPROF_T0
  if constexpr (NT == 32) {
    const int i = tid;
    for (int c = 0; c < w; ++c) {
      const double d = F[cb_col(c, nr) + c];
      if (i == 0) {
        D[f + c] = d;
        if (fabs(d) <= thresh) atomicMin(zp, f + c);
      }
      double l = 0.0;
      if (i > c && i < nr) {
        l = F[cb_col(c, nr) + i] * __drcp_rn(d);
        F[cb_col(c, nr) + i] = l;
      }
      const double dl = d * l;
      for (int c2 = c + 1; c2 < nr; ++c2) {
        const double lc2 = __shfl_sync(kFull, dl, c2);  // d * L(c2, c)
        if (i >= c2 && i < nr) F[cb_col(c2, nr) + i] -= l * lc2;
      }
      __syncwarp();
    }
  } else {
    // blocked right-looking LDLᵀ, panels of kPb = 8 columns:
    //  (a) warp 0 factors the panel's kb x kb diagonal block in registers
    //      (lane l holds block row c0 + l, pivots broadcast by shuffles);
    //  (b) every thread takes one row below the block and finishes its kb
    //      panel entries on its own (row-oriented: for each k, divide by d_k,
    //      then subtract L(i,k) d_k L(k2,k) from the later k2 — the very
    //      operations, in the very order, of the column-oriented update);
    //  (c) all warps apply the rank-8 update F22 -= L21 (D L21)ᵀ to the
    //      trailing lower triangle on the FP64 tensor cores (mma.m8n8k4.f64,
    //      8 x 8 tiles, two k-steps), tiles dealt round-robin to the warps.
    constexpr int kPb = NCL_CTA_PANEL;  // panel width (csrc/cuda/dev.hpp)
#ifdef NCL_DIAG_SHARE
    constexpr bool kDiagShare = true;
#else
    constexpr bool kDiagShare = false;
#endif
#ifdef NCL_NO_LOOKAHEAD
    constexpr bool kLookAhead = false;
#else
    constexpr bool kLookAhead = true;
#endif
    constexpr int nw = NT / 32;
    __shared__ double s_rd[kPb], s_dl[kPb][kPb];  // 1 / d_k and d_k L(k2, k) of the current diagonal block
    const int lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, tg = lane & 3;
    // (a) the kb x kb diagonal block of the panel at c0, by warp 0
    auto diag_block = [&](int c0) {
      const int kb = min(kPb, w - c0);
      double x[kPb];
      const int i = c0 + lane;
#pragma unroll
      for (int k = 0; k < kPb; ++k) x[k] = (k < kb && k <= lane && lane < kb) ? F[cb_col(c0 + k, nr) + i] : 0.0;
      double rk[kPb];  // 1 / d_k, formed by every lane (warp-uniform; no divergent region)
#pragma unroll
      for (int k = 0; k < kPb; ++k) {
        rk[k] = 0.0;
        if (k < kb) {
          const double d = __shfl_sync(kFull, x[k], k);
          rk[k] = __drcp_rn(d);
          if (lane > k && lane < kb) x[k] *= rk[k];
          const double dlo = d * x[k];  // lane k2: d * L(c0 + k2, c0 + k)
#pragma unroll
          for (int k2 = 0; k2 < kPb; ++k2) {  // full range: unrolls with k
            if (k2 > k && k2 < kb) {
              const double dl = __shfl_sync(kFull, dlo, k2);
              if (lane >= k2 && lane < kb) x[k2] -= x[k] * dl;
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kPb; ++k)
        if (k < kb && k <= lane && lane < kb) F[cb_col(c0 + k, nr) + i] = x[k];
      // the rows below need only 1 / d_k and d_k L(k2, k): computed once here
      // (the same product the row update formed per row) so the row chains
      // are multiplies instead of divisions
#pragma unroll
      for (int k = 0; k < kPb; ++k) {
        if (k < kb) {
          const double dk = __shfl_sync(kFull, x[k], k);
          if (lane == k) s_rd[k] = rk[k];  // correctly rounded: = 1.0 / dk, half the latency
          if (lane > k && lane < kb) s_dl[k][lane] = dk * x[k];
        }
      }
      if (lane < kb) {  // lane k's diagonal entry is the pivot d_k
        double dk = 0.0;
#pragma unroll
        for (int k = 0; k < kPb; ++k)
          if (k == lane) dk = x[k];
        D[f + c0 + lane] = dk;
        if (fabs(dk) <= thresh) atomicMin(zp, f + c0 + lane);
      }
    };
    if (warp == 0 && w > 0) diag_block(0);
    __syncthreads();
    for (int c0 = 0; c0 < w; c0 += kPb) {
      const int kb = min(kPb, w - c0);
      DPROF(0)
      DPROF(1)
      // (b) rows below the diagonal block, one per thread: L(i, k) = x_k / d_k
      //     as x_k * (1 / d_k), then x_k2 -= L(i, k) (d_k L(k2, k)) from the
      //     block's precomputed factors (s_rd, s_dl)
      for (int i = c0 + kb + tid; i < nr; i += NT) {
        double x[kPb];
#pragma unroll
        for (int k = 0; k < kPb; ++k) x[k] = k < kb ? F[cb_col(c0 + k, nr) + i] : 0.0;
#pragma unroll
        for (int k = 0; k < kPb; ++k) {
          if (k < kb) {
            x[k] *= s_rd[k];
#pragma unroll
            for (int k2 = 0; k2 < kPb; ++k2)
              if (k2 > k && k2 < kb) x[k2] -= x[k] * s_dl[k][k2];
          }
        }
#pragma unroll
        for (int k = 0; k < kPb; ++k)
          if (k < kb) F[cb_col(c0 + k, nr) + i] = x[k];
      }
      __syncthreads();
      DPROF(2)
      // (c) trailing update of [c1, nr)^2 on the tensor cores; the strip of
      // the next panel (tile column 0) first, then — look-ahead — warp 0
      // factors the next diagonal block while the other warps finish the rest
      const int c1 = c0 + kb, m = nr - c1;
      // look-ahead: warp 0 factors the next diagonal block during the
      // trailing update. A DMMA-issuing neighbour stretches the block's
      // dependent FP64 chain ~2.8x (tools/diag_bench.cu: 1.9 k -> 5.3 k
      // cycles; a DMMA holds the sub-partition's FP64 pipe ~16 cycles), yet
      // the overlap still wins: NCL_NO_LOOKAHEAD (block alone after the
      // update) measured 1.652 vs 1.617 ms per step
      const bool ahead = kLookAhead && c1 < w;
      if (m > 0) {
        const int T = (m + 7) >> 3;
        // this lane's k indices (A column / B row of every m8n8k4 k-step):
        // k = 4 s + tg, s < kPb / 4
        constexpr int kS = kPb / 4;
        const double* Lk[kS];
        double dk[kS];
#pragma unroll
        for (int q = 0; q < kS; ++q) {
          const int k = 4 * q + tg;
          Lk[q] = F + cb_col(c0 + min(k, kb - 1), nr);
          dk[q] = k < kb ? Lk[q][c0 + k] : 0.0;
        }
        // tiles (ti, tj), tj in [tj_lo, ti]: A fragments in registers, four
        // tiles in flight (loads, the rank-kb DMMAs, then the read-modify-writes)
        auto tile_row = [&](int ti, int tj_lo, int tj_hi) {
          const int i = c1 + ti * 8 + g;
          double av[kS];
#pragma unroll
          for (int q = 0; q < kS; ++q) av[q] = (i < nr && 4 * q + tg < kb) ? Lk[q][i] : 0.0;
          for (int tj0 = tj_lo; tj0 <= tj_hi; tj0 += 4) {
            double acc[4][2];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int j = c1 + (tj0 + u) * 8 + g;
              const bool ok = tj0 + u <= tj_hi && j < nr;
              acc[u][0] = acc[u][1] = 0.0;
#pragma unroll
              for (int q = 0; q < kS; ++q) {
                const double bv = ok && 4 * q + tg < kb ? dk[q] * Lk[q][j] : 0.0;
                dmma(acc[u][0], acc[u][1], av[q], bv);
              }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int jj = c1 + (tj0 + u) * 8 + 2 * tg;
              if (tj0 + u <= tj_hi && i < nr) {
                if (jj < nr && i >= jj) F[cb_col(jj, nr) + i] -= acc[u][0];
                if (jj + 1 < nr && i >= jj + 1) F[cb_col(jj + 1, nr) + i] -= acc[u][1];
              }
            }
          }
        };
        if (ahead) {
#ifdef NCL_DENSE_PROF
          const long long sb0 = clock64();
#endif
          for (int ti = warp; ti < T; ti += nw) tile_row(ti, 0, 0);  // the next panel's columns
          __syncthreads();
#ifdef NCL_DENSE_PROF
          if (tid == 0) g_dense_prof[6] += clock64() - sb0;
#endif
        }
        const int tj_lo = ahead ? 1 : 0;
        if (ahead && warp == 0) {
#ifdef NCL_DENSE_PROF
          const long long db0 = clock64();
#endif
          diag_block(c1);
#ifdef NCL_DENSE_PROF
          if (tid == 0) g_dense_prof[5] += clock64() - db0;
#endif
        } else {
          // remaining tile rows dealt in snake order to the working warps.
          // With look-ahead, the warps sharing warp 0's scheduler (warp % 4
          // == 0) stay idle: the diagonal block's dependent FP64 chain would
          // otherwise queue behind their DMMAs in the SM sub-partition's FP64
          // pipe (NCL_DIAG_SHARE=1: A/B, they work too)
          const bool iso = ahead && !kDiagShare;
          const int nwk = !ahead ? nw : iso ? nw - nw / 4 : nw - 1;
          const int wk = !ahead ? warp : iso ? warp - 1 - warp / 4 : warp - 1;
          for (int r = 0; !(iso && (warp & 3) == 0) && r * nwk < T; ++r) {
            const int ti = (r & 1) ? r * nwk + nwk - 1 - wk : r * nwk + wk;
            if (ti >= T || ti < tj_lo) continue;
            tile_row(ti, tj_lo, ti);
          }
        }
      } else if (ahead && warp == 0) {
        diag_block(c1);
      }
      __syncthreads();
      if (!kLookAhead && c1 < w) {
        if (warp == 0) diag_block(c1);
        __syncthreads();
      }
      DPROF(3)
    }
  }
  for (int k = tid; k < w * nr; k += NT) {
    const int c = k / nr, i = k % nr;
    P[k] = i >= c ? F[cb_col(c, nr) + i] : 0.0;
  }
  {
    const int lane = tid & 31, warp = tid >> 5;
    for (int j = warp; j < m2; j += NT / 32) {
      const double* Fj = F + cb_col(w + j, nr) + w;
      double* Cj = C + cb_col(j, m2);
      for (int i = j + lane; i < m2; i += 32) Cj[i] = Fj[i];
    }
  }
  DPROF(4)
}

__device__ unsigned long long* g_phase = nullptr;  // NCL_TASK_TRACE: per-supernode CTA phase stamps [4 * nsn]

template <int NT>
__device__ __forceinline__ void factor_task_smem(const FactorArgs& a, int s, int tid, double thresh, double* F) {
  const DevSymb& S = a.S;
  const int64_t g0 = NT == 32 ? 0 : __ldg(S.gm_ptr + s), g1 = NT == 32 ? 0 : __ldg(S.gm_ptr + s + 1);
  if (g1 > g0) {
    // pull this front's gather map into L2 while the children finish: the
    // assembly then walks it at L2 instead of HBM latency
    const int64_t q0 = __ldg(S.gsp + g0), q1 = __ldg(S.gsp + g1);
    for (int64_t k = g0 + 16 * static_cast<int64_t>(tid); k <= g1; k += 16 * NT) prefetch_l2d(S.gsp + k);
    for (int64_t k = g0 + 32 * static_cast<int64_t>(tid); k < g1; k += 32 * NT) prefetch_l2d(S.gdst + k);
    for (int64_t k = q0 + 16 * static_cast<int64_t>(tid); k < q1; k += 16 * NT) prefetch_l2d(S.gsrc + k);
  }
  unsigned long long* ph = g_phase ? g_phase + 4 * static_cast<int64_t>(s) : nullptr;
  for (int q = __ldg(S.cptr + s) + tid; q < __ldg(S.cptr + s + 1); q += NT) wait_flag(a.flags + __ldg(S.child + q), a.epoch);
  const int f = __ldg(S.sn_first + s);
  const int w = __ldg(S.sn_first + s + 1) - f;
  const int64_t rb = __ldg(S.sn_rptr + s);
  const int nr = static_cast<int>(__ldg(S.sn_rptr + s + 1) - rb);
  const int m2 = nr - w;
  if (ph && tid == 0) ph[0] = gtimer();
  // the front is PACKED lower-triangular (column c at cb_col(c, nr)): 160 rows
  // fit in 100 KB, two CTAs per SM
  for (int k = tid; k < nr * (nr + 1) / 2; k += NT) F[k] = 0.0;
  team_sync<NT>();
  if (g1 > g0) {
    // gather-sum per front entry: A value first, then the children's CB
    // entries in ascending child order (the extend-add order)
    gather4<NT>(S, a.kvals, a.CB, g0, g1, tid, F, nr);
    team_sync<NT>();
  } else {
  for (int64_t e = __ldg(S.aptr + s) + tid; e < __ldg(S.aptr + s + 1); e += NT)
    {
      const int off = __ldg(S.aoff + e);  // panel offset c*nr + r
      F[cb_col(off / nr, nr) + off % nr] = __ldg(a.kvals + __ldg(S.asrc + e));
    }
  team_sync<NT>();
  if constexpr (NT == 32) {
    for (int q = __ldg(S.cptr + s); q < __ldg(S.cptr + s + 1); ++q) {
      const int c = __ldg(S.child + q);
      const int wc = __ldg(S.sn_first + c + 1) - __ldg(S.sn_first + c);
      const int64_t rbc = __ldg(S.sn_rptr + c);
      const int m2c = static_cast<int>(__ldg(S.sn_rptr + c + 1) - rbc) - wc;
      const int* rel = S.relp + rbc + wc;
      const double* Cc = a.CB + __ldg(S.cb_off + c);
      for (int j = 0; j < m2c; ++j) {
        const int rj = __ldg(rel + j);
        for (int i = j + tid; i < m2c; i += 32) F[cb_col(rj, nr) + __ldg(rel + i)] += __ldcg(Cc + cb_col(j, m2c) + i);
      }
      __syncwarp();
    }
  } else {
    // warp `warp` owns front columns [warp*nr/8, (warp+1)*nr/8): every entry
    // has one owner and sees the children in ascending order (deterministic)
    // without a CTA barrier per child
    const int lane = tid & 31, warp = tid >> 5, nw = NT / 32;
    const int cb0 = (warp * nr) / nw, cb1 = ((warp + 1) * nr) / nw;
    for (int q = __ldg(S.cptr + s); q < __ldg(S.cptr + s + 1); ++q) {
      const int c = __ldg(S.child + q);
      const int wc = __ldg(S.sn_first + c + 1) - __ldg(S.sn_first + c);
      const int64_t rbc = __ldg(S.sn_rptr + c);
      const int m2c = static_cast<int>(__ldg(S.sn_rptr + c + 1) - rbc) - wc;
      const int* rel = S.relp + rbc + wc;
      const double* Cc = a.CB + __ldg(S.cb_off + c);
      int lo = 0, hi = m2c;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(rel + mid) < cb0) lo = mid + 1;
        else hi = mid;
      }
      for (int j = lo; j < m2c; ++j) {
        const int rj = __ldg(rel + j);
        if (rj >= cb1) break;
        double* Fj = F + cb_col(rj, nr);
        const double* Cj = Cc + cb_col(j, m2c);
        for (int i = j + lane; i < m2c; i += 32) Fj[__ldg(rel + i)] += __ldcg(Cj + i);
      }
    }
    __syncthreads();
  }
  }  // scatter / extend-add path
  if (ph && tid == 0) ph[1] = gtimer();
  cta_dense<NT>(F, nr, w, f, thresh, a.D, a.zp, a.L + __ldg(S.sn_loff + s), a.CB + __ldg(S.cb_off + s), tid);
  team_sync<NT>();
  if (ph && tid == 0) ph[2] = gtimer();
  if (tid == 0) {
    __threadfence();
    st_release(a.flags + s, a.epoch);
    if (ph) ph[3] = gtimer();
  }
}

// Pull a group program (read in place) into L1 with one prefetch per 128-byte
// line: its record walk then hits L1 instead of paying an L2 round trip per
// dependent read.
__device__ __forceinline__ void prefetch_prog(const int* PG, int lane) {
  const int len = __ldg(PG + 3);
  for (int k = 32 * lane; k < len; k += 32 * 32) asm volatile("prefetch.global.L1 [%0];" ::"l"(PG + k));
}

// cb_col in 32-bit arithmetic for the warp fronts (nr <= 32)
__device__ __forceinline__ int cb32(int j, int m) { return j * m - ((j * (j + 1)) >> 1); }

// Flat position e of a packed lower m x m triangle (column j holds rows
// j..m-1, contiguous, starting at S(j) = j m - j (j - 1) / 2) -> (column j,
// row i), closed form: j = floor((b - sqrt(b^2 - 8 e)) / 2), b = 2 m + 1, from
// a single-precision estimate corrected by one step (exact for m <= 32 and
// any estimate within a few ulp; checked exhaustively). One decode per
// element instead of a data-dependent walk over the columns.
__device__ __forceinline__ void tri_at(int e, int m, int& j, int& i) {
  const float b = static_cast<float>(2 * m + 1);
  const float disc = fmaxf(b * b - 8.0f * static_cast<float>(e), 1.0f);
  int c = static_cast<int>((b - disc * rsqrtf(disc)) * 0.5f);
  auto S = [m](int k) { return k * m - ((k * (k - 1)) >> 1); };
  if (c > 0 && S(c) > e) --c;
  else if (S(c + 1) <= e) ++c;
  j = c;
  i = e - S(c) + c;
}
// zero a packed front with 16-byte stores (warp regions are 16-byte aligned)
__device__ __forceinline__ void zero_front(double* F, int np, int lane) {
  double2* F2 = reinterpret_cast<double2*>(F);
  for (int k = lane; k < (np >> 1); k += 32) F2[k] = make_double2(0.0, 0.0);
  if ((np & 1) && lane == 0) F[np - 1] = 0.0;
}
// lanes copy the Schur complement (front rows/cols >= w, packed nr) to a packed
// m2 block flat: ceil(m2 (m2 + 1) / 64) rounds instead of m2
__device__ __forceinline__ void copy_cb(const double* F, int nr, int w, double* C, int lane) {
  const int m2 = nr - w, ne = m2 * (m2 + 1) / 2;
  for (int e = lane; e < ne; e += 32) {
    int j, i;
    tri_at(e, m2, j, i);
    C[e] = F[cb32(w + j, nr) + w + i];
  }
}
// extend-add of a child's packed m2c block (m2c <= 32, relative rows in lane
// registers `reli`) into the packed front, flat; every front entry receives
// one addition per child, so the order over children is unchanged
__device__ __forceinline__ void extend_add_flat(double* F, int nr, const double* Cc, int m2c, int reli, int lane) {
  const int ne = m2c * (m2c + 1) / 2;
  for (int e0 = 0; e0 < ne; e0 += 32) {
    int j, i;
    tri_at(e0 + lane, m2c, j, i);
    const int rj = __shfl_sync(kFull, reli, min(j, 31)), ri = __shfl_sync(kFull, reli, min(i, 31));
    if (e0 + lane < ne) F[cb32(rj, nr) + ri] += Cc[e0 + lane];
  }
}

// Small front (nr <= 32) by one warp from the packed metadata: lane i owns
// row i; children's metadata is fetched lane-parallel; the relative row map
// of a child sits in registers (lane i holds rel[i]) and its CB columns are
// read contiguously. Inside a subtree group the children were produced by
// this very warp, so there is no flag wait, and only the group's root
// publishes (fence + release). Arithmetic is identical to factor_task_smem<32>.
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void small_task(const FactorArgs& a, int s, int lane, double thresh, double* F,
                                           bool wait_children, bool publish, double* stg) {
  const DevSymb& S = a.S;
  const SnMeta m = S.meta[s];
  const int nr = m.nr, w = m.w, f = m.f, m2 = nr - w;
  if (wait_children)
    for (int q = m.c0 + lane; q < m.c1; q += 32) wait_flag(a.flags + __ldg(S.child + q), a.epoch);
  // the front is PACKED lower (column c at cb_col(c, nr)): half the shared memory
  zero_front(F, nr * (nr + 1) / 2, lane);
  __syncwarp();
  for (int e = lane; e < m.na; e += 32) {
    const int off = __ldg(S.aoff + m.a0 + e);
    F[cb32(off / nr, nr) + off % nr] = __ldg(a.kvals + __ldg(S.asrc + m.a0 + e));
  }
  __syncwarp();
  for (int q0 = m.c0; q0 < m.c1; q0 += 32) {
    // lane k fetches child q0+k's metadata; then children in order
    int cm2 = 0;
    int64_t ccb = 0, crel = 0;
    if (q0 + lane < m.c1) {
      const SnMeta& cmeta = S.meta[__ldg(S.child + q0 + lane)];
      cm2 = cmeta.nr - cmeta.w;
      ccb = cmeta.cboff;
      crel = cmeta.rptr + cmeta.w;
    }
    const int nq = min(32, m.c1 - q0);
    for (int k = 0; k < nq; ++k) {
      const int m2c = __shfl_sync(kFull, cm2, k);
      const long long cbk = __shfl_sync(kFull, static_cast<long long>(ccb), k);
      const long long rlk = __shfl_sync(kFull, static_cast<long long>(crel), k);
      const int reli = lane < m2c ? __ldg(S.relp + rlk + lane) : 0;
      const double* Cc = a.CB + cbk;
      const int ne = m2c * (m2c + 1) / 2;
      if (ne <= kGrpStack) {
        // stage the child's CB in shared memory with async copies (all in
        // flight at once) instead of one dependent global read per column
        for (int e = lane; e < ne; e += 32) cp_async8(stg + e, Cc + e);
        cp_async_wait_all();
        __syncwarp();
        Cc = stg;
      }
      if (ne <= kGrpStack) {  // staged in shared memory
        extend_add_flat(F, nr, stg, m2c, reli, lane);
      } else {
        int co = 0;
        for (int j = 0; j < m2c; ++j) {
          const int relj = __shfl_sync(kFull, reli, j);
          if (lane >= j && lane < m2c) F[cb32(relj, nr) + reli] += __ldcg(Cc + co + lane);
          co += m2c - j - 1;
        }
      }
      __syncwarp();
    }
  }
  const int i = lane;
  for (int c = 0; c < w; ++c) {
    const int offc = cb32(c, nr);
    const double d = F[offc + c];
    if (i == 0) {
      a.D[f + c] = d;
      if (fabs(d) <= thresh) atomicMin(a.zp, f + c);
    }
    double l = 0.0;
    if (i > c && i < nr) {
      l = F[offc + i] * __drcp_rn(d);
      F[offc + i] = l;
    }
    const double dl = d * l;
    int off2 = cb32(c + 1, nr);  // column c2's offset, advanced incrementally
    for (int c2 = c + 1; c2 < nr; ++c2) {
      const double lc2 = __shfl_sync(kFull, dl, c2);
      if (i >= c2 && i < nr) F[off2 + i] -= l * lc2;
      off2 += nr - c2 - 1;
    }
    __syncwarp();
  }
  double* P = a.L + m.loff;
  double* C = a.CB + m.cboff;
  for (int c = 0, fo = 0; c < w; fo += nr - c - 1, ++c)
    if (lane < nr) P[c * nr + lane] = lane >= c ? F[fo + lane] : 0.0;
  copy_cb(F, nr, w, C, lane);
  __syncwarp();
  if (publish && lane == 0) {
    __threadfence();
    st_release(a.flags + s, a.epoch);
  }
}

// Mid-size front (32 < nr <= kMidFront) by one warp in its shared-memory
// region (packed front over the warp's front + stack space): lane l owns rows
// l and l + 32. Children's contribution blocks are read flat (coalesced,
// four loads in flight per lane) with their relative row maps in registers;
// per entry the order is the same as small_task's: A value, then children in
// ascending order, then the column updates in pivot order.
constexpr int kMidFront = 45;  // 45 * 46 / 2 = 1035 <= kGrpFront * (kGrpFront + 1) / 2 + kGrpStack
__device__ __forceinline__ int rel_at(int x, int r0, int r1) {
  const int a = __shfl_sync(kFull, r0, x & 31), b = __shfl_sync(kFull, r1, x & 31);
  return x < 32 ? a : b;
}
__device__ __forceinline__ void mid_task(const FactorArgs& a, int s, int lane, double thresh, double* F) {
  const DevSymb& S = a.S;
  const SnMeta m = S.meta[s];
  const int nr = m.nr, w = m.w, f = m.f, m2 = nr - w;
  for (int q = m.c0 + lane; q < m.c1; q += 32) wait_flag(a.flags + __ldg(S.child + q), a.epoch);
  for (int k = lane; k < nr * (nr + 1) / 2; k += 32) F[k] = 0.0;
  __syncwarp();
  for (int e0 = 0; e0 < m.na; e0 += 128) {
    int off[4];
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + lane + 32 * u;
      off[u] = e < m.na ? __ldg(S.aoff + m.a0 + e) : 0;
      v[u] = e < m.na ? __ldg(a.kvals + __ldg(S.asrc + m.a0 + e)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (e0 + lane + 32 * u < m.na) F[cb32(off[u] / nr, nr) + off[u] % nr] = v[u];
  }
  __syncwarp();
  for (int q = m.c0; q < m.c1; ++q) {
    const SnMeta cm = S.meta[__ldg(S.child + q)];
    const int m2c = cm.nr - cm.w;
    const int64_t rl = cm.rptr + cm.w;
    const int r0 = lane < m2c ? __ldg(S.relp + rl + lane) : 0;
    const int r1 = lane + 32 < m2c ? __ldg(S.relp + rl + lane + 32) : 0;
    const double* Cc = a.CB + cm.cboff;
    const int ne = m2c * (m2c + 1) / 2;
    int j = 0, i = lane;  // packed position lane -> (column j, row i)
    while (i >= m2c && j < m2c) {
      const int ex = i - m2c;
      ++j;
      i = j + ex;
    }
    for (int e0 = 0; e0 < ne; e0 += 128) {
      double v[4];
      int jj[4], ii[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + lane + 32 * u;
        v[u] = e < ne ? __ldcg(Cc + e) : 0.0;
        jj[u] = j;
        ii[u] = i;
        i += 32;
        while (i >= m2c && j < m2c) {
          const int ex = i - m2c;
          ++j;
          i = j + ex;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rj = rel_at(min(jj[u], 63), r0, r1), ri = rel_at(min(ii[u], 63), r0, r1);
        if (e0 + lane + 32 * u < ne) F[cb32(rj, nr) + ri] += v[u];
      }
    }
    __syncwarp();
  }
  const int i0 = lane, i1 = lane + 32;
  for (int c = 0; c < w; ++c) {
    const int offc = cb32(c, nr);
    const double d = F[offc + c];
    if (lane == 0) {
      a.D[f + c] = d;
      if (fabs(d) <= thresh) atomicMin(a.zp, f + c);
    }
    double y0 = 0.0, y1 = 0.0;
    if (i0 > c && i0 < nr) {
      y0 = F[offc + i0] * __drcp_rn(d);
      F[offc + i0] = y0;
    }
    if (i1 > c && i1 < nr) {
      y1 = F[offc + i1] * __drcp_rn(d);
      F[offc + i1] = y1;
    }
    const double dl0 = d * y0, dl1 = d * y1;
    int off2 = cb32(c + 1, nr);
    for (int c2 = c + 1; c2 < nr; ++c2) {
      const double lc2 = c2 < 32 ? __shfl_sync(kFull, dl0, c2) : __shfl_sync(kFull, dl1, c2 - 32);
      if (i0 >= c2 && i0 < nr) F[off2 + i0] -= y0 * lc2;
      if (i1 >= c2 && i1 < nr) F[off2 + i1] -= y1 * lc2;
      off2 += nr - c2 - 1;
    }
    __syncwarp();
  }
  double* P = a.L + m.loff;
  double* C = a.CB + m.cboff;
  for (int c = 0, fo = 0; c < w; fo += nr - c - 1, ++c) {
    if (i0 < nr) P[c * nr + i0] = i0 >= c ? F[fo + i0] : 0.0;
    if (i1 < nr) P[c * nr + i1] = i1 >= c ? F[fo + i1] : 0.0;
  }
  for (int jc = 0, co = 0, fo = cb32(w, nr) + w; jc < m2; co += m2 - jc - 1, fo += nr - w - jc - 1, ++jc) {
    if (i0 >= jc && i0 < m2) C[co + i0] = F[fo + i0];
    if (i1 >= jc && i1 < m2) C[co + i1] = F[fo + i1];
  }
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    st_release(a.flags + s, a.epoch);
  }
}

// A whole subtree group by one warp, entirely in shared memory: the group
// program (csrc/capi.cpp build_layout) and its A values are loaded once,
// children's contribution blocks live on a shared-memory stack (multifrontal
// postorder), and only panels and the group root's CB go to global memory.
// Per node the arithmetic is exactly small_task's.
__device__ __forceinline__ void group_task(const FactorArgs& a, int g, int lane, double thresh, double* F,
                                           double* ST) {
  const DevSymb& S = a.S;
  // the program is read in place (read-only, L1-cached broadcast loads):
  // shared memory holds only the front and the stack, so more warps fit
  const int* __restrict__ PG = a.prog + __ldg(a.gpo + g);
  prefetch_prog(PG, lane);
  const int nnodes = __ldg(PG), nA = __ldg(PG + 1);
  for (int e = lane; e < nA; e += 32) ST[e] = __ldg(a.kvals + PG[4 + nA + e]);
  __syncwarp();
  const int* aoffs = PG + 4;
  double* stack = ST + nA;
  int p = 4 + 2 * nA;
  for (int v = 0; v < nnodes; ++v) {
    const int s = PG[p], f = PG[p + 1], w = PG[p + 2], nr = PG[p + 3], nch = PG[p + 4], push = PG[p + 5],
              af = PG[p + 6], ac = PG[p + 7];
    const int64_t loff = static_cast<int64_t>(static_cast<uint32_t>(PG[p + 8])) |
                         (static_cast<int64_t>(PG[p + 9]) << 32);
    const int64_t cboff = static_cast<int64_t>(static_cast<uint32_t>(PG[p + 10])) |
                          (static_cast<int64_t>(PG[p + 11]) << 32);
    p += 14;
    const int m2 = nr - w;
    zero_front(F, nr * (nr + 1) / 2, lane);  // packed lower front
    __syncwarp();
    for (int e = lane; e < ac; e += 32) F[aoffs[af + e]] = ST[af + e];  // program holds packed offsets
    __syncwarp();
    for (int q = 0; q < nch; ++q) {
      const int m2c = PG[p], off = PG[p + 1];
      const double* Cc = stack + off;
      if (off < 0) {  // external child (register-front phase): its CB in the standard layout
        Cc = a.CB + (static_cast<int64_t>(static_cast<uint32_t>(PG[p + 2])) | (static_cast<int64_t>(PG[p + 3]) << 32));
        if (lane == 0) wait_flag(a.flags + PG[p + 6], a.epoch);  // the register phase may still run (PDL)
        __syncwarp();
        p += 5;  // + CB offset, CV offset, child
      }
      const int reli = lane < m2c ? PG[p + 2 + lane] : 0;
      extend_add_flat(F, nr, Cc, m2c, reli, lane);
      p += 2 + m2c;
      __syncwarp();
    }
    const int i = lane;
    for (int c = 0; c < w; ++c) {
      const int offc = cb32(c, nr);
      const double d = F[offc + c];
      if (i == 0) {
        a.D[f + c] = d;
        if (fabs(d) <= thresh) atomicMin(a.zp, f + c);
      }
      double l = 0.0;
      if (i > c && i < nr) {
        l = F[offc + i] * __drcp_rn(d);
        F[offc + i] = l;
      }
      const double dl = d * l;
      int off2 = cb32(c + 1, nr);  // column c2's offset, advanced incrementally
      for (int c2 = c + 1; c2 < nr; ++c2) {
        const double lc2 = __shfl_sync(kFull, dl, c2);
        if (i >= c2 && i < nr) F[off2 + i] -= l * lc2;
        off2 += nr - c2 - 1;
      }
      __syncwarp();
    }
    double* P = a.L + loff;
    for (int c = 0, fo = 0; c < w; fo += nr - c - 1, ++c)
      if (lane < nr) P[c * nr + lane] = lane >= c ? F[fo + lane] : 0.0;
    double* C = push >= 0 ? stack + push : a.CB + cboff;
    copy_cb(F, nr, w, C, lane);
    __syncwarp();
    if (push < 0 && lane == 0) {  // the group root publishes its CB
      __threadfence();
      st_release(a.flags + s, a.epoch);
    }
  }
}


// ---------------------------------------------------------------------------
// Register-resident fronts (BatchSched, csrc/capi.cpp build_batches): one
// thread per front of a compile-time shape (NR rows, W pivots), the packed
// front in registers (entry (i, j) at PK(i, j), all indices constants).
// Per front entry: the A value (or 0) from the A map, then every child's CB
// entry through its byte map (255 = none), children in ascending order, then
// the pivot columns in order (l = F / d, F(i, c2) -= l_i (d l_c2)) — the
// operations of small_task in the same order, so the factor is bitwise that
// of the warp path. All loads of one source are independent and issued
// together. One persistent launch: warps claim 32 consecutive tasks (the
// list is padded so a warp never spans two levels), threads wait on their
// children's flags and publish their own.
// ---------------------------------------------------------------------------
// acquire every child's flag (the first four ids inline, compile-time indexed
// so the record stays in registers)
__device__ __forceinline__ void wait_children(const FactorArgs& a, const RegInst& I, const int* __restrict__ cid) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (q < I.nch) wait_flag(a.flags + I.cid[q], a.epoch);
  for (int q = 4; q < I.nch; ++q) wait_flag(a.flags + __ldg(cid + I.ccb + q), a.epoch);
}

template <int NR, int W, int R>
__device__ __forceinline__ void reg_front(const FactorArgs& a, const RegInst& I, int r, unsigned tm,
                                          const int* __restrict__ amap, const uint8_t* __restrict__ cmap,
                                          const uint32_t* __restrict__ cmapw, const int64_t* __restrict__ ccb,
                                          const int* __restrict__ cid, double thresh) {
  constexpr int NP = NR * (NR + 1) / 2, NPAD = (NP + 3) & ~3, M2 = NR - W, KR = (NR + R - 1) / R;
  constexpr int PW = W * NR - W * (W - 1) / 2;  // packed entries of the W pivot columns (the A map's length)
  auto PK = [](int i, int j) { return j * NR - j * (j + 1) / 2 + i; };  // packed lower, i >= j
  auto row = [r](int k) { return R == 1 ? k : r + R * k; };            // the lane's k-th row
  // broadcast of a team member's register (R == 1: the value itself)
  auto bcast = [tm](double v, int src) { return R == 1 ? v : __shfl_sync(tm, v, src, R); };
  double F[KR][NR];
  const int* am = amap + I.amap;
  const uint8_t* cm = cmap + I.cmap;
  if constexpr (R == 1) {
    // small fronts: round trip 1 (independent) = A slots + the first PRE
    // children's maps, round trip 2 = the children's flags, round trip 3 = A
    // values + CB entries; larger fronts keep fewer values in flight
    constexpr int PRE = 0;  // measured: preloading children's maps costs more in registers than it saves
    const int npre = min(I.nch, PRE);
    const uint32_t* cmw = cmapw + I.cmap;
    int sl[PW];
#pragma unroll
    for (int p = 0; p < PW; ++p) sl[p] = __ldg(am + 32 * p);
    uint32_t mw[PRE > 0 ? PRE : 1][NPAD / 4];
#pragma unroll
    for (int q = 0; q < PRE; ++q)
#pragma unroll
      for (int w4 = 0; w4 < NPAD / 4; ++w4) mw[q][w4] = q < npre ? __ldg(cmw + (q * (NPAD / 4) + w4) * 32) : 0xffffffffu;
    wait_children(a, I, cid);
#pragma unroll
    for (int j = 0; j < NR; ++j)
#pragma unroll
      for (int i = j; i < NR; ++i) {
        const int sv = j < W ? sl[j < W ? PK(i, j) : 0] : -1;
        F[i][j] = sv >= 0 ? __ldg(a.kvals + sv) : 0.0;
      }
#pragma unroll
    for (int q = 0; q < PRE; ++q) {
      if (q >= npre) break;
      const double* C = a.CB + I.cb[q];
#pragma unroll
      for (int j = 0; j < NR; ++j)
#pragma unroll
        for (int i = j; i < NR; ++i) {
          const uint32_t src = (mw[q][PK(i, j) >> 2] >> (8 * (PK(i, j) & 3))) & 0xffu;
          if (src != 0xffu) F[i][j] += __ldcg(C + src);
        }
    }
    for (int q = npre; q < I.nch; ++q) {
      const double* C = a.CB + __ldg(ccb + I.ccb + q);
      uint32_t w[NPAD / 4];
#pragma unroll
      for (int w4 = 0; w4 < NPAD / 4; ++w4) w[w4] = __ldg(cmw + (q * (NPAD / 4) + w4) * 32);
#pragma unroll
      for (int j = 0; j < NR; ++j)
#pragma unroll
        for (int i = j; i < NR; ++i) {
          const uint32_t src = (w[PK(i, j) >> 2] >> (8 * (PK(i, j) & 3))) & 0xffu;
          if (src != 0xffu) F[i][j] += __ldcg(C + src);
        }
    }
  } else {
    wait_children(a, I, cid);
#pragma unroll
    for (int k = 0; k < KR; ++k)
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        const int i = row(k);
        const int slv = (i < NR && j <= i && j < W) ? __ldg(am + PK(i, j)) : -1;
        F[k][j] = slv >= 0 ? __ldg(a.kvals + slv) : 0.0;
      }
    for (int q = 0; q < I.nch; ++q) {
      const double* C = a.CB + __ldg(ccb + I.ccb + q);
      const uint8_t* cq = cm + q * NPAD;
#pragma unroll
      for (int k = 0; k < KR; ++k)
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          const int i = row(k);
          const uint32_t src = (i < NR && j <= i) ? __ldg(cq + PK(i, j)) : 0xffu;
          if (src != 0xffu) F[k][j] += __ldcg(C + src);
        }
    }
  }
#pragma unroll
  for (int c = 0; c < W; ++c) {
    const double d = bcast(F[c / R][c], c % R);
    if (r == 0) {
      a.D[I.f + c] = d;
      if (fabs(d) <= thresh) atomicMin(a.zp, I.f + c);
    }
#pragma unroll
    for (int k = 0; k < KR; ++k)
      if (row(k) > c && row(k) < NR) F[k][c] *= __drcp_rn(d);
#pragma unroll
    for (int c2 = c + 1; c2 < NR; ++c2) {
      const double lc2 = d * bcast(F[c2 / R][c], c2 % R);
#pragma unroll
      for (int k = 0; k < KR; ++k)
        if (row(k) >= c2 && row(k) < NR) F[k][c2] -= F[k][c] * lc2;
    }
  }
  double* P = a.L + I.loff;
#pragma unroll
  for (int c = 0; c < W; ++c)
#pragma unroll
    for (int k = 0; k < KR; ++k)
      if (row(k) < NR) P[c * NR + row(k)] = row(k) >= c ? F[k][c] : 0.0;
  double* Cs = a.CB + I.cboff;
#pragma unroll
  for (int j = 0; j < M2; ++j)
#pragma unroll
    for (int k = 0; k < KR; ++k)
      if (row(k) >= W + j && row(k) < NR) Cs[j * M2 - j * (j + 1) / 2 + row(k) - W] = F[k][W + j];
}

template <int K0, int... K>
__device__ __forceinline__ void reg_dispatch(const FactorArgs& a, const RegChunk& ch, int lane,
                                             const RegInst* __restrict__ inst, const int* amap, const uint8_t* cmap,
                                             const uint32_t* cmapw, const int64_t* ccb, const int* cid,
                                             double thresh, std::integer_sequence<int, K...>) {
  (((ch.shape == K0 + K) ? [&] {
    constexpr int NR = kRegShapes[K0 + K][0], W = kRegShapes[K0 + K][1], R = kRegShapes[K0 + K][2];
    const int ix = lane / R;
    if (ix < ch.n) {
      const unsigned tm = R == 32 ? kFull : (((1u << R) - 1u) << (ix * R));
      const RegInst I = inst[ch.first + ix];
      reg_front<NR, W, R>(a, I, lane % R, tm, amap, cmap, cmapw, ccb, cid, thresh);
      if constexpr (R > 1) __syncwarp(tm);
      if (lane % R == 0) st_release(a.flags + I.s, a.epoch);  // release: orders this thread's writes
    }
  }()
                    : void()),
   ...);
}

template <int K0, int K1>
__global__ void __launch_bounds__(128) reg_factor_kernel(FactorArgs a, const RegInst* __restrict__ inst,
                                                         const RegChunk* __restrict__ chunks, int nchunk,
                                                         const int* __restrict__ amap,
                                                         const uint8_t* __restrict__ cmap,
                                                         const uint32_t* __restrict__ cmapw,
                                                         const int64_t* __restrict__ ccb, const int* __restrict__ cid) {
  const int lane = threadIdx.x & 31;
  const double thresh = __ldcg(a.thresh);
  const int tail = nchunk - static_cast<int>(gridDim.x) * 4;
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(a.ticket, 1);
    c = __shfl_sync(kFull, c, 0);
    if (lane == 0 && c >= tail) pdl_trigger();
    if (c >= nchunk) break;
    const RegChunk ch = chunks[c];
    reg_dispatch<K0>(a, ch, lane, inst, amap, cmap, cmapw, ccb, cid, thresh,
                     std::make_integer_sequence<int, K1 - K0>{});
  }
}

template <int NT>
__global__ void __launch_bounds__(NT == 32 ? 128 : NT, NT == 32 ? NCL_FK32_MINB : NT == 128 ? NCL_FK128_MINB : 2) factor_kernel(FactorArgs a) {
  __shared__ int s_ticket;
  extern __shared__ double s_front[];
  const int tid = NT == 32 ? (threadIdx.x & 31) : threadIdx.x;
  constexpr int kFrontPk = kGrpFront * (kGrpFront + 1) / 2;              // packed lower 32 x 32
  constexpr int kWarpSmem = kFrontPk + kGrpStack;                         // doubles per warp
  double* F = NT == 32 ? s_front + (threadIdx.x >> 5) * kWarpSmem : s_front;
  double* gST = F + kFrontPk;
  const double thresh = __ldcg(a.thresh);
  Claim<NT> cl;
  const int tail = a.t1 - static_cast<int>(gridDim.x) * (NT == 32 ? 4 : 1);  // the last claims of the launch
  for (;;) {
    const int t = cl.next(a.ticket, a.t0, a.t1, a.nleaf, tid, &s_ticket);
    if (tid == 0 && (t < 0 || t >= tail)) pdl_trigger();
    if (t < 0) break;
    // a task is a whole small subtree in postorder (one warp, no scheduling
    // between its nodes) or a single supernode
    const bool group = t < a.nleaf;  // subtree group: children internal, only the root publishes
    if (a.trace && tid == 0) a.trace[2 * t] = gtimer();
    if constexpr (NT == 32) {
      if (group && a.prog) {
        group_task(a, t, tid, thresh, F, gST);
        if (a.trace && tid == 0) a.trace[2 * t + 1] = gtimer();
        continue;
      }
    }
    const int k0 = __ldg(a.tptr + t), k1 = __ldg(a.tptr + t + 1);
    for (int k = k0; k < k1; ++k) {
      const int s = __ldg(a.tasks + k);
      const int nr = static_cast<int>(__ldg(a.S.sn_rptr + s + 1) - __ldg(a.S.sn_rptr + s));
      if (a.skip_big && __ldg(a.S.big + s)) continue;  // runs on the large-front path
      if (NT == 32 && nr <= kWarpFront) small_task(a, s, tid, thresh, F, !group, !group || k == k1 - 1, F + kFrontPk);
      else if (NT == 32 && !group && nr <= kMidFront) mid_task(a, s, tid, thresh, F);
      else if (NT != 32 && nr <= (NT == 128 ? kCtaFrontS : kCtaFront)) factor_task_smem<NT>(a, s, tid, thresh, F);
      else factor_task<NT>(a, s, tid, thresh, !group, !group || k == k1 - 1);
    }
    if (a.trace && tid == 0) a.trace[2 * t + 1] = gtimer();
  }
}

// Heavy-gather front that fits the CTA path: bf_gather assembled it (many
// children, multi-CTA) into its full-layout scratch; one CTA factors it here
// with the same arithmetic as the CTA smem path.
template <int NT>
__global__ void __launch_bounds__(NT) big_cta_kernel(DevSymb S, const BigDesc* d, const double* Fs, double* L,
                                                     double* CB, double* D, const double* thresh_p, int* zp) {
  extern __shared__ double s_front[];
  const BigDesc b = d[blockIdx.x];
  if (b.npan != 0) return;
  const int nr = b.nr, tid = threadIdx.x;
  const double* G = Fs + b.foff;  // assembled in the packed layout (gdst, nr <= kCtaFront)
  for (int k = tid; k < nr * (nr + 1) / 2; k += NT) s_front[k] = __ldcg(G + k);
  __syncthreads();
  cta_dense<NT>(s_front, nr, b.w, b.f, __ldcg(thresh_p), D, zp, L + __ldg(S.sn_loff + b.s), CB + __ldg(S.cb_off + b.s),
                 tid);
}

// one atomic per block (warp shuffles, then the block's warps through shared
// memory): the per-warp atomics on one address serialised in L2
__global__ void __launch_bounds__(256) maxdiag_kernel(const int* __restrict__ pos, int nd, const double* __restrict__ v,
                                                      double* out) {
  __shared__ double wm[8];
  double m = 0.0;
  // four independent position -> value gathers in flight per thread
  const int stride = gridDim.x * blockDim.x;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < nd; i += 4 * stride) {
    int p[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) p[u] = __ldg(pos + i + u * stride);
    double x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = __ldg(v + p[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) m = fmax(m, fabs(x[u]));
  }
  for (; i < nd; i += stride) m = fmax(m, fabs(__ldg(v + __ldg(pos + i))));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) m = fmax(m, wm[w]);
    atomic_max_nonneg(out, m);
  }
}
__global__ void thresh_kernel(double* scal, double tol, int* istat, int n) {
  // scal[1] = max|diag M| ; scal[0] = pivot_tol * max(1, maxdiag)  (sparse_sym.cpp:286)
  scal[0] = tol * fmax(1.0, scal[1]);
  istat[0] = n;  // no zero pivot yet
  istat[1] = istat[2] = istat[3] = 0;
}

__global__ void __launch_bounds__(256) inertia_kernel(const double* __restrict__ D, int n, const double* scal,
                                                      int* istat, const uint8_t* __restrict__ report) {
  __shared__ int wc[3][8];
  const double th = scal[0];
  int np = 0, nn = 0, nz = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (report && !report[i]) continue;  // sharded: every column counted by exactly one rank
    const double d = __ldg(D + i);
    if (fabs(d) <= th) nz++;
    else if (d > 0.0) np++;
    else nn++;
  }
  for (int o = 16; o > 0; o >>= 1) {
    np += __shfl_xor_sync(kFull, np, o);
    nn += __shfl_xor_sync(kFull, nn, o);
    nz += __shfl_xor_sync(kFull, nz, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) wc[0][w] = np, wc[1][w] = nn, wc[2][w] = nz;
  __syncthreads();
  if (threadIdx.x < 3) {  // one atomic per counter per block
    int t = 0;
    for (int k = 0; k < 8; ++k) t += wc[threadIdx.x][k];
    if (t) atomicAdd(istat + 1 + threadIdx.x, t);
  }
}

// ---------------------------------------------------------------------------
// Solves (K4), same task order and team split as the factorization.
// Forward, multifrontal: supernode s gathers b through the permutation
// (px[k] = b[perm[k]], sparse_sym.cpp:349), extend-adds its children's
// contribution vectors (CV, rows below their columns), runs the unit-lower
// triangular solve of its w columns and leaves -L21 x1 in its own CV.
// Backward, roots first: T_c = sum_{i>=w} L_ic x_{R_i} over ancestor values
// (parallel over columns), then the w x w unit-upper block, D^{-1} fused,
// result scattered through the permutation (sparse_sym.cpp:351-362).
// ---------------------------------------------------------------------------
struct SolveArgs {
  DevSymb S;
  const double* L;
  const double* D;
  double* CV;
  double* xp;
  const double* b;
  double* x;
  int* flags;
  int* ticket;
  int epoch;
  int t0, t1;
  const int* tasks;
  const int* tptr;
  const int* prog;
  const int64_t* gpo;
  int nleaf;
  unsigned long long* trace;  // optional (NCL_SOLVE_TRACE): globaltimer start/end per task
  int pregathered = -1;       // node whose heavy contribution-vector gather ran GPU-wide (fwd_root_gather)
};

__device__ __forceinline__ void prefetch_l2(const double* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

__device__ __forceinline__ int64_t rec64(const int* r) {
  return static_cast<int64_t>(static_cast<uint32_t>(r[0])) | (static_cast<int64_t>(r[1]) << 32);
}

// Forward solve of a subtree group by one warp from its program (same node
// order as the factor): lane i owns row i, children's contribution vectors
// come from a shared-memory stack (at the factor's CB stack offsets), only
// x (pivot rows) and the root's CV go to global memory. Same arithmetic as
// fwd_task<32>.
__device__ void fwd_group(const SolveArgs& a, int g, int lane, double* VS, double* ST) {
  const DevSymb& S = a.S;
  const int* __restrict__ PG = a.prog + __ldg(a.gpo + g);  // read in place (see group_task)
  prefetch_prog(PG, lane);
  const int nnodes = __ldg(PG), nA = __ldg(PG + 1);
  int p = 4 + 2 * nA;
  for (int v = 0; v < nnodes; ++v) {
    const int* R = PG + p;
    const int s = R[0], f = R[1], w = R[2], nr = R[3], nch = R[4], push = R[5];
    const int64_t loff = rec64(R + 8), rb = rec64(R + 12);
    p += 14;
    if (lane < nr) VS[lane] = lane < w ? __ldcg(a.b + __ldg(S.perm + f + lane)) : 0.0;
    __syncwarp();
    for (int q = 0; q < nch; ++q) {
      const int m2c = PG[p], off = PG[p + 1];
      if (off < 0) {  // external child (register-front phase): its CV in the standard layout
        const int64_t cv = rec64(PG + p + 4);
        if (lane == 0) wait_flag(a.flags + PG[p + 6], a.epoch);  // the register phase may still run (PDL)
        __syncwarp();
        if (lane < m2c) VS[PG[p + 7 + lane]] += __ldcg(a.CV + cv + lane);
        p += 7 + m2c;
      } else {
        if (lane < m2c) VS[PG[p + 2 + lane]] += ST[off + lane];
        p += 2 + m2c;
      }
      __syncwarp();
    }
    const double* P = a.L + loff;
    // lane i owns row i in a register; panel columns are fetched eight at a
    // time (all loads in flight), the pivots broadcast by shuffles
    double y = lane < nr ? VS[lane] : 0.0;
    for (int c0 = 0; c0 < w; c0 += 8) {
      double pv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        pv[u] = (c0 + u < w && lane > c0 + u && lane < nr) ? __ldg(P + (c0 + u) * nr + lane) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (c0 + u < w) {
          const double xc = __shfl_sync(kFull, y, c0 + u);
          if (lane > c0 + u && lane < nr) y -= pv[u] * xc;
        }
      }
    }
    if (lane < w) a.xp[f + lane] = y;
    if (lane >= w && lane < nr) {
      if (push >= 0) ST[push + (lane - w)] = y;
      else a.CV[rb + lane] = y;
    }
    __syncwarp();
    if (push < 0 && lane == 0) {
      __threadfence();
      st_release(a.flags + s, a.epoch);
    }
  }
}

// Backward solve of a group (reverse postorder; the root waits for its
// parent, which lies outside the group). Same arithmetic as bwd_task<32>.
__device__ void bwd_group(const SolveArgs& a, int g, int lane) {
  const DevSymb& S = a.S;
  const int* __restrict__ PG = a.prog + __ldg(a.gpo + g);  // read in place (see group_task)
  prefetch_prog(PG, lane);
  const int nnodes = __ldg(PG);
  const int* OFF = PG + __ldg(PG + 2);  // record offsets of the nodes (table after the records)
  for (int v = nnodes - 1; v >= 0; --v) {
    const int* R = PG + OFF[v];
    const int s = R[0], f = R[1], w = R[2], nr = R[3];
    const int64_t loff = rec64(R + 8), rb = rec64(R + 12);
    if (v == nnodes - 1) {
      const int ps = __ldg(S.sn_parent + s);
      if (lane == 0 && ps >= 0) wait_flag(a.flags + ps, a.epoch);
      __syncwarp();
    }
    const double* P = a.L + loff;
    const bool below = lane >= w && lane < nr;
    const double xi = below ? __ldcg(a.xp + __ldg(S.rows + rb + lane)) : 0.0;
    // 1 / d off the column chain (each lane its own pivot, before the chain)
    const double rl = lane < w ? __drcp_rn(__ldg(a.D + f + lane)) : 1.0;
    const int pl = lane < w ? __ldg(S.perm + f + lane) : 0;
    double T = 0.0;  // lane c < w holds T[c]
    for (int c0 = 0; c0 < w; c0 += 8) {  // eight columns' loads and reductions in flight
      double acc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] = (c0 + u < w && below) ? __ldg(P + (c0 + u) * nr + lane) * xi : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] += __shfl_xor_sync(kFull, acc[u], o);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (lane == c0 + u) T = acc[u];
    }
    double xs = lane < w ? a.xp[f + lane] : 0.0;
    for (int c1 = w; c1 > 0; c1 -= 8) {  // upper part: column c of row lane < c, eight at a time
      double pu[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c1 - 1 - u;
        pu[u] = (c >= 0 && lane < c) ? __ldg(P + lane * nr + c) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c1 - 1 - u;
        if (c >= 0) {
          double vv = 0.0;
          if (lane == c) {
            vv = xs * rl - T;
            xs = vv;
            a.xp[f + c] = vv;
            a.x[pl] = vv;
          }
          vv = __shfl_sync(kFull, vv, c);
          if (lane < c) T += pu[u] * vv;
        }
      }
    }
    __syncwarp();
    // the node's x is final: register fronts below it (a later, possibly
    // overlapping launch) wait on this flag
    if (lane == 0) {
      __threadfence();
      st_release(a.flags + s, a.epoch);
    }
  }
}


// Forward triangular part of a single (one warp, nr <= 32 kSl): lane l owns
// rows l + 32 q in registers, pivots by shuffle, panel columns fetched four
// at a time. Same operations and order as the column loop.
template <int kSl>
__device__ __forceinline__ void fwd_warp_reg(const double* __restrict__ P, int nr, int w, double* xs, double* cv,
                                             int tid) {
  double y[kSl];
#pragma unroll
  for (int q = 0; q < kSl; ++q) {
    const int r = tid + 32 * q;
    y[q] = r < nr ? (r < w ? xs[r] : cv[r]) : 0.0;
  }
  for (int c0 = 0; c0 < w; c0 += 4) {
    double pv[4][kSl];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int q = 0; q < kSl; ++q) {
        const int c = c0 + u, r = tid + 32 * q;
        pv[u][q] = (c < w && r > c && r < nr) ? __ldg(P + static_cast<int64_t>(c) * nr + r) : 0.0;
      }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + u;
      if (c < w) {
        const int qc = c >> 5;
        double yc = y[0];
#pragma unroll
        for (int q = 1; q < kSl; ++q) yc = qc == q ? y[q] : yc;
        const double xc = __shfl_sync(kFull, yc, c & 31);
#pragma unroll
        for (int q = 0; q < kSl; ++q) {
          const int r = tid + 32 * q;
          if (r > c && r < nr) y[q] -= pv[u][q] * xc;
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kSl; ++q) {
    const int r = tid + 32 * q;
    if (r < w) xs[r] = y[q];
    else if (r < nr) cv[r] = y[q];
  }
  __syncwarp();
}

// Rows of a node with many contributing children (the separator roots): a
// warp per row, lanes over its sources, fixed xor-butterfly combine, then b
// (deterministic); four rows per warp interleaved so their loads are in
// flight together. Rows k0, k0 + 4 kstep_rows ... of this warp.
__device__ __forceinline__ void heavy_cv_rows(const SolveArgs& a, int s, int f, int w, int nr, int64_t v0, int kfirst,
                                              int kstep, int lane) {
  const DevSymb& S = a.S;
  double* cv = a.CV + __ldg(S.sn_rptr + s);
  double* xs = a.xp + f;
  for (int k0 = kfirst; k0 < nr; k0 += kstep) {
    int64_t qa[4], qb[4];
    double acc[4];
    int64_t len = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + u;
      qa[u] = k < nr ? __ldg(S.cvsp + v0 + k) : 0;
      qb[u] = k < nr ? __ldg(S.cvsp + v0 + k + 1) : 0;
      acc[u] = 0.0;
      len = max(len, qb[u] - qa[u]);
    }
    for (int64_t o = lane; o < len; o += 64) {  // two sources per row per lane in flight
      int64_t src[8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        src[u] = qa[u] + o < qb[u] ? __ldg(S.cvsrc + qa[u] + o) : -1;
        src[u + 4] = qa[u] + o + 32 < qb[u] ? __ldg(S.cvsrc + qa[u] + o + 32) : -1;
      }
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = src[u] >= 0 ? __ldcg(a.CV + src[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (src[u] >= 0) acc[u] += v[u];
        if (src[u + 4] >= 0) acc[u] += v[u + 4];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      for (int o = 16; o > 0; o >>= 1) acc[u] += __shfl_xor_sync(kFull, acc[u], o);
      const int k = k0 + u;
      if (lane == 0 && k < nr) {
        if (k < w) xs[k] = __ldcg(a.b + __ldg(S.perm + f + k)) + acc[u];
        else cv[k] = acc[u];
      }
    }
  }
}

template <int NT>
__device__ __forceinline__ void fwd_task(const SolveArgs& a, int s, int tid) {
  const DevSymb& S = a.S;
  const int f = __ldg(S.sn_first + s);
  const int w = __ldg(S.sn_first + s + 1) - f;
  const int64_t rb = __ldg(S.sn_rptr + s);
  const int nr = static_cast<int>(__ldg(S.sn_rptr + s + 1) - rb);
  const double* P = a.L + __ldg(S.sn_loff + s);
  const int64_t v0 = NT == 32 ? 0 : __ldg(S.cv_ptr + s), v1 = NT == 32 ? 0 : __ldg(S.cv_ptr + s + 1);
  if (NT != 32) {
    // pull the panel and the gather map into L2 while the children finish
    for (int64_t e = 16 * static_cast<int64_t>(tid); e < static_cast<int64_t>(nr) * w; e += 16 * NT) prefetch_l2(P + e);
    if (v1 > v0) {
      const int64_t q0 = __ldg(S.cvsp + v0), q1 = __ldg(S.cvsp + v1);
      for (int64_t k = v0 + 16 * static_cast<int64_t>(tid); k <= v1; k += 16 * NT) prefetch_l2d(S.cvsp + k);
      for (int64_t k = q0 + 16 * static_cast<int64_t>(tid); k < q1; k += 16 * NT) prefetch_l2d(S.cvsrc + k);
    }
  }
  for (int q = __ldg(S.cptr + s) + tid; q < __ldg(S.cptr + s + 1); q += NT) wait_flag(a.flags + __ldg(S.child + q), a.epoch);
  team_sync<NT>();
  double* cv = a.CV + rb;
  double* xs = a.xp + f;
  if (v1 > v0) {
    if (NT != 32 && __ldg(S.cvsp + v1) - __ldg(S.cvsp + v0) > 8 * static_cast<int64_t>(nr)) {
      // many children (the separator roots): a warp per row, lanes over its
      // sources, fixed xor-butterfly combine, then b (deterministic)
      // (four rows per warp interleaved: their loads are in flight together)
      if (a.pregathered != s) heavy_cv_rows(a, s, f, w, nr, v0, 4 * (tid >> 5), 4 * (NT / 32), tid & 31);
    } else {
      // gather per row: b (pivot rows) then the children's CV entries in
      // child order — the sequential extend-add's summation order
      for (int k = tid; k < nr; k += NT) {
        double acc = k < w ? __ldcg(a.b + __ldg(S.perm + f + k)) : 0.0;
        for (int64_t q = __ldg(S.cvsp + v0 + k); q < __ldg(S.cvsp + v0 + k + 1); ++q)
          acc += __ldcg(a.CV + __ldg(S.cvsrc + q));
        if (k < w) xs[k] = acc;
        else cv[k] = acc;
      }
    }
    team_sync<NT>();
  } else {
  for (int k = tid; k < nr; k += NT) {
    if (k < w) xs[k] = __ldcg(a.b + __ldg(S.perm + f + k));
    else cv[k] = 0.0;
  }
  team_sync<NT>();
  for (int q = __ldg(S.cptr + s); q < __ldg(S.cptr + s + 1); ++q) {
    const int c = __ldg(S.child + q);
    const int wc = __ldg(S.sn_first + c + 1) - __ldg(S.sn_first + c);
    const int64_t rbc = __ldg(S.sn_rptr + c);
    const int m2c = static_cast<int>(__ldg(S.sn_rptr + c + 1) - rbc) - wc;
    for (int k = tid; k < m2c; k += NT) {
      const int r = __ldg(S.relp + rbc + wc + k);
      const double v = __ldcg(a.CV + rbc + wc + k);
      if (r < w) xs[r] += v;
      else cv[r] += v;
    }
    team_sync<NT>();
  }
  }  // extend-add path
  if (NT == 32 && nr > kCtaFront) {  // generic warp fallback (no such single in the SCOPF layouts)
    for (int c = 0; c < w; ++c) {
      const double xc = xs[c];
      const double* Pc = P + static_cast<int64_t>(c) * nr;
      for (int i = c + 1 + tid; i < nr; i += NT) {
        const double u = Pc[i] * xc;
        if (i < w) xs[i] -= u;
        else cv[i] -= u;
      }
      team_sync<NT>();
    }
  } else if constexpr (NT == 32) {
    if (nr <= 32) fwd_warp_reg<1>(P, nr, w, xs, cv, tid);
    else fwd_warp_reg<(kCtaFront + 31) / 32>(P, nr, w, xs, cv, tid);
  } else {
    // blocked: warp 0 solves each 32-column diagonal block in registers
    // (no CTA barrier per column), then all threads apply the block to the
    // rows below it
    const int lane = tid & 31;
    for (int c0 = 0; c0 < w; c0 += 32) {
      const int c1 = min(w, c0 + 32);
      if (tid < 32) {
        const int i = c0 + lane;
        double y = i < c1 ? xs[i] : 0.0;
        for (int c = c0; c < c1; c += 8) {
          double pv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            pv[u] = (c + u < c1 && i > c + u && i < c1) ? __ldg(P + static_cast<int64_t>(c + u) * nr + i) : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (c + u < c1) {
              const double xc = __shfl_sync(kFull, y, c + u - c0);
              if (i > c + u && i < c1) y -= pv[u] * xc;
            }
          }
        }
        if (i < c1) xs[i] = y;
      }
      __syncthreads();
      for (int i = c1 + tid; i < nr; i += NT) {
        double acc = 0.0;
        for (int c = c0; c < c1; ++c) acc += P[static_cast<int64_t>(c) * nr + i] * xs[c];
        if (i < w) xs[i] -= acc;
        else cv[i] -= acc;
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    __threadfence();
    st_release(a.flags + s, a.epoch);
  }
}

// Backward part of a single (one warp): registers throughout — lane l holds
// the ancestor values of rows w + l + 32 q and T / x of pivot columns l + 32 q;
// the same operation order as the shared-memory CTA version.
template <int kSl>
__device__ __forceinline__ void bwd_warp_reg(const SolveArgs& a, const double* __restrict__ P, const int* Rs, int f,
                                             int nr, int w, double* xs, int lane) {
  const DevSymb& S = a.S;
  double xi[kSl], Tq[kSl], xq[kSl], dq[kSl];
  int pq[kSl];
#pragma unroll
  for (int q = 0; q < kSl; ++q) {
    const int i = w + lane + 32 * q, c = lane + 32 * q;
    xi[q] = i < nr ? __ldcg(a.xp + __ldg(Rs + i)) : 0.0;
    Tq[q] = 0.0;
    xq[q] = c < w ? xs[c] : 0.0;
    dq[q] = c < w ? __drcp_rn(__ldg(a.D + f + c)) : 1.0;  // 1 / d, off the column chain
    pq[q] = c < w ? __ldg(S.perm + f + c) : 0;
  }
  for (int c0 = 0; c0 < w; c0 += 4) {
    double acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc[u] = 0.0;
      const double* Pc = P + static_cast<int64_t>(c0 + u) * nr;
#pragma unroll
      for (int q = 0; q < kSl; ++q) {
        const int i = w + lane + 32 * q;
        if (c0 + u < w && i < nr) acc[u] += __ldg(Pc + i) * xi[q];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] += __shfl_xor_sync(kFull, acc[u], o);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + u;
#pragma unroll
      for (int q = 0; q < kSl; ++q)
        if (c < w && c == lane + 32 * q) Tq[q] = acc[u];
    }
  }
  for (int c1 = w; c1 > 0; c1 -= 2) {
    double pu[2][kSl];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int q = 0; q < kSl; ++q) {
        const int c = c1 - 1 - u, c2 = lane + 32 * q;
        pu[u][q] = (c >= 0 && c2 < c) ? __ldg(P + static_cast<int64_t>(c2) * nr + c) : 0.0;
      }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int c = c1 - 1 - u;
      if (c >= 0) {
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < kSl; ++q)
          if (c == lane + 32 * q) {
            v = xq[q] * dq[q] - Tq[q];
            xq[q] = v;
            xs[c] = v;
            a.x[pq[q]] = v;
          }
        v = __shfl_sync(kFull, v, c & 31);
#pragma unroll
        for (int q = 0; q < kSl; ++q)
          if (lane + 32 * q < c) Tq[q] += pu[u][q] * v;
      }
    }
  }
  __syncwarp();
}

template <int NT>
__device__ __forceinline__ void bwd_task(const SolveArgs& a, int s, int tid) {
  const DevSymb& S = a.S;
  const int ps = __ldg(S.sn_parent + s);
  const int f = __ldg(S.sn_first + s);
  const int w = __ldg(S.sn_first + s + 1) - f;
  const int64_t rb = __ldg(S.sn_rptr + s);
  const int nr = static_cast<int>(__ldg(S.sn_rptr + s + 1) - rb);
  const int* Rs = S.rows + rb;
  const double* P = a.L + __ldg(S.sn_loff + s);
  if (NT != 32) {  // pull the panel and the row list into L2 while the parent finishes
    for (int64_t e = 16 * static_cast<int64_t>(tid); e < static_cast<int64_t>(nr) * w; e += 16 * NT) prefetch_l2(P + e);
    for (int k = 32 * tid; k < nr; k += 32 * NT) prefetch_l2d(Rs + k);
  }
  if (tid == 0 && ps >= 0) wait_flag(a.flags + ps, a.epoch);
  team_sync<NT>();
  double* T = a.CV + rb;  // the first w CV slots are free during the backward sweep
  double* xs = a.xp + f;
  const int lane = tid & 31, warp = tid >> 5;
  if (NT == 32 && nr > kCtaFront) {  // generic warp fallback (no such single in the SCOPF layouts)
    for (int c = 0; c < w; ++c) {
      const double* Pc = P + static_cast<int64_t>(c) * nr;
      double acc = 0.0;
      for (int i = w + lane; i < nr; i += 32) acc += Pc[i] * __ldcg(a.xp + __ldg(Rs + i));
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
      if (lane == 0) T[c] = acc;
    }
    team_sync<NT>();
    for (int c = w - 1; c >= 0; --c) {
      if (tid == 0) {
        const double v = xs[c] * __drcp_rn(__ldg(a.D + f + c)) - T[c];
        xs[c] = v;
        a.x[__ldg(S.perm + f + c)] = v;
      }
      team_sync<NT>();
      const double v = xs[c];
      for (int c2 = tid; c2 < c; c2 += NT) T[c2] += P[static_cast<int64_t>(c2) * nr + c] * v;
      team_sync<NT>();
    }
  } else if constexpr (NT == 32) {
    if (nr - w <= 32 && w <= 32) bwd_warp_reg<1>(a, P, Rs, f, nr, w, xs, lane);
    else bwd_warp_reg<(kCtaFront + 31) / 32>(a, P, Rs, f, nr, w, xs, lane);
  } else {
  for (int c = warp; c < w; c += NT / 32) {
    const double* Pc = P + static_cast<int64_t>(c) * nr;
    double acc = 0.0;
    for (int i = w + lane; i < nr; i += 32) acc += Pc[i] * __ldcg(a.xp + __ldg(Rs + i));
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if (lane == 0) T[c] = acc;
  }
  team_sync<NT>();
    // blocked from the bottom: warp 0 solves a 32-column block, then all
    // threads fold it into T of the columns above
    for (int c1 = w; c1 > 0; c1 -= 32) {
      const int c0 = max(0, c1 - 32);
      if (tid < 32) {  // the 32-column block in registers: lane l is column c0 + l
        const int c2 = c0 + lane;
        const bool in = c2 < c1;
        double Tl = in ? T[c2] : 0.0, xl = in ? xs[c2] : 0.0;
        const double rl = in ? __drcp_rn(__ldg(a.D + f + c2)) : 1.0;  // 1 / d, off the column chain
        const int pl = in ? __ldg(S.perm + f + c2) : 0;  // loaded up front: off the column chain
        for (int cb = c1 - 1; cb >= c0; cb -= 8) {
          double pu[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int c = cb - u;
            pu[u] = (c >= c0 && c2 < c) ? __ldg(P + static_cast<int64_t>(c2) * nr + c) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int c = cb - u;
            if (c >= c0) {
              double v = 0.0;
              if (c2 == c) {
                v = xl * rl - Tl;
                xl = v;
                a.x[pl] = v;
              }
              v = __shfl_sync(kFull, v, c - c0);
              if (c2 < c) Tl += pu[u] * v;
            }
          }
        }
        if (in) {
          xs[c2] = xl;
          T[c2] = Tl;
        }
      }
      __syncthreads();
      for (int c2 = tid; c2 < c0; c2 += NT) {
        double acc = 0.0;
        const double* Pc2 = P + static_cast<int64_t>(c2) * nr;
        for (int c = c0; c < c1; ++c) acc += Pc2[c] * xs[c];
        T[c2] += acc;
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    __threadfence();
    st_release(a.flags + s, a.epoch);
  }
}

// per warp: VS[32] + stack[kGrpStack] (forward groups)
constexpr int kSolWarp = 32 + kGrpStack;  // doubles

template <int NT>
__global__ void __launch_bounds__(NT == 32 ? 128 : NT, NT == 32 ? NCL_SK32_MINB : 4) fwd_kernel(SolveArgs a) {
  __shared__ int s_ticket;
  extern __shared__ double s_sol[];
  const int tid = NT == 32 ? (threadIdx.x & 31) : threadIdx.x;
  Claim<NT> cl;
  const int tail = a.t1 - static_cast<int>(gridDim.x) * (NT == 32 ? 4 : 1);
  for (;;) {
    const int t = cl.next(a.ticket, a.t0, a.t1, a.nleaf, tid, &s_ticket);
    if (tid == 0 && (t < 0 || t >= tail)) pdl_trigger();
    if (t < 0) break;
    if (a.trace && tid == 0) a.trace[2 * t] = gtimer();
    if (NT == 32 && a.prog && t < a.nleaf) {
      double* VS = s_sol + (threadIdx.x >> 5) * kSolWarp;
      fwd_group(a, t, tid, VS, VS + 32);
    } else {
      for (int k = __ldg(a.tptr + t); k < __ldg(a.tptr + t + 1); ++k) fwd_task<NT>(a, __ldg(a.tasks + k), tid);
    }
    if (a.trace && tid == 0) a.trace[2 * t + 1] = gtimer();
  }
}

// GPU-wide forward gather of the last CTA task's contribution vectors (the
// separator root: one row per warp-quad across many CTAs instead of one
// CTA), the same per-row arithmetic as heavy_cv_rows inside fwd_task; the
// root's own task then skips its gather (SolveArgs::pregathered).
__global__ void __launch_bounds__(256) fwd_root_gather(SolveArgs a, int s) {
  const DevSymb& S = a.S;
  for (int q = __ldg(S.cptr + s) + threadIdx.x; q < __ldg(S.cptr + s + 1); q += blockDim.x)
    wait_flag(a.flags + __ldg(S.child + q), a.epoch);
  __syncthreads();
  const int f = __ldg(S.sn_first + s), w = __ldg(S.sn_first + s + 1) - f;
  const int nr = static_cast<int>(__ldg(S.sn_rptr + s + 1) - __ldg(S.sn_rptr + s));
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), nwg = gridDim.x * (blockDim.x >> 5);
  heavy_cv_rows(a, s, f, w, nr, __ldg(S.cv_ptr + s), 4 * gw, 4 * nwg, threadIdx.x & 31);
}

// tickets in reverse order (roots first); no leaf chunking
template <int NT>
__global__ void __launch_bounds__(NT == 32 ? 128 : NT, NT == 32 ? NCL_SK32_MINB : 4) bwd_kernel(SolveArgs a) {
  __shared__ int s_ticket;
  extern __shared__ double s_sol[];
  const int tid = NT == 32 ? (threadIdx.x & 31) : threadIdx.x;
  for (;;) {
    int t;
    if constexpr (NT == 32) {
      t = 0;
      if (tid == 0) t = atomicAdd(a.ticket, 1);
      t = __shfl_sync(kFull, t, 0);
    } else {
      __syncthreads();
      if (tid == 0) s_ticket = atomicAdd(a.ticket, 1);
      __syncthreads();
      t = s_ticket;
    }
    const int k = a.t1 - 1 - t;
    if (tid == 0 && k < a.t0 + static_cast<int>(gridDim.x) * (NT == 32 ? 4 : 1)) pdl_trigger();
    if (k < a.t0) break;
    if (a.trace && tid == 0) a.trace[2 * k] = gtimer();
    if (NT == 32 && a.prog && k < a.nleaf) {
      double* VS = s_sol + (threadIdx.x >> 5) * kSolWarp;
      bwd_group(a, k, tid);
    } else {
      for (int j = __ldg(a.tptr + k + 1) - 1; j >= __ldg(a.tptr + k); --j) bwd_task<NT>(a, __ldg(a.tasks + j), tid);
    }
    if (a.trace && tid == 0) a.trace[2 * k + 1] = gtimer();
  }
}

// ---------------------------------------------------------------------------
// Register-resident solves of the batched tiny-front forest (BatchSched, the
// same forest reg_factor_kernel factors): one thread per front of a
// compile-time shape (NR rows, W pivots). Forward, in the factor's chunk
// order (children first): b through the permutation, the children's
// contribution vectors extend-added in ascending child order (relative rows
// from relp, every load of a child issued together), the unit-lower solve of
// the W columns, x1 to xp and -L21 x1 to the front's CV. Backward, chunks in
// reverse order (parents first): the ancestor values gathered through the
// row list, T = L21^T x2, then the unit-upper block with D^{-1} fused and the
// result scattered through the permutation. Same operations, in the same
// order, as fwd_group / bwd_warp_reg do for a node.
// ---------------------------------------------------------------------------
template <int NR, int W>
__device__ __forceinline__ void reg_fwd_front(const SolveArgs& a, const RegInst& I, const int* __restrict__ cid,
                                              const uint32_t* __restrict__ smap) {
  const DevSymb& S = a.S;
  static_assert(NR <= 4 * kSmapWords, "solve row map words");
  constexpr int NW = (NR + 3) / 4;
  // everything that does not depend on the children's results first: the
  // panel, b through the permutation, the first four children's CV offsets
  // and row maps — after the flags only the CV loads remain
  const int64_t rb = __ldg(S.sn_rptr + I.s);
  double P[W][NR];
  const double* Pg = a.L + I.loff;
#pragma unroll
  for (int c = 0; c < W; ++c)
#pragma unroll
    for (int i = c + 1; i < NR; ++i) P[c][i] = __ldg(Pg + c * NR + i);
  double v[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) v[i] = i < W ? __ldcg(a.b + __ldg(S.perm + I.f + i)) : 0.0;
  int rel[4];
  uint32_t mw[4][NW];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    rel[q] = q < I.nch ? static_cast<int>(__ldg(smap + (q * kSmapStride + kSmapWords) * 32)) : 0;
#pragma unroll
    for (int w4 = 0; w4 < NW; ++w4) mw[q][w4] = q < I.nch ? __ldg(smap + (q * kSmapStride + w4) * 32) : 0xffffffffu;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (q < I.nch) wait_flag(a.flags + I.cid[q], a.epoch);
  for (int q = 4; q < I.nch; ++q) wait_flag(a.flags + __ldg(cid + I.ccb + q), a.epoch);
  // per parent row (constant index) the child's CV entry or none: v stays in
  // registers; children in ascending order (the extend-add order)
#pragma unroll
  for (int q = 0; q < 4; ++q) {
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const uint32_t k = (mw[q][i >> 2] >> (8 * (i & 3))) & 0xffu;
      if (k != 0xffu) v[i] += __ldcg(a.CV + rel[q] + k);
    }
  }
  for (int q = 4; q < I.nch; ++q) {
    const int rq = static_cast<int>(__ldg(smap + (q * kSmapStride + kSmapWords) * 32));
    uint32_t m[NW];
#pragma unroll
    for (int w4 = 0; w4 < NW; ++w4) m[w4] = __ldg(smap + (q * kSmapStride + w4) * 32);
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const uint32_t k = (m[i >> 2] >> (8 * (i & 3))) & 0xffu;
      if (k != 0xffu) v[i] += __ldcg(a.CV + rq + k);
    }
  }
#pragma unroll
  for (int c = 0; c < W; ++c) {
    const double xc = v[c];
#pragma unroll
    for (int i = c + 1; i < NR; ++i) v[i] -= P[c][i] * xc;
  }
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    if (i < W) a.xp[I.f + i] = v[i];
    else a.CV[rb + i] = v[i];
  }
  st_release(a.flags + I.s, a.epoch);  // release: orders this thread's writes
}

template <int NR, int W>
__device__ __forceinline__ void reg_bwd_front(const SolveArgs& a, const RegInst& I) {
  const DevSymb& S = a.S;
  const int ps = __ldg(S.sn_parent + I.s);
  const int64_t rb = __ldg(S.sn_rptr + I.s);
  int ri[NR];
  double P[W][NR], d[W], xs[W];
  int pl[W];
  const double* Pg = a.L + I.loff;
#pragma unroll
  for (int i = W; i < NR; ++i) ri[i] = __ldg(S.rows + rb + i);
#pragma unroll
  for (int c = 0; c < W; ++c) {
#pragma unroll
    for (int i = 0; i < NR; ++i) P[c][i] = (i > c) ? __ldg(Pg + c * NR + i) : 0.0;
    d[c] = __drcp_rn(__ldg(a.D + I.f + c));  // 1 / d, before the parent wait
    pl[c] = __ldg(S.perm + I.f + c);
    xs[c] = __ldcg(a.xp + I.f + c);
  }
  // the parent may still be running: a register front, or (the launch
  // overlaps the warp phase's tail) a group member / warp single
  if (ps >= 0) wait_flag(a.flags + ps, a.epoch);
  double xi[NR];
#pragma unroll
  for (int i = W; i < NR; ++i) xi[i] = __ldcg(a.xp + ri[i]);
  double T[W];
#pragma unroll
  for (int c = 0; c < W; ++c) {
    double acc = 0.0;
#pragma unroll
    for (int i = W; i < NR; ++i) acc += P[c][i] * xi[i];
    T[c] = acc;
  }
#pragma unroll
  for (int c = W - 1; c >= 0; --c) {
    const double vv = xs[c] * d[c] - T[c];
    a.xp[I.f + c] = vv;
    a.x[pl[c]] = vv;
#pragma unroll
    for (int c2 = 0; c2 < c; ++c2) T[c2] += P[c2][c] * vv;
  }
  st_release(a.flags + I.s, a.epoch);
}

template <bool FWD, int... K>
__device__ __forceinline__ void reg_solve_dispatch(const SolveArgs& a, const RegChunk& ch, int lane,
                                                   const RegInst* __restrict__ inst, const int* cid,
                                                   const uint32_t* smapw, std::integer_sequence<int, K...>) {
  (((ch.shape == K) ? [&] {
    constexpr int NR = kRegShapes[K][0], W = kRegShapes[K][1];
    if (lane < ch.n) {
      const RegInst I = inst[ch.first + lane];
      if constexpr (FWD) reg_fwd_front<NR, W>(a, I, cid, smapw + ch.smap + lane);
      else reg_bwd_front<NR, W>(a, I);
    }
  }()
                    : void()),
   ...);
}

template <bool FWD>
__global__ void __launch_bounds__(128) reg_solve_kernel(SolveArgs a, const RegInst* __restrict__ inst,
                                                        const RegChunk* __restrict__ chunks, int nchunk,
                                                        const int* __restrict__ cid,
                                                        const uint32_t* __restrict__ smapw) {
  const int lane = threadIdx.x & 31;
  const int tail = nchunk - static_cast<int>(gridDim.x) * 4;
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(a.ticket, 1);
    c = __shfl_sync(kFull, c, 0);
    if (lane == 0 && c >= tail) pdl_trigger();
    if (c >= nchunk) break;
    const RegChunk ch = chunks[FWD ? c : nchunk - 1 - c];
    reg_solve_dispatch<FWD>(a, ch, lane, inst, cid, smapw, std::make_integer_sequence<int, kNumRegShapes>{});
  }
}

// SpMV in the reference accumulation order (sparse_sym.cpp:105-115), no FMA.
__global__ void spmv_kernel(int n, const int64_t* __restrict__ ptr, const int* __restrict__ vi,
                            const int* __restrict__ ci, const double* __restrict__ v, const double* __restrict__ x,
                            double* __restrict__ y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p) acc = __dadd_rn(acc, __dmul_rn(v[vi[p]], x[ci[p]]));
    y[i] = acc;
  }
}

__global__ void residual_kernel(int n, const int64_t* __restrict__ ptr, const int* __restrict__ vi,
                                const int* __restrict__ ci, const double* __restrict__ v,
                                const double* __restrict__ b, const double* __restrict__ x, double* __restrict__ r,
                                double* out) {
  double m = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p) acc = __dadd_rn(acc, __dmul_rn(v[vi[p]], x[ci[p]]));
    const double ri = __dsub_rn(b[i], acc);
    r[i] = ri;
    m = fmax(m, fabs(ri));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, m);
}

__global__ void absmax_kernel(const double* __restrict__ v, int64_t n, double* out) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(v[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, m);
}

__global__ void axpy_kernel(double* __restrict__ x, const double* __restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = __dadd_rn(x[i], d[i]);
}

// row sums of |M| in the reference order (sparse_sym.cpp:79-92), then max
__global__ void rowsum_kernel(int n, const int64_t* __restrict__ ptr, const int* __restrict__ vi,
                              const double* __restrict__ v, double* out) {
  double m = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p) acc = __dadd_rn(acc, fabs(v[vi[p]]));
    m = fmax(m, acc);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, m);
}

// Frobenius norm squared: one CTA, each thread strides over columns and sums
// sequentially, then a fixed shared-memory tree (deterministic).
__global__ void frob_kernel(int n, const int* __restrict__ cp, const int* __restrict__ ri,
                            const double* __restrict__ v, double* out) {
  __shared__ double sh[1024];
  double acc = 0.0;
  for (int c = threadIdx.x; c < n; c += blockDim.x)
    for (int p = cp[c]; p < cp[c + 1]; ++p) {
      const double x = v[p] * v[p];
      acc += (ri[p] == c) ? x : 2.0 * x;
    }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sh[0];
}

int g_num_sms = 0;
#define COUNT(n) (g_kernel_launches += (n))
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}


int grid_for(int64_t n, int block) {
  const int64_t g = (n + block - 1) / block;
  const int cap = num_sms() * 8;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

int64_t g_kernel_launches = 0;

void dev_max_abs_diag(const DevPattern& P, const double* kvals, double* out, cudaStream_t st) {
  cudaMemsetAsync(out, 0, sizeof(double), st);
  if (P.ndiag > 0)
    COUNT(1), maxdiag_kernel<<<std::min(grid_for(P.ndiag, 256), 8 * num_sms()), 256, 0, st>>>(P.diag_pos, P.ndiag, kvals, out);
}

template <class K>
int persistent_grid(K fn, int threads, int ntasks, int smem = 0) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
  if (per_sm <= 0) per_sm = 1;
  const int g = num_sms() * per_sm;
  return std::max(1, std::min(g, ntasks));
}

unsigned long long* g_task_trace = nullptr;  // NCL_TASK_TRACE debugging
static unsigned long long* g_solve_trace = nullptr;  // NCL_SOLVE_TRACE debugging
constexpr int kSolSmem = 4 * kSolWarp * sizeof(double);
static int g_fg = 0, g_fg2 = 0, g_fg3 = 0, g_sf = 0, g_sf2 = 0, g_sb = 0, g_sb2 = 0;
constexpr int kFacSmem1 = 4 * (kGrpFront * (kGrpFront + 1) / 2 + kGrpStack) * sizeof(double);
constexpr int kFacSmem2 = kCtaFront * (kCtaFront + 1) / 2 * sizeof(double);  // packed lower front
constexpr int kFacSmem3 = kCtaFrontS * (kCtaFrontS + 1) / 2 * sizeof(double);  // small-CTA segments
// NCL_NO_PDL=1: plain stream-ordered launches (A/B)
static const bool g_pdl = std::getenv("NCL_NO_PDL") == nullptr;
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*k)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, Args&&... args) {
  if (!g_pdl) {
    k<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

static void init_grids() {
  if (g_fg) return;
  cudaFuncSetAttribute(factor_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFacSmem1);
  cudaFuncSetAttribute(factor_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFacSmem2);
  g_fg = persistent_grid(factor_kernel<32>, 128, 1 << 30, kFacSmem1);
  g_fg2 = persistent_grid(factor_kernel<256>, 256, 1 << 30, kFacSmem2);
  cudaFuncSetAttribute(factor_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFacSmem3);
  g_fg3 = persistent_grid(factor_kernel<128>, 128, 1 << 30, kFacSmem3);
  cudaFuncSetAttribute(fwd_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSolSmem);
  cudaFuncSetAttribute(bwd_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSolSmem);
  g_sf = persistent_grid(fwd_kernel<32>, 128, 1 << 30, kSolSmem);
  g_sf2 = persistent_grid(fwd_kernel<256>, 256, 1 << 30);
  g_sb = persistent_grid(bwd_kernel<32>, 128, 1 << 30, kSolSmem);
  g_sb2 = persistent_grid(bwd_kernel<256>, 256, 1 << 30);
}

void dev_big_cta(const DevSymb& S, DevFactor& F, const BigDesc* d, int nf, cudaStream_t st) {
  static int set = 0, nt = 256;
  if (!set) {
    // NCL_ROOT_NT=512|1024 (A/B): threads of the one-CTA heavy fronts (the root)
    const char* e = std::getenv("NCL_ROOT_NT");
    nt = e ? std::atoi(e) : 256;
    cudaFuncSetAttribute(big_cta_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFacSmem2);
    cudaFuncSetAttribute(big_cta_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFacSmem2);
    cudaFuncSetAttribute(big_cta_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFacSmem2);
    set = 1;
  }
  if (nt == 1024) big_cta_kernel<1024><<<nf, 1024, kFacSmem2, st>>>(S, d, F.bigF, F.L, F.CB, F.D, F.scal, F.istat);
  else if (nt == 512) big_cta_kernel<512><<<nf, 512, kFacSmem2, st>>>(S, d, F.bigF, F.L, F.CB, F.D, F.scal, F.istat);
  else big_cta_kernel<256><<<nf, 256, kFacSmem2, st>>>(S, d, F.bigF, F.L, F.CB, F.D, F.scal, F.istat);
  COUNT(1);
}

void dev_factor_begin(const DevSymb& S0, const DevPattern& P, DevFactor& F, const double* kvals, double pivot_tol,
                      cudaStream_t st) {
  DevSymb& S = const_cast<DevSymb&>(S0);
  init_grids();
  dev_max_abs_diag(P, kvals, F.scal + 1, st);
  COUNT(1);
  thresh_kernel<<<1, 1, 0, st>>>(F.scal, pivot_tol, F.istat, S.n);
  S.epoch++;
  cudaMemsetAsync(S.tickets, 0, kTickets * sizeof(int), st);
}

// NCL_FACTOR_PHASES=1: CUDA events around the phases of every factorization
// (batched subtrees | warp tasks | CTA segments), averaged and printed to stderr at
// exit (debug timeline; synchronises the stream once per factorization)
namespace {
struct PhaseTimer {
  bool on = std::getenv("NCL_FACTOR_PHASES") != nullptr;
  cudaEvent_t ev[4]{};
  double acc[3]{};
  int n = 0;
  void mark(int k, cudaStream_t st) {
    if (!on) return;
    if (!ev[k]) cudaEventCreate(&ev[k]);
    cudaEventRecord(ev[k], st);
    if (k == 3) {
      cudaEventSynchronize(ev[3]);
      for (int i = 0; i < 3; ++i) {
        float ms = 0;
        cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
        acc[i] += ms;
      }
      ++n;
    }
  }
  ~PhaseTimer() {
    if (on && n)
      std::fprintf(stderr, "[ncl] factor phases over %d runs (ms): batch %.4f  warp %.4f  cta %.4f\n", n, acc[0] / n,
                   acc[1] / n, acc[2] / n);
  }
} g_ptimer;
}  // namespace

void dev_factor_list(const DevSymb& S, DevFactor& F, const double* kvals, const DevTasks& T, int slot,
                     cudaStream_t st) {
  if (T.n == 0) return;
  g_ptimer.mark(0, st);
  FactorArgs a{S, F.L, F.CB, F.D, kvals, F.scal, F.istat, S.flags, S.tickets + 2 * slot, S.epoch, 0, T.split,
               T.ids, T.tptr, T.prog, T.gpo, T.nleaf, 0, g_task_trace};
  if (T.batch) {
    const BatchSched& bs = *T.batch;
    static int grid1 = 0, grid2 = 0;
    if (!grid1) {
      grid1 = persistent_grid(reg_factor_kernel<0, kRegTier1>, 128, 1 << 30);
      grid2 = persistent_grid(reg_factor_kernel<kRegTier1, kNumRegShapes>, 128, 1 << 30);
    }
    const int n1 = bs.nchunk1, n2 = static_cast<int>(bs.chunks.size()) - bs.nchunk1;
    FactorArgs ra = a;
    if (n1 > 0) {
      ra.ticket = S.tickets + kTicketRegFac1;
      cudaMemsetAsync(ra.ticket, 0, sizeof(int), st);
      COUNT(1);
      reg_factor_kernel<0, kRegTier1><<<std::min(grid1, (n1 + 3) / 4), 128, 0, st>>>(
          ra, bs.dev_inst, bs.dev_chunks, n1, bs.dev_amap, bs.dev_cmap, bs.dev_cmapw, bs.dev_ccb, bs.dev_cid);
    }
    if (n2 > 0) {
      ra.ticket = S.tickets + kTicketRegFac2;
      cudaMemsetAsync(ra.ticket, 0, sizeof(int), st);
      COUNT(1);
      reg_factor_kernel<kRegTier1, kNumRegShapes><<<std::min(grid2, (n2 + 3) / 4), 128, 0, st>>>(
          ra, bs.dev_inst, bs.dev_chunks + n1, n2, bs.dev_amap, bs.dev_cmap, bs.dev_cmapw, bs.dev_ccb, bs.dev_cid);
    }
  }
  g_ptimer.mark(1, st);
  if (T.split > 0 && T.tptr) {
    COUNT(1);
    // groups wait on their external (register-front) children's flags, so
    // the warp phase may overlap the register phase's tail
    launch_pdl(factor_kernel<32>, g_fg, 128, kFacSmem1, st, a);
  }
  g_ptimer.mark(2, st);
  if (T.top && (T.top->any_big || T.top->any_small)) {
    // segment by segment (merged levels): the segment's fronts in one
    // persistent launch (128-thread CTAs when they all fit kCtaFrontS rows),
    // then its large fronts on the multi-CTA path
    const TopSched& ts = *T.top;
    a.skip_big = 1;
    a.nleaf = 0;
    for (size_t L = 0; L < ts.lvl_begin.size(); ++L) {
      const int b = ts.lvl_begin[L], e = ts.lvl_end[L];
      const int nsmall = (e - b) - static_cast<int>(ts.big[L].size());
      if (nsmall > 0) {
        // unsharded: a pre-zeroed ticket per segment and a programmatic
        // dependent launch (every segment task waits on its children's
        // flags); sharded phases reuse one ticket
        const bool pdl = slot == 0 && kTicketSeg0 + static_cast<int>(L) < kTicketRegBwd0;
        if (pdl) {
          a.ticket = S.tickets + kTicketSeg0 + L;
        } else {
          cudaMemsetAsync(S.tickets + kTicketShardSeg, 0, sizeof(int), st);
          a.ticket = S.tickets + kTicketShardSeg;
        }
        a.t0 = b;
        a.t1 = e;
        COUNT(1);
        if (pdl) {
          if (ts.small[L]) launch_pdl(factor_kernel<128>, std::min(g_fg3, e - b), 128, kFacSmem3, st, a);
          else launch_pdl(factor_kernel<256>, std::min(g_fg2, e - b), 256, kFacSmem2, st, a);
        } else {
          if (ts.small[L]) factor_kernel<128><<<std::min(g_fg3, e - b), 128, kFacSmem3, st>>>(a);
          else factor_kernel<256><<<std::min(g_fg2, e - b), 256, kFacSmem2, st>>>(a);
        }
      }
      if (!ts.big[L].empty()) dev_factor_big_batch(S, F, kvals, ts.big[L], ts.big_dev[L], st);
    }
    g_ptimer.mark(3, st);
    return;
  }
  if (T.split < T.n) {
    a.ticket = S.tickets + 2 * slot + 1;
    a.t0 = T.split;
    a.t1 = T.n;
    COUNT(1);
    factor_kernel<256><<<std::min(g_fg2, T.n - T.split), 256, kFacSmem2, st>>>(a);
  }
  g_ptimer.mark(3, st);
}

// NCL_TASK_TRACE: per-supernode phase stamps of the CTA smem path
// (after the wait, after the assembly, after the dense factor, after publish)
void dev_phase_trace(unsigned long long* buf) { cudaMemcpyToSymbol(g_phase, &buf, sizeof(buf)); }

void dev_factor(const DevSymb& S, const DevPattern& P, DevFactor& F, const double* kvals, double pivot_tol,
                cudaStream_t st, const TopSched* top) {
  dev_factor_begin(S, P, F, kvals, pivot_tol, st);
  // NCL_NO_BATCH=1: the layout without batched subtrees (A/B timing only)
  static const bool no_batch = std::getenv("NCL_NO_BATCH") != nullptr;
  DevTasks T = no_batch ? S.tasks : S.ftasks;
  if (top) T.top = top;
  dev_factor_list(S, F, kvals, T, 0, st);
}

void dev_inertia(const DevSymb& S, DevFactor& F, cudaStream_t st, const uint8_t* report) {
  COUNT(1);
  inertia_kernel<<<std::min(grid_for(S.n, 256), 8 * num_sms()), 256, 0, st>>>(F.D, S.n, F.scal, F.istat, report);
}

void dev_solve_begin(const DevSymb& S0, cudaStream_t st) {
  DevSymb& S = const_cast<DevSymb&>(S0);
  init_grids();
  S.epoch++;
  cudaMemsetAsync(S.tickets, 0, kTickets * sizeof(int), st);
}

// the batched forest of a task list (one launch; its chunks, children first)
static void reg_solve(const DevSymb& S, const BatchSched& bs, SolveArgs a, bool fwd, int slot, cudaStream_t st) {
  static int grid = 0;
  if (!grid) grid = persistent_grid(reg_solve_kernel<true>, 128, 1 << 30);
  const int n = static_cast<int>(bs.chunks.size());
  if (n == 0) return;
  if (fwd) {
    a.ticket = S.tickets + kTicketRegFwd;
    cudaMemsetAsync(a.ticket, 0, sizeof(int), st);
  } else {  // zeroed by dev_solve_begin: no memset between it and the warp phase (PDL)
    a.ticket = S.tickets + kTicketRegBwd0 + slot;
  }
  COUNT(1);
  if (fwd)
    reg_solve_kernel<true><<<std::min(grid, (n + 3) / 4), 128, 0, st>>>(a, bs.dev_inst, bs.dev_chunks, n, bs.dev_cid,
                                                                       bs.dev_smapw);
  else  // every front waits on its parent's flag: may overlap the warp phase's tail
    launch_pdl(reg_solve_kernel<false>, std::min(grid, (n + 3) / 4), 128, 0, st, a, bs.dev_inst, bs.dev_chunks, n,
               bs.dev_cid, bs.dev_smapw);
}

void dev_solve_fwd_list(const DevSymb& S, DevFactor& F, const double* b, const DevTasks& T, int slot,
                        cudaStream_t st) {
  if (T.n == 0 && !T.batch) return;
  SolveArgs fa{S, F.L, F.D, F.CV, F.xp, b, nullptr, S.flags + S.nsn, S.tickets + 2 * slot, S.epoch, 0, T.split,
               T.ids, T.tptr, T.prog, T.gpo, T.nleaf, g_solve_trace};
  if (T.batch) reg_solve(S, *T.batch, fa, true, slot, st);
  if (T.split > 0) COUNT(1), launch_pdl(fwd_kernel<32>, g_sf, 128, kSolSmem, st, fa);
  if (T.split < T.n) {
    fa.ticket = S.tickets + 2 * slot + 1;
    fa.t0 = T.split;
    fa.t1 = T.n;
    // the last task (the separator root) gathers its many children's CVs
    // GPU-wide in its own launch, then runs its triangular part
    const int root = T.root_heavy;
    if (root >= 0 && T.n - T.split > 1) fa.t1 = T.n - 1;
    COUNT(1);
    launch_pdl(fwd_kernel<256>, std::min(g_sf2, fa.t1 - fa.t0), 256, 0, st, fa);  // CTA tasks wait on children
    if (root >= 0 && T.n - T.split > 1) {
      const int nr = T.root_nr;
      COUNT(2);
      launch_pdl(fwd_root_gather, std::max(1, std::min(2 * num_sms(), (nr + 31) / 32)), 256, 0, st, fa, root);
      fa.pregathered = root;
      fa.ticket = S.tickets + kTicketRoot;
      cudaMemsetAsync(fa.ticket, 0, sizeof(int), st);
      fa.t0 = T.n - 1;
      fa.t1 = T.n;
      fwd_kernel<256><<<1, 256, 0, st>>>(fa);
    }
  }
}

// backward over one list, roots first (the CTA part first, then the warp part)
void dev_solve_bwd_list(const DevSymb& S, DevFactor& F, double* x, const DevTasks& T, int slot, cudaStream_t st) {
  if (T.n == 0 && !T.batch) return;
  SolveArgs ba{S, F.L, F.D, F.CV, F.xp, nullptr, x, S.flags + 2 * S.nsn, S.tickets + 2 * slot, S.epoch, T.split,
               T.n, T.ids, T.tptr, T.prog, T.gpo, T.nleaf, g_solve_trace ? g_solve_trace + 2 * T.n : nullptr};

  if (T.split < T.n) COUNT(1), bwd_kernel<256><<<std::min(g_sb2, T.n - T.split), 256, 0, st>>>(ba);
  if (T.split > 0) {
    ba.ticket = S.tickets + 2 * slot + 1;
    ba.t0 = 0;
    ba.t1 = T.split;
    COUNT(1);
    launch_pdl(bwd_kernel<32>, g_sb, 128, kSolSmem, st, ba);  // every warp task waits on its parent
  }
  // the batched forest last: every parent is in this list or earlier
  if (T.batch) reg_solve(S, *T.batch, ba, false, slot, st);
}

void dev_solve(const DevSymb& S, DevFactor& F, const double* b, double* x, cudaStream_t st) {
  if (S.n == 0) return;
  // NCL_SOLVE_TRACE=<file>: per-task globaltimer start/end of the 3rd solve
  // (forward then backward, 4 x tasks uint64; debug timeline)
  static const char* trace_path = std::getenv("NCL_SOLVE_TRACE");
  // NCL_SOLVE_NO_BATCH=1: the layout without the register-front forest (A/B timing only)
  static const bool no_batch = std::getenv("NCL_SOLVE_NO_BATCH") != nullptr;
  const DevTasks& T = no_batch ? S.tasks : S.ftasks;
  static int traced = 0;
  const bool tr = trace_path && traced++ == 2;
  if (tr) {
    cudaMalloc(&g_solve_trace, 4 * sizeof(unsigned long long) * T.n);
    cudaMemsetAsync(g_solve_trace, 0, 4 * sizeof(unsigned long long) * T.n, st);
  }
  dev_solve_begin(S, st);
  dev_solve_fwd_list(S, F, b, T, 0, st);
  dev_solve_bwd_list(S, F, x, T, 2, st);
  if (tr) {
    std::vector<unsigned long long> h(4 * static_cast<size_t>(T.n));
    cudaMemcpyAsync(h.data(), g_solve_trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaFree(g_solve_trace);
    g_solve_trace = nullptr;
    if (FILE* fp = std::fopen(trace_path, "wb")) {
      const int hdr[4] = {T.n, T.nleaf, T.split, 0};
      std::fwrite(hdr, sizeof(int), 4, fp);
      std::fwrite(h.data(), sizeof(unsigned long long), h.size(), fp);
      std::fclose(fp);
    }
  }
}

void dev_spmv(const DevPattern& P, const double* kvals, const double* x, double* y, cudaStream_t st) {
  if (P.n > 0) COUNT(1), spmv_kernel<<<grid_for(P.n, 256), 256, 0, st>>>(P.n, P.mv_ptr, P.mv_val, P.mv_col, kvals, x, y);
}

void dev_residual(const DevPattern& P, const double* kvals, const double* b, const double* x, double* r,
                  double* out_max, cudaStream_t st) {
  cudaMemsetAsync(out_max, 0, sizeof(double), st);
  if (P.n > 0)
    COUNT(1), residual_kernel<<<grid_for(P.n, 256), 256, 0, st>>>(P.n, P.mv_ptr, P.mv_val, P.mv_col, kvals, b, x, r, out_max);
}

void dev_absmax(const double* v, int64_t n, double* out, cudaStream_t st) {
  COUNT(1);
  absmax_kernel<<<grid_for(n, 256), 256, 0, st>>>(v, n, out);
}

void dev_axpy_inplace(double* x, const double* d, int64_t n, cudaStream_t st) {
  COUNT(1);
  axpy_kernel<<<grid_for(n, 256), 256, 0, st>>>(x, d, n);
}

void dev_rowsum_max(const DevPattern& P, const double* kvals, double* out, cudaStream_t st) {
  cudaMemsetAsync(out, 0, sizeof(double), st);
  if (P.n > 0) COUNT(1), rowsum_kernel<<<grid_for(P.n, 256), 256, 0, st>>>(P.n, P.mv_ptr, P.mv_val, kvals, out);
}

void dev_frob_sq(const DevPattern& P, const int* colptr, const int* rowind, const double* kvals, double* out,
                 cudaStream_t st) {
  COUNT(1);
  frob_kernel<<<1, 1024, 0, st>>>(P.n, colptr, rowind, kvals, out);
}

int dev_num_sms() { return num_sms(); }

}  // namespace nclb
