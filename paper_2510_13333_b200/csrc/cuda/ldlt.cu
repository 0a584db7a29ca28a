// K3 numeric LDLᵀ, K4 triangular solves, K5 SpMV / residual, K6 norms.
//
// Replaces the reference's sequential up-looking factorization
// (/root/reference/proj/src/sparse_sym.cpp:268-337), solve_in_place (:346-363)
// and SparseSym::multiply/max_abs_diag/norm_inf (:69-115).
//
// Factorization: supernodal LEFT-looking LDLᵀ, 1x1 pivots in the fixed
// symbolic order, no pivoting. One warp owns one supernode panel and gathers
// every descendant update into it in a fixed order (so results are
// deterministic run to run — SPEC.md:69), then factors its dense diagonal
// block and scales the off-diagonal rows. Scheduling is a single persistent
// launch: tasks come from one ticket counter in leaves-first height order
// (leaves in chunks), and each inner task waits on its children's epoch
// flags (release/acquire at gpu scope). Deadlock freedom: the minimum
// outstanding ticket only depends on smaller tickets held by running warps.
#include <cuda_runtime.h>

#include <cstdint>

#include "dev.hpp"

namespace nclb {

namespace {

constexpr int kWarps = 4;          // warps per CTA of the persistent kernels
constexpr int kRelCap = 256;       // cached relative indices per warp
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void wait_flag(const int* f, int epoch) {
  while (ld_acquire(f) != epoch) __nanosleep(32);
}

__device__ __forceinline__ int lower_bound_i(const int* __restrict__ a, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  // non-negative doubles order like their bit patterns
  atomicMax(reinterpret_cast<unsigned long long*>(addr), static_cast<unsigned long long>(__double_as_longlong(v)));
}

// Task queue: one ticket counter for the whole launch. Tickets below
// nleaf_chunks hand out chunks of kLeafChunk leaves (no dependencies); later
// tickets hand out single inner supernodes in leaves-first height order.
// Only running warps take tickets, so the minimum outstanding task always
// has all of its (smaller-ticket) dependencies finished or in progress by a
// running warp: no deadlock even if not every CTA is resident.
constexpr int kLeafChunk = 8;
struct TaskCursor {
  int cur = 0, end = 0;
};
__device__ __forceinline__ int next_task(TaskCursor& tc, int nleaf, int nsn, int* ticket, int lane) {
  if (tc.cur < tc.end) return tc.cur++;
  int t = 0;
  if (lane == 0) t = atomicAdd(ticket, 1);
  t = __shfl_sync(kFull, t, 0);
  const int nchunks = (nleaf + kLeafChunk - 1) / kLeafChunk;
  if (t < nchunks) {
    tc.cur = t * kLeafChunk;
    tc.end = min(nleaf, tc.cur + kLeafChunk);
    return tc.cur++;
  }
  const int s = nleaf + (t - nchunks);
  return s < nsn ? s : -1;
}

struct FactorArgs {
  DevSymb S;
  double* L;
  double* D;
  const double* kvals;
  const double* thresh;
  int* zp;
  int* flags;
  int* ticket;
  int epoch;
};

__global__ void __launch_bounds__(kWarps * 32) factor_kernel(FactorArgs a) {
  __shared__ int s_rel[kWarps][kRelCap];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const DevSymb& S = a.S;
  const double thresh = __ldcg(a.thresh);
  TaskCursor tc;
  int* rel = s_rel[wib];
  for (;;) {
    const int t = next_task(tc, S.nleaf, S.nsn, a.ticket, lane);
    if (t < 0) break;
    const int s = __ldg(S.order + t);
    // wait for children (their subtrees are complete by induction)
    if (lane == 0)
      for (int q = __ldg(S.cptr + s); q < __ldg(S.cptr + s + 1); ++q) wait_flag(a.flags + __ldg(S.child + q), a.epoch);
    __syncwarp();
    const int f = __ldg(S.sn_first + s);
    const int w = __ldg(S.sn_first + s + 1) - f;
    const int64_t rb = __ldg(S.sn_rptr + s);
    const int nr = static_cast<int>(__ldg(S.sn_rptr + s + 1) - rb);
    const int* Rs = S.rows + rb;
    double* P = a.L + __ldg(S.sn_loff + s);
    // zero-fill and scatter A (each panel entry has at most one A entry)
    for (int i = lane; i < w * nr; i += 32) P[i] = 0.0;
    __syncwarp();
    for (int64_t e = __ldg(S.aptr + s) + lane; e < __ldg(S.aptr + s + 1); e += 32)
      P[__ldg(S.aoff + e)] = __ldg(a.kvals + __ldg(S.asrc + e));
    __syncwarp();
    // gather descendant updates in list order
    for (int64_t u = __ldg(S.uptr + s); u < __ldg(S.uptr + s + 1); ++u) {
      const int d = __ldg(S.upd + 3 * u), p0 = __ldg(S.upd + 3 * u + 1), p1 = __ldg(S.upd + 3 * u + 2);
      const int fd = __ldg(S.sn_first + d);
      const int wd = __ldg(S.sn_first + d + 1) - fd;
      const int64_t rbd = __ldg(S.sn_rptr + d);
      const int nd = static_cast<int>(__ldg(S.sn_rptr + d + 1) - rbd);
      const int* Rd = S.rows + rbd;
      const double* Ld = a.L + __ldg(S.sn_loff + d);
      const double* Dd = a.D + fd;
      const int ntail = nd - p0;
      const bool cached = ntail <= kRelCap;
      if (cached) {
        for (int p = lane; p < ntail; p += 32) rel[p] = lower_bound_i(Rs, nr, __ldg(Rd + p0 + p));
      }
      __syncwarp();
      for (int q = p0; q < p1; ++q) {
        const int c = __ldg(Rd + q) - f;
        for (int p = q + lane; p < nd; p += 32) {
          double acc = 0.0;
          for (int k = 0; k < wd; ++k) {
            const double lqk = __ldcg(Ld + static_cast<int64_t>(k) * nd + q);
            const double dk = __ldcg(Dd + k);
            acc += __ldcg(Ld + static_cast<int64_t>(k) * nd + p) * (dk * lqk);
          }
          const int r = cached ? rel[p - p0] : lower_bound_i(Rs, nr, __ldg(Rd + p));
          P[static_cast<int64_t>(c) * nr + r] -= acc;
        }
      }
      __syncwarp();
    }
    // dense LDLᵀ of the panel (right-looking inside the supernode)
    for (int c = 0; c < w; ++c) {
      double* Pc = P + static_cast<int64_t>(c) * nr;
      const double dc = Pc[c];
      if (lane == 0) {
        a.D[f + c] = dc;
        if (fabs(dc) <= thresh) atomicMin(a.zp, f + c);
      }
      for (int i = c + 1 + lane; i < nr; i += 32) Pc[i] = Pc[i] / dc;
      __syncwarp();
      for (int c2 = c + 1; c2 < w; ++c2) {
        const double lc2 = Pc[c2] * dc;
        double* P2 = P + static_cast<int64_t>(c2) * nr;
        for (int i = c2 + lane; i < nr; i += 32) P2[i] -= Pc[i] * lc2;
      }
      __syncwarp();
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      st_release(a.flags + s, a.epoch);
    }
  }
}

__global__ void maxdiag_kernel(const int* __restrict__ pos, int nd, const double* __restrict__ v, double* out) {
  double m = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nd; i += gridDim.x * blockDim.x)
    m = fmax(m, fabs(v[pos[i]]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, m);
}

__global__ void thresh_kernel(double* scal, double tol, int* istat, int n) {
  // scal[1] = max|diag M| ; scal[0] = pivot_tol * max(1, maxdiag)  (sparse_sym.cpp:286)
  scal[0] = tol * fmax(1.0, scal[1]);
  istat[0] = n;  // no zero pivot yet
  istat[1] = istat[2] = istat[3] = 0;
}

__global__ void inertia_kernel(const double* __restrict__ D, int n, const double* scal, int* istat) {
  const double th = scal[0];
  int np = 0, nn = 0, nz = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double d = D[i];
    if (fabs(d) <= th) nz++;
    else if (d > 0.0) np++;
    else nn++;
  }
  for (int o = 16; o > 0; o >>= 1) {
    np += __shfl_xor_sync(kFull, np, o);
    nn += __shfl_xor_sync(kFull, nn, o);
    nz += __shfl_xor_sync(kFull, nz, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(istat + 1, np);
    atomicAdd(istat + 2, nn);
    atomicAdd(istat + 3, nz);
  }
}

// ---------------------------------------------------------------------------
// Solves: forward (with fused gather permutation), backward (with fused D⁻¹
// and scatter un-permutation). Same persistent schedule as the factor.
// ---------------------------------------------------------------------------
struct SolveArgs {
  DevSymb S;
  const double* L;
  const double* D;
  double* xp;
  const double* b;
  double* x;
  int* flags;
  int* ticket;
  int epoch;
};

__global__ void __launch_bounds__(kWarps * 32) fwd_kernel(SolveArgs a) {
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const DevSymb& S = a.S;
  TaskCursor tc;
  for (;;) {
    const int t = next_task(tc, S.nleaf, S.nsn, a.ticket, lane);
    if (t < 0) break;
    const int s = __ldg(S.order + t);
    if (lane == 0)
      for (int q = __ldg(S.cptr + s); q < __ldg(S.cptr + s + 1); ++q) wait_flag(a.flags + __ldg(S.child + q), a.epoch);
    __syncwarp();
    const int f = __ldg(S.sn_first + s);
    const int w = __ldg(S.sn_first + s + 1) - f;
    const int64_t rb = __ldg(S.sn_rptr + s);
    const int nr = static_cast<int>(__ldg(S.sn_rptr + s + 1) - rb);
    const double* P = a.L + __ldg(S.sn_loff + s);
    // gather b through the permutation (px[k] = b[perm[k]], sparse_sym.cpp:349)
    for (int c = lane; c < w; c += 32) a.xp[f + c] = __ldcg(a.b + __ldg(S.perm + f + c));
    __syncwarp();
    for (int64_t u = __ldg(S.uptr + s); u < __ldg(S.uptr + s + 1); ++u) {
      const int d = __ldg(S.upd + 3 * u), p0 = __ldg(S.upd + 3 * u + 1), p1 = __ldg(S.upd + 3 * u + 2);
      const int fd = __ldg(S.sn_first + d);
      const int wd = __ldg(S.sn_first + d + 1) - fd;
      const int64_t rbd = __ldg(S.sn_rptr + d);
      const int nd = static_cast<int>(__ldg(S.sn_rptr + d + 1) - rbd);
      const int* Rd = S.rows + rbd;
      const double* Ld = a.L + __ldg(S.sn_loff + d);
      for (int q = p0 + lane; q < p1; q += 32) {
        double acc = 0.0;
        for (int k = 0; k < wd; ++k) acc += __ldg(Ld + static_cast<int64_t>(k) * nd + q) * __ldcg(a.xp + fd + k);
        const int r = __ldg(Rd + q);
        a.xp[r] -= acc;
      }
      __syncwarp();
    }
    // unit-lower diagonal block
    for (int c = 0; c < w; ++c) {
      const double xc = a.xp[f + c];
      for (int c2 = c + 1 + lane; c2 < w; c2 += 32) a.xp[f + c2] -= P[static_cast<int64_t>(c) * nr + c2] * xc;
      __syncwarp();
    }
    if (lane == 0) {
      __threadfence();
      st_release(a.flags + s, a.epoch);
    }
  }
}

__global__ void __launch_bounds__(kWarps * 32) bwd_kernel(SolveArgs a) {
  const int lane = threadIdx.x & 31;
  const DevSymb& S = a.S;
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1);
    t = __shfl_sync(kFull, t, 0);
    if (t >= S.nsn) break;
    const int s = __ldg(S.order + (S.nsn - 1 - t));  // roots first
    const int ps = __ldg(S.sn_parent + s);
    if (lane == 0 && ps >= 0) wait_flag(a.flags + ps, a.epoch);
    __syncwarp();
    const int f = __ldg(S.sn_first + s);
    const int w = __ldg(S.sn_first + s + 1) - f;
    const int64_t rb = __ldg(S.sn_rptr + s);
    const int nr = static_cast<int>(__ldg(S.sn_rptr + s + 1) - rb);
    const int* Rs = S.rows + rb;
    const double* P = a.L + __ldg(S.sn_loff + s);
    for (int c = w - 1; c >= 0; --c) {
      const double* Pc = P + static_cast<int64_t>(c) * nr;
      double acc = 0.0;
      for (int i = c + 1 + lane; i < nr; i += 32) acc += Pc[i] * __ldcg(a.xp + __ldg(Rs + i));
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
      if (lane == 0) {
        const double v = a.xp[f + c] / __ldg(a.D + f + c) - acc;
        a.xp[f + c] = v;
        a.x[__ldg(S.perm + f + c)] = v;
      }
      __syncwarp();
    }
    if (lane == 0) {
      __threadfence();
      st_release(a.flags + s, a.epoch);
    }
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

int persistent_grid(const void* fn) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kWarps * 32, 0);
  if (per_sm <= 0) per_sm = 1;
  return num_sms() * per_sm;
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
  if (P.ndiag > 0) COUNT(1), maxdiag_kernel<<<grid_for(P.ndiag, 256), 256, 0, st>>>(P.diag_pos, P.ndiag, kvals, out);
}

void dev_factor(const DevSymb& S0, const DevPattern& P, DevFactor& F, const double* kvals, double pivot_tol,
                cudaStream_t st) {
  DevSymb& S = const_cast<DevSymb&>(S0);
  dev_max_abs_diag(P, kvals, F.scal + 1, st);
  COUNT(1);
  thresh_kernel<<<1, 1, 0, st>>>(F.scal, pivot_tol, F.istat, S.n);
  S.epoch++;
  cudaMemsetAsync(S.tickets, 0, 4 * sizeof(int), st);
  FactorArgs a{S, F.L, F.D, kvals, F.scal, F.istat, S.flags, S.tickets + 0, S.epoch};
  static int grid = 0;
  if (!grid) grid = persistent_grid(reinterpret_cast<const void*>(factor_kernel));
  if (S.nsn > 0) COUNT(1), factor_kernel<<<grid, kWarps * 32, 0, st>>>(a);
}

void dev_inertia(const DevSymb& S, DevFactor& F, cudaStream_t st) {
  COUNT(1);
  inertia_kernel<<<grid_for(S.n, 256), 256, 0, st>>>(F.D, S.n, F.scal, F.istat);
}

void dev_solve(const DevSymb& S0, DevFactor& F, const double* b, double* x, cudaStream_t st) {
  DevSymb& S = const_cast<DevSymb&>(S0);
  if (S.n == 0) return;
  S.epoch++;
  cudaMemsetAsync(S.tickets + 1, 0, 2 * sizeof(int), st);
  static int gf = 0, gb = 0;
  if (!gf) gf = persistent_grid(reinterpret_cast<const void*>(fwd_kernel));
  if (!gb) gb = persistent_grid(reinterpret_cast<const void*>(bwd_kernel));
  SolveArgs a{S, F.L, F.D, F.xp, b, x, S.flags + S.nsn, S.tickets + 1, S.epoch};
  COUNT(2);
  fwd_kernel<<<gf, kWarps * 32, 0, st>>>(a);
  SolveArgs bb{S, F.L, F.D, F.xp, b, x, S.flags + 2 * S.nsn, S.tickets + 2, S.epoch};
  bwd_kernel<<<gb, kWarps * 32, 0, st>>>(bb);
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
