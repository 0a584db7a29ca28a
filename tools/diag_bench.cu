// Micro-benchmark (debug tool, not part of the library): cycles of the CTA
// path's 8 x 8 diagonal-block chain (the shuffle form of cta_dense's
// diag_block, ldlt.cu) run by warp 0 while the other warps of the CTA are
// idle / issue DMMAs / shared-memory read-modify-writes / DFMAs — which
// shared resource slows the look-ahead chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/diag_bench.cu -o tools/diag_bench.bin
#include <cstdio>

constexpr unsigned kFull = 0xffffffffu;
constexpr int kPb = 8;

__device__ __forceinline__ void dmma(double& c0, double& c1, double av, double bv) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(av), "d"(bv));
}

__device__ __forceinline__ void diag_block(double* F, int ld, int lane, double* s_rd, double (*s_dl)[kPb], double* D) {
  const int kb = kPb;
  double x[kPb];
#pragma unroll
  for (int k = 0; k < kPb; ++k) x[k] = (k <= lane && lane < kb) ? F[k * ld + lane] : 0.0;
  double rk[kPb];
#pragma unroll
  for (int k = 0; k < kPb; ++k) {
    const double d = __shfl_sync(kFull, x[k], k);
    rk[k] = __drcp_rn(d);
    if (lane > k && lane < kb) x[k] *= rk[k];
    const double dlo = d * x[k];
#pragma unroll
    for (int k2 = k + 1; k2 < kPb; ++k2) {
      const double dl = __shfl_sync(kFull, dlo, k2);
      if (lane >= k2 && lane < kb) x[k2] -= x[k] * dl;
    }
  }
#pragma unroll
  for (int k = 0; k < kPb; ++k)
    if (k <= lane && lane < kb) F[k * ld + lane] = x[k];
#pragma unroll
  for (int k = 0; k < kPb; ++k) {
    const double dk = __shfl_sync(kFull, x[k], k);
    if (lane == k) s_rd[k] = rk[k];
    if (lane > k && lane < kb) s_dl[k][lane] = dk * x[k];
  }
  if (lane < kb) {
    double dk = 0.0;
#pragma unroll
    for (int k = 0; k < kPb; ++k)
      if (k == lane) dk = x[k];
    D[lane] = dk;
  }
}

__global__ void __launch_bounds__(256) bench(int mode, int reps, long long* out, double* D, double* sink) {
  __shared__ double F[kPb * 40];
  __shared__ double W[8][512];
  __shared__ double s_rd[kPb], s_dl[kPb][kPb];
  __shared__ volatile int done;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) done = 0;
  for (int i = tid; i < kPb * 40; i += 256) F[i] = (i % 41 == 0) ? 10.0 : 0.01 * (i % 7);
  for (int i = tid; i < 8 * 512; i += 256) (&W[0][0])[i] = 0.001 * i;
  __syncthreads();
  if (warp == 0) {
    long long t = 0;
    for (int r = 0; r < reps; ++r) {
      for (int i = lane; i < kPb * 40; i += 32) F[i] = (i % 41 == 0) ? 10.0 + r : 0.01 * (i % 7);
      __syncwarp();
      const long long t0 = clock64();
      diag_block(F, 40, lane, s_rd, s_dl, D);
      __syncwarp();
      t += clock64() - t0;
    }
    if (lane == 0) out[0] = t / reps, done = 1;
  } else {
    double a0 = 0, a1 = 0, b0 = 0, b1 = 0, c0 = 0, c1 = 0, e0 = 0, e1 = 0, av = lane * 0.5, bv = 1.0 / (lane + 1);
    int it = 0;
    while (!done) {
      if (mode == 1) {
        for (int u = 0; u < 8; ++u) {
          dmma(a0, a1, av, bv);
          dmma(b0, b1, bv, av);
          dmma(c0, c1, av, av);
          dmma(e0, e1, bv, bv);
        }
      } else if (mode == 2) {
        double* Wr = W[warp];
        for (int u = 0; u < 8; ++u) {
          const int j = (lane * 2 + u * 64 + it) & 511;
          Wr[j] -= Wr[(j + 37) & 511] * 0.5;
        }
      } else if (mode == 3) {
        for (int u = 0; u < 8; ++u) {
          a0 = fma(a0, bv, av);
          b0 = fma(b0, av, bv);
          c0 = fma(c0, bv, bv);
          e0 = fma(e0, av, av);
        }
      }
      ++it;
    }
    sink[tid] = a0 + a1 + b0 + b1 + c0 + c1 + e0 + e1;
  }
}

int main() {
  long long* out;
  double *D, *sink;
  cudaMalloc(&out, 8);
  cudaMalloc(&D, 64 * 8);
  cudaMalloc(&sink, 256 * 8);
  const char* names[] = {"idle", "dmma", "smem rmw", "dfma"};
  for (int mode = 0; mode < 4; ++mode) {
    bench<<<1, 256>>>(mode, 5, out, D, sink);
    bench<<<1, 256>>>(mode, 200, out, D, sink);
    long long c = 0;
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    std::printf("other warps %-9s: diag block %lld cycles  (%s)\n", names[mode], c, cudaGetErrorString(cudaGetLastError()));
  }
  int main2();
  return main2();
}

// DMMA latency (one dependent chain) and per-warp issue rate (8 chains), and
// the same for DFMA, one warp / 8 warps per CTA
__global__ void dmma_lat(int n, int chains8, long long* out, double* sink) {
  const int lane = threadIdx.x & 31;
  double a[8][2], av = lane * 0.5, bv = 1.0 / (lane + 1);
  for (int c = 0; c < 8; ++c) a[c][0] = a[c][1] = 0.0;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (chains8) {
#pragma unroll
      for (int c = 0; c < 8; ++c) dmma(a[c][0], a[c][1], av, bv);
    } else {
      dmma(a[0][0], a[0][1], av, bv);
    }
  }
  const long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < 8; ++c) s += a[c][0] + a[c][1];
  sink[threadIdx.x] = s;
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
__global__ void dfma_lat(int n, int chains8, long long* out, double* sink) {
  const int lane = threadIdx.x & 31;
  double a[8], av = lane * 0.5, bv = 1.0 / (lane + 1);
  for (int c = 0; c < 8; ++c) a[c] = 0.0;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (chains8) {
#pragma unroll
      for (int c = 0; c < 8; ++c) a[c] = fma(a[c], bv, av);
    } else {
      a[0] = fma(a[0], bv, av);
    }
  }
  const long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < 8; ++c) s += a[c];
  sink[threadIdx.x] = s;
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
int main2() {
  long long* out;
  double* sink;
  cudaMalloc(&out, 8);
  cudaMalloc(&sink, 1024 * 8);
  const int n = 4096;
  for (int warps : {1, 4, 8}) {
    for (int c8 : {0, 1}) {
      long long c = 0;
      dmma_lat<<<1, 32 * warps>>>(n, c8, out, sink);
      dmma_lat<<<1, 32 * warps>>>(n, c8, out, sink);
      cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
      const double per = double(c) / n / (c8 ? 8 : 1);
      long long f = 0;
      dfma_lat<<<1, 32 * warps>>>(n, c8, out, sink);
      dfma_lat<<<1, 32 * warps>>>(n, c8, out, sink);
      cudaMemcpy(&f, out, 8, cudaMemcpyDeviceToHost);
      std::printf("warps %d %s: DMMA %.1f cycles/op (warp 0)  DFMA %.1f cycles/op\n", warps,
                  c8 ? "8 independent chains" : "1 dependent chain   ", per, double(f) / n / (c8 ? 8 : 1));
    }
  }
  return 0;
}
