// Latency probe 2 (debug tool): the diagonal-block step chain of cta_dense.
#include <cstdio>
__device__ __forceinline__ double divz(double x, double d) {
  const bool z = x == 0.0;
  double xs = z ? 1.0 : x;
  asm("mov.b64 %0, %0;" : "+d"(xs));  // opaque: keeps x == 0 off the division's slow path
  const double q = xs / d;
  return z ? 0.0 : q;
}
template <int kPb>
__global__ void diag(double* F, int kb, long long* cyc, int reps) {
  const int lane = threadIdx.x;
  double x[kPb];
#pragma unroll
  for (int k = 0; k < kPb; ++k) x[k] = F[k * 32 + lane];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int k = 0; k < kPb; ++k) {
      if (k < kb) {
        const double d = __shfl_sync(0xffffffffu, x[k], k);
        if (lane > k && lane < kb) x[k] = divz(x[k], d);
        const double dlo = d * x[k];
#pragma unroll
        for (int k2 = 0; k2 < kPb; ++k2) {
          if (k2 > k && k2 < kb) {
            const double dl = __shfl_sync(0xffffffffu, dlo, k2);
            if (lane >= k2 && lane < kb) x[k2] -= x[k] * dl;
          }
        }
      }
    }
  }
  long long t1 = clock64();
#pragma unroll
  for (int k = 0; k < kPb; ++k) F[k * 32 + lane] = x[k];
  if (lane == 0) cyc[0] = (t1 - t0) / reps;
}
int main() {
  double* F; long long* c; cudaMalloc(&F, 8 * 32 * 8); cudaMalloc(&c, 8);
  double h[256]; for (int i = 0; i < 256; ++i) h[i] = (i % 33 == 0) ? 40.0 : 0.01 * (i % 7);
  for (int kb : {4, 8}) {
    cudaMemcpy(F, h, sizeof(h), cudaMemcpyHostToDevice);
    diag<8><<<1, 32>>>(F, kb, c, 10);
    cudaMemcpy(F, h, sizeof(h), cudaMemcpyHostToDevice);
    diag<8><<<1, 32>>>(F, kb, c, 10);
    long long v; cudaMemcpy(&v, c, 8, cudaMemcpyDeviceToHost);
    printf("diag block kb=%d: %lld cycles per block\n", kb, v);
  }
  return 0;
}
