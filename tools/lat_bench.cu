// Latency probe (debug tool): dependent chains of FP64 div / rcp / fma / shfl.
#include <cstdio>
__global__ void lat(double* out, double a, double b, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) x = b / x;
  long long t1 = clock64();
  double y = a;
  for (int i = 0; i < 256; ++i) y = fma(y, b, a);
  long long t2 = clock64();
  double z = a;
  for (int i = 0; i < 256; ++i) z = __shfl_sync(0xffffffffu, z, (threadIdx.x + 1) & 31) + 1.0;
  long long t3 = clock64();
  double r = a;
  for (int i = 0; i < 256; ++i) r = __drcp_rn(r);
  long long t4 = clock64();
  double q = a;
  for (int i = 0; i < 256; ++i) q = q * b;
  long long t5 = clock64();
  float fx = (float)a;
  for (int i = 0; i < 256; ++i) fx = (float)b / fx;
  long long t6 = clock64();
  out[threadIdx.x] = x + y + z + r + q + fx;
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / 256; cyc[1] = (t2 - t1) / 256; cyc[2] = (t3 - t2) / 256;
    cyc[3] = (t4 - t3) / 256; cyc[4] = (t5 - t4) / 256; cyc[5] = (t6 - t5) / 256;
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64);
  for (int rep = 0; rep < 2; ++rep) lat<<<1, 32>>>(o, 1.7, 1.3, c);
  long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  printf("cycles per dependent op: ddiv %lld  dfma %lld  shfl64+dadd %lld  drcp_rn %lld  dmul %lld  fdiv %lld\n", h[0], h[1], h[2], h[3], h[4], h[5]);
  return 0;
}
