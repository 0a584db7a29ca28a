// FP64 peak microbenchmark (B200, sm_100a): the DMMA tensor pipe
// (mma.sync.aligned.m8n8k4.row.col.f64 — tcgen05 has no f64 kind) and the
// FFMA.F64 pipe, every SM busy, CUDA-event timed. The measured numbers are the
// denominators of the FP64 roofline fractions in DESIGN.md / profiles/.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kAcc = 8;  // independent accumulator tiles per warp (hide DMMA latency)

__global__ void __launch_bounds__(256) dmma_loop(double* out, double a0, double b0) {
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  double c[kAcc][2];
#pragma unroll
  for (int t = 0; t < kAcc; ++t) c[t][0] = c[t][1] = 0.0;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int t = 0; t < kAcc; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < kAcc; ++t) s += c[t][0] + c[t][1];
  if (s == 1234.5) out[threadIdx.x] = s;  // keep the chain alive
}

__global__ void __launch_bounds__(256) ffma_loop(double* out, double a0, double b0) {
  double a = a0 + threadIdx.x * 1e-9, b = b0;
  double c[kAcc];
#pragma unroll
  for (int t = 0; t < kAcc; ++t) c[t] = t;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int t = 0; t < kAcc; ++t) c[t] = fma(c[t], a, b);
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < kAcc; ++t) s += c[t];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <class K>
double run(K kern, int blocks, double flop_per_thread_iter) {
  double* o;
  cudaMalloc(&o, 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, 256>>>(o, 1.0, 0.5);  // warm-up
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) kern<<<blocks, 256>>>(o, 1.0, 0.5);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(o);
  const double flop = flop_per_thread_iter * kIters * kAcc * 256.0 * blocks * reps;
  return flop / (ms * 1e-3) / 1e12;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // one m8n8k4 f64 MMA = 8*8*4*2 = 512 flop per warp = 16 flop per thread
  double best_d = 0, best_f = 0;
  for (int per_sm : {2, 4, 8}) {
    const double d = run(dmma_loop, sms * per_sm, 16.0);
    const double f = run(ffma_loop, sms * per_sm, 2.0);
    std::printf("{\"blocks_per_sm\": %d, \"dmma_tflops\": %.3f, \"ffma_f64_tflops\": %.3f}\n", per_sm, d, f);
    if (d > best_d) best_d = d;
    if (f > best_f) best_f = f;
  }
  std::printf("{\"sms\": %d, \"fp64_dmma_tflops\": %.3f, \"fp64_ffma_tflops\": %.3f}\n", sms, best_d, best_f);
  return 0;
}
