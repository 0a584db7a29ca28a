// Micro-benchmark of the one-CTA dense front factorization (ldlt.cu
// cta_dense<256>) on synthetic diagonally dominant fronts: per-phase clock
// counts (panel vs trailing update) for a few (nr, w). Debug tool, not part
// of the library:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//     -Ipaper_2510_13333_b200/csrc -Iinclude --expt-relaxed-constexpr \
//     tools/front_bench.cu paper_2510_13333_b200/csrc/cuda/bigfront.cu -o tools/front_bench.bin
#define NCL_DENSE_PROF
#include "../paper_2510_13333_b200/csrc/cuda/ldlt.cu"

#include <cstdio>
#include <random>
#include <vector>

using namespace nclb;

template <int NT>
__global__ void __launch_bounds__(NT) front_kernel(const double* G, int nr, int w, double* L, double* CB, double* D,
                                                    int* zp, int reps, long long* cyc) {
  extern __shared__ double s_front[];
  const int tid = threadIdx.x;
  long long t0 = 0, tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int c = tid >> 5; c < nr; c += NT / 32)
      for (int i = c + (tid & 31); i < nr; i += 32) s_front[cb_col(c, nr) + i] = G[static_cast<int64_t>(c) * nr + i];
    __syncthreads();
    t0 = clock64();
    cta_dense<NT>(s_front, nr, w, 0, 0.0, D, zp, L, CB, tid);
    __syncthreads();
    tot += clock64() - t0;
  }
  if (tid == 0) cyc[blockIdx.x] = tot / reps;
}

template <int NT>
void run(bool root_only) {
  std::printf("threads %d\n", NT);
  const int cases[][2] = {{27, 4}, {48, 6}, {84, 10}, {133, 22}, {155, 155}, {160, 64}};
  for (auto& cs : cases) {
    if (root_only && cs[0] != 155) continue;
    const int nr = cs[0], w = cs[1];
    std::vector<double> h(static_cast<size_t>(nr) * nr, 0.0);
    std::mt19937_64 rng(nr);
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    for (int c = 0; c < nr; ++c)
      for (int i = c; i < nr; ++i) h[static_cast<size_t>(c) * nr + i] = (i == c) ? nr + 1.0 : (rng() % 3 ? 0.0 : U(rng));
    double *G, *L, *CB, *D;
    int* zp;
    long long* cyc;
    cudaMalloc(&G, h.size() * 8);
    cudaMalloc(&L, h.size() * 8);
    cudaMalloc(&CB, h.size() * 8);
    cudaMalloc(&D, nr * 8);
    cudaMalloc(&zp, 4);
    cudaMalloc(&cyc, 148 * 8);
    cudaMemcpy(G, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    const int smem = 160 * 161 / 2 * 8;
    cudaFuncSetAttribute(front_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    front_kernel<NT><<<1, NT, smem>>>(G, nr, w, L, CB, D, zp, 3, cyc);
    cudaDeviceSynchronize();
    long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_dense_prof, z, sizeof(z));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    front_kernel<NT><<<1, NT, smem>>>(G, nr, w, L, CB, D, zp, 20, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpyFromSymbol(z, g_dense_prof, sizeof(z));
    std::printf("   per rep: diag block %lld  barrier %lld  rows %lld  trailing %lld (look-ahead diag %lld, strip %lld)  writeout %lld cycles\n", z[0] / 20,
                z[1] / 20, z[2] / 20, z[3] / 20, z[5] / 20, z[6] / 20, z[4] / 20);
    std::printf("nr=%3d w=%3d  cta_dense %8lld cycles (%.2f us at 1.965 GHz)  kernel %.1f us/rep  err=%s\n", nr, w, c,
                c / 1965.0, ms * 1000 / 20, cudaGetErrorString(cudaGetLastError()));
    cudaFree(G);
    cudaFree(L);
    cudaFree(CB);
    cudaFree(D);
    cudaFree(zp);
    cudaFree(cyc);
  }
}

int main(int argc, char** argv) {
  // "root": the 155 x 155 root front only, 256 threads (ncu source capture)
  const bool root_only = argc > 1;
  run<256>(root_only);
  if (!root_only) run<512>(false);
  return 0;
}
