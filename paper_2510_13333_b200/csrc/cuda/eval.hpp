// Device structures of the template evaluator (K1).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../host/expr.hpp"

namespace nclb {

struct DevFam {
  int64_t ninst = 0;
  int64_t block0 = 0;  // first block of this family in the merged launch
  int64_t base = 0;    // contribution buffer offset
  int nv = 0, np = 0, G = 0, H = 0, obj = 0;
  const int* vars = nullptr;       // [nv][ninst]
  const double* params = nullptr;  // [np][ninst]
  const int* rows = nullptr;       // [ninst]
  const int* hess_hi = nullptr;
  const int* hess_lo = nullptr;
  const Instr* prog[4] = {nullptr, nullptr, nullptr, nullptr};
  const int* outs[4] = {nullptr, nullptr, nullptr, nullptr};
  int plen[4] = {0, 0, 0, 0};
};

struct DevModel {
  const DevFam* fams = nullptr;  // device array
  int nfam = 0;
  int nblocks = 0;
  int maxregs[4] = {0, 0, 0, 0};
  double* contrib = nullptr;
  unsigned long long* err = nullptr;  // min (family<<40 | inst<<2 | code), ~0 = none
};

void dev_eval(const DevModel& M, int kind, const double* w, double sigma, const double* lam, cudaStream_t st);
void dev_gather64(int64_t nslots, const int64_t* ptr, const int* idx, const double* src, double* dst,
                  cudaStream_t st);
// out[r] = sum_{p in ptr[r]..ptr[r+1]} vals[k] * x[xi[k]], k = kidx ? kidx[p] : p
void dev_csr_mv(int64_t nrows, const int64_t* ptr, const int* kidx, const int* xi, const double* vals,
                const double* x, double* out, cudaStream_t st);

}  // namespace nclb
