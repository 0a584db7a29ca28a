// Launch entry points of the IPM vector kernels (csrc/cuda/ipm.cu).
#pragma once

#include <cuda_runtime.h>

#include "../host/ipm_elem.hpp"

namespace nclb {

enum IpmElemOp {
  IE_INIT_X = 0,
  IE_INIT_ROW,
  IE_NEWTON,
  IE_RHS_X,
  IE_RECOVER,
  IE_TRIAL,
  IE_ACCEPT,
  IE_RESTORE_ROW,
  IE_UPDATE_MULT
};
enum IpmRedOp { IR_KKT = 0, IR_FTB, IR_MERIT, IR_DPHI, IR_RINF };

// asynchronous on st
void dev_ipm_elem(int op, const ipm::Vecs& V, const ipm::Scal& S, cudaStream_t st);
// part: kRedBlocks * 8 + 1 doubles of scratch, zeroed once (the last slot is
// the completion ticket); out: up to 8 doubles
void dev_ipm_reduce(int which, const ipm::Vecs& V, const ipm::Scal& S, double* part, double* out, cudaStream_t st);

}  // namespace nclb
