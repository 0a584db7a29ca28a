// Host side of model_ad: ModelBuilder semantics and the fixed index maps
// (/root/reference/proj/include/nclopf/model.hpp:29-97,
//  /root/reference/proj/src/model.cpp:28-128). Evaluation itself is GPU-only
// (csrc/cuda/eval.cu); this file produces the per-family instance tables,
// the compiled register programs and the reference-order gather lists the
// kernels consume.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "expr.hpp"

namespace nclb {

constexpr int kMaxSlots = 40;  // model.cpp:12

struct HFamily {
  Template tmpl;
  bool objective = false;
  bool used = false;
  int64_t ninst = 0;
  int np = 0;                   // max params over instances (padded)
  std::vector<int> vars;        // AoS during building: [inst][nv]
  std::vector<double> params;   // AoS: [inst][np_i] ragged
  std::vector<int64_t> pstart;  // [ninst+1] ragged param offsets
  std::vector<int> rows;
  explicit HFamily(Template t) : tmpl(std::move(t)) {}
};

struct BuiltModel {
  int n = 0, m = 0;
  std::vector<HFamily> fams;
  std::vector<std::pair<int, int>> jac_coords, hess_coords;
  // per family: SoA tables and programs
  struct F {
    int64_t ninst = 0;
    int nv = 0, np = 0, G = 0, H = 0;
    bool objective = false;
    std::vector<int> vars;       // [nv][ninst]
    std::vector<double> params;  // [np][ninst]
    std::vector<int> rows;       // [ninst]
    std::vector<int> hess_hi, hess_lo;  // template slots per Hessian entry
    Program prog[PK_N];
    int nregs[PK_N] = {0, 0, 0, 0};
    int64_t base = 0;  // offset into the contribution buffer
  };
  std::vector<F> f;
  int64_t ncontrib = 0;
  // reference-order gather lists: output slot -> contribution indices
  std::vector<int64_t> c_ptr, j_ptr, h_ptr, g_ptr, o_ptr;
  std::vector<int64_t> c_idx, j_idx, h_idx, g_idx, o_idx;
  // jac_times / jac_trans_times gathers (model.cpp:211-223)
  std::vector<int64_t> jt_ptr;  // by column: k indices ascending
  std::vector<int> jt_idx;
  std::vector<int64_t> jr_ptr;  // by row (jac_coords is row-sorted)
  std::vector<int> jcol, jrow;
};

class HostBuilder {
 public:
  explicit HostBuilder(int n) : n_(n) {}
  int num_vars() const { return n_; }
  int num_rows() const { return m_; }
  int add_template(Template t);
  int add_rows(int count);
  void add_terms(int tid, bool objective, int64_t count, const int* rows, int nv, const int* vars, int np,
                 const double* params);
  BuiltModel build();

 private:
  int n_ = 0, m_ = 0;
  std::vector<HFamily> fams_;
};

// Register allocation: rewrites a CSE program so registers are reused after
// their last use; returns the number of physical registers.
int allocate_registers(Program& p);

}  // namespace nclb
