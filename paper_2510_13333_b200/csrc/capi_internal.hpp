// Internal helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <chrono>

#include <cmath>
#include <cstdint>
#include <limits>
#include <string>
#include <vector>

namespace nclb {

struct CudaError {
  std::string msg;
};

extern cudaStream_t g_stream;
extern thread_local std::string g_err;
void ck(cudaError_t e, const char* what);
void ensure_init();
void check_launch(const char* what);
int set_err(int code, const std::string& msg);
int map_exc();

// upload accounting (printed under NCL_ANALYZE_TIMING): nanoseconds in
// cudaMalloc, nanoseconds in the copies, bytes copied (any thread)
inline std::atomic<int64_t> g_upload_stats[3] = {0, 0, 0};

// Owning device buffer (cudaMalloc/cudaFree), sized in elements.
template <class T>
struct DevBuf {
  T* p = nullptr;
  int64_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(int64_t count) {
    if (count <= n && p) return;
    release();
    const int64_t bytes = std::max<int64_t>(count, 1) * static_cast<int64_t>(sizeof(T));
    ck(cudaMalloc(reinterpret_cast<void**>(&p), bytes), "cudaMalloc");
    n = std::max<int64_t>(count, 1);
  }
  void upload(const std::vector<T>& v) {
    const auto t0 = std::chrono::steady_clock::now();
    alloc(static_cast<int64_t>(v.size()));
    const auto t1 = std::chrono::steady_clock::now();
    if (!v.empty())
      ck(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, g_stream), "upload");
    ck(cudaStreamSynchronize(g_stream), "upload sync");
    g_upload_stats[0] += std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
    g_upload_stats[1] += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t1).count();
    g_upload_stats[2] += static_cast<int64_t>(v.size() * sizeof(T));
  }
  void download(std::vector<T>& v, int64_t count) const {
    v.resize(count);
    if (count > 0) ck(cudaMemcpyAsync(v.data(), p, count * sizeof(T), cudaMemcpyDeviceToHost, g_stream), "download");
    ck(cudaStreamSynchronize(g_stream), "download sync");
  }
};

}  // namespace nclb

#include "../../include/nclopf_b200.h"
namespace nclb {
// the condensed-KKT matrix's device maps (capi_kkt.cpp), built ahead of its
// first assembly: NCL_OK or an error code (message in this thread's g_err)
int kkt_prepare_device(ncl_kkt_t K);
// the symbolic factor's device copy (capi.cpp upload_symb), otherwise made by
// the first factorization: NCL_OK or an error code
int symb_prepare_device(ncl_symb_t S);
}  // namespace nclb
#include "cuda/dev.hpp"
#include "host/sparse.hpp"

// SparseSym handle (shared by the C-ABI translation units).
struct ncl_sym {
  nclb::SymPattern pat;
  nclb::DevBuf<double> vals;
  nclb::DevBuf<int> colptr, rowind;
  nclb::DevBuf<int> diag_pos, mv_val, mv_col;
  nclb::DevBuf<int64_t> mv_ptr;
  nclb::DevBuf<int> slot_ptr, slot_trip;
  nclb::DevBuf<double> trip_vals;
  nclb::DevBuf<double> scratch;
  nclb::DevBuf<double> rowsum;
  nclb::DevBuf<double> mvx, mvy;  // host-path multiply staging (allocated once)
  nclb::DevPattern dp;
  uint64_t hash = 0;
  bool dev_ready = false;  // pattern + values uploaded (lazy: host-only use needs no GPU)
  explicit ncl_sym(int n) : pat(n) {}
};

namespace nclb {
uint64_t pattern_hash(const std::vector<int>& cp, const std::vector<int>& ri);
void upload_pattern(ncl_sym* M);
void ensure_dev(ncl_sym* M, const char* what);
}  // namespace nclb
