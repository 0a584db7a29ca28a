// C-ABI for the sparse_core part of the boundary (include/nclopf_b200.h).
// Host code: handle bookkeeping, one-time symbolic analysis (csrc/host),
// uploads; every numeric operation is a CUDA kernel from csrc/cuda.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/nclopf_b200.h"
#include "capi_internal.hpp"
#include "cuda/dev.hpp"
#include "host/sparse.hpp"

using nclb::Error;

namespace nclb {
thread_local std::string g_err;
cudaStream_t g_stream = nullptr;
int g_device = -1;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int map_exc() {
  try {
    throw;
  } catch (const Error& e) {
    return set_err(e.code, e.msg);
  } catch (const CudaError& e) {
    return set_err(NCL_E_CUDA, e.msg);
  } catch (const std::bad_alloc&) {
    return set_err(NCL_E_NOMEM, "out of memory");
  } catch (const std::exception& e) {
    return set_err(NCL_E_INTERNAL, e.what());
  }
}
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError{std::string(what) + ": " + cudaGetErrorString(e)};
}
void ensure_init() {
  if (!g_stream) {
    int rc = ncl_init(-1);
    if (rc != NCL_OK) throw CudaError{g_err};
  }
}
void check_launch(const char* what) {
  ck(cudaGetLastError(), what);
}
}  // namespace nclb

using namespace nclb;

#define API extern "C" __attribute__((visibility("default")))
#define GUARD(...)    \
  try {               \
    __VA_ARGS__;      \
  } catch (...) {     \
    return map_exc(); \
  }                   \
  return NCL_OK;

// ----------------------------------------------------------------------------
API int ncl_init(int device) {
  try {
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
      return set_err(NCL_E_CUDA, "ncl_init: no CUDA device (the B200 path has no CPU fallback)");
    if (device < 0) {
      ck(cudaGetDevice(&device), "cudaGetDevice");
    }
    ck(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major < 10)
      return set_err(NCL_E_CUDA, "ncl_init: device is not sm_100 class (built for sm_100a only)");
    if (!g_stream) ck(cudaStreamCreateWithFlags(&g_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    g_device = device;
  } catch (...) {
    return map_exc();
  }
  return NCL_OK;
}
API int ncl_synchronize(void) { GUARD(ensure_init(); ck(cudaStreamSynchronize(g_stream), "sync")); }
API const char* ncl_last_error(void) { return g_err.c_str(); }
API void* ncl_stream(void) {
  try {
    ensure_init();
  } catch (...) {
    map_exc();
    return nullptr;
  }
  return g_stream;
}
API int ncl_device_alloc(void** ptr, int64_t bytes) {
  GUARD(ensure_init(); ck(cudaMalloc(ptr, std::max<int64_t>(bytes, 8)), "cudaMalloc"));
}
API int ncl_device_free(void* ptr) { GUARD(ck(cudaFree(ptr), "cudaFree")); }
API int ncl_memcpy(void* dst, const void* src, int64_t bytes, int kind) {
  GUARD({
    ensure_init();
    const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice : kind == 1 ? cudaMemcpyDeviceToHost
                                                                            : cudaMemcpyDeviceToDevice;
    if (bytes > 0) ck(cudaMemcpyAsync(dst, src, bytes, k, g_stream), "cudaMemcpyAsync");
    ck(cudaStreamSynchronize(g_stream), "sync");
  });
}
API int64_t ncl_kernel_launches(void) { return g_kernel_launches; }

// ---------------------------------------------------------------------------
// SparseSym
// ---------------------------------------------------------------------------
namespace nclb {
uint64_t pattern_hash(const std::vector<int>& cp, const std::vector<int>& ri) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  };
  for (int v : cp) mix(static_cast<uint32_t>(v));
  for (int v : ri) mix(static_cast<uint32_t>(v));
  return h;
}

void require_finalized(const ncl_sym* M, const char* what) {
  if (!M->pat.finalized()) throw Error{NCL_E_LOGIC, std::string(what) + ": matrix not finalized"};
}

// Upload pattern-level device data (first device use after finalize()).
void upload_pattern(ncl_sym* M) {
  if (M->dev_ready) return;
  ensure_init();
  const int n = M->pat.dim();
  const auto& cp = M->pat.col_ptr();
  const auto& ri = M->pat.row_ind();
  const int nnz = M->pat.nnz();
  M->colptr.upload(cp);
  M->rowind.upload(ri);
  M->vals.upload(M->pat.values());
  // diagonal slots
  std::vector<int> dpos;
  for (int c = 0; c < n; ++c)
    for (int p = cp[c]; p < cp[c + 1]; ++p)
      if (ri[p] == c) dpos.push_back(p);
  M->diag_pos.upload(dpos);
  // symmetric SpMV gather in reference order: row i = lower-row entries
  // (i,c), c<i ascending; then column i's entries in storage order.
  std::vector<int64_t> ptr(n + 1, 0);
  for (int c = 0; c < n; ++c)
    for (int p = cp[c]; p < cp[c + 1]; ++p) {
      const int r = ri[p];
      if (r != c) ptr[r + 1]++;  // (r,c) contributes to row r via the lower part
      ptr[c + 1]++;              // column c's own entries contribute to row c
    }
  for (int i = 0; i < n; ++i) ptr[i + 1] += ptr[i];
  std::vector<int> mval(ptr[n]), mcol(ptr[n]);
  {
    std::vector<int64_t> fp(ptr.begin(), ptr.end() - 1);
    // pass over columns ascending: for row r>c the (r,c) entry lands in row r
    // before r's own column entries (which come at column r > c).
    for (int c = 0; c < n; ++c) {
      for (int p = cp[c]; p < cp[c + 1]; ++p) {
        const int r = ri[p];
        if (r != c) {
          mval[fp[r]] = p;
          mcol[fp[r]] = c;
          fp[r]++;
        }
      }
      for (int p = cp[c]; p < cp[c + 1]; ++p) {
        const int r = ri[p];
        mval[fp[c]] = p;
        mcol[fp[c]] = r;  // y[c] += v x[r] (r==c for the diagonal: y[r] += v x[c])
        fp[c]++;
      }
    }
  }
  M->mv_ptr.upload(ptr);
  M->mv_val.upload(mval);
  M->mv_col.upload(mcol);
  M->scratch.alloc(8);
  M->dp.n = n;
  M->dp.nnz = nnz;
  M->dp.diag_pos = M->diag_pos.p;
  M->dp.ndiag = static_cast<int>(dpos.size());
  M->dp.mv_ptr = M->mv_ptr.p;
  M->dp.mv_val = M->mv_val.p;
  M->dp.mv_col = M->mv_col.p;
  M->dev_ready = true;
}
void ensure_dev(ncl_sym* M, const char* what) {
  if (!M->pat.finalized()) throw Error{NCL_E_LOGIC, std::string(what) + ": matrix not finalized"};
  upload_pattern(M);
}
// the triplet -> slot gather of the GPU refill (built on first use: matrices
// whose values are assembled on the device, like the condensed K, never need it)
void ensure_refill_map(ncl_sym* M) {
  if (M->slot_ptr.p) return;
  std::vector<int> sptr, sidx;
  M->pat.slot_trip_csr(sptr, sidx);
  M->slot_ptr.upload(sptr);
  M->slot_trip.upload(sidx);
}
}  // namespace nclb

API int ncl_sym_create(int n, ncl_sym_t* out) {
  GUARD({
    if (n < 0) throw Error{NCL_E_INVALID, "SparseSym: negative dimension"};
    *out = new ncl_sym(n);
  });
}
API void ncl_sym_destroy(ncl_sym_t M) { delete M; }
API int ncl_sym_add(ncl_sym_t M, int64_t count, const int* rows, const int* cols, const double* vals) {
  GUARD(for (int64_t k = 0; k < count; ++k) M->pat.add(rows[k], cols[k], vals[k]));
}
API int ncl_sym_finalize(ncl_sym_t M) {
  GUARD({
    M->pat.finalize();
    M->hash = pattern_hash(M->pat.col_ptr(), M->pat.row_ind());
  });
}
API int ncl_sym_begin_refill(ncl_sym_t M) { GUARD(M->pat.begin_refill()); }
API int ncl_sym_refill(ncl_sym_t M) {
  GUARD({
    if (!M->pat.finalized()) throw Error{NCL_E_LOGIC, "SparseSym::refill: not finalized"};
    ensure_dev(M, "SparseSym::refill");
    ensure_refill_map(M);
    M->trip_vals.upload(M->pat.trip_vals());
    dev_gather_sum(M->pat.nnz(), M->slot_ptr.p, M->slot_trip.p, M->trip_vals.p, M->vals.p, g_stream);
    check_launch("refill");
  });
}
API int ncl_sym_refill_values(ncl_sym_t M, const double* tv, int where) {
  GUARD({
    if (!M->pat.finalized()) throw Error{NCL_E_LOGIC, "SparseSym::refill: not finalized"};
    ensure_dev(M, "SparseSym::refill");
    ensure_refill_map(M);
    const int64_t nt = M->pat.num_trips();
    const double* src = tv;
    if (where == NCL_HOST) {
      M->trip_vals.alloc(nt);
      ck(cudaMemcpyAsync(M->trip_vals.p, tv, nt * sizeof(double), cudaMemcpyHostToDevice, g_stream), "H2D");
      src = M->trip_vals.p;
    }
    dev_gather_sum(M->pat.nnz(), M->slot_ptr.p, M->slot_trip.p, src, M->vals.p, g_stream);
    check_launch("refill_values");
    if (where == NCL_HOST) ck(cudaStreamSynchronize(g_stream), "sync");
  });
}
API int ncl_sym_dim(ncl_sym_t M) { return M->pat.dim(); }
API int ncl_sym_nnz(ncl_sym_t M) { return M->pat.nnz(); }
API int64_t ncl_sym_num_triplets(ncl_sym_t M) { return M->pat.num_trips(); }
API int ncl_sym_finalized(ncl_sym_t M) { return M->pat.finalized() ? 1 : 0; }
API int ncl_sym_get_csc(ncl_sym_t M, int* colptr, int* rowind, double* vals) {
  GUARD({
    const auto& cp = M->pat.col_ptr();
    const auto& ri = M->pat.row_ind();
    if (colptr && !cp.empty()) std::memcpy(colptr, cp.data(), cp.size() * sizeof(int));
    if (rowind && !ri.empty()) std::memcpy(rowind, ri.data(), ri.size() * sizeof(int));
    if (vals && M->pat.nnz() > 0 && !M->dev_ready) {
      std::memcpy(vals, M->pat.values().data(), M->pat.nnz() * sizeof(double));
    } else if (vals && M->pat.nnz() > 0) {
      require_finalized(M, "SparseSym::values");
      ck(cudaMemcpyAsync(vals, M->vals.p, M->pat.nnz() * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
      ck(cudaStreamSynchronize(g_stream), "sync");
    }
  });
}
API int ncl_sym_set_values(ncl_sym_t M, const double* v, int where) {
  GUARD({
    ensure_dev(M, "SparseSym::set_values");
    const int64_t nz = M->pat.nnz();
    ck(cudaMemcpyAsync(M->vals.p, v, nz * sizeof(double),
                       where == NCL_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, g_stream),
       "set_values");
    if (where == NCL_HOST) ck(cudaStreamSynchronize(g_stream), "sync");
  });
}
API double* ncl_sym_device_values(ncl_sym_t M) {
  try {
    ensure_dev(M, "SparseSym::device_values");
  } catch (...) {
    map_exc();
    return nullptr;
  }
  return M->vals.p;
}

static int scalar_op(ncl_sym_t M, double* out, int which) {
  GUARD({
    ensure_dev(M, "SparseSym");
    double* d = M->scratch.p;
    if (which == 0) dev_max_abs_diag(M->dp, M->vals.p, d, g_stream);
    else if (which == 1) dev_rowsum_max(M->dp, M->vals.p, d, g_stream);
    else dev_frob_sq(M->dp, M->colptr.p, M->rowind.p, M->vals.p, d, g_stream);
    check_launch("norm");
    double h = 0;
    ck(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
    ck(cudaStreamSynchronize(g_stream), "sync");
    *out = which == 2 ? std::sqrt(h) : h;
  });
}
API int ncl_sym_max_abs_diag(ncl_sym_t M, double* out) { return scalar_op(M, out, 0); }
API int ncl_sym_norm_inf(ncl_sym_t M, double* out) { return scalar_op(M, out, 1); }
API int ncl_sym_frobenius_norm(ncl_sym_t M, double* out) { return scalar_op(M, out, 2); }

API int ncl_sym_multiply(ncl_sym_t M, const double* x, double* y, int where) {
  GUARD({
    ensure_dev(M, "SparseSym::multiply");
    const int n = M->pat.dim();
    if (where == NCL_DEVICE) {
      dev_spmv(M->dp, M->vals.p, x, y, g_stream);
      check_launch("spmv");
      return NCL_OK;
    }
    M->mvx.alloc(n);  // no-ops after the first call
    M->mvy.alloc(n);
    ck(cudaMemcpyAsync(M->mvx.p, x, n * sizeof(double), cudaMemcpyHostToDevice, g_stream), "H2D");
    dev_spmv(M->dp, M->vals.p, M->mvx.p, M->mvy.p, g_stream);
    check_launch("spmv");
    ck(cudaMemcpyAsync(y, M->mvy.p, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
    ck(cudaStreamSynchronize(g_stream), "sync");
  });
}
API int ncl_sym_same_pattern(ncl_sym_t A, ncl_sym_t B) {
  return A->pat.dim() == B->pat.dim() && A->pat.col_ptr() == B->pat.col_ptr() && A->pat.row_ind() == B->pat.row_ind();
}
API int ncl_sym_write_matrix_market(ncl_sym_t M, char* buf, int64_t cap, int64_t* len) {
  GUARD({
    const int n = M->pat.dim();
    std::vector<double> v(M->pat.values());
    if (M->dev_ready && !v.empty()) {
      ck(cudaMemcpyAsync(v.data(), M->vals.p, v.size() * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
      ck(cudaStreamSynchronize(g_stream), "sync");
    }
    std::ostringstream os;
    os << "%%MatrixMarket matrix coordinate real symmetric\n";
    os << n << " " << n << " " << M->pat.nnz() << "\n";
    char line[64];
    const auto& cp = M->pat.col_ptr();
    const auto& ri = M->pat.row_ind();
    for (int c = 0; c < n && M->pat.finalized(); ++c)
      for (int p = cp[c]; p < cp[c + 1]; ++p) {
        std::snprintf(line, sizeof(line), "%d %d %.17g\n", ri[p] + 1, c + 1, v[p]);
        os << line;
      }
    const std::string s = os.str();
    *len = static_cast<int64_t>(s.size());
    if (buf && cap > 0) std::memcpy(buf, s.data(), std::min<int64_t>(cap, *len));
  });
}

// ---------------------------------------------------------------------------
// Symbolic analysis
// ---------------------------------------------------------------------------
// device copy of one TaskLayout
struct LayoutDev {
  DevBuf<int> nodes, tptr, prog, bamap;
  DevBuf<uint8_t> bcmap;
  DevBuf<uint32_t> bcmapw, bsmapw;
  DevBuf<int64_t> bccb;
  DevBuf<int> bcid;
  DevBuf<RegChunk> bchunks;
  DevBuf<RegInst> binst;
  DevBuf<int64_t> gpo;
  std::vector<DevBuf<BigDesc>> top;
};

struct ncl_symb {
  SymbolicCore core;
  Supernodal Z;
  TaskLayout flay;  // task layout of factor and solves: register-front forest + subtree groups + singles
  TaskLayout lay;   // the same list unbatched (built only for the NCL_*NO_BATCH A/B switches)
  uint64_t hash = 0;
  int nnz = 0;
  DevSymb d;
  DevBuf<int> perm, sn_first, sn_parent, rows, relp, cptr, child, order, asrc, aoff, flags, tickets;
  DevBuf<int64_t> sn_rptr, sn_loff, cb_off, aptr, gm_ptr, gsp, gsrc, cv_ptr, cvsp, cvsrc;
  DevBuf<int> gdst;
  DevBuf<uint8_t> big;
  DevBuf<int> lay_nodes, lay_tptr, lay_prog;
  DevBuf<int64_t> lay_gpo;
  LayoutDev fdev;  // device copy of flay
  DevBuf<int> aoffp;
  DevBuf<SnMeta> meta;
  DevBuf<ChildRec> chrec;
  std::vector<DevBuf<BigDesc>> top_dev;
  bool dev_ready = false;
};

namespace {
void build_batches(const Supernodal& Z, const std::vector<int>& list, int split, const std::vector<uint8_t>& inlist,
                   std::vector<uint8_t>& batched, BatchSched& B) {
  const int nsn = Z.nsn;
  auto i32 = [](int64_t v) {  // RegInst offsets are int32
    if (v < 0 || v >= (int64_t(1) << 31)) throw Error{NCL_E_INVALID, "analyze: register-front offsets exceed int32"};
    return static_cast<int>(v);
  };
  auto wof = [&](int s) { return Z.sn_first[s + 1] - Z.sn_first[s]; };
  auto nrof = [&](int s) { return static_cast<int>(Z.sn_rptr[s + 1] - Z.sn_rptr[s]); };
  auto shape_of = [&](int s) {
    for (int k = 0; k < kNumRegShapes; ++k)
      if (kRegShapes[k][0] == nrof(s) && kRegShapes[k][1] == wof(s)) return k;  // first match
    return -1;
  };
  // levels of the register-front forest (list order: children before
  // parents); tier 1 (shapes < kRegTier1) is closed under children on its own
  std::vector<int> lev(nsn, -1), shp(nsn, -1), tier(nsn, 0);
  int nlev = 0;
  for (int i = 0; i < split; ++i) {
    const int s = list[i], k = shape_of(s);
    if (k < 0) continue;
    int l = 0, t = k < kRegTier1 ? 1 : 2;
    bool ok = true;
    for (int q = Z.cptr[s]; q < Z.cptr[s + 1] && ok; ++q) {
      const int c = Z.child[q];
      if (!inlist[c]) continue;  // finished by an earlier phase (sharded lists): its standard CB
      if (lev[c] < 0) ok = false;
      else l = std::max(l, lev[c] + 1), t = std::max(t, tier[c]);
    }
    if (ok) lev[s] = l, shp[s] = k, tier[s] = t, nlev = std::max(nlev, l + 1);
  }
  std::vector<std::vector<std::vector<int>>> bucket(2 * nlev, std::vector<std::vector<int>>(kNumRegShapes));
  for (int i = 0; i < split; ++i)
    if (lev[list[i]] >= 0) bucket[(tier[list[i]] - 1) * nlev + lev[list[i]]][shp[list[i]]].push_back(list[i]);
  nlev *= 2;
  for (int l = 0; l < nlev; ++l) {
    for (int k = 0; k < kNumRegShapes; ++k) {
      auto& v = bucket[l][k];
      if (v.empty()) continue;
      // same child count next to each other: the child loop stays converged
      std::stable_sort(v.begin(), v.end(),
                       [&](int x, int y) { return Z.cptr[x + 1] - Z.cptr[x] < Z.cptr[y + 1] - Z.cptr[y]; });
      const int nr = kRegShapes[k][0], per = 32 / kRegShapes[k][2];
      const int np = nr * (nr + 1) / 2, npad = (np + 3) & ~3;
      const int R = kRegShapes[k][2], nw = npad / 4;
      const int wk = kRegShapes[k][1], pw = wk * nr - wk * (wk - 1) / 2;  // packed entries of the W pivot columns
      const size_t chunk0 = B.chunks.size();
      for (size_t x = 0; x < v.size(); x += per)
        B.chunks.push_back(RegChunk{k, static_cast<int>(std::min<size_t>(per, v.size() - x)),
                                    static_cast<int>(B.inst.size() + x), -1});
      static_assert(kSmapWords * 4 >= 12, "solve row maps cover 12 rows");
      int64_t abase = 0, wbase = 0;  // R == 1: per-chunk blocks interleaved over the 32 lanes
      for (size_t x = 0; x < v.size(); ++x) {
        const int s = v[x];
        const int ix = static_cast<int>(x % 32);
        const int ixc = static_cast<int>(x % per);  // front index inside its chunk (the solve's lane)
        if (ixc == 0) {
          int maxnch = 0;
          for (size_t y = x; y < std::min(v.size(), x + per); ++y)
            maxnch = std::max(maxnch, Z.cptr[v[y] + 1] - Z.cptr[v[y]]);
          if (R == 1) {
            abase = static_cast<int64_t>(B.amap.size());
            B.amap.resize(B.amap.size() + static_cast<size_t>(pw) * 32, -1);
            wbase = static_cast<int64_t>(B.cmapw.size());
            B.cmapw.resize(B.cmapw.size() + static_cast<size_t>(maxnch) * nw * 32, 0xffffffffu);
          }
          B.chunks[chunk0 + x / per].smap = static_cast<int>(B.smapw.size());
          B.smapw.resize(B.smapw.size() + static_cast<size_t>(maxnch) * kSmapStride * 32, 0xffffffffu);
        }
        batched[s] = 1;
        RegInst I{};
        I.loff = i32(Z.sn_loff[s]);
        I.cboff = i32(Z.cb_off[s]);
        I.s = s;
        I.f = Z.sn_first[s];
        I.nch = Z.cptr[s + 1] - Z.cptr[s];
        const int64_t ast = R == 1 ? 32 : 1;  // A-map stride
        if (R == 1) {
          I.amap = i32(abase + ix);
          I.cmap = i32(wbase + ix);
        } else {
          I.amap = i32(static_cast<int64_t>(B.amap.size()));
          B.amap.resize(B.amap.size() + pw, -1);
          I.cmap = i32(static_cast<int64_t>(B.cmap.size()));
        }
        for (int64_t e = Z.a_ptr[s]; e < Z.a_ptr[s + 1]; ++e) {
          const int64_t pp = cb_col(Z.a_off[e] / nr, nr) + Z.a_off[e] % nr;
          if (pp >= pw) throw Error{NCL_E_INTERNAL, "analyze: A entry outside the pivot columns"};
          B.amap[I.amap + ast * pp] = Z.a_src[e];
        }
        I.ccb = i32(static_cast<int64_t>(B.ccb.size()));
        for (int q = Z.cptr[s]; q < Z.cptr[s + 1]; ++q) {
          const int c = Z.child[q], qi = q - Z.cptr[s];
          const int m2c = nrof(c) - wof(c);
          const int* rel = Z.relp.data() + Z.sn_rptr[c] + wof(c);
          {
            // forward solve (one thread per front, any R): parent row rel[kk] <- the child's CV entry kk
            const int64_t sb = B.chunks[chunk0 + x / per].smap;
            for (int kk = 0; kk < m2c; ++kk) {
              uint32_t& wd = B.smapw[sb + (static_cast<int64_t>(qi) * kSmapStride + rel[kk] / 4) * 32 + ixc];
              wd = (wd & ~(0xffu << (8 * (rel[kk] % 4)))) | (static_cast<uint32_t>(kk) << (8 * (rel[kk] % 4)));
            }
            const int64_t cvo = Z.sn_rptr[c] + wof(c);
            if (cvo >= (int64_t(1) << 31)) throw Error{NCL_E_INVALID, "analyze: row list exceeds int32 addressing"};
            B.smapw[sb + (static_cast<int64_t>(qi) * kSmapStride + kSmapWords) * 32 + ixc] = static_cast<uint32_t>(cvo);
          }
          if (R == 1) {
            for (int j = 0; j < m2c; ++j)
              for (int ii = j; ii < m2c; ++ii) {
                const int64_t pp = cb_col(rel[j], nr) + rel[ii];
                uint32_t& wd = B.cmapw[I.cmap + (static_cast<int64_t>(qi) * nw + pp / 4) * 32];
                wd = (wd & ~(0xffu << (8 * (pp % 4)))) | (static_cast<uint32_t>(cb_col(j, m2c) + ii) << (8 * (pp % 4)));
              }
          } else {
            const size_t base = B.cmap.size();
            B.cmap.resize(base + npad, 255);
            for (int j = 0; j < m2c; ++j)
              for (int ii = j; ii < m2c; ++ii)
                B.cmap[base + cb_col(rel[j], nr) + rel[ii]] = static_cast<uint8_t>(cb_col(j, m2c) + ii);
          }
          B.ccb.push_back(Z.cb_off[c]);
          B.cid.push_back(c);
          if (qi < 4) I.cid[qi] = c, I.cb[qi] = i32(Z.cb_off[c]);
        }
        B.inst.push_back(I);
        B.nodes++;
      }
    }
    if (l == nlev / 2 - 1) B.nchunk1 = static_cast<int>(B.chunks.size());
  }
}

// Task layout of a list (leaves-first height order, CTA part from `split`):
// every warp-part supernode whose subtree has <= kGroup supernodes and whose
// parent does not qualify roots a GROUP task (its subtree in postorder,
// processed by one warp without scheduling between nodes); the remaining
// warp-part supernodes and the CTA part are single-node tasks. Order: groups
// (dependency-free), warp singles by height, CTA singles by height.
//
// With `batch`, warp-part supernodes of the register-front shapes
// (kRegShapes) whose children in the list are such fronts too are factored
// level by level, one thread per front (BatchSched), and leave the group /
// single tasks.
void build_batches(const Supernodal& Z, const std::vector<int>& list, int split, const std::vector<uint8_t>& inlist,
                   std::vector<uint8_t>& batched, BatchSched& B);

TaskLayout build_layout(const Supernodal& Z, const std::vector<int>& list, int split, bool batch = false) {
  const int nsn = Z.nsn;
  TaskLayout L;
  std::vector<uint8_t> warp(nsn, 0), inlist(nsn, 0), batched(nsn, 0);
  for (int i = 0; i < split; ++i) warp[list[i]] = 1;
  for (int s : list) inlist[s] = 1;
  if (batch) build_batches(Z, list, split, inlist, batched, L.batch);
  // Groups are maximal warp-part subtrees whose whole multifrontal working
  // set fits one warp's shared memory: every front nr <= kGrpFront, the
  // program (records + relative maps + A entries) <= kGrpProg ints, the A
  // values plus the peak contribution-block stack <= kGrpStack doubles.
  auto wof = [&](int s) { return Z.sn_first[s + 1] - Z.sn_first[s]; };
  auto nrof = [&](int s) { return static_cast<int>(Z.sn_rptr[s + 1] - Z.sn_rptr[s]); };
  auto cbof = [&](int s) {
    const int64_t m2 = nrof(s) - wof(s);
    return m2 * (m2 + 1) / 2;
  };
  std::vector<uint8_t> fits(nsn, 0);
  std::vector<int64_t> prog(nsn, 0), na(nsn, 0), stk(nsn, 0);
  for (int i = 0; i < split; ++i) {
    const int s = list[i];
    // batched (register-front) nodes are never grouped; a group reads their
    // CBs as EXTERNAL children from the standard CB layout (they finished in
    // an earlier launch)
    bool ok = nrof(s) <= kGrpFront && !batched[s];
    int64_t pr = 14 + 2 * (Z.a_ptr[s + 1] - Z.a_ptr[s]), a = Z.a_ptr[s + 1] - Z.a_ptr[s], pk = 0, run = 0;
    for (int q = Z.cptr[s]; q < Z.cptr[s + 1]; ++q) {
      const int c = Z.child[q];
      if (batched[c]) {
        pr += 7 + (nrof(c) - wof(c));
        continue;
      }
      ok = ok && fits[c];
      pr += prog[c] + 2 + (nrof(c) - wof(c));
      a += na[c];
      pk = std::max(pk, run + stk[c]);
      run += cbof(c);
    }
    pk = std::max(pk, run);
    prog[s] = pr;
    na[s] = a;
    stk[s] = pk;
    fits[s] = ok && pr + 4 <= kGrpProg && pk + a <= kGrpStack;
  }
  L.tptr.push_back(0);
  L.gpo.push_back(0);
  std::vector<std::pair<int, int>> st;  // (node, next child cursor)
  std::vector<int> post;
  std::vector<int> cboff(nsn, -1);  // stack offset of a pushed CB (set before its parent reads it)
  for (int i = 0; i < split; ++i) {
    const int r = list[i], p = Z.sn_parent[r];
    if (!fits[r] || (p >= 0 && warp[p] && fits[p])) continue;
    post.clear();
    st.emplace_back(r, Z.cptr[r]);  // postorder DFS, children ascending
    while (!st.empty()) {
      auto& top = st.back();
      if (top.second < Z.cptr[top.first + 1]) {
        const int c = Z.child[top.second++];
        if (!batched[c]) st.emplace_back(c, Z.cptr[c]);  // external children are not group members
      } else {
        post.push_back(top.first);
        st.pop_back();
      }
    }
    L.nodes.insert(L.nodes.end(), post.begin(), post.end());
    L.tptr.push_back(static_cast<int>(L.nodes.size()));
    // program: [nnodes, nA, tab, len] [aoff x nA] [asrc x nA] then per node
    // [s, f, w, nr, nch, push_off(-1 = root), a_first, a_cnt, loff lo/hi, cboff lo/hi, rptr lo/hi] and per child
    // [m2c, stack_off, rel x m2c] ([m2c, -1, cboff lo/hi, cvoff lo/hi, child, rel x m2c] for an external child),
    // then the record offsets [tab .. tab + nnodes);
    // stack offsets from a postorder simulation
    const size_t base = L.prog.size();
    const int nA = static_cast<int>(na[r]);
    L.prog.insert(L.prog.end(), {static_cast<int>(post.size()), nA, 0, 0});
    const size_t aoff0 = L.prog.size();
    L.prog.resize(aoff0 + 2 * static_cast<size_t>(nA));
    int top = 0, afirst = 0;
    std::vector<int> rec_off;  // node record offsets (table appended after the records)
    rec_off.reserve(post.size());
    for (int s : post) {
      const int acnt = static_cast<int>(Z.a_ptr[s + 1] - Z.a_ptr[s]);
      for (int e = 0; e < acnt; ++e) {
        const int off = Z.a_off[Z.a_ptr[s] + e], nr_s = nrof(s);  // panel offset -> packed-lower front offset
        L.prog[aoff0 + afirst + e] = static_cast<int>(cb_col(off / nr_s, nr_s)) + off % nr_s;
        L.prog[aoff0 + nA + afirst + e] = Z.a_src[Z.a_ptr[s] + e];
      }
      int pop = 0;
      for (int q = Z.cptr[s]; q < Z.cptr[s + 1]; ++q)
        if (!batched[Z.child[q]]) pop += static_cast<int>(cbof(Z.child[q]));
      const int push = s == r ? -1 : top - pop;
      const int64_t lo = Z.sn_loff[s], cbo = Z.cb_off[s], rp = Z.sn_rptr[s];
      rec_off.push_back(static_cast<int>(L.prog.size() - base));
      L.prog.insert(L.prog.end(), {s, Z.sn_first[s], wof(s), nrof(s), Z.cptr[s + 1] - Z.cptr[s], push, afirst, acnt,
                                   static_cast<int>(lo & 0xffffffff), static_cast<int>(lo >> 32),
                                   static_cast<int>(cbo & 0xffffffff), static_cast<int>(cbo >> 32),
                                   static_cast<int>(rp & 0xffffffff), static_cast<int>(rp >> 32)});
      for (int q = Z.cptr[s]; q < Z.cptr[s + 1]; ++q) {
        const int c = Z.child[q];
        const int m2c = nrof(c) - wof(c);
        L.prog.push_back(m2c);
        if (batched[c]) {
          // external child: its CB (factor) and its CV (forward solve) in the
          // standard layouts
          const int64_t cv = Z.sn_rptr[c] + wof(c);
          L.prog.push_back(-1);
          L.prog.push_back(static_cast<int>(Z.cb_off[c] & 0xffffffff));
          L.prog.push_back(static_cast<int>(Z.cb_off[c] >> 32));
          L.prog.push_back(static_cast<int>(cv & 0xffffffff));
          L.prog.push_back(static_cast<int>(cv >> 32));
          L.prog.push_back(c);  // its completion flag (the group may start before the register phase ends)
        } else {
          L.prog.push_back(cboff[c]);
        }
        for (int k = 0; k < m2c; ++k) L.prog.push_back(Z.relp[Z.sn_rptr[c] + wof(c) + k]);
      }
      top -= pop;
      if (s != r) {
        cboff[s] = top;
        top += static_cast<int>(cbof(s));
      }
      afirst += acnt;
    }
    L.prog[base + 2] = static_cast<int>(L.prog.size() - base);  // [2]: offset of the record-offset table
    L.prog.insert(L.prog.end(), rec_off.begin(), rec_off.end());
    L.prog[base + 3] = static_cast<int>(L.prog.size() - base);
    L.gpo.push_back(static_cast<int64_t>(L.prog.size()));
  }
  L.nleaf = static_cast<int>(L.tptr.size()) - 1;
  std::vector<uint8_t> grouped(nsn, 0);
  for (int s : L.nodes) grouped[s] = 1;
  for (int i = 0; i < split; ++i)
    if (!grouped[list[i]] && !batched[list[i]]) {
      L.nodes.push_back(list[i]);
      L.tptr.push_back(static_cast<int>(L.nodes.size()));
    }
  L.split = static_cast<int>(L.tptr.size()) - 1;
  for (int i = split; i < static_cast<int>(list.size()); ++i) {
    L.nodes.push_back(list[i]);
    L.tptr.push_back(static_cast<int>(L.nodes.size()));
  }
  // level schedule of the CTA part (task indices), large fronts per level
  TopSched& t = L.top;
  const int ntask = static_cast<int>(L.tptr.size()) - 1;
  auto node_of = [&](int task) { return L.nodes[L.tptr[task]]; };  // CTA-part tasks are single nodes
  for (int i = L.split; i < ntask;) {
    const int h = Z.height[node_of(i)];
    int e = i;
    std::vector<BigDesc> big;
    int lvl_max_nr = 0;
    while (e < ntask && Z.height[node_of(e)] == h) {
      const int s = node_of(e);
      const int nr = static_cast<int>(Z.sn_rptr[s + 1] - Z.sn_rptr[s]);
      if (!Z.big[s]) lvl_max_nr = std::max(lvl_max_nr, nr);
      if (Z.big[s]) {
        BigDesc b{};
        b.s = s;
        b.f = Z.sn_first[s];
        b.w = Z.sn_first[s + 1] - Z.sn_first[s];
        b.nr = nr;
        // panel width: 32 (the diagonal block is one warp, the rows below
        // stream through registers: no shared-memory cap on nr); the
        // NCL_BF_PANEL=1 A/B path stages the whole panel and keeps the cap
        static const bool staged = std::getenv("NCL_BF_PANEL") != nullptr;
        b.pw = 32;
        while (staged && b.pw > 8 && static_cast<int64_t>(nr) * b.pw * 8 > 220 * 1024) b.pw /= 2;
        b.npan = nr <= kCtaFront ? 0 : (b.w + b.pw - 1) / b.pw;  // one CTA (dev_big_cta)
        b.g0 = Z.gm_ptr[s];
        b.g1 = Z.gm_ptr[s + 1];
        // lanes per front entry in the assembly: ~4 sources per lane
        const int64_t nsrc = b.g1 > b.g0 ? Z.gsp[b.g1] - Z.gsp[b.g0] : 0;
        const int64_t per = b.g1 > b.g0 ? nsrc / (b.g1 - b.g0) : 0;
        b.gsz = 1;
        while (b.gsz < 32 && 4 * b.gsz < per) b.gsz *= 2;
        big.push_back(b);
        t.any_big = true;
        t.max_nr = std::max(t.max_nr, nr);
      }
      ++e;
    }
    // merge levels without large fronts into one segment (one persistent
    // launch, flags order them); a segment closes at a level holding large
    // fronts, which run (as one batch) after that level's small fronts
    // Levels whose fronts all fit kCtaFrontS rows form their own segments
    // (small CTAs, several per SM).
    const char small = lvl_max_nr <= kCtaFrontS;
    if (small) t.any_small = true;
    if (!t.lvl_begin.empty() && t.big.back().empty() && t.small.back() == small) {
      t.lvl_end.back() = e;
      t.big.back() = std::move(big);
    } else {
      t.lvl_begin.push_back(i);
      t.lvl_end.push_back(e);
      t.big.push_back(std::move(big));
      t.small.push_back(small);
    }
    i = e;
  }
  for (auto& seg : t.big) {  // scratch layout of each batch
    int64_t fo = 0, wo = 0;
    for (auto& b : seg) {
      b.foff = fo;
      b.woff = wo;
      fo += static_cast<int64_t>(b.nr) * b.nr;
      wo += static_cast<int64_t>(b.nr) * 32;
    }
    t.scratch_f = std::max(t.scratch_f, fo);
    t.scratch_w = std::max(t.scratch_w, wo);
  }
  return L;
}

// device copies of the per-segment large-front descriptors
void upload_top(TopSched& t, std::vector<DevBuf<BigDesc>>& store) {
  store.clear();
  store.resize(t.big.size());
  t.big_dev.assign(t.big.size(), nullptr);
  for (size_t k = 0; k < t.big.size(); ++k)
    if (!t.big[k].empty()) {
      store[k].upload(t.big[k]);
      t.big_dev[k] = store[k].p;
    }
}

DevTasks upload_layout(TaskLayout& L, LayoutDev& D, const Supernodal& Z) {
  upload_top(L.top, D.top);
  D.nodes.upload(L.nodes);
  D.tptr.upload(L.tptr);
  D.prog.upload(L.prog);
  D.gpo.upload(L.gpo);
  const bool has_batch = !L.batch.inst.empty();
  if (has_batch) {
    D.binst.upload(L.batch.inst);
    D.bamap.upload(L.batch.amap);
    D.bcmap.upload(L.batch.cmap);
    D.bcmapw.upload(L.batch.cmapw);
    L.batch.dev_cmapw = D.bcmapw.p;
    D.bccb.upload(L.batch.ccb);
    D.bcid.upload(L.batch.cid);
    D.bchunks.upload(L.batch.chunks);
    D.bsmapw.upload(L.batch.smapw);
    L.batch.dev_smapw = D.bsmapw.p;
    L.batch.dev_cid = D.bcid.p;
    L.batch.dev_chunks = D.bchunks.p;
    L.batch.dev_inst = D.binst.p;
    L.batch.dev_amap = D.bamap.p;
    L.batch.dev_cmap = D.bcmap.p;
    L.batch.dev_ccb = D.bccb.p;
  }
  DevTasks T{D.nodes.p, D.tptr.p, D.prog.p, D.gpo.p, static_cast<int>(L.tptr.size()) - 1, L.nleaf, L.split,
             &L.top, has_batch ? &L.batch : nullptr};
  // a last CTA task with many contributing children (the separator root)
  // gathers its contribution vectors GPU-wide in the forward solve
  if (T.n > T.split + 1) {
    const int s = L.nodes[L.tptr[T.n - 1]];
    if (s < static_cast<int>(Z.cv_ptr.size()) - 1 && Z.cv_ptr[s + 1] > Z.cv_ptr[s]) {
      const int nr = static_cast<int>(Z.sn_rptr[s + 1] - Z.sn_rptr[s]);
      const int64_t nsrc = Z.cvsp[Z.cv_ptr[s + 1]] - Z.cvsp[Z.cv_ptr[s]];
      if (nsrc > 32 * static_cast<int64_t>(nr) && nsrc >= 8192) {
        T.root_heavy = s;
        T.root_nr = nr;
      }
    }
  }
  return T;
}

void upload_symb(ncl_symb* S) {
  if (S->dev_ready) return;
  ensure_init();
  static const bool timing = std::getenv("NCL_ANALYZE_TIMING") != nullptr;
  auto t = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[upload]    %-16s %.3f s  (so far: cudaMalloc %.3f s, copies %.3f s, %.1f MB)\n", what,
                 std::chrono::duration<double>(now - t).count(), g_upload_stats[0] * 1e-9, g_upload_stats[1] * 1e-9,
                 g_upload_stats[2] * 1e-6);
    t = now;
  };
  const Supernodal& Z = S->Z;
  S->perm.upload(S->core.perm);
  S->sn_first.upload(Z.sn_first);
  S->sn_parent.upload(Z.sn_parent);
  S->rows.upload(Z.rows);
  S->relp.upload(Z.relp);
  S->cptr.upload(Z.cptr);
  S->child.upload(Z.child);
  S->order.upload(Z.order);
  S->sn_rptr.upload(Z.sn_rptr);
  S->sn_loff.upload(Z.sn_loff);
  S->cb_off.upload(Z.cb_off);
  S->gm_ptr.upload(Z.gm_ptr);
  S->gdst.upload(Z.gdst);
  S->gsp.upload(Z.gsp);
  S->gsrc.upload(Z.gsrc);
  S->big.upload(Z.big);
  S->cv_ptr.upload(Z.cv_ptr);
  S->cvsp.upload(Z.cvsp);
  S->cvsrc.upload(Z.cvsrc);
  lap("symbolic arrays");
  if (!S->lay.tptr.empty()) {  // the unbatched layout exists only for NCL_*NO_BATCH A/B runs
    upload_top(S->lay.top, S->top_dev);
    S->lay_nodes.upload(S->lay.nodes);
    S->lay_prog.upload(S->lay.prog);
    S->lay_gpo.upload(S->lay.gpo);
    S->lay_tptr.upload(S->lay.tptr);
  }
  // A entries grouped by target supernode (Supernodal::a_ptr/a_src/a_off)
  const int nsn = Z.nsn;
  const std::vector<int64_t>& aptr = Z.a_ptr;
  S->aptr.upload(Z.a_ptr);
  S->asrc.upload(Z.a_src);
  S->aoff.upload(Z.a_off);
  {
    std::vector<int> ap(Z.a_off.size());
    for (int s = 0; s < nsn; ++s) {
      const int nr = static_cast<int>(Z.sn_rptr[s + 1] - Z.sn_rptr[s]);
      for (int64_t e = aptr[s]; e < aptr[s + 1]; ++e)
        ap[e] = static_cast<int>(cb_col(Z.a_off[e] / nr, nr) + Z.a_off[e] % nr);
    }
    S->aoffp.upload(ap);
  }
  lap("A maps");
  {
    std::vector<SnMeta> mv(nsn);
    for (int s = 0; s < nsn; ++s) {
      SnMeta& m = mv[s];
      m.loff = Z.sn_loff[s];
      m.cboff = Z.cb_off[s];
      m.rptr = Z.sn_rptr[s];
      m.a0 = aptr[s];
      m.na = static_cast<int>(aptr[s + 1] - aptr[s]);
      m.f = Z.sn_first[s];
      m.w = Z.sn_first[s + 1] - Z.sn_first[s];
      m.nr = static_cast<int>(Z.sn_rptr[s + 1] - Z.sn_rptr[s]);
      m.c0 = Z.cptr[s];
      m.c1 = Z.cptr[s + 1];
      m.parent = Z.sn_parent[s];
      m.pad = 0;
    }
    S->meta.upload(mv);
    std::vector<ChildRec> cr(Z.child.size());
    for (size_t q = 0; q < Z.child.size(); ++q) {
      const int c = Z.child[q];
      cr[q].cboff = Z.cb_off[c];
      cr[q].rel = static_cast<int>(Z.sn_rptr[c] + (Z.sn_first[c + 1] - Z.sn_first[c]));
      cr[q].m2c = static_cast<int>(Z.sn_rptr[c + 1] - Z.sn_rptr[c]) - (Z.sn_first[c + 1] - Z.sn_first[c]);
    }
    S->chrec.upload(cr);
  }
  lap("records");
  S->flags.alloc(3 * std::max(1, nsn));
  ck(cudaMemsetAsync(S->flags.p, 0, 3 * std::max(1, nsn) * sizeof(int), g_stream), "memset");
  S->tickets.alloc(kTickets);
  DevSymb& d = S->d;
  d.n = S->core.n;
  d.nsn = nsn;
  d.nleaf = Z.nleaf;
  d.nsplit = Z.nsplit;
  d.cb_storage = Z.cb_storage;
  d.nnz = S->nnz;
  d.l_storage = Z.l_storage;
  d.perm = S->perm.p;
  d.sn_first = S->sn_first.p;
  d.sn_parent = S->sn_parent.p;
  d.sn_rptr = S->sn_rptr.p;
  d.rows = S->rows.p;
  d.sn_loff = S->sn_loff.p;
  d.relp = S->relp.p;
  d.cb_off = S->cb_off.p;
  d.gm_ptr = S->gm_ptr.p;
  d.gdst = S->gdst.p;
  d.gsp = S->gsp.p;
  d.gsrc = S->gsrc.p;
  d.big = S->big.p;
  d.cv_ptr = S->cv_ptr.p;
  d.cvsp = S->cvsp.p;
  d.cvsrc = S->cvsrc.p;
  d.meta = S->meta.p;
  d.ftasks = upload_layout(S->flay, S->fdev, Z);
  lap("layout");
  d.tasks = S->lay.tptr.empty()
                ? d.ftasks
                : DevTasks{S->lay_nodes.p, S->lay_tptr.p, S->lay_prog.p, S->lay_gpo.p,
                           static_cast<int>(S->lay.tptr.size()) - 1, S->lay.nleaf, S->lay.split, &S->lay.top};
  d.cptr = S->cptr.p;
  d.child = S->child.p;
  d.chrec = S->chrec.p;
  d.order = S->order.p;
  d.aptr = S->aptr.p;
  d.asrc = S->asrc.p;
  d.aoff = S->aoff.p;
  d.aoffp = S->aoffp.p;
  d.flags = S->flags.p;
  d.tickets = S->tickets.p;
  d.epoch = 0;
  if (Z.l_storage >= (int64_t(1) << 31) || static_cast<int64_t>(Z.amap.size()) >= (int64_t(1) << 31) ||
      static_cast<int64_t>(Z.rows.size()) >= (int64_t(1) << 31))
    throw Error{NCL_E_INVALID, "analyze: factor exceeds int32 panel addressing"};
  S->dev_ready = true;
}
}  // namespace

namespace nclb {
int symb_prepare_device(ncl_symb_t S) {
  try {
    upload_symb(S);
  } catch (...) {
    return map_exc();
  }
  return NCL_OK;
}
}  // namespace nclb

API int ncl_symbolic_order(ncl_sym_t M, int* perm) {
  GUARD({
    if (!M->pat.finalized()) throw Error{NCL_E_LOGIC, "symbolic_order: pattern not finalized"};
    auto p = symbolic_order(M->pat.dim(), M->pat.col_ptr(), M->pat.row_ind());
    if (!p.empty()) std::memcpy(perm, p.data(), p.size() * sizeof(int));
  });
}

ncl_symb* analyze_impl(ncl_sym_t M, const int* perm) {
  if (!M->pat.finalized()) throw Error{NCL_E_LOGIC, "analyze: matrix not finalized"};
  const int n = M->pat.dim();
  // NCL_ANALYZE_TIMING=1: per-phase host seconds on stderr
  static const bool timing = std::getenv("NCL_ANALYZE_TIMING") != nullptr;
  auto t = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[analyze] %-16s %.3f s\n", what, std::chrono::duration<double>(now - t).count());
    t = now;
  };
  std::vector<int> p = perm ? std::vector<int>(perm, perm + n)
                            : symbolic_order(n, M->pat.col_ptr(), M->pat.row_ind());
  lap("symbolic_order");
  auto S = std::make_unique<ncl_symb>();
  S->core = analyze_core(n, M->pat.col_ptr(), M->pat.row_ind(), std::move(p));
  lap("analyze_core");
  S->Z = build_supernodes(S->core, M->pat.col_ptr(), M->pat.row_ind());
  lap("build_supernodes");
  // factor and solves run on the batched layout (register fronts split off);
  // the unbatched one is built only for the NCL_NO_BATCH / NCL_SOLVE_NO_BATCH
  // A/B switches
  static const bool unbatched = std::getenv("NCL_NO_BATCH") || std::getenv("NCL_SOLVE_NO_BATCH");
  if (unbatched) S->lay = build_layout(S->Z, S->Z.order, S->Z.nsplit);
  S->flay = build_layout(S->Z, S->Z.order, S->Z.nsplit, true);
  lap("build_layout");
  S->hash = M->hash;
  S->nnz = M->pat.nnz();
  return S.release();
}

API int ncl_analyze(ncl_sym_t M, const int* perm, ncl_symb_t* out) { GUARD(*out = analyze_impl(M, perm)); }
API void ncl_symb_destroy(ncl_symb_t S) { delete S; }
API int ncl_symb_info_get(ncl_symb_t S, ncl_symb_info* info) {
  GUARD({
    info->n = S->core.n;
    info->l_nnz = S->core.l_nnz;
    info->nsupernodes = S->Z.nsn;
    info->max_height = S->Z.max_height;
    info->max_width = S->Z.max_w;
    info->max_rows = S->Z.max_nr;
    info->l_storage = S->Z.l_storage;
    info->flops = S->Z.flops;
    info->cb_storage = S->Z.cb_storage;
    info->nsplit = S->Z.nsplit;
    int nb = 0;
    for (const auto& lv : S->flay.top.big) nb += static_cast<int>(lv.size());
    info->n_big = nb;
    info->n_tasks = static_cast<int>(S->flay.tptr.size()) - 1 + static_cast<int>(S->flay.batch.inst.size());
  });
}
API int ncl_symb_supernodes(ncl_symb_t S, int* sn_first, int64_t* sn_rptr, int* sn_parent, int* height,
                            int* order) {
  GUARD({
    const Supernodal& Z = S->Z;
    auto cp = [](auto* dst, const auto& v) {
      if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(sn_first, Z.sn_first);
    cp(sn_rptr, Z.sn_rptr);
    cp(sn_parent, Z.sn_parent);
    cp(height, Z.height);
    cp(order, Z.order);
  });
}
API int ncl_symb_get(ncl_symb_t S, int* perm, int* iperm, int* parent, int* up_colptr, int* up_rowind,
                     int* entry_map, int* l_colcount) {
  GUARD({
    auto cp = [](int* dst, const std::vector<int>& v) {
      if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(int));
    };
    cp(perm, S->core.perm);
    cp(iperm, S->core.iperm);
    cp(parent, S->core.parent);
    cp(up_colptr, S->core.up_colptr);
    cp(up_rowind, S->core.up_rowind);
    cp(entry_map, S->core.entry_map);
    cp(l_colcount, S->core.l_colcount);
  });
}

// ---------------------------------------------------------------------------
// Numeric factorization
// ---------------------------------------------------------------------------
struct ncl_fact {
  ncl_symb* S = nullptr;
  std::unique_ptr<ncl_symb> owned;
  DevFactor F;
  DevBuf<double> L, CB, CV, D, xp, scal, work1, work2, work3, bigF, bigW;
  DevBuf<int> istat;
  // > 1 after a sharded refactorization of a world > 1 run: L / D hold only
  // this rank's supernodes (plus the shared separator), so the whole-factor
  // getters refuse it
  int sharded_world = 1;
};

namespace {
void check_match(ncl_sym_t M, ncl_symb* S) {
  if (M->pat.dim() != S->core.n || M->pat.nnz() != S->nnz)
    throw Error{NCL_E_INVALID, "factorize: matrix does not match symbolic analysis"};
  if (M->hash != S->hash) throw Error{NCL_E_INVALID, "factorize: matrix pattern differs from the analyzed pattern"};
}
void alloc_fact(ncl_fact* f) {
  const int n = f->S->core.n;
  f->L.alloc(std::max<int64_t>(1, f->S->Z.l_storage));
  f->CB.alloc(std::max<int64_t>(1, f->S->Z.cb_storage));
  f->CV.alloc(std::max<int64_t>(1, static_cast<int64_t>(f->S->Z.rows.size())));
  f->D.alloc(std::max(1, n));
  f->xp.alloc(std::max(1, n));
  f->scal.alloc(8);
  f->istat.alloc(8);
  f->work1.alloc(std::max(1, n));
  f->work2.alloc(std::max(1, n));
  f->work3.alloc(std::max(1, n));
  f->F.L = f->L.p;
  f->F.CB = f->CB.p;
  f->F.CV = f->CV.p;
  if (f->S->flay.top.any_big) {  // scratch of the batched large-front path
    f->bigF.alloc(f->S->flay.top.scratch_f);
    f->bigW.alloc(f->S->flay.top.scratch_w);
    f->F.bigF = f->bigF.p;
    f->F.bigW = f->bigW.p;
  }
  f->F.D = f->D.p;
  f->F.xp = f->xp.p;
  f->F.scal = f->scal.p;
  f->F.istat = f->istat.p;
}
void run_factor(ncl_fact* f, ncl_sym_t M, double tol) {
  // NCL_TASK_TRACE=<file>: per-task globaltimer start/end of the next
  // factorization (debug timeline of the persistent schedule)
  static const char* trace_path = std::getenv("NCL_TASK_TRACE");
  static int traced = 0;
  static DevBuf<unsigned long long> tbuf, pbuf;
  const int ntask = f->S->d.ftasks.n;
  const int64_t nsn = static_cast<int64_t>(f->S->Z.sn_first.size()) - 1;
  if (trace_path && traced == 2) {
    tbuf.alloc(2 * static_cast<int64_t>(ntask));
    ck(cudaMemsetAsync(tbuf.p, 0, 2 * ntask * sizeof(unsigned long long), g_stream), "memset");
    g_task_trace = tbuf.p;
    pbuf.alloc(4 * nsn);
    ck(cudaMemsetAsync(pbuf.p, 0, 4 * nsn * sizeof(unsigned long long), g_stream), "memset");
    dev_phase_trace(pbuf.p);
  }
  dev_factor(f->S->d, M->dp, f->F, M->vals.p, tol, g_stream, nullptr);
  if (trace_path && traced++ == 2) {
    g_task_trace = nullptr;
    std::vector<unsigned long long> h;
    tbuf.download(h, 2 * static_cast<int64_t>(ntask));
    if (FILE* fp = std::fopen(trace_path, "wb")) {
      const int hdr[4] = {ntask, f->S->d.ftasks.nleaf, f->S->d.ftasks.split, 0};
      std::fwrite(hdr, sizeof(int), 4, fp);
      std::fwrite(h.data(), sizeof(unsigned long long), h.size(), fp);
      std::fwrite(f->S->flay.tptr.data(), sizeof(int), f->S->flay.tptr.size(), fp);
      std::fwrite(f->S->flay.nodes.data(), sizeof(int), f->S->flay.nodes.size(), fp);
      std::fclose(fp);
    }
    dev_phase_trace(nullptr);
    std::vector<unsigned long long> hp;
    pbuf.download(hp, 4 * nsn);
    if (FILE* fp = std::fopen((std::string(trace_path) + ".phase").c_str(), "wb")) {
      std::fwrite(hp.data(), sizeof(unsigned long long), hp.size(), fp);
      std::fclose(fp);
    }
  }
  dev_inertia(f->S->d, f->F, g_stream);
  check_launch("factorize");
}
}  // namespace

API int ncl_factorize(ncl_sym_t M, ncl_symb_t S, double pivot_tol, ncl_fact_t* out) {
  GUARD({
    if (!M->pat.finalized()) throw Error{NCL_E_LOGIC, "factorize: matrix not finalized"};
    auto f = std::make_unique<ncl_fact>();
    if (S) {
      f->S = S;
    } else {
      f->owned.reset(analyze_impl(M, nullptr));
      f->S = f->owned.get();
    }
    check_match(M, f->S);
    // NCL_ANALYZE_TIMING=1: the one-time costs of the first factorization
    static const bool timing = std::getenv("NCL_ANALYZE_TIMING") != nullptr;
    auto t = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
      if (!timing) return;
      ck(cudaStreamSynchronize(g_stream), "sync");
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[factorize] %-16s %.3f s\n", what, std::chrono::duration<double>(now - t).count());
      t = now;
    };
    ensure_dev(M, "factorize");
    lap("matrix upload");
    upload_symb(f->S);
    lap("symbolic upload");
    alloc_fact(f.get());
    lap("factor alloc");
    run_factor(f.get(), M, pivot_tol);
    ck(cudaStreamSynchronize(g_stream), "factorize");
    lap("first factor");
    *out = f.release();
  });
}
API int ncl_refactorize(ncl_fact_t F, ncl_sym_t M, double pivot_tol) {
  GUARD({
    check_match(M, F->S);
    ensure_dev(M, "factorize");
    run_factor(F, M, pivot_tol);
    F->sharded_world = 1;
  });
}
API void ncl_fact_destroy(ncl_fact_t F) { delete F; }
API int ncl_fact_status(ncl_fact_t F, int* status, int* zpi, int* np, int* nn, int* nz) {
  GUARD({
    int h[4];
    ck(cudaMemcpyAsync(h, F->istat.p, sizeof(h), cudaMemcpyDeviceToHost, g_stream), "D2H");
    ck(cudaStreamSynchronize(g_stream), "sync");
    const int n = F->S->core.n;
    if (h[0] < n) {
      *status = 1;
      *zpi = F->S->core.perm[h[0]];
      *np = *nn = *nz = 0;
    } else {
      *status = 0;
      *zpi = -1;
      *np = h[1];
      *nn = h[2];
      *nz = h[3];
    }
  });
}
API int ncl_fact_diagonal(ncl_fact_t F, double* d) {
  GUARD({
    if (F->sharded_world > 1)
      throw Error{NCL_E_LOGIC, "diagonal: factor of a sharded world > 1 run (use ncl_shard_diagonal)"};
    const int n = F->S->core.n;
    if (n > 0) ck(cudaMemcpyAsync(d, F->D.p, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
    ck(cudaStreamSynchronize(g_stream), "sync");
  });
}
namespace {
bool fact_ok_sync(ncl_fact_t F) {
  int h = 0;
  ck(cudaMemcpyAsync(&h, F->istat.p, sizeof(int), cudaMemcpyDeviceToHost, g_stream), "D2H");
  ck(cudaStreamSynchronize(g_stream), "sync");
  return h >= F->S->core.n;
}
}  // namespace
API int ncl_fact_solve(ncl_fact_t F, double* x, int where) {
  GUARD({
    if (F->sharded_world > 1) throw Error{NCL_E_LOGIC, "solve: factor of a sharded world > 1 run (use ncl_shard_solve)"};
    const int n = F->S->core.n;
    if (where == NCL_DEVICE) {
      dev_solve(F->S->d, F->F, x, x, g_stream);
      check_launch("solve");
      return NCL_OK;
    }
    ck(cudaMemcpyAsync(F->work1.p, x, n * sizeof(double), cudaMemcpyHostToDevice, g_stream), "H2D");
    dev_solve(F->S->d, F->F, F->work1.p, F->work1.p, g_stream);
    check_launch("solve");
    ck(cudaMemcpyAsync(x, F->work1.p, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
    ck(cudaStreamSynchronize(g_stream), "sync");
  });
}

// solve_refined (sparse_sym.cpp:371-401): x = F\b; up to max_sweeps
// refinement sweeps while ||b - Mx||_inf / max(1,||b||_inf) > target.
// The residual norm decision needs one scalar D2H per sweep.
int solve_refined_dev(ncl_fact_t F, ncl_sym_t M, const double* db, double* dx, double target, int max_sweeps,
                      double* residual, int* sweeps, int* converged) {
  const int n = F->S->core.n;
  double* r = F->work2.p;
  double* sc = F->scal.p + 4;  // [4]=bnorm [5]=rnorm
  dev_solve(F->S->d, F->F, db, dx, g_stream);
  ck(cudaMemsetAsync(sc, 0, sizeof(double), g_stream), "memset");
  dev_absmax(db, n, sc, g_stream);
  double bnorm = 0;
  ck(cudaMemcpyAsync(&bnorm, sc, sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
  ck(cudaStreamSynchronize(g_stream), "sync");
  const double scale = std::max(1.0, bnorm);
  *converged = 0;
  *residual = std::numeric_limits<double>::infinity();
  for (int sweep = 0; sweep <= max_sweeps; ++sweep) {
    dev_residual(M->dp, M->vals.p, db, dx, r, sc + 1, g_stream);
    double rn = 0;
    ck(cudaMemcpyAsync(&rn, sc + 1, sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
    ck(cudaStreamSynchronize(g_stream), "sync");
    *residual = rn / scale;
    *sweeps = sweep;
    if (*residual <= target) {
      *converged = 1;
      return NCL_OK;
    }
    if (sweep == max_sweeps) break;
    dev_solve(F->S->d, F->F, r, r, g_stream);
    dev_axpy_inplace(dx, r, n, g_stream);
  }
  check_launch("solve_refined");
  return NCL_OK;
}

API int ncl_solve_refined(ncl_fact_t F, ncl_sym_t M, const double* b, double target, int max_sweeps, double* x,
                          int where, double* residual, int* sweeps, int* converged) {
  GUARD({
    if (F->sharded_world > 1) throw Error{NCL_E_LOGIC, "solve_refined: factor of a sharded world > 1 run"};
    if (!fact_ok_sync(F)) throw Error{NCL_E_LOGIC, "solve_refined: factorization not usable"};
    check_match(M, F->S);
    ensure_dev(M, "solve_refined");
    const int n = F->S->core.n;
    if (where == NCL_DEVICE) {
      solve_refined_dev(F, M, b, x, target, max_sweeps, residual, sweeps, converged);
      return NCL_OK;
    }
    ck(cudaMemcpyAsync(F->work3.p, b, n * sizeof(double), cudaMemcpyHostToDevice, g_stream), "H2D");
    solve_refined_dev(F, M, F->work3.p, F->work1.p, target, max_sweeps, residual, sweeps, converged);
    ck(cudaMemcpyAsync(x, F->work1.p, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
    ck(cudaStreamSynchronize(g_stream), "sync");
  });
}

// One factor + solve from host buffers with a single synchronisation: the
// values' H2D and the factorization on the library stream, the right-hand
// side's H2D on a copy stream underneath the factorization, then the solve,
// the D2H of x and of the status words.
API int ncl_factor_solve_host(ncl_fact_t F, ncl_sym_t M, const double* vals, const double* b, double* x,
                              double pivot_tol, int* status, int* zero_pivot_index, int* n_pos, int* n_neg,
                              int* n_zero) {
  GUARD({
    if (F->sharded_world > 1) throw Error{NCL_E_LOGIC, "factor_solve: factor of a sharded world > 1 run"};
    check_match(M, F->S);
    ensure_dev(M, "factor_solve");
    static cudaStream_t cs = nullptr;
    static cudaEvent_t eb = nullptr;
    if (!cs) {
      ck(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "cudaStreamCreate");
      ck(cudaEventCreateWithFlags(&eb, cudaEventDisableTiming), "event");
    }
    const int n = F->S->core.n;
    const int64_t nz = M->pat.nnz();
    // the copy stream may only overwrite work1 once the previous solve is done
    ck(cudaEventRecord(eb, g_stream), "event");
    ck(cudaStreamWaitEvent(cs, eb, 0), "wait");
    if (n > 0) ck(cudaMemcpyAsync(F->work1.p, b, n * sizeof(double), cudaMemcpyHostToDevice, cs), "H2D b");
    ck(cudaEventRecord(eb, cs), "event");
    ck(cudaMemcpyAsync(M->vals.p, vals, nz * sizeof(double), cudaMemcpyHostToDevice, g_stream), "H2D values");
    run_factor(F, M, pivot_tol);
    F->sharded_world = 1;
    ck(cudaStreamWaitEvent(g_stream, eb, 0), "wait");
    dev_solve(F->S->d, F->F, F->work1.p, F->work1.p, g_stream);
    if (n > 0) ck(cudaMemcpyAsync(x, F->work1.p, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H x");
    int h[4];
    ck(cudaMemcpyAsync(h, F->istat.p, sizeof(h), cudaMemcpyDeviceToHost, g_stream), "D2H status");
    ck(cudaStreamSynchronize(g_stream), "sync");
    check_launch("factor_solve");
    if (h[0] < n) {
      *status = 1;
      *zero_pivot_index = F->S->core.perm[h[0]];
      *n_pos = *n_neg = *n_zero = 0;
    } else {
      *status = 0;
      *zero_pivot_index = -1;
      *n_pos = h[1];
      *n_neg = h[2];
      *n_zero = h[3];
    }
  });
}

API int ncl_fact_get_L(ncl_fact_t F, int* lp, int* li, double* lx) {
  GUARD({
    if (F->sharded_world > 1) throw Error{NCL_E_LOGIC, "get_L: factor of a sharded world > 1 run"};
    const Supernodal& Z = F->S->Z;
    const int n = F->S->core.n;
    std::vector<double> Lh(Z.l_storage);
    if (Z.l_storage > 0)
      ck(cudaMemcpyAsync(Lh.data(), F->L.p, Z.l_storage * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
    ck(cudaStreamSynchronize(g_stream), "sync");
    // reference layout: only the true structure of L (amalgamated panels
    // also hold explicit zeros outside it)
    std::vector<int64_t> tp;
    std::vector<int> ti;
    true_L_structure(F->S->core, tp, ti);
    for (int j = 0; j <= n; ++j)
      if (lp) lp[j] = static_cast<int>(tp[j]);
    for (int j = 0; j < n; ++j) {
      const int s = Z.sn_of_col[j], f = Z.sn_first[s];
      const int64_t rb = Z.sn_rptr[s];
      const int nr = static_cast<int>(Z.sn_rptr[s + 1] - rb);
      const int* R = Z.rows.data() + rb;
      int q = 0;
      for (int64_t p = tp[j]; p < tp[j + 1]; ++p) {
        const int r = ti[p];
        while (R[q] < r) ++q;
        if (li) li[p] = r;
        if (lx) lx[p] = Lh[Z.sn_loff[s] + static_cast<int64_t>(j - f) * nr + q];
      }
    }
  });
}

// ---------------------------------------------------------------------------
// Multi-GPU: NCCL (dlopen'd, so the library shares the process's libnccl.so.2
// with torch) and the contingency-sharded factor / solve (csrc/host/shard.hpp)
// ---------------------------------------------------------------------------
#include <dlfcn.h>
#include <nccl.h>

#include "../../include/nclopf_dist.h"
#include "host/shard.hpp"

namespace {
struct Nccl {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) get_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGetErrorString) err = nullptr;
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0;
};
Nccl g_nccl;
void nccl_load() {
  if (g_nccl.h) return;
  g_nccl.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!g_nccl.h) throw Error{NCL_E_CUDA, std::string("NCCL not loadable: ") + dlerror()};
  auto sym = [](const char* n) {
    void* p = dlsym(g_nccl.h, n);
    if (!p) throw Error{NCL_E_CUDA, std::string("NCCL symbol missing: ") + n};
    return p;
  };
  g_nccl.get_id = reinterpret_cast<decltype(g_nccl.get_id)>(sym("ncclGetUniqueId"));
  g_nccl.init_rank = reinterpret_cast<decltype(g_nccl.init_rank)>(sym("ncclCommInitRank"));
  g_nccl.all_gather = reinterpret_cast<decltype(g_nccl.all_gather)>(sym("ncclAllGather"));
  g_nccl.all_reduce = reinterpret_cast<decltype(g_nccl.all_reduce)>(sym("ncclAllReduce"));
  g_nccl.destroy = reinterpret_cast<decltype(g_nccl.destroy)>(sym("ncclCommDestroy"));
  g_nccl.err = reinterpret_cast<decltype(g_nccl.err)>(sym("ncclGetErrorString"));
}
void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error{NCL_E_CUDA, std::string(what) + ": " + g_nccl.err(r)};
}
}  // namespace

API int ncl_dist_get_unique_id(char* id) {
  GUARD({
    nccl_load();
    ncclUniqueId u;
    nck(g_nccl.get_id(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  });
}
API int ncl_dist_init(int world, int rank, const char* id) {
  GUARD({
    ensure_init();
    nccl_load();
    if (g_nccl.comm) throw Error{NCL_E_LOGIC, "ncl_dist_init: already initialised"};
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    nck(g_nccl.init_rank(&g_nccl.comm, world, u, rank), "ncclCommInitRank");
    g_nccl.world = world;
    g_nccl.rank = rank;
  });
}
API int ncl_dist_finalize(void) {
  GUARD({
    if (g_nccl.comm) g_nccl.destroy(g_nccl.comm);
    g_nccl.comm = nullptr;
    g_nccl.world = 1;
    g_nccl.rank = 0;
  });
}

struct ncl_shard {
  ShardPlan P;
  ncl_symb* S = nullptr;
  bool dev_ready = false;
  DevBuf<int> bids, bowner;
  DevBuf<int64_t> cb_off, cv_off;
  DevBuf<uint8_t> report;
  DevBuf<double> send, recv;
  DevBuf<int> unrep;  // original indices this rank does not report (zeroed before the x all-reduce)
  TaskLayout flayA, flayB;  // phase A / B task layouts (register fronts split off)
  LayoutDev fdevA, fdevB;
  DevTasks ftA{}, ftB{};
  int64_t nunrep = 0;
};

namespace {
void shard_upload(ncl_shard* sh) {
  if (sh->dev_ready) return;
  ensure_init();
  upload_symb(sh->S);
  sh->ftA = upload_layout(sh->flayA, sh->fdevA, sh->S->Z);
  sh->ftB = upload_layout(sh->flayB, sh->fdevB, sh->S->Z);
  sh->bids.upload(sh->P.boundary);
  sh->bowner.upload(sh->P.bowner);
  sh->cb_off.upload(sh->P.cb_pack_off);
  sh->cv_off.upload(sh->P.cv_pack_off);
  sh->report.upload(sh->P.col_report);
  {
    std::vector<int> u;
    const auto& perm = sh->S->core.perm;
    for (size_t j = 0; j < sh->P.col_report.size(); ++j)
      if (!sh->P.col_report[j]) u.push_back(perm[j]);
    sh->nunrep = static_cast<int64_t>(u.size());
    sh->unrep.upload(u);
  }
  const int64_t chunk = std::max(sh->P.cb_chunk, sh->P.cv_chunk);
  sh->send.alloc(std::max<int64_t>(1, chunk));
  sh->recv.alloc(std::max<int64_t>(1, chunk * sh->P.world));
  sh->dev_ready = true;
}
void grow_scratch(ncl_fact* F, ncl_shard* sh) {
  const int64_t nf = std::max(sh->flayA.top.scratch_f, sh->flayB.top.scratch_f);
  const int64_t nw = std::max(sh->flayA.top.scratch_w, sh->flayB.top.scratch_w);
  if (nf > 0) {
    F->bigF.alloc(std::max<int64_t>(nf, F->bigF.n));
    F->bigW.alloc(std::max<int64_t>(nw, F->bigW.n));
    F->F.bigF = F->bigF.p;
    F->F.bigW = F->bigW.p;
  }
}
void need_comm(const ncl_shard* sh) {
  if (sh->P.world == 1) return;
  if (!g_nccl.comm || g_nccl.world != sh->P.world || g_nccl.rank != sh->P.rank)
    throw Error{NCL_E_LOGIC, "sharded call needs ncl_dist_init with the plan's world/rank"};
}
// The boundary exchange in three steps so that the transport is pluggable:
// pack (device kernel) -> all-gather of `chunk` doubles per rank (NCCL here,
// or the caller's own transport in the split-phase API) -> unpack (device
// kernel, publishes the separator's completion flags).
int64_t xchunk(const ncl_shard* sh, int cv) { return cv ? sh->P.cv_chunk : sh->P.cb_chunk; }
void pack_blocks(ncl_shard* sh, const double* base, int cv) {
  const ShardPlan& P = sh->P;
  const int nb = static_cast<int>(P.boundary.size());
  if (nb == 0 || xchunk(sh, cv) == 0) return;
  dev_shard_pack(sh->S->d, base, sh->bids.p, sh->bowner.p, cv ? sh->cv_off.p : sh->cb_off.p, nb, P.rank, cv,
                 sh->send.p, g_stream);
}
void unpack_blocks(ncl_shard* sh, double* base, int cv, int* flags, int epoch, const double* recv) {
  const ShardPlan& P = sh->P;
  const int nb = static_cast<int>(P.boundary.size());
  if (nb == 0 || xchunk(sh, cv) == 0) return;
  dev_shard_unpack(sh->S->d, base, sh->bids.p, sh->bowner.p, cv ? sh->cv_off.p : sh->cb_off.p, nb, P.rank, cv, recv,
                   xchunk(sh, cv), flags, epoch, g_stream);
}
void allgather_blocks(ncl_shard* sh, double* base, int cv, int* flags, int epoch) {
  const int64_t chunk = xchunk(sh, cv);
  if (sh->P.boundary.empty() || chunk == 0) return;
  pack_blocks(sh, base, cv);
  nck(g_nccl.all_gather(sh->send.p, sh->recv.p, chunk, ncclFloat64, g_nccl.comm, g_stream), "ncclAllGather");
  unpack_blocks(sh, base, cv, flags, epoch, sh->recv.p);
}
// caller-side buffers of the split-phase API (host or device)
void copy_out(double* dst, const double* src, int64_t n, int where) {
  if (n > 0)
    ck(cudaMemcpyAsync(dst, src, n * sizeof(double),
                       where == NCL_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, g_stream),
       "copy out");
}
const double* stage_in(ncl_shard* sh, const double* src, int64_t n, int where) {
  if (where != NCL_HOST) return src;
  if (n > 0) ck(cudaMemcpyAsync(sh->recv.p, src, n * sizeof(double), cudaMemcpyHostToDevice, g_stream), "H2D");
  return sh->recv.p;
}
void shard_factor_a(ncl_fact* F, ncl_sym_t M, ncl_shard* sh, double tol) {
  if (sh->S != F->S) throw Error{NCL_E_INVALID, "shard plan built for another symbolic factor"};
  check_match(M, F->S);
  ensure_dev(M, "factorize");
  shard_upload(sh);
  grow_scratch(F, sh);
  DevSymb& d = F->S->d;
  dev_factor_begin(d, M->dp, F->F, M->vals.p, tol, g_stream);
  dev_factor_list(d, F->F, M->vals.p, sh->ftA, 0, g_stream);
  F->sharded_world = sh->P.world;
}
void shard_factor_b(ncl_fact* F, ncl_sym_t M, ncl_shard* sh) {
  DevSymb& d = F->S->d;
  dev_factor_list(d, F->F, M->vals.p, sh->ftB, 1, g_stream);
  // istat = [zero-pivot position, npos, nneg, nzero] over the pivots this rank reports
  dev_inertia(d, F->F, g_stream, sh->P.world > 1 ? sh->report.p : nullptr);
}
double* shard_x(ncl_fact* F, double* x, int where) { return where == NCL_HOST ? F->work1.p : x; }
void shard_solve_a(ncl_fact* F, ncl_shard* sh, double* x, int where) {
  if (sh->S != F->S) throw Error{NCL_E_INVALID, "shard plan built for another symbolic factor"};
  shard_upload(sh);
  const int n = F->S->core.n;
  double* dx = shard_x(F, x, where);
  if (where == NCL_HOST && n > 0)
    ck(cudaMemcpyAsync(dx, x, n * sizeof(double), cudaMemcpyHostToDevice, g_stream), "H2D");
  DevSymb& d = F->S->d;
  dev_solve_begin(d, g_stream);
  dev_solve_fwd_list(d, F->F, dx, sh->ftA, 0, g_stream);
}
void shard_solve_b(ncl_fact* F, ncl_shard* sh, double* dx) {
  DevSymb& d = F->S->d;
  dev_solve_fwd_list(d, F->F, dx, sh->ftB, 1, g_stream);
  dev_solve_bwd_list(d, F->F, dx, sh->ftB, 2, g_stream);
  dev_solve_bwd_list(d, F->F, dx, sh->ftA, 3, g_stream);
  // every rank keeps only the entries it reports: the sum over ranks is x
  if (sh->P.world > 1) dev_zero_indexed(dx, sh->unrep.p, sh->nunrep, g_stream);
}
}  // namespace

API int ncl_shard_create(ncl_symb_t S, const int* var_group, int ngroups, int world, int rank, ncl_shard_t* out) {
  GUARD({
    auto sh = std::make_unique<ncl_shard>();
    sh->S = S;
    std::vector<int> g(var_group, var_group + S->core.n);
    sh->P = build_shard_plan(S->Z, S->core, g, ngroups, world, rank);
    sh->flayA = build_layout(S->Z, sh->P.listA, sh->P.splitA, true);
    sh->flayB = build_layout(S->Z, sh->P.listB, sh->P.splitB, true);
    *out = sh.release();
  });
}
API void ncl_shard_destroy(ncl_shard_t P) { delete P; }
API int ncl_shard_info_get(ncl_shard_t sh, ncl_shard_info* info) {
  GUARD({
    const ShardPlan& P = sh->P;
    info->world = P.world;
    info->rank = P.rank;
    info->owned_supernodes = P.owned_supernodes;
    info->shared_supernodes = P.shared_supernodes;
    info->n_phase_a = static_cast<int>(P.listA.size());
    info->n_phase_b = static_cast<int>(P.listB.size());
    info->n_boundary = static_cast<int>(P.boundary.size());
    info->cb_chunk = P.cb_chunk;
    info->cv_chunk = P.cv_chunk;
    int64_t rc = 0;
    for (uint8_t v : P.col_report) rc += v;
    info->report_cols = rc;
  });
}
API int ncl_shard_owners(ncl_shard_t sh, int* owner) {
  GUARD(std::memcpy(owner, sh->P.owner.data(), sh->P.owner.size() * sizeof(int)));
}
API int ncl_shard_boundary(ncl_shard_t sh, int* ids, int* owner, int64_t* cb_off, int64_t* cv_off) {
  GUARD({
    const ShardPlan& P = sh->P;
    const size_t nb = P.boundary.size();
    if (ids) std::memcpy(ids, P.boundary.data(), nb * sizeof(int));
    if (owner) std::memcpy(owner, P.bowner.data(), nb * sizeof(int));
    if (cb_off) std::memcpy(cb_off, P.cb_pack_off.data(), nb * sizeof(int64_t));
    if (cv_off) std::memcpy(cv_off, P.cv_pack_off.data(), nb * sizeof(int64_t));
  });
}

API int ncl_shard_refactorize(ncl_fact_t F, ncl_sym_t M, ncl_shard_t sh, double tol) {
  GUARD({
    need_comm(sh);
    shard_factor_a(F, M, sh, tol);
    DevSymb& d = F->S->d;
    if (sh->P.world > 1) allgather_blocks(sh, F->F.CB, 0, d.flags, d.epoch);
    shard_factor_b(F, M, sh);
    if (sh->P.world > 1) {
      nck(g_nccl.all_reduce(F->F.istat, F->F.istat, 1, ncclInt32, ncclMin, g_nccl.comm, g_stream), "allreduce");
      nck(g_nccl.all_reduce(F->F.istat + 1, F->F.istat + 1, 3, ncclInt32, ncclSum, g_nccl.comm, g_stream),
          "allreduce");
    }
    check_launch("shard factorize");
  });
}

// Split-phase sharded factorization / solve: the same kernels and the same
// pack / unpack as ncl_shard_refactorize / ncl_shard_solve, with the two
// collectives (the all-gather of boundary blocks and the final reduction)
// left to the caller's transport.
API int ncl_shard_factor_phase_a(ncl_fact_t F, ncl_sym_t M, ncl_shard_t sh, double tol, double* send, int where) {
  GUARD({
    shard_factor_a(F, M, sh, tol);
    pack_blocks(sh, F->F.CB, 0);
    copy_out(send, sh->send.p, sh->P.cb_chunk, where);
    if (where == NCL_HOST) ck(cudaStreamSynchronize(g_stream), "sync");
    check_launch("shard factor phase A");
  });
}
API int ncl_shard_factor_phase_b(ncl_fact_t F, ncl_sym_t M, ncl_shard_t sh, const double* recv, int where,
                                 int* istat) {
  GUARD({
    check_match(M, F->S);
    DevSymb& d = F->S->d;
    const int64_t chunk = sh->P.cb_chunk;
    if (sh->P.world > 1 && chunk > 0)
      unpack_blocks(sh, F->F.CB, 0, d.flags, d.epoch, stage_in(sh, recv, chunk * sh->P.world, where));
    shard_factor_b(F, M, sh);
    ck(cudaMemcpyAsync(istat, F->istat.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, g_stream), "D2H");
    ck(cudaStreamSynchronize(g_stream), "sync");
    check_launch("shard factor phase B");
  });
}
API int ncl_shard_set_status(ncl_fact_t F, const int* istat) {
  GUARD(ck(cudaMemcpyAsync(F->istat.p, istat, 4 * sizeof(int), cudaMemcpyHostToDevice, g_stream), "H2D");
        ck(cudaStreamSynchronize(g_stream), "sync"));
}
API int ncl_shard_solve_phase_a(ncl_fact_t F, ncl_shard_t sh, double* x, int where, double* send, int swhere) {
  GUARD({
    shard_solve_a(F, sh, x, where);
    pack_blocks(sh, F->F.CV, 1);
    copy_out(send, sh->send.p, sh->P.cv_chunk, swhere);
    if (swhere == NCL_HOST) ck(cudaStreamSynchronize(g_stream), "sync");
    check_launch("shard solve phase A");
  });
}
API int ncl_shard_solve_phase_b(ncl_fact_t F, ncl_shard_t sh, double* x, int where, const double* recv, int rwhere) {
  GUARD({
    DevSymb& d = F->S->d;
    const int64_t chunk = sh->P.cv_chunk;
    double* dx = shard_x(F, x, where);
    if (sh->P.world > 1 && chunk > 0)
      unpack_blocks(sh, F->F.CV, 1, d.flags + d.nsn, d.epoch, stage_in(sh, recv, chunk * sh->P.world, rwhere));
    shard_solve_b(F, sh, dx);
    const int n = F->S->core.n;
    if (where == NCL_HOST && n > 0) {
      ck(cudaMemcpyAsync(x, dx, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
      ck(cudaStreamSynchronize(g_stream), "sync");
    }
    check_launch("shard solve phase B");
  });
}
API int ncl_shard_diagonal(ncl_fact_t F, ncl_shard_t sh, double* d) {
  GUARD({
    if (sh->S != F->S) throw Error{NCL_E_INVALID, "shard plan built for another symbolic factor"};
    const int n = F->S->core.n;
    if (n > 0) ck(cudaMemcpyAsync(d, F->D.p, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
    ck(cudaStreamSynchronize(g_stream), "sync");
    const double nan = std::numeric_limits<double>::quiet_NaN();
    if (sh->P.world > 1)
      for (int k = 0; k < n; ++k)
        if (!sh->P.col_report[k]) d[k] = nan;
  });
}

// Single-GPU emulation of a world-G run: every rank's phase A on one device
// (they write disjoint CBs, so no exchange is needed), then phase B once.
API int ncl_shard_refactorize_emulated(ncl_fact_t F, ncl_sym_t M, ncl_shard_t* plans, int G, double tol) {
  GUARD({
    if (G < 1 || 2 * (G + 1) > kTicketSeg0) throw Error{NCL_E_INVALID, "emulated shards: bad G"};
    check_match(M, F->S);
    ensure_dev(M, "factorize");
    for (int r = 0; r < G; ++r) {
      if (plans[r]->S != F->S || plans[r]->P.world != G || plans[r]->P.rank != r)
        throw Error{NCL_E_INVALID, "emulated shards: plans must be ranks 0..G-1 of one world"};
      shard_upload(plans[r]);
    }
    DevSymb& d = F->S->d;
    for (int r = 0; r < G; ++r) grow_scratch(F, plans[r]);
    dev_factor_begin(d, M->dp, F->F, M->vals.p, tol, g_stream);
    for (int r = 0; r < G; ++r) dev_factor_list(d, F->F, M->vals.p, plans[r]->ftA, r, g_stream);
    dev_factor_list(d, F->F, M->vals.p, plans[0]->ftB, G, g_stream);
    dev_inertia(d, F->F, g_stream);
    F->sharded_world = 1;
    check_launch("emulated shard factorize");
  });
}


API int ncl_shard_solve(ncl_fact_t F, ncl_shard_t sh, double* x, int where) {
  GUARD({
    need_comm(sh);
    shard_solve_a(F, sh, x, where);
    DevSymb& d = F->S->d;
    double* dx = shard_x(F, x, where);
    if (sh->P.world > 1) allgather_blocks(sh, F->F.CV, 1, d.flags + d.nsn, d.epoch);
    shard_solve_b(F, sh, dx);
    if (sh->P.world > 1) nck(g_nccl.all_reduce(dx, dx, F->S->core.n, ncclFloat64, ncclSum, g_nccl.comm, g_stream),
                             "allreduce x");
    const int n = F->S->core.n;
    if (where == NCL_HOST && n > 0) {
      ck(cudaMemcpyAsync(x, dx, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream), "D2H");
      ck(cudaStreamSynchronize(g_stream), "sync");
    }
    check_launch("shard solve");
  });
}
