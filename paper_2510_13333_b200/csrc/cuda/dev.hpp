// Device-side data structures and launch entry points for the sparse
// LDLᵀ path (K3 factor, K4 solve, K5 SpMV/refinement, K6 norms).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../limits.hpp"

namespace nclb {

// Contribution blocks are packed lower-triangular, column-major: column j of
// an m x m block holds rows j..m-1 contiguously; entry (i, j) is at
// cb_col(j, m) + i.
__host__ __device__ inline int64_t cb_col(int j, int m) {
  return static_cast<int64_t>(j) * m - static_cast<int64_t>(j) * (j + 1) / 2;
}

// Number of library kernel launches issued so far (evidence for the bench's
// gpu_launches key). Incremented by every dev_* wrapper.
extern int64_t g_kernel_launches;

// Host-side schedule of the CTA part of a list when it holds fronts too large
// for shared memory: per height level the [begin, end) index range in the
// list and the large supernodes (s, f, w, nr) that run the blocked DMMA path.
// One large front of a batch (csrc/cuda/bigfront.cu)
struct BigDesc {
  int s, f, w, nr, pw, npan;  // supernode, first column, width, rows, panel width, panels (0: one-CTA front)
  int gsz, pad_;              // lanes summing one front entry's gather sources (power of two)
  int64_t g0, g1;             // gather-map entry range
  int64_t foff, woff;         // offsets of its scratch front (nr^2) and W (nr * pw)
};
constexpr int kCtaFrontS = 80;  // front cap of the small-CTA segments (packed lower: 25.9 KB)
struct TopSched {
  std::vector<int> lvl_begin, lvl_end;   // segments of the CTA part (task index ranges)
  std::vector<std::vector<BigDesc>> big;  // per segment: its large fronts (run as one batch)
  std::vector<const BigDesc*> big_dev;    // per segment: device copy of `big`
  std::vector<char> small;                // per segment: every front <= kCtaFrontS rows (128-thread CTAs)
  bool any_big = false, any_small = false;
  int max_nr = 0;
  int64_t scratch_f = 0, scratch_w = 0;   // largest per-segment scratch (doubles)
};
// Register-resident fronts of a task list (csrc/capi.cpp build_batches).
// The wide bottom of the tree is a handful of tiny front shapes (500x256:
// (nr, w) = (7,1) 185 k, (8,2) 86 k, (10,2) 73 k, (8,1) 55 k, ... of 560 k
// supernodes). For the shapes in kRegShapes every index of the front is a
// compile-time constant, so a team of R lanes (R = 1 for the smallest
// shapes) factors one front held in registers: no shared memory, nothing but
// the arithmetic, one predicated load per front entry per source and, for
// R > 1, one shuffle per pivot entry. Supernodes of these shapes whose
// children in the list are such fronts too form a dependency-closed forest
// that runs as ONE persistent launch before the other tasks: warps claim
// chunks (up to 32 / R fronts of one shape and level; chunks sorted by
// level), lanes wait on their children's flags (acquire) and publish their
// own (release). Per front entry the operations
// are small_task's in the same order (A value, children ascending, pivot
// columns in order): the factor is bitwise that of the warp path.
struct alignas(16) RegInst {  // 64 bytes: four 16-byte loads per front
  int loff, cboff;  // panel, contribution-block offsets (doubles; analyze checks both < 2^31)
  int amap;         // offset (ints) of the A map: per packed entry of the front's first W columns (the
                    // only ones A reaches) the K value slot, -1 = none
  int cmap;         // children's maps: per child, per packed front entry the source position in the
                    // child's packed CB, 255 = none. R > 1: byte offset in `cmap` (rows padded to 4
                    // bytes); R == 1: word offset in `cmapw`, words interleaved over the chunk's 32 lanes
                    // (word w of child q at cmap + (q * words + w) * 32), and the A map interleaved the
                    // same way (entry p at amap + 32 p): coalesced
  int ccb;          // offset of the children's CB offsets (int64 each) and supernode ids (int each)
  int s, f, nch;
  int cid[4];       // the first four children inline (supernode ids, CB offsets): one round trip less
  int cb[4];
};
static_assert(sizeof(RegInst) == 64, "RegInst is four 16-byte loads");
struct RegChunk {
  int shape, n, first;  // n fronts inst[first .. first + n) of one shape
  int smap;             // word offset of the chunk's forward-solve child records in smapw: for front lane
                        // l and child q, word w < kSmapWords (rows 4w .. 4w + 3) at
                        // smap + (q * kSmapStride + w) * 32 + l holds the child's CV entry index per parent
                        // row (255 = none), word kSmapWords the child's CV offset (int32)
};
constexpr int kSmapWords = 3;                // rows of a register front <= 12
constexpr int kSmapStride = kSmapWords + 1;  // + the child's CV offset
struct BatchSched {
  std::vector<RegInst> inst;
  std::vector<int> amap;
  std::vector<uint8_t> cmap;
  std::vector<uint32_t> cmapw;
  std::vector<int64_t> ccb;
  std::vector<int> cid;      // children's supernode ids (same index as ccb)
  std::vector<uint32_t> smapw;   // forward-solve row maps (RegChunk::smap)
  std::vector<RegChunk> chunks;  // tier-1 chunks in level order, then tier-2 chunks in level order
  int nchunk1 = 0;               // chunks of tier 1
  int64_t nodes = 0;         // supernodes covered
  const RegInst* dev_inst = nullptr;
  const int* dev_amap = nullptr;
  const uint8_t* dev_cmap = nullptr;
  const uint32_t* dev_cmapw = nullptr;
  const int64_t* dev_ccb = nullptr;
  const int* dev_cid = nullptr;
  const RegChunk* dev_chunks = nullptr;
  const uint32_t* dev_smapw = nullptr;
};
// Per child slot q of the children CSR (child[q]): what a parent needs to
// extend-add that child's contribution block (one 16-byte load)
struct alignas(16) ChildRec {
  int64_t cboff;  // the child's CB offset
  int rel;        // index in relp of the child's first CB row (rptr + w)
  int m2c;        // CB order nr - w
};
// Packed per-supernode metadata (one 64-byte record, four 16-byte loads):
// everything a small-front task needs before touching the numbers.
struct alignas(16) SnMeta {
  int64_t loff;   // panel offset (L)
  int64_t cboff;  // contribution-block offset (CB)
  int64_t rptr;   // row-list offset (rows / relp / CV)
  int64_t a0;     // first A entry (aptr)
  int na;         // number of A entries
  int f, w, nr;   // first column, width, rows
  int c0, c1;     // children range in child[]
  int parent, pad;
};
static_assert(sizeof(SnMeta) == 64, "SnMeta must stay one 64-byte record");

// A task list: `ids` holds supernodes, task t covers ids[tptr[t] .. tptr[t+1])
// (a whole small subtree in postorder, or one supernode). Tasks are in
// dependency order; the first `nleaf` have no external dependencies, tasks
// from `split` on are single supernodes run CTA-per-task.
struct DevTasks {
  const int* ids = nullptr;
  const int* tptr = nullptr;
  const int* prog = nullptr;       // group programs (factor)
  const int64_t* gpo = nullptr;    // [ngroups+1]
  int n = 0, nleaf = 0, split = 0;  // counts / indices in TASKS
  const TopSched* top = nullptr;    // host pointer; nullptr or !any_big -> one persistent launch
  const BatchSched* batch = nullptr;  // host pointer; batched subtrees run before the task list (factor)
  int root_heavy = -1;  // the last task's node when its forward CV gather runs GPU-wide (fwd_root_gather)
  int root_nr = 0;
};

// Symbolic schedule resident in HBM (built once from host Supernodal).
struct DevSymb {
  int n = 0, nsn = 0, nleaf = 0, nsplit = 0;
  int64_t nnz = 0, l_storage = 0;
  int* perm = nullptr;       // [n]
  int* sn_first = nullptr;   // [nsn+1]
  int* sn_parent = nullptr;  // [nsn]
  int64_t* sn_rptr = nullptr;
  int* rows = nullptr;
  int64_t* sn_loff = nullptr;
  int* relp = nullptr;       // [rows] child row -> position in the parent's row list
  int64_t* cb_off = nullptr; // [nsn+1] contribution-block offsets ((nr-w)^2 each)
  int64_t cb_storage = 0;
  int64_t* gm_ptr = nullptr;  // [nsn+1] gather-map entry ranges (CTA-part fronts)
  int* gdst = nullptr;        // front position of each gather entry
  int64_t* gsp = nullptr;     // [entries+1] source ranges
  int64_t* gsrc = nullptr;    // ~A slot or global CB index
  uint8_t* big = nullptr;     // [nsn] 1 = large-front path
  int64_t* cv_ptr = nullptr;  // forward-solve gather (CTA-part fronts)
  int64_t* cvsp = nullptr;
  int64_t* cvsrc = nullptr;
  int* cptr = nullptr;  // children CSR
  int* child = nullptr;
  const ChildRec* chrec = nullptr;  // [child slots]
  int* order = nullptr;  // ticket order, leaves first
  int64_t* aptr = nullptr;   // [nsn+1] A entries per supernode
  int* asrc = nullptr;       // source value slot
  int* aoff = nullptr;       // offset inside panel
  int* aoffp = nullptr;      // offset inside the packed-lower front (cb_col(off / nr, nr) + off % nr)
  // scheduling state
  DevTasks tasks;           // default (unsharded) task list (solves)
  DevTasks ftasks;          // the same list with its batched subtrees split off (factor)
  const SnMeta* meta = nullptr;  // [nsn]
  int* flags = nullptr;     // [3*nsn] epoch flags: factor, fwd, bwd
  int* tickets = nullptr;   // [4]
  int epoch = 0;
};

// Pattern-level device data of one SparseSym (independent of the ordering).
struct DevPattern {
  int n = 0;
  int64_t nnz = 0;
  int* diag_pos = nullptr;  // value slots of the stored diagonal entries
  int ndiag = 0;
  // bit-exact symmetric SpMV row gather in the reference multiply order
  // (sparse_sym.cpp:105-115): row i lists (value slot, x index)
  int64_t* mv_ptr = nullptr;  // [n+1]
  int* mv_val = nullptr;
  int* mv_col = nullptr;
};

struct DevFactor {
  double* L = nullptr;  // panels
  double* CB = nullptr; // contribution blocks (multifrontal Schur updates)
  double* CV = nullptr; // [rows] forward-solve contribution vectors
  double* bigF = nullptr;  // scratch front of the blocked large-front path (max_nr^2)
  double* bigW = nullptr;  // scratch W = L21 D (max_nr x 32)
  double* D = nullptr;  // [n] by pivot position
  double* xp = nullptr;  // [n] permuted work vector
  double* scal = nullptr;  // [4]: thresh, maxdiag, scratch
  int* istat = nullptr;    // [4]: zp position, npos, nneg, nzero
};

// A task list: supernode ids in leaves-first height order; the first
// `nleaf` are leaves, tasks from `split` on run CTA-per-task.
// Host copy of a task layout (see build_layout in capi.cpp)
struct TaskLayout {
  std::vector<int> nodes, tptr;
  int nleaf = 0, split = 0;
  TopSched top;
  BatchSched batch;  // empty unless built with batched subtrees
  // group programs (one per group task, see build_layout): int stream
  std::vector<int> prog;
  std::vector<int64_t> gpo;  // [ngroups+1]
};
// per-warp shared-memory budget of a group task (csrc/cuda/ldlt.cu)
constexpr int kGrpFront = 32;       // fronts of group nodes: nr <= 32 (packed lower: 528 doubles)
constexpr int kGrpStack = 512;      // doubles: A values + contribution-block stack
constexpr int kGrpProg = 1280;      // ints: the group program (read in place: bounds group size only)

// Ticket counters per symbolic handle:
//   [0, 40)             2 per task-list slot (warp / CTA phases of factor and solves)
//   [40, 56)            the unsharded factorization's CTA segments (zeroed once per
//                       factorization: consecutive segment launches have no memset
//                       between them — programmatic dependent launch, ldlt.cu)
//   [56, 60)            backward register-front solve per slot (zeroed by dev_solve_begin)
//   60                  forward register-front solve
//   61, 62              register-front factor phases
//   63                  sharded CTA segments
//   64                  the forward solve's separator-root task (after its GPU-wide gather)
constexpr int kTickets = 72;
constexpr int kTicketSeg0 = 40;
constexpr int kTicketRegBwd0 = 56, kTicketRegFwd = 60, kTicketRegFac1 = 61, kTicketRegFac2 = 62,
              kTicketShardSeg = 63, kTicketRoot = 64;
// panel width of the one-CTA dense front factorization (ldlt.cu cta_dense):
// the diagonal block is factored by one warp in registers, the trailing
// update is a rank-NCL_CTA_PANEL DMMA update (kPb / 4 k-steps per tile)
#ifndef NCL_CTA_PANEL
#define NCL_CTA_PANEL 8
#endif

extern unsigned long long* g_task_trace;  // device buffer [2 * tasks] or nullptr
void dev_phase_trace(unsigned long long* buf);  // device buffer [4 * nsn] or nullptr

// all launches are asynchronous on `st`
// sharded pieces: begin (threshold, epoch, tickets) -> list(s) -> inertia
void dev_factor_begin(const DevSymb& S, const DevPattern& P, DevFactor& F, const double* kvals, double pivot_tol,
                      cudaStream_t st);
void dev_factor_list(const DevSymb& S, DevFactor& F, const double* kvals, const DevTasks& T, int slot,
                     cudaStream_t st);
void dev_solve_begin(const DevSymb& S, cudaStream_t st);
void dev_solve_fwd_list(const DevSymb& S, DevFactor& F, const double* b, const DevTasks& T, int slot,
                        cudaStream_t st);
void dev_solve_bwd_list(const DevSymb& S, DevFactor& F, double* x, const DevTasks& T, int slot, cudaStream_t st);
// exchange helpers (csrc/cuda/shard.cu): pack my boundary CBs (or CVs) into
// send; unpack the others' from recv (G chunks) and publish their flags
void dev_shard_pack(const DevSymb& S, const double* src, const int* bids, const int* bowner, const int64_t* pack_off,
                    int nb, int rank, int cv, double* send, cudaStream_t st);
void dev_shard_unpack(const DevSymb& S, double* dst, const int* bids, const int* bowner, const int64_t* pack_off,
                      int nb, int rank, int cv, const double* recv, int64_t chunk, int* flags, int epoch,
                      cudaStream_t st);
// all large fronts of one segment, batched (same arithmetic per front as one at a time)
// one CTA per heavy-gather front with nr <= the CTA front cap (npan == 0):
// scratch front (full layout, assembled) -> shared memory -> cta_dense
void dev_big_cta(const DevSymb& S, DevFactor& F, const BigDesc* d, int nf, cudaStream_t st);
void dev_factor_big_batch(const DevSymb& S, DevFactor& F, const double* kvals, const std::vector<BigDesc>& h,
                          const BigDesc* d, cudaStream_t st);
void dev_zero_indexed(double* x, const int* idx, int64_t n, cudaStream_t st);
void dev_factor(const DevSymb& S, const DevPattern& P, DevFactor& F, const double* kvals, double pivot_tol,
                cudaStream_t st, const TopSched* top = nullptr);
void dev_inertia(const DevSymb& S, DevFactor& F, cudaStream_t st, const uint8_t* report = nullptr);
// x := M^{-1} b (in place allowed: x may alias b)
void dev_solve(const DevSymb& S, DevFactor& F, const double* b, double* x, cudaStream_t st);
void dev_spmv(const DevPattern& P, const double* kvals, const double* x, double* y, cudaStream_t st);
// r = b - M x ; *out_max = max|r| (zeroed here), fused
void dev_residual(const DevPattern& P, const double* kvals, const double* b, const double* x, double* r,
                  double* out_max, cudaStream_t st);
void dev_absmax(const double* v, int64_t n, double* out, cudaStream_t st);  // out must be zeroed
void dev_axpy_inplace(double* x, const double* d, int64_t n, cudaStream_t st);  // x += d
void dev_max_abs_diag(const DevPattern& P, const double* kvals, double* out, cudaStream_t st);
void dev_rowsum_max(const DevPattern& P, const double* kvals, double* out, cudaStream_t st);
// sum over stored entries of (diag ? v^2 : 2 v^2), deterministic two-level tree
void dev_frob_sq(const DevPattern& P, const int* colptr, const int* rowind, const double* kvals, double* out,
                 cudaStream_t st);
int dev_num_sms();
void dev_gather_sum(int64_t nslots, const int* ptr, const int* idx, const double* src, double* dst,
                    cudaStream_t st);
// compact K2 (csrc/cuda/assemble.cu): bitwise the same K as dev_kkt_assemble
void dev_kkt_assemble_compact(int64_t nnz, const int* slot_h, const uint64_t* dgmask, const int* dgrank,
                              const uint32_t* tp, const int* ta, const uint8_t* td, const int* jrow, const double* H,
                              const double* J, const double* sigx, double dw, const double* D, double* K,
                              cudaStream_t st);
void dev_kkt_assemble(int64_t nnz, const int* slot_h, const int* slot_diag, const int64_t* jptr, const int* jterm,
                      const double* H, const double* J, const double* sigx, double dw, const double* D, double* K,
                      cudaStream_t st);

}  // namespace nclb
