/* nclopf_dist.h — multi-GPU C-ABI: NCCL communicator and the contingency-
 * sharded multifrontal factor / solve.
 *
 * The reference is single-threaded (no MPI/NCCL anywhere in
 * /root/reference/proj); SPEC.md:76-77 only allows distinct factorizations
 * to run concurrently. This extends factorize / solve_in_place
 * (sparse_sym.hpp:90-126) to G ranks, one per GPU: every rank factors the
 * supernodes of its own contingencies, the contribution blocks of the
 * subtree roots are all-gathered over NVLink (NCCL), and the top separator
 * is factored redundantly. L, D and x are bitwise identical for every G.
 */
#ifndef NCLOPF_DIST_H
#define NCLOPF_DIST_H

#include <stdint.h>

#include "nclopf_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* 128-byte NCCL unique id (ncclGetUniqueId) for rank 0 to broadcast */
int ncl_dist_get_unique_id(char* id);
/* one communicator per process on the library's device (ncclCommInitRank) */
int ncl_dist_init(int world, int rank, const char* id);
int ncl_dist_finalize(void);

typedef struct ncl_shard* ncl_shard_t;
typedef struct ncl_shard_info {
  int world, rank;
  int64_t owned_supernodes, shared_supernodes;
  int n_phase_a, n_phase_b, n_boundary;
  int64_t cb_chunk, cv_chunk; /* doubles per rank in the two all-gathers */
  int64_t report_cols;        /* pivot columns whose D / x this rank reports */
} ncl_shard_info;

/* var_group[i] (n = S's dimension): 0 = base case, 1..ngroups-1 = contingency
 * of ORIGINAL variable i. Contingencies go to ranks in contiguous blocks. */
int ncl_shard_create(ncl_symb_t S, const int* var_group, int ngroups, int world, int rank, ncl_shard_t* out);
void ncl_shard_destroy(ncl_shard_t P);
int ncl_shard_info_get(ncl_shard_t P, ncl_shard_info* info);
int ncl_shard_owners(ncl_shard_t P, int* owner); /* per supernode: rank or -1 (shared) */
int ncl_shard_boundary(ncl_shard_t P, int* ids, int* owner, int64_t* cb_off, int64_t* cv_off);
/* sharded refactorize of M's device values into F (asynchronous); world > 1
 * needs ncl_dist_init(world, rank). Status / inertia via ncl_fact_status are
 * global (all-reduced). */
int ncl_shard_refactorize(ncl_fact_t F, ncl_sym_t M, ncl_shard_t P, double pivot_tol);
/* sharded solve_in_place; the full x ends up on every rank */
int ncl_shard_solve(ncl_fact_t F, ncl_shard_t P, double* x, int where);
/* Split-phase form of the two calls above, for callers that bring their own
 * transport (and for single-GPU tests of the exchange): the same kernels and
 * the same pack / unpack, with the collectives done by the caller.
 *   factor:  phase_a (own + base-only supernodes, then pack this rank's
 *            boundary contribution blocks into `send`, cb_chunk doubles)
 *            -> caller all-gathers send into recv (world * cb_chunk doubles,
 *               rank-major, as ncclAllGather lays it out)
 *            -> phase_b (unpack, separator, this rank's pivot report into
 *               istat[4] = {zero-pivot position or n, npos, nneg, nzero})
 *            -> caller reduces istat over ranks (min, sum, sum, sum) and
 *               stores it with ncl_shard_set_status.
 *   solve:   phase_a (forward over own subtrees, pack boundary contribution
 *            vectors, cv_chunk doubles) -> all-gather -> phase_b (rest of
 *            the solve; x holds only this rank's reported entries, zeros
 *            elsewhere) -> caller sums x over ranks.
 * `where` / `swhere` / `rwhere` say whether x / send / recv are host or
 * device pointers; device buffers are read and written asynchronously on the
 * library stream (ncl_stream), host buffers are complete on return. After a world > 1 factorization the whole-factor getters
 * (ncl_fact_diagonal, ncl_fact_get_L, ncl_fact_solve, ncl_solve_refined)
 * return NCL_E_LOGIC; ncl_shard_diagonal returns this rank's reported D
 * entries (NaN elsewhere). */
int ncl_shard_factor_phase_a(ncl_fact_t F, ncl_sym_t M, ncl_shard_t P, double pivot_tol, double* send, int where);
int ncl_shard_factor_phase_b(ncl_fact_t F, ncl_sym_t M, ncl_shard_t P, const double* recv, int where, int* istat);
int ncl_shard_set_status(ncl_fact_t F, const int* istat);
int ncl_shard_solve_phase_a(ncl_fact_t F, ncl_shard_t P, double* x, int where, double* send, int swhere);
int ncl_shard_solve_phase_b(ncl_fact_t F, ncl_shard_t P, double* x, int where, const double* recv, int rwhere);
int ncl_shard_diagonal(ncl_fact_t F, ncl_shard_t P, double* d);
/* single-GPU emulation of a world-G factorization (plans = ranks 0..G-1) */
int ncl_shard_refactorize_emulated(ncl_fact_t F, ncl_sym_t M, ncl_shard_t* plans, int G, double pivot_tol);

#ifdef __cplusplus
}
#endif
#endif
