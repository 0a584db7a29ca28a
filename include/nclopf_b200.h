/* nclopf_b200.h — C-ABI of the B200-native NCL/IPM hot path.
 *
 * Drop-in boundary for the reference C++ API under /root/reference/proj
 * (C++20, namespace nclopf). The reference has no FFI of its own; these are
 * the entry points a binding of that API binds (see INTEGRATION.md for the
 * nclopf::-compatible C++ façade and the ctypes binding). Plain pointers,
 * sizes and opaque handles only; no torch or CUDA types in any signature.
 *
 * Conventions
 *  - Return value: NCL_OK (0) or a negative NCL_E_* code; the message of the
 *    last error on this thread is ncl_last_error(). Codes map 1:1 to the
 *    reference's exceptions (see nclopf_expr_program.h).
 *  - Arrays are caller-owned. `where` = NCL_HOST (0) for host memory
 *    (reference std::span semantics, synchronous), NCL_DEVICE (1) for device
 *    memory on the library stream (asynchronous, the device-resident fast
 *    path used by the IPM).
 *  - All indices are 0-based int32 as in the reference; l_nnz is int64.
 *  - Everything numeric runs on the GPU. There is no CPU fallback: if no
 *    sm_100 device is present every compute entry point fails with
 *    NCL_E_CUDA.
 */
#ifndef NCLOPF_B200_H
#define NCLOPF_B200_H

#include <stdint.h>

#include "nclopf_expr_program.h"

#ifdef __cplusplus
extern "C" {
#endif

#define NCL_HOST 0
#define NCL_DEVICE 1

typedef struct ncl_sym* ncl_sym_t;     /* nclopf::SparseSym        (sparse_sym.hpp:20-66)   */
typedef struct ncl_symb* ncl_symb_t;   /* nclopf::SymbolicFactor   (sparse_sym.hpp:74-85)   */
typedef struct ncl_fact* ncl_fact_t;   /* nclopf::Factorization    (sparse_sym.hpp:97-121)  */

/* ---- library ------------------------------------------------------------ */
int ncl_init(int device);               /* select device, create the library stream */
int ncl_synchronize(void);
const char* ncl_last_error(void);
void* ncl_stream(void);                 /* cudaStream_t of the library (opaque) */
int ncl_device_alloc(void** ptr, int64_t bytes);
int ncl_device_free(void* ptr);
int ncl_memcpy(void* dst, const void* src, int64_t bytes, int kind); /* kind: 0 H2D 1 D2H 2 D2D, on stream, sync */
int64_t ncl_kernel_launches(void);      /* count of library kernel launches so far */

/* ---- SparseSym: sparse_sym.hpp:20-66, sparse_sym.cpp:12-131 -------------- */
int ncl_sym_create(int n, ncl_sym_t* out);                                 /* SparseSym(int n) */
void ncl_sym_destroy(ncl_sym_t M);
int ncl_sym_add(ncl_sym_t M, int64_t count, const int* rows, const int* cols,
                const double* vals);                                       /* add() x count   */
int ncl_sym_finalize(ncl_sym_t M);                                         /* finalize()      */
int ncl_sym_begin_refill(ncl_sym_t M);                                     /* begin_refill()  */
int ncl_sym_refill(ncl_sym_t M);                                           /* refill() on GPU */
/* Device fast path of refill(): trip_vals[k] is the value of triplet k of
 * the original assembly; merged on the GPU in triplet order (bit-exact with
 * sparse_sym.cpp:63-67). */
int ncl_sym_refill_values(ncl_sym_t M, const double* trip_vals, int where);
int ncl_sym_dim(ncl_sym_t M);
int ncl_sym_nnz(ncl_sym_t M);
int64_t ncl_sym_num_triplets(ncl_sym_t M);
int ncl_sym_finalized(ncl_sym_t M);
int ncl_sym_get_csc(ncl_sym_t M, int* colptr, int* rowind, double* vals);  /* col_ptr/row_ind/values */
int ncl_sym_set_values(ncl_sym_t M, const double* vals, int where);        /* overwrite values (nnz) */
double* ncl_sym_device_values(ncl_sym_t M);                                 /* device-resident values */
int ncl_sym_max_abs_diag(ncl_sym_t M, double* out);                        /* max_abs_diag()  */
int ncl_sym_norm_inf(ncl_sym_t M, double* out);                            /* norm_inf()      */
int ncl_sym_frobenius_norm(ncl_sym_t M, double* out);                      /* frobenius_norm()*/
int ncl_sym_multiply(ncl_sym_t M, const double* x, double* y, int where);  /* multiply()      */
int ncl_sym_same_pattern(ncl_sym_t A, ncl_sym_t B);                        /* same_pattern()  */
/* write_matrix_market(): writes at most cap bytes into buf, *len = full size */
int ncl_sym_write_matrix_market(ncl_sym_t M, char* buf, int64_t cap, int64_t* len);

/* ---- symbolic analysis: sparse_sym.hpp:68-88, sparse_sym.cpp:139-262 ----- */
int ncl_symbolic_order(ncl_sym_t M, int* perm);                 /* symbolic_order(), bit-exact */
int ncl_analyze(ncl_sym_t M, const int* perm, ncl_symb_t* out); /* analyze(M) / analyze(M, perm) */
void ncl_symb_destroy(ncl_symb_t S);
typedef struct ncl_symb_info {
  int n;
  int64_t l_nnz;          /* SymbolicFactor::l_nnz */
  int nsupernodes;
  int max_height;         /* supernodal etree height */
  int max_width;          /* widest supernode */
  int max_rows;           /* tallest supernode panel */
  int64_t l_storage;      /* doubles in the dense supernode panels */
  double flops;           /* sum_j (c_j^2 + 2 c_j) */
} ncl_symb_info;
int ncl_symb_info_get(ncl_symb_t S, ncl_symb_info* info);
int ncl_symb_get(ncl_symb_t S, int* perm, int* iperm, int* parent, int* up_colptr, int* up_rowind,
                 int* entry_map, int* l_colcount);

/* ---- numeric factorization: sparse_sym.hpp:90-126, sparse_sym.cpp:268-344 */
/* factorize(M, symb, pivot_tol); S == NULL -> factorize(M, pivot_tol) which
 * analyzes and owns the symbolic factor. Synchronous; status via
 * ncl_fact_status. */
int ncl_factorize(ncl_sym_t M, ncl_symb_t S, double pivot_tol, ncl_fact_t* out);
/* Device fast path: refactor M's current device values into F's buffers
 * (same symbolic), asynchronous. */
int ncl_refactorize(ncl_fact_t F, ncl_sym_t M, double pivot_tol);
void ncl_fact_destroy(ncl_fact_t F);
/* status: 0 ok, 1 zero_pivot (FactorizeStatus); zero_pivot_index original
 * 0-based index or -1; inertia (0,0,0) on zero_pivot. Synchronizes. */
int ncl_fact_status(ncl_fact_t F, int* status, int* zero_pivot_index, int* n_pos, int* n_neg, int* n_zero);
int ncl_fact_diagonal(ncl_fact_t F, double* d);                   /* diagonal(), pivot order */
int ncl_fact_solve(ncl_fact_t F, double* x, int where);           /* solve_in_place() */
/* solve_refined(F, M, b, target, max_sweeps) -> RefinedSolve */
int ncl_solve_refined(ncl_fact_t F, ncl_sym_t M, const double* b, double target, int max_sweeps, double* x,
                      int where, double* residual, int* sweeps, int* converged);
/* test/inspection only: L as reference-layout CSC over permuted indices
 * (lp[n+1], li[l_nnz], lx[l_nnz]) */
int ncl_fact_get_L(ncl_fact_t F, int* lp, int* li, double* lx);

#ifdef __cplusplus
}
#endif
#endif
