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
  int64_t cb_storage;     /* doubles in the multifrontal contribution blocks */
  int nsplit;             /* supernodes below this ticket run warp-per-task, above CTA-per-task */
  int n_big;              /* fronts on the multi-CTA gather + blocked DMMA path */
  int n_tasks;            /* scheduled tasks (subtree groups + single supernodes) */
} ncl_symb_info;
int ncl_symb_info_get(ncl_symb_t S, ncl_symb_info* info);
/* inspection: supernode partition (nsn+1 firsts, nsn+1 row offsets), parent
 * supernodes, heights, ticket order (nsn each); any may be NULL */
int ncl_symb_supernodes(ncl_symb_t S, int* sn_first, int64_t* sn_rptr, int* sn_parent, int* height, int* order);
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
/* refill(values) + factorize + solve of a host caller in one call: M's
 * values (nnz) and b (n) from host memory, x (n) back; the rhs upload runs
 * on a copy stream underneath the factorization, one synchronisation at the
 * end (pinned host buffers for the overlap). status / zero_pivot_index /
 * inertia as ncl_fact_status; x is meaningful only when status == 0. */
int ncl_factor_solve_host(ncl_fact_t F, ncl_sym_t M, const double* vals, const double* b, double* x,
                          double pivot_tol, int* status, int* zero_pivot_index, int* n_pos, int* n_neg, int* n_zero);
/* test/inspection only: L as reference-layout CSC over permuted indices
 * (lp[n+1], li[l_nnz], lx[l_nnz]) */
int ncl_fact_get_L(ncl_fact_t F, int* lp, int* li, double* lx);

/* ---- model_ad: model.hpp:29-109, model.cpp, expr.hpp:108-135 ------------- */
typedef struct ncl_builder* ncl_builder_t; /* nclopf::ModelBuilder   (model.hpp:74-97) */
typedef struct ncl_model* ncl_model_t;     /* nclopf::ModelFunctions (model.hpp:29-71) */

int ncl_builder_create(int num_vars, ncl_builder_t* out);                  /* ModelBuilder(int) */
void ncl_builder_destroy(ncl_builder_t B);
int ncl_builder_num_vars(ncl_builder_t B);
int ncl_builder_num_rows(ncl_builder_t B);
/* add_template(ExpressionTemplate(f, num_var_slots, name)); f as a node program */
int ncl_builder_add_template(ncl_builder_t B, int nnodes, const ncl_expr_node* nodes, int num_var_slots,
                             const char* name, int* tmpl_id);
int ncl_builder_add_rows(ncl_builder_t B, int count, int* first_row);       /* add_rows() */
/* add_objective_term x count: vars[count*nv], params[count*np] (np may be 0) */
int ncl_builder_add_objective_terms(ncl_builder_t B, int tmpl_id, int64_t count, int nv, const int* vars, int np,
                                    const double* params);
/* add_constraint_term x count: rows[count] */
int ncl_builder_add_constraint_terms(ncl_builder_t B, int tmpl_id, int64_t count, const int* rows, int nv,
                                     const int* vars, int np, const double* params);
/* build() && : consumes the builder's content (B stays valid but empty) */
int ncl_builder_build(ncl_builder_t B, ncl_model_t* out);

void ncl_model_destroy(ncl_model_t M);
int ncl_model_sizes(ncl_model_t M, int* num_vars, int* num_cons, int64_t* nnz_jac, int64_t* nnz_hess);
int ncl_model_jac_coords(ncl_model_t M, int* rows, int* cols);   /* jac_coords()  */
int ncl_model_hess_coords(ncl_model_t M, int* rows, int* cols);  /* hess_coords() */
int ncl_model_eval_objective(ncl_model_t M, const double* w, double* out, int where);
int ncl_model_eval_grad_objective(ncl_model_t M, const double* w, double* grad, int where);
int ncl_model_eval_constraints(ncl_model_t M, const double* w, double* c, int where);
int ncl_model_eval_jacobian(ncl_model_t M, const double* w, double* vals, int where);
int ncl_model_eval_hessian_lag(ncl_model_t M, const double* w, double sigma, const double* lam, double* vals,
                               int where);
/* hessian_lag(): a finalized SparseSym of sigma*H_phi + sum lam_k H_k */
int ncl_model_hessian_lag(ncl_model_t M, const double* w, double sigma, const double* lam, ncl_sym_t* out);
int ncl_model_jac_times(ncl_model_t M, const double* jac_vals, const double* v, double* out, int where);
int ncl_model_jac_trans_times(ncl_model_t M, const double* jac_vals, const double* y, double* out, int where);
/* Device fast path used by the IPM: one launch evaluates value, gradient and
 * Hessian programs of every family; gathers into obj[1], grad[n], c[m],
 * jac[nnz_jac], hess[nnz_hess] (any may be NULL). Asynchronous. */
int ncl_model_eval_all_device(ncl_model_t M, const double* w, double sigma, const double* lam, double* obj,
                              double* grad, double* c, double* jac, double* hess);
/* Device fast path of eval_objective + eval_constraints (trial points of the
 * line search): value programs only. Asynchronous. */
int ncl_model_eval_values_device(ncl_model_t M, const double* w, double* obj, double* c);
/* Pending DomainError of device-path evaluations: returns NCL_E_DOMAIN (and
 * clears it) if any evaluation left the smooth domain. Synchronizes. */
int ncl_model_check_domain(ncl_model_t M);
/* fd_check(m, w, seed, tol) (model.hpp:99-109): errs[3] = grad/jac/hess */
int ncl_fd_check(ncl_model_t M, const double* w, unsigned seed, double tol, double* errs, int* pass);

/* ---- condensed Newton matrix (ipm.assemble_newton) ------ */
/* K = H + Sigma_x + delta_w I + J^T D J over the fixed pattern
 * hess_coords U diag U {J^T J}, assembled in a fixed triplet order (see
 * csrc/host/kkt.hpp) so a reference SparseSym fed the same triplets
 * (ncl_kkt_triplets) refills to bit-identical values. */
typedef struct ncl_kkt* ncl_kkt_t;
int ncl_kkt_create(int n, int m, int64_t nnz_hess, const int* hess_rows, const int* hess_cols, int64_t nnz_jac,
                   const int* jac_rows, const int* jac_cols, ncl_kkt_t* out);
int ncl_kkt_create_for_model(ncl_model_t M, ncl_kkt_t* out);
void ncl_kkt_destroy(ncl_kkt_t K);
ncl_sym_t ncl_kkt_matrix(ncl_kkt_t K);            /* borrowed; values live on the device */
int64_t ncl_kkt_num_triplets(ncl_kkt_t K);
int ncl_kkt_triplets(ncl_kkt_t K, int* rows, int* cols);
/* all vectors on the device (where=NCL_DEVICE, async) or host (synchronous):
 * hess[nnz_hess], jac[nnz_jac], sigma_x[n], D[m] */
int ncl_kkt_assemble(ncl_kkt_t K, const double* hess, const double* jac, const double* sigma_x, double delta_w,
                     const double* D, int where);

/* ---- scopf_builder (Eq. 2-4) -------------------- */
/* Host-side problem generation: a corrective AC-SCOPF with complementarity
 * recourse in the paper's variable layout, as a neutral spec (templates +
 * instances + bounds) that any ModelBuilder (this library's or the
 * reference's) can consume. grid: 0 = MATPOWER case9, 1 = seeded geometric
 * synthetic grid (nb, nl, ng, seed). K non-islanding line outages. */
typedef struct ncl_scopf* ncl_scopf_t;
typedef struct ncl_scopf_info {
  int n, m, nfam, K, nb, nl, ng, ncomp;
  int nvar_scen, ncon_scen;
} ncl_scopf_info;
int ncl_scopf_create(int grid, int nb, int nl, int ng, uint64_t seed, int K, ncl_scopf_t* out);
/* explicit contingency list (e.g. a screened list);
 * branch_ids == NULL -> the first K non-islanding outages. An id is
 * l + nl * j: the outage of non-islanding branch l with the post-contingency
 * loads scaled by 1 - 0.015 j, j < 4 (j = 0: the plain N-1 outage; j > 0
 * gives outage x load-scenario contingencies, csrc/host/scopf.hpp) */
int ncl_scopf_create_list(int grid, int nb, int nl, int ng, uint64_t seed, int K, const int* branch_ids,
                          ncl_scopf_t* out);
void ncl_scopf_destroy(ncl_scopf_t S);
int ncl_scopf_get_info(ncl_scopf_t S, ncl_scopf_info* info);
/* family f: name (<=63 chars), node count, slots, params per instance,
 * objective flag, instance count */
int ncl_scopf_family_info(ncl_scopf_t S, int f, char* name, int* nnodes, int* nslots, int* np, int* objective,
                          int64_t* ninst);
int ncl_scopf_family_data(ncl_scopf_t S, int f, ncl_expr_node* nodes, int* rows, int* vars, double* params);
/* variable bounds/start (n), row bounds (m); +-inf for absent bounds */
int ncl_scopf_bounds(ncl_scopf_t S, double* xl, double* xu, double* x0, double* gl, double* gu);
int ncl_scopf_contingencies(ncl_scopf_t S, int* branch_ids);
/* scenario of every variable (n): 0 = base case, k = contingency k — the
 * var_group input of the sharded factorization (nclopf_dist.h) */
int ncl_scopf_var_groups(ncl_scopf_t S, int* groups);
/* every non-islanding single-branch outage of the grid (ascending); ids may be NULL */
int ncl_scopf_candidates(ncl_scopf_t S, int* ids, int* count);
int ncl_scopf_build_model(ncl_scopf_t S, ncl_model_t* out); /* this library's ModelBuilder */
/* screening system (Eq. 5): the K contingency
 * scenarios of `base`'s grid with the base set points fixed — pg0[ng]
 * generator outputs, v0[nb] bus voltages (read at generator buses) — and no
 * objective; the scenarios are independent row/variable blocks of equal size,
 * so one NCL solve screens them all. ids as
 * ncl_scopf_create_list (NULL: the first K non-islanding outages). */
int ncl_scopf_create_screening(ncl_scopf_t base, const double* pg0, const double* v0, int K, const int* ids,
                               ncl_scopf_t* out);

#ifdef __cplusplus
}
#endif
#endif
