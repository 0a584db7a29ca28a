/* nclopf_ipm.h — options/result structs and C-ABI of the NCL + IPM solve.
 *
 * The reference defines these only as SPEC text (no code exists under
 * /root/reference/proj): NclParams, the IPM constants
 * (SPEC.md:336, 346, 379-380), RunConfig/CLI flags,
 * NclResult and the JSON-lines traces (SPEC.md:386-387,
 * 452-453). Filter-line-search constants are unpinned by the paper
 * (SPEC.md:393); the defaults are Ipopt's (Wächter & Biegler 2006), which
 * MadNLP follows. Shared verbatim by the product and the CPU oracle so both
 * take identical branch decisions.
 */
#ifndef NCLOPF_IPM_H
#define NCLOPF_IPM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ncl_options {
  /* NclParams */
  double rho0;          /* 100 */
  double rho_growth;    /* 10 */
  double rho_max;       /* 1e12 */
  double eta_star;      /* 1e-6 outer feasibility tolerance */
  double omega_star;    /* 1e-6 stationarity tolerance */
  double eta0, omega0;  /* 0.1, 0.1; eta_n = max(eta*, 0.1 eta_{n-1}) */
  double lambda_max;    /* 1e12 multiplier guard */
  int max_outer;        /* 40 */
  int max_inner;        /* total IPM iteration cap (3000) */
  /* IPM */
  double mu_init;       /* 0.1 */
  double mu_min;        /* 1e-7 */
  double kappa_mu, theta_mu, kappa_eps;  /* 0.2, 1.5, 10 */
  double tau_min;       /* 0.99, tau = max(tau_min, 1 - mu) */
  double bound_push, bound_frac;  /* 1e-2, 1e-2 */
  double kappa_sigma;   /* 1e10 */
  double s_max;         /* 100 (KKT error scaling) */
  double obj_max_grad;  /* 100: sf = min(1, obj_max_grad / |grad f(x0)|_inf) */
  /* filter line search (Ipopt defaults) */
  double gamma_theta, gamma_phi, eta_phi, delta, s_theta, s_phi, alpha_min_frac;
  int max_backtrack;
  /* inertia correction */
  double dw_first_rel;  /* 1e-8: first dw = dw_first_rel * max(1, |H|_inf) */
  double dw_growth;     /* 10 */
  double dw_decrease;   /* 1/3: next iteration starts from dw_last / 3 */
  double dw_max;        /* 1e40 -> RegularizationExhausted */
  double dc_base, kappa_c;  /* dc = dc_base * mu^kappa_c on a zero pivot: 1e-8, 0.25 */
  int dw_reuse;         /* 1: start from dw_last/3 when the last iteration needed dw > 0 */
  double pivot_tol;     /* 1e-14 for the condensed K (sparse_sym.hpp:125 default 1e-12 is for O(1) diagonals) */
  /* linear solve (sparse_sym.hpp:136-139) */
  double refine_target; /* 1e-8 */
  int refine_max_sweeps;/* 2 (solve_refined's own default is 5) */
  double mu_warm_frac;  /* warm start mu = max(mu_min, mu_warm_frac * omega_n) */
  double acceptable_factor; /* Ipopt 'acceptable' exit: E_0 <= acceptable_factor * omega_n ... */
  int acceptable_iter;      /* ... for this many consecutive iterations (10, 15) */
  int verbose;          /* 1: keep the per-iteration JSON-lines trace */
} ncl_options;

enum ncl_solve_status {
  NCL_SOLVE_OPTIMAL = 0,
  NCL_SOLVE_INFEASIBLE = 1,
  NCL_SOLVE_ITERATION_LIMIT = 2,
  NCL_SOLVE_REG_EXHAUSTED = 3,
  NCL_SOLVE_RESTORATION_FAILED = 4,
  /* |r|_inf <= eta* but the last subproblem stopped on the 'acceptable'
   * rule (E_0 <= acceptable_factor * omega*), not on E_0 <= omega* */
  NCL_SOLVE_ACCEPTABLE = 5
};

typedef struct ncl_result {
  int status;           /* enum ncl_solve_status */
  int outer_iters, inner_iters, factorizations, restorations;
  double objective;     /* unscaled f(x) */
  double r_inf;         /* |r|_inf (includes t on complementarity rows) */
  double inf_pr, inf_du, compl_;  /* final subproblem KKT residuals */
  double rho, mu;
  int multiplier_warning; /* set when a multiplier update leaves |lamN|_inf > lambda_max */
  /* wall-clock seconds (host timer around synchronous backend calls) */
  double t_total, t_init, t_eval, t_factor, t_solve, t_linesearch, t_other;
  double final_e0;      /* scaled KKT error E_0 at the last subproblem's exit */
} ncl_result;

/* One Newton step of the NCL subproblem at a caller-given interior state
 * (assemble_newton + recover_directions; acceptance
 * criterion 6). Host arrays: x, zl, zu (n), r, s, y, vl, vu,
 * lamN (m); s is ignored (held at gl) on equality rows, bound duals of
 * infinite bounds must be 0. */
typedef struct ncl_ipm_state {
  const double *x, *zl, *zu, *r, *s, *y, *vl, *vu, *lamN;
  double mu, rho, sf, dw, dc;
} ncl_ipm_state;
/* outputs: dx, dzl, dzu (n), dr, ds, dy, dvl, dvu (m) — any may be NULL */
typedef struct ncl_newton_step {
  double *dx, *dzl, *dzu, *dr, *ds, *dy, *dvl, *dvu;
  double residual;      /* solve_refined's final relative residual */
  int sweeps, converged;
  int status, npos, nneg, nzero;  /* factorization of the condensed K */
} ncl_newton_step;

/* ---- B200 solve (libnclopf_b200.so) -------------------------------------
 * ncl_solve over a ModelFunctions handle (nclopf_b200.h)
 * with variable bounds xl/xu, start x0 (n) and row bounds gl/gu (m; gl == gu
 * marks an equality row, +-1e20 or beyond means no bound). Host arrays,
 * copied once; the whole iteration then stays in HBM. */
typedef struct ncl_model* ncl_model_handle;
typedef struct ncl_solver* ncl_solver_t;
int ncl_options_default(ncl_options* o);
int ncl_solver_create(ncl_model_handle M, const double* xl, const double* xu, const double* x0, const double* gl,
                      const double* gu, ncl_solver_t* out);
void ncl_solver_destroy(ncl_solver_t S);
int ncl_solver_solve(ncl_solver_t S, const ncl_options* opt, ncl_result* res);
/* final x (n), y (m), r (m); any may be NULL */
int ncl_solver_solution(ncl_solver_t S, double* x, double* y, double* r);
/* one Newton step (see ncl_ipm_state) at the given state; opt supplies
 * pivot_tol / refine_target / refine_max_sweeps (NULL = defaults). Runs the
 * same device path as an IPM iteration: eval -> newton -> K2 assembly -> K3
 * factor -> K4 refined solve -> recovery. */
int ncl_solver_newton_step(ncl_solver_t S, const ncl_ipm_state* st, const ncl_options* opt, ncl_newton_step* out);
/* JSON-lines trace; *len = full size */
int ncl_solver_trace(ncl_solver_t S, char* buf, int64_t cap, int64_t* len);
/* variable-bound multipliers (zl, zu: n) at the last solution and the
 * objective scale sf of the scaled Lagrangian sf f + y'(c - r - s) - zl'(x - xl)
 * - zu'(xu - x) - ... (csrc/host/ipm_elem.hpp); the inputs of mpcc_check */
int ncl_solver_bound_duals(ncl_solver_t S, double* zl, double* zu, double* sf);

#ifdef __cplusplus
}
#endif
#endif
