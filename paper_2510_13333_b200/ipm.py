"""NCL + IPM solve on the B200 backend (C-ABI include/nclopf_ipm.h).

Mirrors SPEC.md's `ncl_solve(model, params) -> NclResult`:
the host C++ control flow runs inside libnclopf_b200.so and keeps the whole
iteration in HBM; Python only passes the bounds once and reads scalars back.
"""
from __future__ import annotations

import ctypes as C
import json
import re
from dataclasses import dataclass

import numpy as np

from ._lib import P, check, i32, i64, lib, register
from .sparse import _f64, _ptr

f64 = C.c_double

_OPT_FIELDS = [
    ("rho0", f64), ("rho_growth", f64), ("rho_max", f64), ("eta_star", f64), ("omega_star", f64),
    ("eta0", f64), ("omega0", f64), ("lambda_max", f64), ("max_outer", i32), ("max_inner", i32),
    ("mu_init", f64), ("mu_min", f64), ("kappa_mu", f64), ("theta_mu", f64), ("kappa_eps", f64),
    ("tau_min", f64), ("bound_push", f64), ("bound_frac", f64), ("kappa_sigma", f64), ("s_max", f64),
    ("obj_max_grad", f64),
    ("gamma_theta", f64), ("gamma_phi", f64), ("eta_phi", f64), ("delta", f64), ("s_theta", f64), ("s_phi", f64),
    ("alpha_min_frac", f64), ("max_backtrack", i32),
    ("dw_first_rel", f64), ("dw_growth", f64), ("dw_decrease", f64), ("dw_max", f64), ("dc_base", f64),
    ("kappa_c", f64), ("dw_reuse", i32), ("pivot_tol", f64), ("refine_target", f64), ("refine_max_sweeps", i32),
    ("mu_warm_frac", f64), ("acceptable_factor", f64), ("acceptable_iter", i32), ("verbose", i32),
]


class NclOptions(C.Structure):
    """ncl_options (NclParams SPEC.md:401-404 + IPM constants SPEC.md:336-380)."""
    _fields_ = _OPT_FIELDS


class NclResult(C.Structure):
    _fields_ = [
        ("status", i32), ("outer_iters", i32), ("inner_iters", i32), ("factorizations", i32), ("restorations", i32),
        ("objective", f64), ("r_inf", f64), ("inf_pr", f64), ("inf_du", f64), ("compl_", f64), ("rho", f64),
        ("mu", f64), ("multiplier_warning", i32),
        ("t_total", f64), ("t_init", f64), ("t_eval", f64), ("t_factor", f64), ("t_solve", f64),
        ("t_linesearch", f64), ("t_other", f64), ("final_e0", f64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class IpmState(C.Structure):
    """ncl_ipm_state: a primal-dual point of the NCL subproblem (host arrays)."""
    _fields_ = [(k, C.c_void_p) for k in ("x", "zl", "zu", "r", "s", "y", "vl", "vu", "lamN")] + [
        (k, f64) for k in ("mu", "rho", "sf", "dw", "dc")]


class NewtonStep(C.Structure):
    """ncl_newton_step: the recovered Newton direction + solve/factor report."""
    _fields_ = [(k, C.c_void_p) for k in ("dx", "dzl", "dzu", "dr", "ds", "dy", "dvl", "dvu")] + [
        ("residual", f64), ("sweeps", i32), ("converged", i32), ("status", i32), ("npos", i32), ("nneg", i32),
        ("nzero", i32)]


STEP_X = ("dx", "dzl", "dzu")
STEP_ROW = ("dr", "ds", "dy", "dvl", "dvu")


def pack_state(state: dict, n: int, m: int):
    """(IpmState, keep-alive arrays) from a dict with x, zl, zu (n), r, s, y,
    vl, vu, lamN (m) and scalars mu, rho, sf, dw, dc."""
    keep = {k: _f64(state[k]) for k in ("x", "zl", "zu", "r", "s", "y", "vl", "vu", "lamN")}
    for k in ("x", "zl", "zu"):
        assert keep[k].shape == (n,), k
    for k in ("r", "s", "y", "vl", "vu", "lamN"):
        assert keep[k].shape == (m,), k
    st = IpmState(**{k: keep[k].ctypes.data for k in keep},
                  **{k: float(state.get(k, d)) for k, d in (("mu", 0.1), ("rho", 100.0), ("sf", 1.0),
                                                             ("dw", 0.0), ("dc", 0.0))})
    return st, keep


def alloc_step(n: int, m: int):
    arrs = {k: np.zeros(n) for k in STEP_X} | {k: np.zeros(m) for k in STEP_ROW}
    return NewtonStep(**{k: a.ctypes.data for k, a in arrs.items()}), arrs


STATUS = {0: "optimal", 1: "infeasible", 2: "iteration_limit", 3: "regularization_exhausted",
          4: "restoration_failed", 5: "acceptable"}

register({
    "ncl_options_default": (i32, [C.POINTER(NclOptions)]),
    "ncl_solver_create": (i32, [P, P, P, P, P, P, C.POINTER(P)]),
    "ncl_solver_destroy": (None, [P]),
    "ncl_solver_solve": (i32, [P, C.POINTER(NclOptions), C.POINTER(NclResult)]),
    "ncl_solver_solution": (i32, [P, P, P, P]),
    "ncl_solver_bound_duals": (i32, [P, P, P, C.POINTER(f64)]),
    "ncl_solver_trace": (i32, [P, C.c_char_p, i64, C.POINTER(i64)]),
    "ncl_solver_newton_step": (i32, [P, C.POINTER(IpmState), C.POINTER(NclOptions), C.POINTER(NewtonStep)]),
})


def default_options(**overrides) -> NclOptions:
    o = NclOptions()
    check(lib.ncl_options_default(C.byref(o)))
    for k, v in overrides.items():
        setattr(o, k, v)
    return o


_NONFINITE = re.compile(r"(?<=[:\s])(-?)(inf|nan)\b")


def parse_trace(text: str):
    """JSON-lines trace; printf's inf/nan become JSON Infinity/NaN."""
    fix = lambda l: _NONFINITE.sub(lambda m: m.group(1) + "Infinity" if m.group(2) == "inf" else "NaN", l)
    return [json.loads(fix(l)) for l in text.splitlines() if l.strip()]


@dataclass
class SolveOutput:
    result: dict
    status: str
    x: np.ndarray
    y: np.ndarray
    r: np.ndarray
    trace: list


class NclSolver:
    """ncl_solve on the GPU: model = ModelFunctions (paper_2510_13333_b200.model),
    bounds = dict(xl, xu, x0, gl, gu) (host arrays)."""

    def __init__(self, model, bounds):
        self.model = model
        self.n, self.m = model.n, model.m
        arrs = [_f64(bounds[k]) for k in ("xl", "xu", "x0", "gl", "gu")]
        h = C.c_void_p()
        check(lib.ncl_solver_create(model.handle, *[_ptr(a) for a in arrs], C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.ncl_solver_destroy(h)
            self._h = None

    def bound_duals(self):
        """(zl, zu, sf) of the last solve: variable-bound multipliers and the
        objective scale of the scaled Lagrangian (csrc/host/ipm_elem.hpp)"""
        n = self.n
        zl, zu, sf = np.empty(n), np.empty(n), C.c_double()
        check(lib.ncl_solver_bound_duals(self._h, _ptr(zl), _ptr(zu), C.byref(sf)))
        return zl, zu, sf.value

    def solve(self, options: NclOptions | None = None) -> SolveOutput:
        o = options if options is not None else default_options()
        res = NclResult()
        check(lib.ncl_solver_solve(self._h, C.byref(o), C.byref(res)))
        x, y, r = np.empty(self.n), np.empty(self.m), np.empty(self.m)
        check(lib.ncl_solver_solution(self._h, _ptr(x), _ptr(y), _ptr(r)))
        ln = C.c_int64()
        check(lib.ncl_solver_trace(self._h, None, 0, C.byref(ln)))
        buf = C.create_string_buffer(ln.value + 1)
        check(lib.ncl_solver_trace(self._h, buf, ln.value + 1, C.byref(ln)))
        d = res.as_dict()
        return SolveOutput(d, STATUS.get(res.status, str(res.status)), x, y, r, parse_trace(buf.value.decode()))


    def newton_step(self, state: dict, options: NclOptions | None = None) -> dict:
        """One Newton step at `state` (ncl_solver_newton_step): the recovered
        direction dx, dzl, dzu, dr, ds, dy, dvl, dvu plus the factor/solve report."""
        o = options if options is not None else default_options()
        st, keep = pack_state(state, self.n, self.m)
        out, arrs = alloc_step(self.n, self.m)
        check(lib.ncl_solver_newton_step(self._h, C.byref(st), C.byref(o), C.byref(out)))
        del keep
        return arrs | {k: getattr(out, k) for k in ("residual", "sweeps", "converged", "status", "npos", "nneg",
                                                     "nzero")}


def solve_scopf(scopf, options: NclOptions | None = None) -> SolveOutput:
    """Build the model of a Scopf instance and run ncl_solve on the GPU."""
    M = scopf.build_model()
    s = NclSolver(M, scopf.bounds())
    out = s.solve(options)
    del s
    return out
