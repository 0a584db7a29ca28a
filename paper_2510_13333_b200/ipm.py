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


STATUS = {0: "optimal", 1: "infeasible", 2: "iteration_limit", 3: "regularization_exhausted",
          4: "restoration_failed", 5: "acceptable"}

register({
    "ncl_options_default": (i32, [C.POINTER(NclOptions)]),
    "ncl_solver_create": (i32, [P, P, P, P, P, P, C.POINTER(P)]),
    "ncl_solver_destroy": (None, [P]),
    "ncl_solver_solve": (i32, [P, C.POINTER(NclOptions), C.POINTER(NclResult)]),
    "ncl_solver_solution": (i32, [P, P, P, P]),
    "ncl_solver_trace": (i32, [P, C.c_char_p, i64, C.POINTER(i64)]),
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


def solve_scopf(scopf, options: NclOptions | None = None) -> SolveOutput:
    """Build the model of a Scopf instance and run ncl_solve on the GPU."""
    M = scopf.build_model()
    s = NclSolver(M, scopf.bounds())
    out = s.solve(options)
    del s
    return out
