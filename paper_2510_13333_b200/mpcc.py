"""mpcc_check (Eq. 6-11) over the C-ABI
(include/nclopf_mpcc.h): index sets, MPCC-multiplier recovery and the
strong-stationarity certificate, plus the certificate of a GPU SCOPF solve."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import P, InvalidArgument, check, f64, i32, lib, register
from .sparse import _ptr

PLUS_ZERO, ZERO_PLUS, ZERO_ZERO = 0, 1, 2


class MpccCert(C.Structure):
    _fields_ = [("n_p0", i32), ("n_0p", i32), ("n_00", i32), ("grad_residual", f64), ("feas_residual", f64),
                ("comp_residual", f64), ("inactive_violations", i32), ("sign_violations", i32),
                ("first_violation", i32), ("strong", i32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


register({
    "ncl_mpcc_index_sets": (i32, [i32, P, P, f64, P, C.POINTER(i32)]),
    "ncl_mpcc_recover": (i32, [i32, P, P, P, P, P, P, P]),
    "ncl_mpcc_certify": (i32, [i32, P, P, P, P, f64, f64, f64, f64, P, C.POINTER(MpccCert)]),
    "ncl_scopf_comp_pairs": (i32, [P, P, P, P, P, P]),
})


class BothPositive(InvalidArgument):
    """index_sets: complementarity violated at `index`."""

    def __init__(self, code, msg, index):
        super().__init__(code, msg)
        self.index = index


def _a(x):
    return np.ascontiguousarray(x, np.float64)


def index_sets(w1, w2, tol_act=1e-6):
    """(I+0, I0+, I00) as index arrays"""
    w1, w2 = _a(w1), _a(w2)
    p = len(w1)
    cls = np.empty(p, np.int8)
    bad = C.c_int(-1)
    rc = lib.ncl_mpcc_index_sets(p, _ptr(w1), _ptr(w2), float(tol_act), _ptr(cls), C.byref(bad))
    if rc != 0 and bad.value >= 0:
        raise BothPositive(rc, f"BothPositive({bad.value})", bad.value)
    check(rc)
    return tuple(np.flatnonzero(cls == k) for k in (PLUS_ZERO, ZERO_PLUS, ZERO_ZERO))


def recover(nu0, nu1, nu2, w1, w2):
    """(mu1, mu2) = (nu1 - nu0 o w2, nu2 - nu0 o w1)"""
    arrs = [_a(v) for v in (nu0, nu1, nu2, w1, w2)]
    p = len(arrs[0])
    mu1, mu2 = np.empty(p), np.empty(p)
    check(lib.ncl_mpcc_recover(p, *[_ptr(v) for v in arrs], _ptr(mu1), _ptr(mu2)))
    return mu1, mu2


def certify(w1, w2, mu1, mu2, grad_residual, feas_residual, tol=1e-6, tol_act=1e-6) -> dict:
    """certify_strong"""
    arrs = [_a(v) for v in (w1, w2, mu1, mu2)]
    p = len(arrs[0])
    cls = np.empty(p, np.int8)
    out = MpccCert()
    check(lib.ncl_mpcc_certify(p, *[_ptr(v) for v in arrs], float(grad_residual), float(feas_residual), float(tol),
                               float(tol_act), _ptr(cls), C.byref(out)))
    d = out.as_dict()
    d["strong"] = bool(d["strong"])
    d["cls"] = cls
    return d


@dataclass
class CompPairs:
    rows: np.ndarray
    w1var: np.ndarray
    xvar: np.ndarray
    side: np.ndarray
    bound: np.ndarray


def scopf_pairs(scopf) -> CompPairs:
    p = scopf.info.ncomp
    rows, w1, xv, side = (np.empty(p, np.int32) for _ in range(4))
    bound = np.empty(p)
    check(lib.ncl_scopf_comp_pairs(scopf.handle, _ptr(rows), _ptr(w1), _ptr(xv), _ptr(side), _ptr(bound)))
    return CompPairs(rows, w1, xv, side, bound)


def certify_scopf(scopf, solver, out, tol=1e-6, tol_act=1e-6) -> dict:
    """Certificate of a GPU NCL solve of a SCOPF (ipm.NclSolver after solve):
    w1 = recourse variable, w2 = distance of the generator output to the
    limit it is paired with; nu0 = multiplier of the row w1 w2 <= 0 (y >= 0
    under the scaled Lagrangian of ipm_elem.hpp), nu1, nu2 = the bound
    multipliers of w1 >= 0 and of the limit; all divided by the objective
    scale sf. grad_residual is the NLP's dual infeasibility (equal to
    ||grad L^MPCC|| by the recovery identity), feas_residual the NCL ||r||."""
    cp = scopf_pairs(scopf)
    x, y = out.x, out.y
    zl, zu, sf = solver.bound_duals()
    w1 = x[cp.w1var]
    w2 = cp.side * (x[cp.xvar] - cp.bound)
    nu0 = y[cp.rows] / sf
    nu1 = zl[cp.w1var] / sf
    nu2 = np.where(cp.side < 0, zu[cp.xvar], zl[cp.xvar]) / sf
    mu1, mu2 = recover(nu0, nu1, nu2, w1, w2)
    d = certify(w1, w2, mu1, mu2, out.result["inf_du"], out.result["r_inf"], tol, tol_act)
    d.update(w1=w1, w2=w2, mu1=mu1, mu2=mu2, nu0=nu0)
    return d


__all__ = ["index_sets", "recover", "certify", "certify_scopf", "scopf_pairs", "BothPositive", "PLUS_ZERO",
           "ZERO_PLUS", "ZERO_ZERO"]
