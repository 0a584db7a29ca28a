"""ORACLE loader — test infrastructure only.

Loads oracle/_ref/libnclopf_ref.so (the UNMODIFIED reference C++ sources of
/root/reference/proj/src compiled by oracle/Makefile, plus the extern "C"
shim oracle/ref_capi.cpp). Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference arm may import this module. The
product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libnclopf_ref.so")


def build(force: bool = False) -> str:
    """Build oracle/_ref from /root/reference (only possible where it exists)."""
    if force or not os.path.exists(LIB):
        if not os.path.isdir("/root/reference/proj/src"):
            raise RuntimeError("oracle/_ref missing and /root/reference absent: cannot build the oracle here")
        subprocess.run(["make", "-C", HERE, "-j8"], check=True, capture_output=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        P, i32, i64, f64 = C.c_void_p, C.c_int, C.c_int64, C.c_double
        pi, pd = C.POINTER(C.c_int), C.POINTER(C.c_double)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_sym_new": (P, [i32]), "ref_sym_free": (None, [P]),
            "ref_sym_add_many": (i32, [P, i64, P, P, P]), "ref_sym_finalize": (i32, [P]),
            "ref_sym_begin_refill": (i32, [P]), "ref_sym_refill": (i32, [P]),
            "ref_sym_dim": (i32, [P]), "ref_sym_nnz": (i32, [P]),
            "ref_sym_get_csc": (None, [P, P, P, P]),
            "ref_sym_max_abs_diag": (f64, [P]), "ref_sym_norm_inf": (f64, [P]), "ref_sym_frobenius": (f64, [P]),
            "ref_sym_multiply": (i32, [P, P, P]),
            "ref_sym_write_mm": (i32, [P, C.c_char_p, i64, C.POINTER(i64)]),
            "ref_symbolic_order": (i32, [P, P]),
            "ref_analyze": (i32, [P, P, C.POINTER(P)]), "ref_symb_free": (None, [P]),
            "ref_symb_lnnz": (i64, [P]), "ref_symb_get": (None, [P, P, P, P, P, P, P, P]),
            "ref_factorize": (i32, [P, P, f64, C.POINTER(P)]), "ref_fact_free": (None, [P]),
            "ref_fact_status": (i32, [P, pi, pi, pi, pi]), "ref_fact_diag": (None, [P, P]),
            "ref_fact_get_L": (None, [P, P, P, P]), "ref_fact_solve_in_place": (i32, [P, P, i32]),
            "ref_solve_refined": (i32, [P, P, P, f64, i32, P, pd, pi, pi]),
            "ref_mb_new": (P, [i32]), "ref_mb_free": (None, [P]),
            "ref_mb_add_template": (i32, [P, i32, P, i32, C.c_char_p, pi]),
            "ref_mb_add_rows": (i32, [P, i32]),
            "ref_mb_add_terms": (i32, [P, i32, i32, i64, i32, P, i32, P, P]),
            "ref_mb_build": (i32, [P, C.POINTER(P)]), "ref_mf_free": (None, [P]),
            "ref_mf_sizes": (None, [P, pi, pi, C.POINTER(i64), C.POINTER(i64)]),
            "ref_mf_jac_coords": (None, [P, P, P]), "ref_mf_hess_coords": (None, [P, P, P]),
            "ref_mf_eval_objective": (i32, [P, P, pd]), "ref_mf_eval_grad": (i32, [P, P, P]),
            "ref_mf_eval_cons": (i32, [P, P, P]), "ref_mf_eval_jac": (i32, [P, P, P]),
            "ref_mf_eval_hess": (i32, [P, P, f64, P, P]),
            "ref_mf_jac_times": (i32, [P, P, P, P]), "ref_mf_jac_trans_times": (i32, [P, P, P, P]),
            "ref_mf_fd_check": (i32, [P, P, C.c_uint, f64, P, pi]),
        }
        for k, (r, a) in sig.items():
            fn = getattr(L, k)
            fn.restype = r
            fn.argtypes = a
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _chk(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class RefSparseSym:
    """The reference nclopf::SparseSym."""

    def __init__(self, n, rows=None, cols=None, vals=None, finalize=True):
        self.h = lib().ref_sym_new(int(n))
        self.n = int(n)
        if rows is not None:
            self.add_many(rows, cols, vals)
            if finalize:
                self.finalize()

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_sym_free(self.h)
            self.h = None

    def add_many(self, rows, cols, vals):
        r = np.ascontiguousarray(rows, np.int32)
        c = np.ascontiguousarray(cols, np.int32)
        v = np.ascontiguousarray(vals, np.float64)
        _chk(lib().ref_sym_add_many(self.h, len(r), _p(r), _p(c), _p(v)))

    def finalize(self):
        _chk(lib().ref_sym_finalize(self.h))

    def begin_refill(self):
        _chk(lib().ref_sym_begin_refill(self.h))

    def refill(self):
        _chk(lib().ref_sym_refill(self.h))

    def nnz(self):
        return lib().ref_sym_nnz(self.h)

    def csc(self):
        cp = np.empty(self.n + 1, np.int32)
        ri = np.empty(self.nnz(), np.int32)
        v = np.empty(self.nnz(), np.float64)
        lib().ref_sym_get_csc(self.h, _p(cp), _p(ri), _p(v))
        return cp, ri, v

    def max_abs_diag(self):
        return lib().ref_sym_max_abs_diag(self.h)

    def norm_inf(self):
        return lib().ref_sym_norm_inf(self.h)

    def frobenius_norm(self):
        return lib().ref_sym_frobenius(self.h)

    def multiply(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(self.n, np.float64)
        _chk(lib().ref_sym_multiply(self.h, _p(x), _p(y)))
        return y

    def write_matrix_market(self):
        n = C.c_int64()
        _chk(lib().ref_sym_write_mm(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _chk(lib().ref_sym_write_mm(self.h, buf, n.value, C.byref(n)))
        return buf.raw[: n.value].decode()


def ref_symbolic_order(M: RefSparseSym):
    perm = np.empty(M.n, np.int32)
    _chk(lib().ref_symbolic_order(M.h, _p(perm)))
    return perm


class RefSymbolic:
    def __init__(self, M: RefSparseSym, perm=None):
        h = C.c_void_p()
        p = None if perm is None else np.ascontiguousarray(perm, np.int32)
        _chk(lib().ref_analyze(M.h, _p(p), C.byref(h)))
        self.h = h
        n, nz = M.n, M.nnz()
        self.perm, self.iperm, self.parent, self.l_colcount = (np.empty(n, np.int32) for _ in range(4))
        self.up_colptr = np.empty(n + 1, np.int32)
        self.up_rowind, self.entry_map = np.empty(nz, np.int32), np.empty(nz, np.int32)
        lib().ref_symb_get(h, _p(self.perm), _p(self.iperm), _p(self.parent), _p(self.up_colptr),
                           _p(self.up_rowind), _p(self.entry_map), _p(self.l_colcount))
        self.l_nnz = lib().ref_symb_lnnz(h)
        self.n = n

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_symb_free(self.h)
            self.h = None


class RefFactorization:
    def __init__(self, M: RefSparseSym, S: RefSymbolic | None = None, pivot_tol=1e-12):
        h = C.c_void_p()
        _chk(lib().ref_factorize(M.h, None if S is None else S.h, float(pivot_tol), C.byref(h)))
        self.h, self.M, self.S, self.n = h, M, S, M.n
        zp, a, b, c = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        st = lib().ref_fact_status(h, C.byref(zp), C.byref(a), C.byref(b), C.byref(c))
        self.status = "ok" if st == 0 else "zero_pivot"
        self.zero_pivot_index = zp.value
        self.inertia = (a.value, b.value, c.value)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_fact_free(self.h)
            self.h = None

    def ok(self):
        return self.status == "ok"

    def diagonal(self):
        d = np.empty(self.n, np.float64)
        lib().ref_fact_diag(self.h, _p(d))
        return d

    def L_csc(self, l_nnz):
        lp = np.empty(self.n + 1, np.int32)
        li = np.empty(l_nnz, np.int32)
        lx = np.empty(l_nnz, np.float64)
        lib().ref_fact_get_L(self.h, _p(lp), _p(li), _p(lx))
        return lp, li, lx

    def solve(self, b):
        x = np.array(b, np.float64, copy=True)
        _chk(lib().ref_fact_solve_in_place(self.h, _p(x), self.n))
        return x

    def solve_refined(self, b, target=1e-8, max_sweeps=5):
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty(self.n, np.float64)
        r, s, cv = C.c_double(), C.c_int(), C.c_int()
        _chk(lib().ref_solve_refined(self.h, self.M.h, _p(b), float(target), int(max_sweeps), _p(x), C.byref(r),
                                     C.byref(s), C.byref(cv)))
        return x, r.value, s.value, bool(cv.value)
