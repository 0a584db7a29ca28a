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
# NCL_REF_VARIANT=fma loads oracle/_ref_fma (the same reference sources built
# with FMA contraction, oracle/Makefile) — used only by tools/oracle_solve.py
_VARIANT = os.environ.get("NCL_REF_VARIANT", "")
LIB = os.path.join(HERE, "_ref" + (f"_{_VARIANT}" if _VARIANT else ""), "libnclopf_ref.so")


def build(force: bool = False) -> str:
    """Build oracle/_ref from /root/reference (only possible where it exists)."""
    if force or not os.path.exists(LIB):
        if not os.path.isdir("/root/reference/proj/src"):
            raise RuntimeError("oracle/_ref missing and /root/reference absent: cannot build the oracle here")
        subprocess.run(["make", "-C", HERE, "-j8"] + ([f"VARIANT={_VARIANT}"] if _VARIANT else []), check=True,
                       capture_output=True)
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
            "ref_ipm_last_error": (C.c_char_p, []),
            "ref_ipm_default_options": (None, [P]),
            "ref_ncl_solve": (i32, [P, P, P, P, P, P, P, P, P, P, P, P, C.c_char_p, i64, C.POINTER(i64)]),
            "ref_scopf_last_error": (C.c_char_p, []),
            "ref_scopf_new": (i32, [i32, i32, i32, i32, C.c_uint64, i32, P, C.POINTER(P), pi, pi]),
            "ref_scopf_free": (None, [P]),
            "ref_scopf_bounds": (None, [P, P, P, P, P, P]),
            "ref_scopf_model": (i32, [P, C.POINTER(P)]),
            "ref_condensed_kkt": (i32, [P, P, P, P, f64, P, C.POINTER(P)]),
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


class RefModel:
    """The reference nclopf::ModelFunctions, built from the same spec
    (template node programs + instances) as the product model."""

    def __init__(self, h):
        self.h = h
        n, m, nj, nh = C.c_int(), C.c_int(), C.c_int64(), C.c_int64()
        lib().ref_mf_sizes(h, C.byref(n), C.byref(m), C.byref(nj), C.byref(nh))
        self.n, self.m, self.nnzj, self.nnzh = n.value, m.value, nj.value, nh.value

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_mf_free(self.h)
            self.h = None

    @staticmethod
    def from_families(n, m, families):
        """families: iterable of objects with name, nodes (ctypes array),
        nslots, np, objective, rows, vars[ninst, nslots], params[ninst, np]."""
        L = lib()
        b = L.ref_mb_new(int(n))
        try:
            if m:
                L.ref_mb_add_rows(b, int(m))
            for F in families:
                tid = C.c_int()
                _chk(L.ref_mb_add_template(b, len(F.nodes), C.cast(F.nodes, C.c_void_p), int(F.nslots),
                                           F.name.encode(), C.byref(tid)))
                cnt = F.vars.shape[0] if F.nslots else len(F.rows)
                if cnt == 0:
                    continue
                v = np.ascontiguousarray(F.vars, np.int32)
                p = np.ascontiguousarray(F.params, np.float64) if F.np else None
                r = None if F.objective else np.ascontiguousarray(F.rows, np.int32)
                _chk(L.ref_mb_add_terms(b, tid.value, 1 if F.objective else 0, cnt, int(F.nslots), _p(v),
                                        int(F.np), _p(p), _p(r)))
            h = C.c_void_p()
            _chk(L.ref_mb_build(b, C.byref(h)))
        finally:
            L.ref_mb_free(b)
        return RefModel(h)

    def jac_coords(self):
        r, c = np.empty(self.nnzj, np.int32), np.empty(self.nnzj, np.int32)
        lib().ref_mf_jac_coords(self.h, _p(r), _p(c))
        return r, c

    def hess_coords(self):
        r, c = np.empty(self.nnzh, np.int32), np.empty(self.nnzh, np.int32)
        lib().ref_mf_hess_coords(self.h, _p(r), _p(c))
        return r, c

    def eval_objective(self, w):
        o = C.c_double()
        _chk(lib().ref_mf_eval_objective(self.h, _p(np.ascontiguousarray(w, np.float64)), C.byref(o)))
        return o.value

    def _v(self, fn, w, size, *extra):
        out = np.empty(size)
        _chk(fn(self.h, _p(np.ascontiguousarray(w, np.float64)), *extra, _p(out)))
        return out

    def eval_grad_objective(self, w): return self._v(lib().ref_mf_eval_grad, w, self.n)
    def eval_constraints(self, w): return self._v(lib().ref_mf_eval_cons, w, self.m)
    def eval_jacobian(self, w): return self._v(lib().ref_mf_eval_jac, w, self.nnzj)

    def eval_hessian_lag(self, w, sigma, lam):
        return self._v(lib().ref_mf_eval_hess, w, self.nnzh, float(sigma),
                       _p(np.ascontiguousarray(lam, np.float64)))

    def jac_times(self, jv, v):
        out = np.empty(self.m)
        _chk(lib().ref_mf_jac_times(self.h, _p(np.ascontiguousarray(jv)), _p(np.ascontiguousarray(v)), _p(out)))
        return out

    def jac_trans_times(self, jv, y):
        out = np.empty(self.n)
        _chk(lib().ref_mf_jac_trans_times(self.h, _p(np.ascontiguousarray(jv)), _p(np.ascontiguousarray(y)),
                                          _p(out)))
        return out

    def fd_check(self, w, seed, tol=1e-6):
        errs = np.zeros(3)
        ok = C.c_int()
        _chk(lib().ref_mf_fd_check(self.h, _p(np.ascontiguousarray(w, np.float64)), int(seed), float(tol), _p(errs),
                                   C.byref(ok)))
        return dict(grad_err=errs[0], jac_err=errs[1], hess_err=errs[2], pass_=bool(ok.value))


class RefScopf:
    """The SCOPF instance (csrc/host/scopf.cpp compiled into the oracle) with
    its reference ModelFunctions — no product library involved. grid: 0 =
    case9, 1 = synthetic (nb, nl, ng, seed); ids: contingency ids or None."""

    def __init__(self, grid, nb, nl, ng, seed, K, ids=None):
        h, n, m = C.c_void_p(), C.c_int(), C.c_int()
        idp = None if ids is None else np.ascontiguousarray(ids, np.int32)
        if lib().ref_scopf_new(int(grid), int(nb), int(nl), int(ng), int(seed), int(K), _p(idp), C.byref(h),
                               C.byref(n), C.byref(m)):
            raise RefError(1, lib().ref_scopf_last_error().decode())
        self.h, self.n, self.m = h, n.value, m.value

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_scopf_free(self.h)
            self.h = None

    def bounds(self):
        xl, xu, x0 = (np.empty(self.n) for _ in range(3))
        gl, gu = np.empty(self.m), np.empty(self.m)
        lib().ref_scopf_bounds(self.h, _p(xl), _p(xu), _p(x0), _p(gl), _p(gu))
        return dict(xl=xl, xu=xu, x0=x0, gl=gl, gu=gu)

    def model(self) -> "RefModel":
        h = C.c_void_p()
        _chk(lib().ref_scopf_model(self.h, C.byref(h)))
        return RefModel(h)


def ref_condensed_kkt(model: "RefModel", hess, jac, sig, dw, D) -> RefSparseSym:
    """K = H + diag(sig + dw) + J' diag(D) J assembled by the reference
    SparseSym in the product's triplet order (oracle/ref_scopf.cpp)."""
    h = C.c_void_p()
    a = [np.ascontiguousarray(v, np.float64) for v in (hess, jac, sig)]
    Dv = np.ascontiguousarray(D, np.float64)
    if lib().ref_condensed_kkt(model.h, _p(a[0]), _p(a[1]), _p(a[2]), float(dw), _p(Dv), C.byref(h)):
        raise RefError(1, lib().ref_scopf_last_error().decode())
    K = RefSparseSym.__new__(RefSparseSym)
    K.h, K.n = h, model.n
    return K


def ref_newton_step(model: RefModel, bounds, state: dict, options=None) -> dict:
    """One Newton step at `state` on the reference CPU backend (the oracle side
    of ncl_solver_newton_step)."""
    from paper_2510_13333_b200.ipm import NclOptions, NewtonStep, IpmState, alloc_step, pack_state

    L = lib()
    if not hasattr(L, "_ns_sig"):
        L.ref_newton_step.restype = C.c_int
        L.ref_newton_step.argtypes = [C.c_void_p] * 6 + [C.POINTER(IpmState), C.POINTER(NclOptions),
                                                         C.POINTER(NewtonStep)]
        L._ns_sig = True
    if options is None:
        options = NclOptions()
        L.ref_ipm_default_options(C.byref(options))
    arrs = [np.ascontiguousarray(bounds[k], np.float64) for k in ("xl", "xu", "x0", "gl", "gu")]
    st, keep = pack_state(state, model.n, model.m)
    out, res = alloc_step(model.n, model.m)
    rc = L.ref_newton_step(model.h, *[_p(a) for a in arrs], C.byref(st), C.byref(options), C.byref(out))
    if rc != 0:
        raise RefError(rc, L.ref_ipm_last_error().decode())
    del keep
    return res | {k: getattr(out, k) for k in ("residual", "sweeps", "converged", "status", "npos", "nneg", "nzero")}


def ref_ncl_solve(model: RefModel, bounds, perm=None, options=None, trace_cap=1 << 26):
    """ncl_solve over the reference CPU backend (oracle/ref_ipm.cpp): the same
    host NCL/IPM control flow driving the UNMODIFIED reference model_ad and
    sparse_core. `options` is a paper_2510_13333_b200.ipm.NclOptions (the
    ctypes mirror of include/nclopf_ipm.h) or None for the defaults."""
    import json

    from paper_2510_13333_b200.ipm import STATUS, NclOptions, NclResult

    L = lib()
    if options is None:
        options = NclOptions()
        L.ref_ipm_default_options(C.byref(options))
    arrs = [np.ascontiguousarray(bounds[k], np.float64) for k in ("xl", "xu", "x0", "gl", "gu")]
    pm = None if perm is None else np.ascontiguousarray(perm, np.int32)
    res = NclResult()
    x, y, r = np.empty(model.n), np.empty(model.m), np.empty(model.m)
    buf = C.create_string_buffer(trace_cap)
    ln = C.c_int64()
    rc = L.ref_ncl_solve(model.h, *[_p(a) for a in arrs], _p(pm), C.byref(options), C.byref(res), _p(x), _p(y),
                         _p(r), buf, trace_cap, C.byref(ln))
    if rc != 0:
        raise RefError(rc, L.ref_ipm_last_error().decode())
    from paper_2510_13333_b200.ipm import parse_trace

    trace = parse_trace(buf.value.decode())
    return dict(result=res.as_dict(), status=STATUS.get(res.status, str(res.status)), x=x, y=y, r=r, trace=trace)
