"""Python mirror of the reference model_ad API over the B200 C-ABI.

``Expr`` builds expression DAGs with the operators of nclopf::Expr
(/root/reference/proj/include/nclopf/expr.hpp:46-81); ``program()`` lowers one
to the C-ABI node array (include/nclopf_expr_program.h) which both the
product and the oracle replay through their smart constructors.
``ModelBuilder``/``ModelFunctions``/``fd_check`` mirror model.hpp:29-109.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import P, check, f64, i32, i64, lib, register
from .sparse import HOST, SparseSym, _f64, _i32, _ptr

CONST, VAR, PARAM, ADD, SUB, MUL, DIV, POW, NEG, SIN, COS = range(11)


class ExprNode(C.Structure):
    _fields_ = [("op", C.c_int32), ("a", C.c_int32), ("b", C.c_int32), ("slot", C.c_int32), ("value", C.c_double)]


register({
    "ncl_builder_create": (i32, [i32, C.POINTER(P)]),
    "ncl_builder_destroy": (None, [P]),
    "ncl_builder_num_vars": (i32, [P]),
    "ncl_builder_num_rows": (i32, [P]),
    "ncl_builder_add_template": (i32, [P, i32, P, i32, C.c_char_p, C.POINTER(i32)]),
    "ncl_builder_add_rows": (i32, [P, i32, C.POINTER(i32)]),
    "ncl_builder_add_objective_terms": (i32, [P, i32, i64, i32, P, i32, P]),
    "ncl_builder_add_constraint_terms": (i32, [P, i32, i64, P, i32, P, i32, P]),
    "ncl_builder_build": (i32, [P, C.POINTER(P)]),
    "ncl_model_destroy": (None, [P]),
    "ncl_model_sizes": (i32, [P, C.POINTER(i32), C.POINTER(i32), C.POINTER(i64), C.POINTER(i64)]),
    "ncl_model_jac_coords": (i32, [P, P, P]),
    "ncl_model_hess_coords": (i32, [P, P, P]),
    "ncl_model_eval_objective": (i32, [P, P, P, i32]),
    "ncl_model_eval_grad_objective": (i32, [P, P, P, i32]),
    "ncl_model_eval_constraints": (i32, [P, P, P, i32]),
    "ncl_model_eval_jacobian": (i32, [P, P, P, i32]),
    "ncl_model_eval_hessian_lag": (i32, [P, P, f64, P, P, i32]),
    "ncl_model_hessian_lag": (i32, [P, P, f64, P, C.POINTER(P)]),
    "ncl_model_jac_times": (i32, [P, P, P, P, i32]),
    "ncl_model_jac_trans_times": (i32, [P, P, P, P, i32]),
    "ncl_model_eval_all_device": (i32, [P, P, f64, P, P, P, P, P, P]),
    "ncl_model_eval_values_device": (i32, [P, P, P, P]),
    "ncl_model_check_domain": (i32, [P]),
    "ncl_fd_check": (i32, [P, P, C.c_uint, f64, P, C.POINTER(i32)]),
})


class Expr:
    """Expression DAG node (same operator set as nclopf::Expr)."""

    __slots__ = ("op", "a", "b", "slot", "value")

    def __init__(self, op, a=None, b=None, slot=-1, value=0.0):
        self.op, self.a, self.b, self.slot, self.value = op, a, b, slot, float(value)

    @staticmethod
    def constant(v):
        return Expr(CONST, value=v)

    @staticmethod
    def var(slot):
        return Expr(VAR, slot=slot)

    @staticmethod
    def param(slot):
        return Expr(PARAM, slot=slot)

    @staticmethod
    def _w(x):
        return x if isinstance(x, Expr) else Expr.constant(x)

    def __add__(self, o): return Expr(ADD, self, Expr._w(o))
    def __radd__(self, o): return Expr(ADD, Expr._w(o), self)
    def __sub__(self, o): return Expr(SUB, self, Expr._w(o))
    def __rsub__(self, o): return Expr(SUB, Expr._w(o), self)
    def __mul__(self, o): return Expr(MUL, self, Expr._w(o))
    def __rmul__(self, o): return Expr(MUL, Expr._w(o), self)
    def __truediv__(self, o): return Expr(DIV, self, Expr._w(o))
    def __rtruediv__(self, o): return Expr(DIV, Expr._w(o), self)
    def __neg__(self): return Expr(NEG, self)
    def __pow__(self, e): return Expr(POW, self, value=float(e))

    def program(self):
        """Post-order node array (root last), shared subtrees emitted once."""
        out, index = [], {}
        stack = [(self, False)]
        while stack:
            e, done = stack.pop()
            if id(e) in index:
                continue
            if not done:
                stack.append((e, True))
                if e.b is not None:
                    stack.append((e.b, False))
                if e.a is not None:
                    stack.append((e.a, False))
                continue
            a = index[id(e.a)] if e.a is not None else -1
            b = index[id(e.b)] if e.b is not None else -1
            index[id(e)] = len(out)
            out.append((e.op, a, b, e.slot, e.value))
        arr = (ExprNode * len(out))()
        for k, (op, a, b, s, v) in enumerate(out):
            arr[k].op, arr[k].a, arr[k].b, arr[k].slot, arr[k].value = op, a, b, s, v
        return arr


def sin(x): return Expr(SIN, Expr._w(x))
def cos(x): return Expr(COS, Expr._w(x))


class ModelFunctions:
    """nclopf::ModelFunctions (model.hpp:29-71), evaluated on the GPU."""

    def __init__(self, h):
        self._h = h
        n, m, nj, nh = C.c_int(), C.c_int(), C.c_int64(), C.c_int64()
        check(lib.ncl_model_sizes(h, C.byref(n), C.byref(m), C.byref(nj), C.byref(nh)))
        self.n, self.m, self.nnzj, self.nnzh = n.value, m.value, nj.value, nh.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.ncl_model_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def num_vars(self): return self.n
    def num_cons(self): return self.m

    def jac_coords(self):
        r, c = np.empty(self.nnzj, np.int32), np.empty(self.nnzj, np.int32)
        check(lib.ncl_model_jac_coords(self._h, _ptr(r), _ptr(c)))
        return r, c

    def hess_coords(self):
        r, c = np.empty(self.nnzh, np.int32), np.empty(self.nnzh, np.int32)
        check(lib.ncl_model_hess_coords(self._h, _ptr(r), _ptr(c)))
        return r, c

    def eval_objective(self, w):
        out = np.zeros(1)
        check(lib.ncl_model_eval_objective(self._h, _ptr(_f64(w)), _ptr(out), HOST))
        return float(out[0])

    def _vec(self, fn, w, size, *extra):
        out = np.empty(size)
        check(fn(self._h, _ptr(_f64(w)), *extra, _ptr(out), HOST))
        return out

    def eval_grad_objective(self, w): return self._vec(lib.ncl_model_eval_grad_objective, w, self.n)
    def eval_constraints(self, w): return self._vec(lib.ncl_model_eval_constraints, w, self.m)
    def eval_jacobian(self, w): return self._vec(lib.ncl_model_eval_jacobian, w, self.nnzj)

    def eval_hessian_lag(self, w, sigma, lam):
        out = np.empty(self.nnzh)
        check(lib.ncl_model_eval_hessian_lag(self._h, _ptr(_f64(w)), float(sigma), _ptr(_f64(lam)), _ptr(out),
                                             HOST))
        return out

    def hessian_lag(self, w, sigma, lam) -> SparseSym:
        h = C.c_void_p()
        check(lib.ncl_model_hessian_lag(self._h, _ptr(_f64(w)), float(sigma), _ptr(_f64(lam)), C.byref(h)))
        S = SparseSym.__new__(SparseSym)
        S._h = h
        return S

    def jac_times(self, jv, v):
        out = np.empty(self.m)
        check(lib.ncl_model_jac_times(self._h, _ptr(_f64(jv)), _ptr(_f64(v)), _ptr(out), HOST))
        return out

    def jac_trans_times(self, jv, y):
        out = np.empty(self.n)
        check(lib.ncl_model_jac_trans_times(self._h, _ptr(_f64(jv)), _ptr(_f64(y)), _ptr(out), HOST))
        return out


class ModelBuilder:
    """nclopf::ModelBuilder (model.hpp:74-97)."""

    def __init__(self, num_vars: int):
        h = C.c_void_p()
        check(lib.ncl_builder_create(int(num_vars), C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.ncl_builder_destroy(h)
            self._h = None

    def num_vars(self): return lib.ncl_builder_num_vars(self._h)
    def num_rows(self): return lib.ncl_builder_num_rows(self._h)

    def add_template(self, f: Expr, num_var_slots: int, name: str = "") -> int:
        prog = f.program() if isinstance(f, Expr) else f
        tid = C.c_int()
        check(lib.ncl_builder_add_template(self._h, len(prog), prog, int(num_var_slots), name.encode(),
                                           C.byref(tid)))
        return tid.value

    def add_rows(self, count: int) -> int:
        first = C.c_int()
        check(lib.ncl_builder_add_rows(self._h, int(count), C.byref(first)))
        return first.value

    def add_objective_terms(self, tid, vars_, params=None):
        v = _i32(np.atleast_2d(vars_))
        cnt, nv = v.shape
        p = None if params is None else _f64(np.atleast_2d(params))
        np_ = 0 if p is None else p.shape[1]
        check(lib.ncl_builder_add_objective_terms(self._h, tid, cnt, nv, _ptr(v), np_, _ptr(p)))

    def add_objective_term(self, tid, vars_, params=()):
        self.add_objective_terms(tid, [list(vars_)], [list(params)] if len(params) else None)

    def add_constraint_terms(self, tid, rows, vars_, params=None):
        r = _i32(np.atleast_1d(rows))
        v = _i32(np.asarray(vars_).reshape(len(r), -1))
        p = None if params is None else _f64(np.asarray(params, dtype=np.float64).reshape(len(r), -1))
        np_ = 0 if p is None else p.shape[1]
        check(lib.ncl_builder_add_constraint_terms(self._h, tid, len(r), _ptr(r), v.shape[1], _ptr(v), np_,
                                                   _ptr(p)))

    def add_constraint_term(self, tid, row, vars_, params=()):
        self.add_constraint_terms(tid, [row], [list(vars_)], [list(params)] if len(params) else None)

    def build(self) -> ModelFunctions:
        h = C.c_void_p()
        check(lib.ncl_builder_build(self._h, C.byref(h)))
        return ModelFunctions(h)


def fd_check(m: ModelFunctions, w, seed: int, tol: float = 1e-6):
    errs = np.zeros(3)
    ok = C.c_int()
    check(lib.ncl_fd_check(m.handle, _ptr(_f64(w)), int(seed), float(tol), _ptr(errs), C.byref(ok)))
    return dict(grad_err=errs[0], jac_err=errs[1], hess_err=errs[2], pass_=bool(ok.value))
