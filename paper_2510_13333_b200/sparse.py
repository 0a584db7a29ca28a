"""Python mirror of the reference linear-solver API over the B200 C-ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/nclopf/sparse_sym.hpp:20-139:
``SparseSym``, ``symbolic_order``, ``analyze``, ``factorize``,
``Factorization.solve/solve_in_place/diagonal``, ``solve_refined``.
Host arrays are numpy; device arrays are any object exposing ``data_ptr()``
(e.g. torch CUDA tensors), used for the device-resident fast path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import SymbInfo, check, lib

HOST, DEVICE = 0, 1


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class SparseSym:
    """nclopf::SparseSym (sparse_sym.hpp:20-66)."""

    def __init__(self, n: int):
        h = C.c_void_p()
        check(lib.ncl_sym_create(int(n), C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.ncl_sym_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def dim(self) -> int:
        return lib.ncl_sym_dim(self._h)

    def nnz(self) -> int:
        return lib.ncl_sym_nnz(self._h)

    def finalized(self) -> bool:
        return bool(lib.ncl_sym_finalized(self._h))

    def add(self, row: int, col: int, value: float) -> None:
        self.add_many([row], [col], [value])

    def add_many(self, rows, cols, vals) -> None:
        r, c, v = _i32(rows), _i32(cols), _f64(vals)
        check(lib.ncl_sym_add(self._h, len(r), _ptr(r), _ptr(c), _ptr(v)))

    def finalize(self) -> None:
        check(lib.ncl_sym_finalize(self._h))

    def begin_refill(self) -> None:
        check(lib.ncl_sym_begin_refill(self._h))

    def refill(self) -> None:
        check(lib.ncl_sym_refill(self._h))

    def refill_values(self, trip_vals, where: int = HOST) -> None:
        v = _f64(trip_vals) if where == HOST else trip_vals
        check(lib.ncl_sym_refill_values(self._h, _ptr(v), where))

    def col_ptr(self) -> np.ndarray:
        cp = np.empty(self.dim() + 1, np.int32)
        check(lib.ncl_sym_get_csc(self._h, _ptr(cp), None, None))
        return cp

    def row_ind(self) -> np.ndarray:
        ri = np.empty(self.nnz(), np.int32)
        check(lib.ncl_sym_get_csc(self._h, None, _ptr(ri), None))
        return ri

    def values(self) -> np.ndarray:
        v = np.empty(self.nnz(), np.float64)
        check(lib.ncl_sym_get_csc(self._h, None, None, _ptr(v)))
        return v

    def set_values(self, vals, where: int = HOST) -> None:
        v = vals if (where != HOST or hasattr(vals, "data_ptr")) else _f64(vals)
        check(lib.ncl_sym_set_values(self._h, _ptr(v), where))

    def device_values_ptr(self) -> int:
        return lib.ncl_sym_device_values(self._h)

    def _scalar(self, fn) -> float:
        out = C.c_double()
        check(fn(self._h, C.byref(out)))
        return out.value

    def max_abs_diag(self) -> float:
        return self._scalar(lib.ncl_sym_max_abs_diag)

    def norm_inf(self) -> float:
        return self._scalar(lib.ncl_sym_norm_inf)

    def frobenius_norm(self) -> float:
        return self._scalar(lib.ncl_sym_frobenius_norm)

    def multiply(self, x, y=None, where: int = HOST):
        if where == HOST:
            x = _f64(x)
            y = np.empty(self.dim(), np.float64) if y is None else y
        check(lib.ncl_sym_multiply(self._h, _ptr(x), _ptr(y), where))
        return y

    def same_pattern(self, other: "SparseSym") -> bool:
        return bool(lib.ncl_sym_same_pattern(self._h, other._h))

    def write_matrix_market(self) -> str:
        n = C.c_int64()
        check(lib.ncl_sym_write_matrix_market(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(lib.ncl_sym_write_matrix_market(self._h, buf, n.value, C.byref(n)))
        return buf.raw[: n.value].decode()


def symbolic_order(M: SparseSym) -> np.ndarray:
    """symbolic_order (sparse_sym.hpp:68-70): exact minimum degree, bit-exact."""
    perm = np.empty(M.dim(), np.int32)
    check(lib.ncl_symbolic_order(M.handle, _ptr(perm)))
    return perm


@dataclass
class SymbolicInfo:
    n: int
    l_nnz: int
    nsupernodes: int
    max_height: int
    max_width: int
    max_rows: int
    l_storage: int
    flops: float
    cb_storage: int = 0
    nsplit: int = 0
    n_big: int = 0
    n_tasks: int = 0


class SymbolicFactor:
    """nclopf::SymbolicFactor (sparse_sym.hpp:74-85) + the supernodal schedule."""

    def __init__(self, h, M: SparseSym):
        self._h = h
        self._n = M.dim()
        self._nnz = M.nnz()
        self._cache = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.ncl_symb_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def _fields(self):
        if self._cache is None:
            n, nz = self._n, self._nnz
            perm, iperm, parent, lcc = (np.empty(n, np.int32) for _ in range(4))
            upc = np.empty(n + 1, np.int32)
            upr, em = np.empty(nz, np.int32), np.empty(nz, np.int32)
            check(lib.ncl_symb_get(self._h, _ptr(perm), _ptr(iperm), _ptr(parent), _ptr(upc), _ptr(upr),
                                   _ptr(em), _ptr(lcc)))
            self._cache = dict(perm=perm, iperm=iperm, parent=parent, up_colptr=upc, up_rowind=upr,
                               entry_map=em, l_colcount=lcc)
        return self._cache

    n = property(lambda self: self._n)
    perm = property(lambda self: self._fields()["perm"])
    iperm = property(lambda self: self._fields()["iperm"])
    parent = property(lambda self: self._fields()["parent"])
    up_colptr = property(lambda self: self._fields()["up_colptr"])
    up_rowind = property(lambda self: self._fields()["up_rowind"])
    entry_map = property(lambda self: self._fields()["entry_map"])
    l_colcount = property(lambda self: self._fields()["l_colcount"])

    @property
    def l_nnz(self) -> int:
        return self.info().l_nnz

    def info(self) -> SymbolicInfo:
        s = SymbInfo()
        check(lib.ncl_symb_info_get(self._h, C.byref(s)))
        return SymbolicInfo(s.n, s.l_nnz, s.nsupernodes, s.max_height, s.max_width, s.max_rows, s.l_storage,
                            s.flops, s.cb_storage, s.nsplit, s.n_big, s.n_tasks)


def supernodes(S: "SymbolicFactor"):
    """Supernode partition / parents / heights / ticket order (inspection)."""
    info = S.info()
    ns = info.nsupernodes
    first = np.empty(ns + 1, np.int32)
    rptr = np.empty(ns + 1, np.int64)
    par, h, order = (np.empty(ns, np.int32) for _ in range(3))
    check(lib.ncl_symb_supernodes(S.handle, _ptr(first), _ptr(rptr), _ptr(par), _ptr(h), _ptr(order)))
    return dict(first=first, rptr=rptr, parent=par, height=h, order=order)


def analyze(M: SparseSym, perm=None) -> SymbolicFactor:
    """analyze(M) / analyze(M, perm) (sparse_sym.hpp:87-88), bit-exact."""
    h = C.c_void_p()
    p = None if perm is None else _i32(perm)
    if p is not None and len(p) != M.dim():
        from ._lib import InvalidArgument
        raise InvalidArgument(-1, "analyze: bad permutation")
    check(lib.ncl_analyze(M.handle, _ptr(p), C.byref(h)))
    return SymbolicFactor(h, M)


@dataclass
class Inertia:
    n_pos: int = 0
    n_neg: int = 0
    n_zero: int = 0


class Factorization:
    """nclopf::Factorization (sparse_sym.hpp:97-121), device-resident."""

    def __init__(self, h, n: int, symb):
        self._h = h
        self._n = n
        self._symb = symb  # keep the symbolic factor alive (raw pointer semantics)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.ncl_fact_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def _status(self):
        st, zp, a, b, c = (C.c_int() for _ in range(5))
        check(lib.ncl_fact_status(self._h, C.byref(st), C.byref(zp), C.byref(a), C.byref(b), C.byref(c)))
        return st.value, zp.value, Inertia(a.value, b.value, c.value)

    @property
    def status(self) -> str:
        return "ok" if self._status()[0] == 0 else "zero_pivot"

    def ok(self) -> bool:
        return self._status()[0] == 0

    @property
    def zero_pivot_index(self) -> int:
        return self._status()[1]

    @property
    def inertia(self) -> Inertia:
        return self._status()[2]

    def diagonal(self) -> np.ndarray:
        d = np.empty(self._n, np.float64)
        check(lib.ncl_fact_diagonal(self._h, _ptr(d)))
        return d

    def solve_in_place(self, x, where: int = HOST) -> None:
        if where == HOST:
            if hasattr(x, "data_ptr"):  # pinned torch CPU tensor
                assert str(x.dtype) == "torch.float64" and x.is_contiguous() and not x.is_cuda
            else:
                assert x.dtype == np.float64 and x.flags.c_contiguous
        check(lib.ncl_fact_solve(self._h, _ptr(x), where))

    def solve(self, b) -> np.ndarray:
        x = np.array(b, dtype=np.float64, copy=True)
        self.solve_in_place(x)
        return x

    def refactorize(self, M: SparseSym, pivot_tol: float = 1e-12) -> None:
        check(lib.ncl_refactorize(self._h, M.handle, float(pivot_tol)))

    def factor_solve_host(self, M: SparseSym, vals, b, x, pivot_tol: float = 1e-12):
        """ncl_factor_solve_host: M's values and b from host buffers (numpy
        or pinned torch CPU tensors), x back, one synchronisation; returns
        (status, zero_pivot_index, Inertia)"""
        st, zp, a, bb, c = (C.c_int() for _ in range(5))
        check(lib.ncl_factor_solve_host(self._h, M.handle, _ptr(vals), _ptr(b), _ptr(x), float(pivot_tol),
                                        C.byref(st), C.byref(zp), C.byref(a), C.byref(bb), C.byref(c)))
        return ("ok" if st.value == 0 else "zero_pivot"), zp.value, Inertia(a.value, bb.value, c.value)

    def L_csc(self):
        """Test-only: L in the reference's CSC layout (permuted indices)."""
        info = self._symb.info() if self._symb is not None else None
        lnnz = info.l_nnz
        lp = np.empty(self._n + 1, np.int32)
        li = np.empty(lnnz, np.int32)
        lx = np.empty(lnnz, np.float64)
        check(lib.ncl_fact_get_L(self._h, _ptr(lp), _ptr(li), _ptr(lx)))
        return lp, li, lx


def factorize(M: SparseSym, symb: SymbolicFactor | None = None, pivot_tol: float = 1e-12) -> Factorization:
    """factorize(M, symb, pivot_tol) / factorize(M, pivot_tol) (sparse_sym.hpp:125-126)."""
    h = C.c_void_p()
    if symb is None:
        symb_owned = analyze(M)
        check(lib.ncl_factorize(M.handle, symb_owned.handle, float(pivot_tol), C.byref(h)))
        return Factorization(h, M.dim(), symb_owned)
    check(lib.ncl_factorize(M.handle, symb.handle, float(pivot_tol), C.byref(h)))
    return Factorization(h, M.dim(), symb)


@dataclass
class RefinedSolve:
    x: np.ndarray
    residual: float
    sweeps: int
    converged: bool


def solve_refined(F: Factorization, M: SparseSym, b, target: float = 1e-8, max_sweeps: int = 5) -> RefinedSolve:
    """solve_refined (sparse_sym.hpp:136-139)."""
    b = _f64(b)
    x = np.empty(M.dim(), np.float64)
    res, sw, cv = C.c_double(), C.c_int(), C.c_int()
    check(lib.ncl_solve_refined(F.handle, M.handle, _ptr(b), float(target), int(max_sweeps), _ptr(x), HOST,
                                C.byref(res), C.byref(sw), C.byref(cv)))
    return RefinedSolve(x, res.value, sw.value, bool(cv.value))
