"""Condensed Newton matrix K = H + Σ_x + δ_w I + Jᵀ D J (C-ABI ncl_kkt_*)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import P, check, f64, i32, i64, lib, register
from .sparse import HOST, SparseSym, _f64, _ptr

register({
    "ncl_kkt_create": (i32, [i32, i32, i64, P, P, i64, P, P, C.POINTER(P)]),
    "ncl_kkt_create_for_model": (i32, [P, C.POINTER(P)]),
    "ncl_kkt_destroy": (None, [P]),
    "ncl_kkt_matrix": (P, [P]),
    "ncl_kkt_num_triplets": (i64, [P]),
    "ncl_kkt_triplets": (i32, [P, P, P]),
    "ncl_kkt_assemble": (i32, [P, P, P, P, f64, P, i32]),
})


class _Borrowed(SparseSym):
    """SparseSym view of a handle owned by someone else (never destroyed here)."""

    def __init__(self, h, owner):
        self._h = C.c_void_p(h)
        self._owner = owner

    def __del__(self):
        self._h = None


class Kkt:
    def __init__(self, model):
        h = C.c_void_p()
        check(lib.ncl_kkt_create_for_model(model.handle, C.byref(h)))
        self._h = h
        self.n, self.m = model.n, model.m
        self.matrix = _Borrowed(lib.ncl_kkt_matrix(h), self)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self.matrix = None
            lib.ncl_kkt_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def triplets(self):
        nt = lib.ncl_kkt_num_triplets(self._h)
        r, c = np.empty(nt, np.int32), np.empty(nt, np.int32)
        check(lib.ncl_kkt_triplets(self._h, _ptr(r), _ptr(c)))
        return r, c

    def assemble(self, hess, jac, sigma_x, delta_w, D, where=HOST):
        if where == HOST:
            hess, jac, sigma_x, D = _f64(hess), _f64(jac), _f64(sigma_x), _f64(D)
        check(lib.ncl_kkt_assemble(self._h, _ptr(hess), _ptr(jac), _ptr(sigma_x), float(delta_w), _ptr(D), where))


def reference_triplet_values(kkt: Kkt, jac_rows, hess, jac, sigma_x, delta_w, D):
    """Triplet values in the assembly order (for feeding a reference SparseSym):
    H entries, Σ_x+δ_w, then D_r J_a J_b for every row and pair a>=b."""
    vals = [np.asarray(hess, np.float64), np.asarray(sigma_x, np.float64) + delta_w]
    jr = np.asarray(jac_rows)
    m = kkt.m
    starts = np.searchsorted(jr, np.arange(m + 1))
    out = []
    for r in range(m):
        a0, a1 = starts[r], starts[r + 1]
        for a in range(a0, a1):
            for b in range(a0, a + 1):
                out.append(D[r] * jac[a] * jac[b])
    vals.append(np.array(out, np.float64))
    return np.concatenate(vals)
