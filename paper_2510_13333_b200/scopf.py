"""SCOPF problem generator binding (C-ABI ncl_scopf_*): the paper-layout
corrective AC-SCOPF on MATPOWER case9 or seeded synthetic geometric grids."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import P, check, i32, i64, lib, register
from .model import ExprNode, ModelFunctions
from .sparse import _ptr


class ScopfInfo(C.Structure):
    _fields_ = [("n", i32), ("m", i32), ("nfam", i32), ("K", i32), ("nb", i32), ("nl", i32), ("ng", i32),
                ("ncomp", i32), ("nvar_scen", i32), ("ncon_scen", i32)]


register({
    "ncl_scopf_create_network": (i32, [P, i32, P, C.POINTER(P)]),
    "ncl_scopf_create_screening": (i32, [P, P, P, i32, P, C.POINTER(P)]),
    "ncl_scopf_create": (i32, [i32, i32, i32, i32, C.c_uint64, i32, C.POINTER(P)]),
    "ncl_scopf_create_list": (i32, [i32, i32, i32, i32, C.c_uint64, i32, P, C.POINTER(P)]),
    "ncl_scopf_destroy": (None, [P]),
    "ncl_scopf_get_info": (i32, [P, C.POINTER(ScopfInfo)]),
    "ncl_scopf_family_info": (i32, [P, i32, C.c_char_p, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32),
                                    C.POINTER(i32), C.POINTER(i64)]),
    "ncl_scopf_family_data": (i32, [P, i32, P, P, P, P]),
    "ncl_scopf_bounds": (i32, [P, P, P, P, P, P]),
    "ncl_scopf_contingencies": (i32, [P, P]),
    "ncl_scopf_candidates": (i32, [P, P, C.POINTER(i32)]),
    "ncl_scopf_build_model": (i32, [P, C.POINTER(P)]),
})

# Grid sizes of the BASELINE.json configs
GRIDS = {
    "case9": (0, 9, 9, 3),
    "case118": (1, 118, 186, 54),        # same-size synthetic (no MATPOWER data offline)
    "activsg500": (1, 500, 597, 56),
    "activsg2000": (1, 2000, 3206, 432),
}


def screened(grid: str, seed: int = 2510):
    """Committed list of N-1 contingencies that passed screening (each one
    solved alone as a K=1 SCOPF to optimality), ascending branch order."""
    import json
    import os
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", f"screened_{grid}_{seed}.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f)["feasible"]


LOAD_LEVELS = 4  # csrc/host/scopf.hpp kLoadLevels: id = branch + nl * level, loads x (1 - 0.015 level)


def contingency_ids(grid: str, K: int, seed: int = 2510):
    """The first K contingency ids of a grid: the screened N-1 outages
    (level 0) first, then the same outages at load levels 1, 2, 3
    (outage x load-scenario contingencies; see include/nclopf_b200.h
    ncl_scopf_create_list). None when the grid has no screened list."""
    base = screened(grid, seed)
    if base is None:
        return None
    nl = GRIDS[grid][2]
    ids = [l + nl * j for j in range(LOAD_LEVELS) for l in base]
    if len(ids) < K:
        raise ValueError(f"only {len(ids)} contingencies ({len(base)} screened outages x {LOAD_LEVELS} load levels) "
                         f"for {grid}")
    return ids[:K]


@dataclass
class Family:
    name: str
    nodes: object
    nslots: int
    np: int
    objective: bool
    rows: np.ndarray
    vars: np.ndarray
    params: np.ndarray


class Scopf:
    def __init__(self, grid: str = "case9", K: int = 0, seed: int = 2510, contingencies=None, network=None):
        """contingencies: explicit contingency ids (branch + nl * load level);
        default = contingency_ids(grid, K, seed): the committed screened
        outages (data/screened_<grid>_<seed>.json,
        tools/screen_contingencies.py), then the same outages at lower load
        levels, when a screened list exists, else the first K non-islanding
        branches."""
        h = C.c_void_p()
        if network is not None:  # a parsed MATPOWER case (paper_2510_13333_b200.matpower)
            ids = None if contingencies is None else np.ascontiguousarray(np.asarray(contingencies)[:K], np.int32)
            check(lib.ncl_scopf_create_network(network.handle, K, _ptr(ids), C.byref(h)))
            self._finish(h, network.name)
            return
        kind, nb, nl, ng = GRIDS[grid]
        if contingencies is None and K > 0:
            contingencies = contingency_ids(grid, K, seed)
        if contingencies is None:
            check(lib.ncl_scopf_create(kind, nb, nl, ng, seed, K, C.byref(h)))
        else:
            ids = np.ascontiguousarray(np.asarray(contingencies)[:K], np.int32)
            check(lib.ncl_scopf_create_list(kind, nb, nl, ng, seed, K, _ptr(ids), C.byref(h)))
        self._finish(h, grid)

    @classmethod
    def screening(cls, base: "Scopf", pg0, v0, ids) -> "Scopf":
        """Eq. 5 screening system of `base`'s grid: the contingencies `ids`
        with the base set points pg0 (ng) and v0 (nb) fixed, no objective;
        K equal blocks of n / K variables and m / K rows."""
        obj = cls.__new__(cls)
        pg0, v0 = np.ascontiguousarray(pg0, np.float64), np.ascontiguousarray(v0, np.float64)
        ids = np.ascontiguousarray(ids, np.int32)
        h = C.c_void_p()
        check(lib.ncl_scopf_create_screening(base.handle, _ptr(pg0), _ptr(v0), len(ids), _ptr(ids), C.byref(h)))
        obj._finish(h, base.grid)
        return obj

    def _finish(self, h, grid):
        self._h = h
        s = ScopfInfo()
        check(lib.ncl_scopf_get_info(h, C.byref(s)))
        self.info = s
        self.n, self.m, self.K = s.n, s.m, s.K
        self.grid = grid

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.ncl_scopf_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def families(self):
        out = []
        for f in range(self.info.nfam):
            name = C.create_string_buffer(64)
            nn, ns, np_, obj, ni = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int64()
            check(lib.ncl_scopf_family_info(self._h, f, name, C.byref(nn), C.byref(ns), C.byref(np_), C.byref(obj),
                                            C.byref(ni)))
            nodes = (ExprNode * nn.value)()
            rows = np.empty(0 if obj.value else ni.value, np.int32)
            vars_ = np.empty(ni.value * ns.value, np.int32)
            params = np.empty(ni.value * np_.value, np.float64)
            check(lib.ncl_scopf_family_data(self._h, f, nodes, _ptr(rows), _ptr(vars_), _ptr(params)))
            out.append(Family(name.value.decode(), nodes, ns.value, np_.value, bool(obj.value), rows,
                              vars_.reshape(ni.value, ns.value), params.reshape(ni.value, np_.value)))
        return out

    def bounds(self):
        xl, xu, x0 = (np.empty(self.n) for _ in range(3))
        gl, gu = np.empty(self.m), np.empty(self.m)
        check(lib.ncl_scopf_bounds(self._h, _ptr(xl), _ptr(xu), _ptr(x0), _ptr(gl), _ptr(gu)))
        return dict(xl=xl, xu=xu, x0=x0, gl=gl, gu=gu)

    def contingencies(self):
        ids = np.empty(self.K, np.int32)
        check(lib.ncl_scopf_contingencies(self._h, _ptr(ids)))
        return ids

    def candidates(self):
        """All non-islanding single-branch outages of the grid, ascending."""
        cnt = C.c_int()
        check(lib.ncl_scopf_candidates(self._h, None, C.byref(cnt)))
        ids = np.empty(cnt.value, np.int32)
        check(lib.ncl_scopf_candidates(self._h, _ptr(ids), C.byref(cnt)))
        return ids

    def build_model(self) -> ModelFunctions:
        h = C.c_void_p()
        check(lib.ncl_scopf_build_model(self._h, C.byref(h)))
        return ModelFunctions(h)
