"""Multi-GPU contingency sharding of the KKT factor / solve (C-ABI
include/nclopf_dist.h). torch.distributed is plumbing only: it carries the
128-byte NCCL unique id from rank 0; the data path is the library's own NCCL
communicator (all-gather of subtree-root contribution blocks over NVLink)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import P, check, i32, i64, lib, register
from .sparse import DEVICE, HOST, _ptr


class ShardInfo(C.Structure):
    _fields_ = [("world", i32), ("rank", i32), ("owned_supernodes", i64), ("shared_supernodes", i64),
                ("n_phase_a", i32), ("n_phase_b", i32), ("n_boundary", i32), ("cb_chunk", i64), ("cv_chunk", i64),
                ("report_cols", i64)]


register({
    "ncl_dist_get_unique_id": (i32, [C.c_char_p]),
    "ncl_dist_init": (i32, [i32, i32, C.c_char_p]),
    "ncl_dist_finalize": (i32, []),
    "ncl_shard_create": (i32, [P, P, i32, i32, i32, C.POINTER(P)]),
    "ncl_shard_destroy": (None, [P]),
    "ncl_shard_info_get": (i32, [P, C.POINTER(ShardInfo)]),
    "ncl_shard_owners": (i32, [P, P]),
    "ncl_shard_boundary": (i32, [P, P, P, P, P]),
    "ncl_shard_refactorize": (i32, [P, P, P, C.c_double]),
    "ncl_shard_solve": (i32, [P, P, P, i32]),
    "ncl_shard_refactorize_emulated": (i32, [P, P, P, i32, C.c_double]),
    "ncl_shard_factor_phase_a": (i32, [P, P, P, C.c_double, P, i32]),
    "ncl_shard_factor_phase_b": (i32, [P, P, P, P, i32, P]),
    "ncl_shard_set_status": (i32, [P, P]),
    "ncl_shard_solve_phase_a": (i32, [P, P, P, i32, P, i32]),
    "ncl_shard_solve_phase_b": (i32, [P, P, P, i32, P, i32]),
    "ncl_shard_diagonal": (i32, [P, P, P]),
    "ncl_scopf_var_groups": (i32, [P, P]),
})


def var_groups(scopf) -> np.ndarray:
    g = np.empty(scopf.n, np.int32)
    check(lib.ncl_scopf_var_groups(scopf.handle, _ptr(g)))
    return g


def init_nccl(world: int, rank: int, torch_dist) -> None:
    """Create the library's NCCL communicator; the unique id travels over the
    already-initialised torch.distributed group (any backend)."""
    import torch
    buf = C.create_string_buffer(128)
    if rank == 0:
        check(lib.ncl_dist_get_unique_id(buf))
    t = torch.tensor(list(buf.raw), dtype=torch.uint8)
    if torch_dist.get_backend() == "nccl":
        t = t.cuda()
    torch_dist.broadcast(t, 0)
    check(lib.ncl_dist_init(world, rank, bytes(t.cpu().tolist())))


def finalize_nccl() -> None:
    check(lib.ncl_dist_finalize())


@dataclass
class Boundary:
    ids: np.ndarray
    owner: np.ndarray
    cb_off: np.ndarray
    cv_off: np.ndarray


class ShardPlan:
    """Owner/phase plan of one rank (host side, no GPU needed)."""

    def __init__(self, symb, groups, ngroups: int, world: int, rank: int):
        g = np.ascontiguousarray(groups, np.int32)
        h = C.c_void_p()
        check(lib.ncl_shard_create(symb.handle, _ptr(g), int(ngroups), int(world), int(rank), C.byref(h)))
        self._h, self._symb = h, symb
        self.world, self.rank = world, rank

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.ncl_shard_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def info(self) -> ShardInfo:
        s = ShardInfo()
        check(lib.ncl_shard_info_get(self._h, C.byref(s)))
        return s

    def owners(self) -> np.ndarray:
        o = np.empty(self._symb.info().nsupernodes, np.int32)
        check(lib.ncl_shard_owners(self._h, _ptr(o)))
        return o

    def boundary(self) -> Boundary:
        nb = self.info().n_boundary
        ids, own = np.empty(nb, np.int32), np.empty(nb, np.int32)
        cb, cv = np.empty(nb, np.int64), np.empty(nb, np.int64)
        check(lib.ncl_shard_boundary(self._h, _ptr(ids), _ptr(own), _ptr(cb), _ptr(cv)))
        return Boundary(ids, own, cb, cv)

    def refactorize(self, F, M, pivot_tol: float = 1e-12) -> None:
        check(lib.ncl_shard_refactorize(F.handle, M.handle, self._h, float(pivot_tol)))

    def solve_in_place(self, F, x, where: int = HOST) -> None:
        check(lib.ncl_shard_solve(F.handle, self._h, _ptr(x), where))

    # split-phase form (include/nclopf_dist.h): the caller moves the bytes
    @staticmethod
    def _where(a) -> int:
        return DEVICE if (hasattr(a, "is_cuda") and a.is_cuda) else HOST

    def factor_phase_a(self, F, M, send, pivot_tol: float = 1e-12) -> None:
        """own + base-only supernodes, boundary CBs packed into send (cb_chunk doubles)"""
        check(lib.ncl_shard_factor_phase_a(F.handle, M.handle, self._h, float(pivot_tol), _ptr(send),
                                           self._where(send)))

    def factor_phase_b(self, F, M, recv) -> np.ndarray:
        """unpack the all-gathered blocks (world * cb_chunk), separator; returns
        this rank's [zero-pivot position, npos, nneg, nzero]"""
        ist = np.zeros(4, np.int32)
        check(lib.ncl_shard_factor_phase_b(F.handle, M.handle, self._h, _ptr(recv), self._where(recv), _ptr(ist)))
        return ist

    @staticmethod
    def set_status(F, istat) -> None:
        ist = np.ascontiguousarray(istat, np.int32)
        check(lib.ncl_shard_set_status(F.handle, _ptr(ist)))

    def solve_phase_a(self, F, x, send) -> None:
        check(lib.ncl_shard_solve_phase_a(F.handle, self._h, _ptr(x), self._where(x), _ptr(send), self._where(send)))

    def solve_phase_b(self, F, x, recv) -> None:
        check(lib.ncl_shard_solve_phase_b(F.handle, self._h, _ptr(x), self._where(x), _ptr(recv), self._where(recv)))

    def diagonal(self, F) -> np.ndarray:
        """D by pivot position on the columns this rank reports, NaN elsewhere"""
        d = np.empty(F._n, np.float64)
        check(lib.ncl_shard_diagonal(F.handle, self._h, _ptr(d)))
        return d


def combine_status(istats) -> np.ndarray:
    """the reduction ncl_shard_refactorize does with NCCL: min of the zero-pivot
    position, sums of the inertia counts"""
    a = np.asarray(istats, np.int64)
    return np.array([a[:, 0].min(), a[:, 1].sum(), a[:, 2].sum(), a[:, 3].sum()], np.int32)


def refactorize_emulated(F, M, plans, pivot_tol: float = 1e-12) -> None:
    arr = (C.c_void_p * len(plans))(*[p.handle.value for p in plans])
    check(lib.ncl_shard_refactorize_emulated(F.handle, M.handle, arr, len(plans), float(pivot_tol)))


__all__ = ["ShardPlan", "ShardInfo", "combine_status", "var_groups", "init_nccl", "finalize_nccl", "refactorize_emulated",
           "DEVICE", "HOST"]
