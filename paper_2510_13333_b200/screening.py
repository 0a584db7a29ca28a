"""Contingency screening (Eq. 5).

screen_all fixes the base-case set points of a converged base OPF (K = 0
solve) and measures every contingency's infeasibility ||r||^2 + ||t||^2 — the
NCL regularisation r on the scenario's rows (t is r on its complementarity
rows, csrc/host/ipm_elem.hpp) at the NCL solution of its Eq. 5 system.
Batched: the Eq. 5 systems of a whole batch of contingencies are independent
blocks of ONE problem (csrc/host/scopf.cpp screening mode), solved by one
B200 NCL solve; because the blocks share no variable or row, the minimiser
of the batch is the per-block minimisers side by side (each block's residual
is its own), so a batch of B contingencies costs one solve of B blocks
instead of B solves. select_representative picks the hardest feasible ones."""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .ipm import NclSolver, default_options
from .scopf import Scopf

FEAS_TOL = 1e-8   # squared objective
HARD_CAP = 1e-2   # structural-infeasibility cap


@dataclass
class Record:
    id: int
    status: str
    objective: float
    iters: int
    structural: bool = False


@dataclass
class ScreeningReport:
    records: list = field(default_factory=list)

    @property
    def ranking(self):
        """contingency ids by nonincreasing objective"""
        return [r.id for r in sorted(self.records, key=lambda r: (-r.objective, r.id))]

    def by_id(self):
        return {r.id: r for r in self.records}


def base_set_points(base: Scopf, options=None):
    """(pg0, v0, output) of the base OPF (K = 0): generator outputs and bus
    voltages of the paper-layout base scenario (v: x[0:nb], pg: x[2nb:2nb+ng])"""
    assert base.K == 0
    out = NclSolver(base.build_model(), base.bounds()).solve(options or default_options())
    nb, ng = base.info.nb, base.info.ng
    return out.x[2 * nb:2 * nb + ng].copy(), out.x[:nb].copy(), out


def solve_batch(base: Scopf, pg0, v0, ids, options=None):
    """one NCL solve of the Eq. 5 systems of `ids` side by side; returns the
    per-contingency objectives, the solve's status and iterations"""
    s = Scopf.screening(base, pg0, v0, ids)
    out = NclSolver(s.build_model(), s.bounds()).solve(options or default_options(verbose=0))
    K = len(ids)
    r = out.r.reshape(K, -1)  # equal blocks of m / K rows, contingency order
    return np.sum(r * r, axis=1), out.status, out.result["inner_iters"]


def screen_all(grid: str = "case118", ids=None, batch: int | None = None, seed: int = 2510, options=None,
               base_options=None) -> ScreeningReport:
    """screen_all: `ids` default = every non-islanding
    single-branch outage; batch = contingencies per NCL solve (None: all in
    one). Islanding outages are structurally infeasible (never solved)."""
    base = Scopf(grid, 0, seed=seed)
    pg0, v0, _ = base_set_points(base, base_options)
    cand = [int(c) for c in base.candidates()]
    ids = cand if ids is None else [int(i) for i in ids]
    ok = set(cand)
    solvable = [i for i in ids if (i % base.info.nl) in ok]
    rep = ScreeningReport()
    for i in ids:
        if i not in solvable:
            rep.records.append(Record(i, "structural", float("inf"), 0, True))
    B = len(solvable) if not batch else batch
    for k in range(0, len(solvable), max(1, B)):
        chunk = solvable[k:k + B]
        obj, status, iters = solve_batch(base, pg0, v0, chunk, options)
        for i, o in zip(chunk, obj):
            rep.records.append(Record(i, status, float(o), iters, bool(o > HARD_CAP)))
    rep.records.sort(key=lambda r: r.id)
    return rep


class NotEnoughFeasible(ValueError):
    pass


def select_representative(report: ScreeningReport, K: int):
    """select_representative: the K highest-objective
    contingencies that are not structurally infeasible (islanding or objective
    above the hard cap), hardest first"""
    ok = [r for r in report.records if not r.structural and r.objective <= HARD_CAP]
    if K > len(ok):
        raise NotEnoughFeasible(f"{K} requested, {len(ok)} not structurally infeasible")
    ok.sort(key=lambda r: (-r.objective, r.id))
    return [r.id for r in ok[:K]]


__all__ = ["screen_all", "select_representative", "solve_batch", "base_set_points", "ScreeningReport", "Record",
           "NotEnoughFeasible", "FEAS_TOL", "HARD_CAP"]
