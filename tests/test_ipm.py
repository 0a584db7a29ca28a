"""NCL outer loop + IPM.

CPU (oracle, the same host control flow over the reference sparse_core /
model_ad): SPEC's toy examples and the MATPOWER case9 known optimum.
GPU: the B200 solve against the oracle on the same instance — identical
status, outer/inner iteration counts, objective and infeasibilities within
1e-6 relative (BASELINE.json north_star parity bar).
"""
import numpy as np
import pytest

from oracle.ref import RefModel, ref_ncl_solve
from paper_2510_13333_b200.ipm import default_options
from paper_2510_13333_b200.model import Expr
from paper_2510_13333_b200.scopf import Scopf
from tests.test_model import Fam, both_models

INF = float("inf")


def _bounds(n, m, xl=None, xu=None, x0=None, gl=None, gu=None):
    return dict(xl=np.full(n, -INF) if xl is None else np.asarray(xl, float),
                xu=np.full(n, INF) if xu is None else np.asarray(xu, float),
                x0=np.zeros(n) if x0 is None else np.asarray(x0, float),
                gl=np.zeros(m) if gl is None else np.asarray(gl, float),
                gu=np.zeros(m) if gu is None else np.asarray(gu, float))


def test_toy_feasible_multiplier():
    """min w^2 s.t. w = 1 -> w = 1, multiplier -2."""
    w = Expr.var(0)
    fams = [Fam("obj", w * w, 1, True, None, [0]), Fam("c", w + 0.0, 1, False, [0], [0])]
    R = RefModel.from_families(1, 1, fams)
    out = ref_ncl_solve(R, _bounds(1, 1, gl=[1.0], gu=[1.0]))
    assert out["status"] == "optimal"
    assert abs(out["x"][0] - 1.0) < 1e-6
    # L = f + y c: 2 w + y = 0 at w = 1 (the objective is scaled by sf = 1 here: |grad| = 0 < 100)
    assert abs(out["y"][0] + 2.0) < 1e-4
    assert out["result"]["r_inf"] <= 1e-6


def test_toy_infeasible():
    """w = 0 and w = 1 -> infeasible, w = 0.5 (Eq. 13 least squares)."""
    w = Expr.var(0)
    fams = [Fam("c", w + 0.0, 1, False, [0, 1], [0, 0])]
    R = RefModel.from_families(1, 2, fams)
    out = ref_ncl_solve(R, _bounds(1, 2, gl=[0.0, 1.0], gu=[0.0, 1.0]), options=default_options(max_outer=40))
    assert out["status"] == "infeasible"
    assert abs(out["x"][0] - 0.5) < 1e-4
    assert abs(out["result"]["r_inf"] - 0.5) < 1e-4


def test_toy_bounds_and_inequality():
    """min (w0-2)^2 + (w1-2)^2 s.t. w0 + w1 <= 2, 0 <= w <= 10 -> w = (1, 1)."""
    a, b = Expr.var(0), Expr.var(1)
    fams = [Fam("obj", (a - 2.0) * (a - 2.0) + (b - 2.0) * (b - 2.0), 2, True, None, [0, 1]),
            Fam("lin", a + b, 2, False, [0], [0, 1])]
    R = RefModel.from_families(2, 1, fams)
    out = ref_ncl_solve(R, _bounds(2, 1, xl=[0, 0], xu=[10, 10], x0=[0.5, 3.0], gl=[-INF], gu=[2.0]))
    assert out["status"] == "optimal"
    np.testing.assert_allclose(out["x"], [1.0, 1.0], atol=1e-5)


def test_case9_known_optimum():
    """MATPOWER case9 ACOPF: published optimal cost 5296.69 $/h (config C1)."""
    s = Scopf("case9", 0)
    R = RefModel.from_families(s.n, s.m, s.families())
    out = ref_ncl_solve(R, s.bounds())
    assert out["status"] == "optimal"
    assert abs(out["result"]["objective"] - 5296.69) < 0.01
    assert out["result"]["r_inf"] <= 1e-6


def test_trace_schema():
    s = Scopf("case9", 0)
    R = RefModel.from_families(s.n, s.m, s.families())
    out = ref_ncl_solve(R, s.bounds())
    inner = [t for t in out["trace"] if "iter" in t]
    outer = [t for t in out["trace"] if "outer_summary" in t]
    assert len(inner) == out["result"]["inner_iters"]
    assert len(outer) == out["result"]["outer_iters"]
    assert {"mu", "inf_pr", "inf_du", "dw", "alpha_pr"} <= set(inner[0])
    rhos = [t["rho"] for t in outer]
    assert all(b >= a for a, b in zip(rhos, rhos[1:]))  # penalty monotone


# ------------------------------------------------------------------ GPU parity
def _compare(g, r):
    gr, rr = g.result, r["result"]
    assert g.status == r["status"]
    assert gr["outer_iters"] == rr["outer_iters"]
    assert gr["inner_iters"] == rr["inner_iters"]
    assert abs(gr["objective"] - rr["objective"]) <= 1e-6 * abs(rr["objective"])
    for k in ("r_inf", "inf_pr"):
        assert abs(gr[k] - rr[k]) <= 1e-6 * max(1.0, abs(rr[k])), k


@pytest.mark.gpu
@pytest.mark.parametrize("grid,K", [("case9", 0), ("case9", 2), ("case118", 4), ("case118", 16), ("activsg500", 16)])
def test_gpu_solve_matches_oracle(gpu, grid, K):
    from paper_2510_13333_b200.ipm import solve_scopf
    s = Scopf(grid, K)
    R = RefModel.from_families(s.n, s.m, s.families())
    ref = ref_ncl_solve(R, s.bounds())
    out = solve_scopf(s)
    _compare(out, ref)
    if grid == "case9" and K == 0:
        assert abs(out.result["objective"] - 5296.69) < 0.01


@pytest.mark.gpu
def test_gpu_toy_models(gpu):
    from paper_2510_13333_b200.ipm import NclSolver
    a, b = Expr.var(0), Expr.var(1)
    fams = [Fam("obj", (a - 2.0) * (a - 2.0) + (b - 2.0) * (b - 2.0), 2, True, None, [0, 1]),
            Fam("lin", a + b, 2, False, [0], [0, 1])]
    M, R = both_models(2, 1, fams)
    bd = _bounds(2, 1, xl=[0, 0], xu=[10, 10], x0=[0.5, 3.0], gl=[-INF], gu=[2.0])
    out = NclSolver(M, bd).solve()
    ref = ref_ncl_solve(R, bd)
    _compare(out, ref)
    np.testing.assert_allclose(out.x, [1.0, 1.0], atol=1e-5)
