"""Condensation + recovery against the full, uncondensed Newton system
(SPEC.md:316-333 assemble_newton / recover_directions; SPEC.md:373
"condensation exactness"; acceptance criterion 6).

The IPM solves the condensed K = W + Sigma_x + dw + J'DJ (north_star step
(2)) and recovers dr, ds, dy and the bound-dual steps element-wise
(csrc/host/ipm_elem.hpp). Both backends run that same code, so GPU-vs-oracle
parity cannot catch a sign error in it. Here the direction each backend
returns (ncl_solver_newton_step / ref_newton_step) is checked against a
dense solve of the FULL primal-dual Newton linearisation, written out
independently below from the Lagrangian of the NCL subproblem

  L = sf f + lamN'r + rho/2 r'r + y'(c - r - s) - zl'(x-xl) - zu'(xu-x)
      - vl'(s-gl) - vu'(gu-s)

with unknowns (dx, dr, ds[ineq rows], dy, dzl, dzu, dvl, dvu):
  (W + dw I) dx + J'dy - dzl + dzu        = -(sf grad f + J'y - zl + zu)
  rho dr - dy                             = -(lamN + rho r - y)
  -dy - dvl + dvu            (ineq rows)  = -(-y - vl + vu)
  J dx - dr - ds - dc dy                  = -(c - r - s)
  zl dx + (x-xl) dzl = mu - (x-xl) zl,   -zu dx + (xu-x) dzu = mu - (xu-x) zu
  vl ds + (s-gl) dvl = mu - (s-gl) vl,   -vu ds + (gu-s) dvu = mu - (gu-s) vu
Bar: relative error <= 1e-10 on both backends.
"""
import numpy as np
import pytest

from oracle.ref import RefModel, ref_newton_step
from paper_2510_13333_b200.ipm import default_options
from paper_2510_13333_b200.model import Expr, cos, sin
from paper_2510_13333_b200.scopf import Scopf
from tests.test_model import Fam, both_models

INF = 1e30  # beyond kBig = 1e20: no bound


def _toy(rng, n=10):
    """10 variables, 6 rows (3 equalities, 3 inequalities with lower / upper
    / two-sided bounds), nonlinear objective and constraints, mixed bounds."""
    a, b, c = Expr.var(0), Expr.var(1), Expr.var(2)
    p = Expr.param(0)
    fams = [
        Fam("obj2", p * a * a + a * b + sin(b), 2, True, None, [[i, (i + 3) % n] for i in range(n)],
            rng.uniform(0.5, 2.0, (n, 1))),
        Fam("bil", a * b + c * c - p, 3, False, [0, 1, 2], [[0, 1, 2], [3, 4, 5], [6, 7, 8]], [[0.3], [0.1], [-0.2]]),
        Fam("trig", sin(a) * b + cos(c), 3, False, [3, 4, 5], [[9, 0, 4], [2, 5, 7], [1, 8, 3]]),
    ]
    xl = rng.uniform(-2, -1, n)
    xu = rng.uniform(1, 2, n)
    xl[[1, 6]] = -INF  # upper only
    xu[[2, 7]] = INF  # lower only
    xl[4], xu[4] = -INF, INF  # free
    gl = np.array([0.0, 0.0, 0.0, -1.0, -INF, -0.5])
    gu = np.array([0.0, 0.0, 0.0, INF, 1.0, 2.5])
    return n, 6, fams, dict(xl=xl, xu=xu, x0=np.zeros(n), gl=gl, gu=gu)


def _state(rng, bd, n, m, mu=0.1, rho=30.0, dw=0.0, dc=0.0):
    xl, xu, gl, gu = bd["xl"], bd["xu"], bd["gl"], bd["gu"]
    lo, up = xl > -1e20, xu < 1e20
    x = rng.uniform(-0.8, 0.8, n)
    zl = np.where(lo, rng.uniform(0.05, 2.0, n), 0.0)
    zu = np.where(up, rng.uniform(0.05, 2.0, n), 0.0)
    eq = gl == gu
    glo, gup = (gl > -1e20) & ~eq, (gu < 1e20) & ~eq
    s = np.where(eq, gl, 0.0)
    for i in range(m):
        if not eq[i]:
            a = gl[i] if gl[i] > -1e20 else gu[i] - 3.0
            b = gu[i] if gu[i] < 1e20 else gl[i] + 3.0
            s[i] = rng.uniform(a + 0.1 * (b - a), b - 0.1 * (b - a))
    vl = np.where(glo, rng.uniform(0.05, 2.0, m), 0.0)
    vu = np.where(gup, rng.uniform(0.05, 2.0, m), 0.0)
    return dict(x=x, zl=zl, zu=zu, r=0.1 * rng.standard_normal(m), s=s, y=rng.standard_normal(m), vl=vl, vu=vu,
                lamN=rng.standard_normal(m), mu=mu, rho=rho, sf=1.0, dw=dw, dc=dc)


def full_newton(R: RefModel, bd, st):
    """Dense solve of the uncondensed system (module docstring); J, W, c,
    grad from the reference model functions."""
    n, m = R.n, R.m
    x = st["x"]
    J = np.zeros((m, n))
    for i, j, v in zip(*R.jac_coords(), R.eval_jacobian(x)):
        J[i, j] += v
    W = np.zeros((n, n))
    for i, j, v in zip(*R.hess_coords(), R.eval_hessian_lag(x, st["sf"], st["y"])):
        W[i, j] += v
        if i != j:
            W[j, i] += v
    c, g = R.eval_constraints(x), R.eval_grad_objective(x)
    xl, xu, gl, gu = bd["xl"], bd["xu"], bd["gl"], bd["gu"]
    lo, up = np.flatnonzero(xl > -1e20), np.flatnonzero(xu < 1e20)
    eq = gl == gu
    ineq = np.flatnonzero(~eq)
    slo = np.flatnonzero((gl > -1e20) & ~eq)
    sup = np.flatnonzero((gu < 1e20) & ~eq)
    s = np.where(eq, gl, st["s"])
    zl, zu, vl, vu, y, r = st["zl"], st["zu"], st["vl"], st["vu"], st["y"], st["r"]
    mu, rho = st["mu"], st["rho"]
    sizes = dict(dx=n, dr=m, ds=len(ineq), dy=m, dzl=len(lo), dzu=len(up), dvl=len(slo), dvu=len(sup))
    off, o = {}, 0
    for k, v in sizes.items():
        off[k], o = o, o + v
    N = o
    A, rhs = np.zeros((N, N)), np.zeros(N)
    row = 0
    # stationarity in x
    A[row:row + n, off["dx"]:off["dx"] + n] = W + st["dw"] * np.eye(n)
    A[row:row + n, off["dy"]:off["dy"] + m] = J.T
    for k, i in enumerate(lo):
        A[row + i, off["dzl"] + k] = -1.0
    for k, i in enumerate(up):
        A[row + i, off["dzu"] + k] = 1.0
    rhs[row:row + n] = -(st["sf"] * g + J.T @ y - zl + zu)
    row += n
    # stationarity in r
    for i in range(m):
        A[row + i, off["dr"] + i] = rho
        A[row + i, off["dy"] + i] = -1.0
    rhs[row:row + m] = -(st["lamN"] + rho * r - y)
    row += m
    # stationarity in s (inequality rows)
    for k, i in enumerate(ineq):
        A[row + k, off["dy"] + i] = -1.0
        if i in slo:
            A[row + k, off["dvl"] + list(slo).index(i)] = -1.0
        if i in sup:
            A[row + k, off["dvu"] + list(sup).index(i)] = 1.0
        rhs[row + k] = -(-y[i] - vl[i] + vu[i])
    row += len(ineq)
    # primal feasibility c - r - s = 0
    A[row:row + m, off["dx"]:off["dx"] + n] = J
    for i in range(m):
        A[row + i, off["dr"] + i] = -1.0
        A[row + i, off["dy"] + i] = -st["dc"]
    for k, i in enumerate(ineq):
        A[row + i, off["ds"] + k] = -1.0
    rhs[row:row + m] = -(c - r - s)
    row += m
    # complementarity
    for k, i in enumerate(lo):
        A[row, off["dx"] + i], A[row, off["dzl"] + k] = zl[i], x[i] - xl[i]
        rhs[row] = mu - (x[i] - xl[i]) * zl[i]
        row += 1
    for k, i in enumerate(up):
        A[row, off["dx"] + i], A[row, off["dzu"] + k] = -zu[i], xu[i] - x[i]
        rhs[row] = mu - (xu[i] - x[i]) * zu[i]
        row += 1
    ipos = {i: k for k, i in enumerate(ineq)}
    for k, i in enumerate(slo):
        A[row, off["ds"] + ipos[i]], A[row, off["dvl"] + k] = vl[i], s[i] - gl[i]
        rhs[row] = mu - (s[i] - gl[i]) * vl[i]
        row += 1
    for k, i in enumerate(sup):
        A[row, off["ds"] + ipos[i]], A[row, off["dvu"] + k] = -vu[i], gu[i] - s[i]
        rhs[row] = mu - (gu[i] - s[i]) * vu[i]
        row += 1
    assert row == N
    z = np.linalg.solve(A, rhs)
    out = {k: z[off[k]:off[k] + v] for k, v in sizes.items()}
    # scatter the reduced blocks back to full length (zeros where absent)
    full = dict(dx=out["dx"], dr=out["dr"], dy=out["dy"], ds=np.zeros(m), dzl=np.zeros(n), dzu=np.zeros(n),
                dvl=np.zeros(m), dvu=np.zeros(m))
    full["ds"][ineq] = out["ds"]
    full["dzl"][lo] = out["dzl"]
    full["dzu"][up] = out["dzu"]
    full["dvl"][slo] = out["dvl"]
    full["dvu"][sup] = out["dvu"]
    return full


KEYS = ("dx", "dr", "ds", "dy", "dzl", "dzu", "dvl", "dvu")


def _relerr(step, ref):
    scale = max(1.0, max(np.max(np.abs(ref[k])) for k in KEYS))
    return max(np.max(np.abs(step[k] - ref[k])) for k in KEYS) / scale


def _opts():
    # a tight refinement target so the comparison measures the condensation,
    # not the stopping rule of solve_refined
    return default_options(refine_target=1e-15, refine_max_sweeps=5)


CASES = [dict(), dict(dw=0.5), dict(dc=1e-3), dict(mu=1e-4, rho=1e4), dict(dw=1e-3, dc=1e-6, mu=1e-2)]


@pytest.mark.parametrize("kw", CASES)
@pytest.mark.parametrize("seed", [0, 1])
def test_oracle_step_matches_full_newton(kw, seed):
    rng = np.random.default_rng(seed)
    n, m, fams, bd = _toy(rng)
    R = RefModel.from_families(n, m, fams)
    st = _state(rng, bd, n, m, **kw)
    step = ref_newton_step(R, bd, st, _opts())
    assert step["status"] == 0
    assert _relerr(step, full_newton(R, bd, st)) <= 1e-10


def test_oracle_step_case9_scopf():
    """The same check on a real SCOPF model (case9 x 2 contingencies, paper layout)."""
    s = Scopf("case9", 2)
    R = RefModel.from_families(s.n, s.m, s.families())
    bd = s.bounds()
    rng = np.random.default_rng(3)
    st = _scopf_state(rng, bd, s.n, s.m)
    step = ref_newton_step(R, bd, st, _opts())
    assert step["status"] == 0
    assert _relerr(step, full_newton(R, bd, st)) <= 1e-10


def _scopf_state(rng, bd, n, m):
    xl, xu = bd["xl"], bd["xu"]
    lo, up = xl > -1e20, xu < 1e20
    a = np.where(lo, xl, np.where(up, xu - 2.0, -1.0))
    b = np.where(up, xu, np.where(lo, xl + 2.0, 1.0))
    x = a + (b - a) * rng.uniform(0.2, 0.8, n)
    st = _state(rng, bd, n, m, mu=1e-2, rho=100.0, dw=1e-4)
    st["x"] = x
    return st


def test_spec_centered_examples():
    """at an exactly centred, stationary state the step is
    zero — dx = 0 gives dnu_i = 0 (W_i V_i e = mu e), and lambda = lambda^n +
    rho r with dlambda = 0 gives dr = 0. Problem: min |x - t|^2 s.t.
    x0 - t0 = 0, state x = t, y = lamN = 0.7, r = 0; the bound duals satisfy
    zl - zu = J'y (stationarity) and (x - xl) zl = (xu - x) zu = mu."""
    n, mu, yv = 3, 0.01, 0.7
    t = np.array([0.25, -0.5, 0.75])
    a, p = Expr.var(0), Expr.param(0)
    fams = [Fam("obj", (a - p) * (a - p), 1, True, None, [[i] for i in range(n)], t.reshape(-1, 1)),
            Fam("lin", a - p, 1, False, [0], [[0]], [[t[0]]])]
    R = RefModel.from_families(n, 1, fams)
    zu = np.full(n, mu)
    zl = np.full(n, mu)
    zl[0] += yv
    xl, xu = t - mu / zl, t + mu / zu
    bd = dict(xl=xl, xu=xu, x0=t.copy(), gl=np.zeros(1), gu=np.zeros(1))
    st = dict(x=t.copy(), zl=zl, zu=zu, r=np.zeros(1), s=np.zeros(1), y=np.array([yv]), vl=np.zeros(1),
              vu=np.zeros(1), lamN=np.array([yv]), mu=mu, rho=50.0, sf=1.0, dw=0.0, dc=0.0)
    step = ref_newton_step(R, bd, st, _opts())
    assert step["status"] == 0
    for k in KEYS:
        assert np.max(np.abs(step[k])) <= 1e-13, (k, step[k])


@pytest.mark.gpu
@pytest.mark.parametrize("kw", CASES)
def test_gpu_step_matches_full_newton(gpu, kw):
    from paper_2510_13333_b200.ipm import NclSolver
    rng = np.random.default_rng(11)
    n, m, fams, bd = _toy(rng)
    M, R = both_models(n, m, fams)
    st = _state(rng, bd, n, m, **kw)
    step = NclSolver(M, bd).newton_step(st, _opts())
    assert step["status"] == 0
    assert _relerr(step, full_newton(R, bd, st)) <= 1e-10
    ref = ref_newton_step(R, bd, st, _opts())
    assert _relerr(step, ref) <= 1e-12


@pytest.mark.gpu
def test_gpu_step_case9_scopf(gpu):
    from paper_2510_13333_b200.ipm import NclSolver
    s = Scopf("case9", 2)
    R = RefModel.from_families(s.n, s.m, s.families())
    bd = s.bounds()
    st = _scopf_state(np.random.default_rng(3), bd, s.n, s.m)
    step = NclSolver(s.build_model(), bd).newton_step(st, _opts())
    assert step["status"] == 0
    assert _relerr(step, full_newton(R, bd, st)) <= 1e-10
