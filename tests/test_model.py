"""model_ad + scopf_builder: oracle KATs (CPU) and product-vs-reference
parity of the GPU evaluator / condensed KKT assembly (GPU)."""
import numpy as np
import pytest

from oracle.ref import RefModel, RefSparseSym
from paper_2510_13333_b200 import model as pm
from paper_2510_13333_b200.scopf import Scopf
from paper_2510_13333_b200.model import Expr, cos, sin


class Fam:
    def __init__(self, name, expr, nslots, objective, rows, vars_, params=None):
        self.name, self.nodes, self.nslots, self.objective = name, expr.program(), nslots, objective
        self.rows = np.asarray(rows if rows is not None else [], np.int32)
        self.vars = np.asarray(vars_, np.int32).reshape(-1, nslots)
        self.params = np.zeros((len(self.vars), 0)) if params is None else np.asarray(params, float).reshape(
            len(self.vars), -1)
        self.np = self.params.shape[1]


def both_models(n, m, fams):
    R = RefModel.from_families(n, m, fams)
    B = pm.ModelBuilder(n)
    if m:
        B.add_rows(m)
    for F in fams:
        tid = B.add_template(F.nodes, F.nslots, F.name)
        if F.objective:
            B.add_objective_terms(tid, F.vars, F.params if F.np else None)
        else:
            B.add_constraint_terms(tid, F.rows, F.vars, F.params if F.np else None)
    return B.build(), R


# ---------------- oracle KATs, CPU ----------------------
def test_oracle_model_kats():
    x0, x1 = Expr.var(0), Expr.var(1)
    R = RefModel.from_families(2, 0, [Fam("phi", x0 * x0 + x1, 2, True, None, [0, 1])])
    assert R.eval_objective([1.0, 1.0]) == 2.0
    p = Expr.var(0)
    cost = Expr.param(0) * p * p + Expr.param(1) * p
    R = RefModel.from_families(1, 0, [Fam("cost", cost, 1, True, None, [0], [[0.1, 20.0]])])
    assert abs(R.eval_objective([1.5]) - 30.225) < 1e-12
    R = RefModel.from_families(2, 1, [Fam("bil", x0 * x1, 2, False, [0], [0, 1])])
    J = R.eval_jacobian([3.0, 4.0])
    np.testing.assert_array_equal(J, [4.0, 3.0])
    H = R.eval_hessian_lag([3.0, 4.0], 0.0, [2.0])
    hr, hc = R.hess_coords()
    assert (hr[0], hc[0], H[0]) == (1, 0, 2.0)
    # aliased slots w0*w0 -> H(0,0)=4 with lambda=2 (model.cpp:121-123)
    R = RefModel.from_families(1, 1, [Fam("alias", x0 * x1, 2, False, [0], [0, 0])])
    assert R.eval_hessian_lag([3.0], 0.0, [2.0])[0] == 4.0
    assert R.eval_jacobian([3.0])[0] == 6.0
    f = sin(x0) * cos(x1)
    R = RefModel.from_families(2, 0, [Fam("sc", f, 2, True, None, [0, 1])])
    assert R.fd_check([0.3, 0.7], 1)["pass_"]


@pytest.mark.parametrize("grid,K", [("case9", 0), ("case9", 1), ("case118", 16), ("activsg500", 4),
                                    ("activsg500", 8)])
def test_scopf_layout_matches_paper(grid, K):
    """nvar/ncon follow the layout fitted to Tables II-III."""
    s = Scopf(grid, K)
    i = s.info
    B = 2 * i.nb + 2 * i.ng + 4 * i.nl
    Cc = 1 + 2 * i.nb + 6 * i.nl
    assert s.n == B + K * (B + 1 + 4 * i.ng)
    assert s.m == Cc + K * (Cc + 6 * i.ng - 2)
    assert i.ncomp == 4 * i.ng * K  # p = 4 n_g K pairs
    if grid == "activsg500":
        assert (s.n, s.m) == {4: (18400, 24251), 8: (33300, 43919)}[K]
    if grid == "case9" and K == 0:
        assert (s.n, s.m) == (60, 73)


def test_contingencies_do_not_island():
    s = Scopf("activsg500", 32)
    ids = s.contingencies()
    assert len(ids) == 32 and np.all(np.diff(ids) > 0)


# ---------------- GPU parity ------------------------------------------------
def _relerr(a, b):
    return float(np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b)))) if len(b) else 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("grid,K", [("case9", 0), ("case9", 2), ("case118", 4), ("activsg500", 2)])
def test_scopf_eval_parity(gpu, grid, K):
    s = Scopf(grid, K)
    fams = s.families()
    R = RefModel.from_families(s.n, s.m, fams)
    M = s.build_model()
    for a, b in zip(M.jac_coords(), R.jac_coords()):
        np.testing.assert_array_equal(a, b)
    for a, b in zip(M.hess_coords(), R.hess_coords()):
        np.testing.assert_array_equal(a, b)
    bd = s.bounds()
    rng = np.random.default_rng(0)
    lo = np.where(np.isfinite(bd["xl"]), bd["xl"], -1.0)
    hi = np.where(np.isfinite(bd["xu"]), bd["xu"], 1.0)
    for trial in range(3):
        w = lo + (hi - lo) * rng.random(s.n)
        lam = rng.standard_normal(s.m)
        lam[rng.random(s.m) < 0.1] = 0.0  # weight-0 instances are skipped
        assert abs(M.eval_objective(w) - R.eval_objective(w)) <= 1e-14 * abs(R.eval_objective(w))
        assert np.array_equal(M.eval_grad_objective(w), R.eval_grad_objective(w))
        # sin/cos may differ by an ulp between CUDA and glibc: 1e-14 relative
        assert _relerr(M.eval_constraints(w), R.eval_constraints(w)) < 1e-14
        jv = M.eval_jacobian(w)
        assert _relerr(jv, R.eval_jacobian(w)) < 1e-14
        assert _relerr(M.eval_hessian_lag(w, 0.7, lam), R.eval_hessian_lag(w, 0.7, lam)) < 1e-14
        v = rng.standard_normal(s.n)
        y = rng.standard_normal(s.m)
        assert np.array_equal(M.jac_times(jv, v), R.jac_times(jv, v))
        assert np.array_equal(M.jac_trans_times(jv, y), R.jac_trans_times(jv, y))


@pytest.mark.gpu
def test_generic_templates_bit_exact_and_fd(gpu):
    x0, x1, x2 = Expr.var(0), Expr.var(1), Expr.var(2)
    fams = [
        Fam("poly", x0 * x1 * x2 + Expr.param(0) * x0 * x0 - x2 / (x1 + 3.0), 3, False, [0, 1, 0],
            [[0, 1, 2], [2, 1, 0], [1, 1, 2]], [[0.5], [-1.5], [2.0]]),
        Fam("pw", (x0 * x0 + 1.0) ** 1.5 + x1 ** 2, 2, False, [1, 2], [[0, 3], [3, 2]]),
        Fam("obj", x0 * x0 - 3.0 * x1, 2, True, None, [[0, 1], [2, 3]]),
    ]
    M, R = both_models(4, 3, fams)
    w = np.array([0.3, -0.4, 1.2, 0.8])
    lam = np.array([1.0, 0.0, -2.0])
    assert np.array_equal(M.eval_constraints(w)[[0]], R.eval_constraints(w)[[0]])
    assert _relerr(M.eval_constraints(w), R.eval_constraints(w)) < 1e-15
    assert np.array_equal(M.eval_jacobian(w)[:6], R.eval_jacobian(w)[:6]) or \
        _relerr(M.eval_jacobian(w), R.eval_jacobian(w)) < 1e-15
    assert _relerr(M.eval_hessian_lag(w, 1.3, lam), R.eval_hessian_lag(w, 1.3, lam)) < 1e-15
    rep = pm.fd_check(M, w, 3)
    ref = R.fd_check(w, 3)
    assert rep["pass_"] and ref["pass_"]


@pytest.mark.gpu
def test_domain_error(gpu):
    from paper_2510_13333_b200._lib import DomainError
    x0 = Expr.var(0)
    M, R = both_models(1, 1, [Fam("inv", 1.0 / x0, 1, False, [0], [[0]])])
    with pytest.raises(DomainError):
        M.eval_constraints(np.array([0.0]))


@pytest.mark.gpu
@pytest.mark.parametrize("grid,K", [("case9", 1), ("case118", 2)])
def test_kkt_assembly_bit_exact(gpu, grid, K):
    from paper_2510_13333_b200.kkt import Kkt, reference_triplet_values
    s = Scopf(grid, K)
    M = s.build_model()
    kk = Kkt(M)
    rng = np.random.default_rng(1)
    hess = rng.standard_normal(M.nnzh)
    jac = rng.standard_normal(M.nnzj)
    sig = rng.random(M.n)
    D = 1.0 / (0.01 + rng.random(M.m))
    kk.assemble(hess, jac, sig, 1e-4, D)
    jr, _ = M.jac_coords()
    tv = reference_triplet_values(kk, jr, hess, jac, sig, 1e-4, D)
    tr, tc = kk.triplets()
    ref = RefSparseSym(M.n, tr, tc, tv)
    cp, ri, rv = ref.csc()
    np.testing.assert_array_equal(kk.matrix.col_ptr(), cp)
    np.testing.assert_array_equal(kk.matrix.row_ind(), ri)
    assert np.array_equal(kk.matrix.values(), rv)
