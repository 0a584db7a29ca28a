"""mpcc_check: index sets, MPCC-multiplier recovery and the
strong-stationarity certificate — the SPEC's examples on the host functions,
the recovery identity on random points, and (GPU) the certificate of a
corrective SCOPF solved by the B200 NCL solver."""
import numpy as np
import pytest

from paper_2510_13333_b200 import mpcc


def test_index_sets_spec_examples():
    # SPEC.md:479-482
    p0, z0, zz = mpcc.index_sets([1, 0, 0], [0, 2, 0], 1e-6)
    assert list(p0) == [0] and list(z0) == [1] and list(zz) == [2]
    p0, z0, zz = mpcc.index_sets(np.zeros(5), np.zeros(5))
    assert len(p0) == len(z0) == 0 and list(zz) == list(range(5))
    with pytest.raises(mpcc.BothPositive) as e:
        mpcc.index_sets([1.0], [1.0])
    assert e.value.index == 0
    # the sets partition {0..p-1} at feasible points
    rng = np.random.default_rng(1)
    w1 = np.where(rng.random(200) < 0.5, rng.random(200), 0.0)
    w2 = np.where(w1 > 0, 0.0, np.where(rng.random(200) < 0.5, rng.random(200), 0.0))
    sets = mpcc.index_sets(w1, w2)
    assert sorted(np.concatenate(sets).tolist()) == list(range(200))


def test_recovery_spec_examples_and_gradient_identity():
    rng = np.random.default_rng(2)
    p = 50
    w1, w2 = rng.random(p), rng.random(p)
    nu1, nu2 = rng.random(p), rng.random(p)
    # nu0 = 0 -> mu = nu
    mu1, mu2 = mpcc.recover(np.zeros(p), nu1, nu2, w1, w2)
    assert np.array_equal(mu1, nu1) and np.array_equal(mu2, nu2)
    # gradient equivalence: with L = f + nu0'(w1 o w2) - nu1'w1 -
    # nu2'w2 and L^MPCC = f - mu1'w1 - mu2'w2, grad_w of the two agree
    nu0 = rng.random(p)
    mu1, mu2 = mpcc.recover(nu0, nu1, nu2, w1, w2)
    g1_nlp, g2_nlp = nu0 * w2 - nu1, nu0 * w1 - nu2
    assert np.max(np.abs(g1_nlp - (-mu1))) <= 1e-12 and np.max(np.abs(g2_nlp - (-mu2))) <= 1e-12
    # i in I+0 with w2 = 0: mu1 = nu1, mu2 = nu2 - nu0 w1
    mu1, mu2 = mpcc.recover([0.5], [0.0], [3.0], [2.0], [0.0])
    assert mu1[0] == 0.0 and mu2[0] == 3.0 - 1.0


def test_certify_spec_examples():
    # min w1 + w2 over the pair: (0, 0) with mu1 = mu2 = 1 -> strong
    c = mpcc.certify([0.0], [0.0], [1.0], [1.0], 0.0, 0.0)
    assert c["strong"] and c["n_00"] == 1
    # min w1 - w2 s.t. w2 <= 1: (0, 1), I0+, mu1 free, mu2 = 0 -> strong
    c = mpcc.certify([0.0], [1.0], [-3.0], [0.0], 0.0, 0.0)
    assert c["strong"] and c["n_0p"] == 1
    # I00 index with mu1 = -1 -> weak / unclassified
    c = mpcc.certify([0.0], [0.0], [-1.0], [0.5], 0.0, 0.0)
    assert not c["strong"] and c["sign_violations"] == 1 and c["first_violation"] == 0
    # toy MPCC min (w1 - 1)^2 + (w2 - 1)^2 at (1, 0): the
    # w2-branch is optimal; grad_w2 f = -2 = mu2 * (-1)... mu2 = -2 on I+0 is
    # sign-free, mu1 = 0: strong
    c = mpcc.certify([1.0], [0.0], [0.0], [-2.0], 0.0, 0.0)
    assert c["strong"] and c["n_p0"] == 1
    # a gradient residual above tol is not strong
    assert not mpcc.certify([1.0], [0.0], [0.0], [-2.0], 1e-3, 0.0)["strong"]


@pytest.mark.gpu
@pytest.mark.parametrize("grid,K", [("case118", 4), ("activsg500", 4)])
def test_scopf_solution_certificate(gpu, grid, K):
    """the droop / PV-PQ complementarity pairs of a solved corrective SCOPF:
    a valid partition, complementarity at solver accuracy, the recovery
    identity at the solution, and the Eq. 11 verdict (recorded)."""
    from paper_2510_13333_b200.ipm import NclSolver, default_options
    from paper_2510_13333_b200.scopf import Scopf
    s = Scopf(grid, K)
    S = NclSolver(s.build_model(), s.bounds())
    out = S.solve(default_options())
    assert out.status == "optimal"
    # NCL meets w1 w2 <= 0 up to r (|r| <= eta* = 1e-7), so the pairs are
    # complementary to ~sqrt(1e-7) componentwise: activity at 1e-3
    d = mpcc.certify_scopf(s, S, out, tol=1e-5, tol_act=1e-3)
    p = s.info.ncomp
    assert p == 4 * s.info.ng * K
    assert d["n_p0"] + d["n_0p"] + d["n_00"] == p
    assert d["comp_residual"] <= 1e-6
    # the multipliers of an interior solution: nu >= 0 up to the barrier
    assert np.min(d["nu0"]) >= -1e-8
    # every pair is classified and the certificate is internally consistent
    if d["strong"]:
        assert d["sign_violations"] == 0 and d["inactive_violations"] == 0
    print(grid, K, {k: d[k] for k in ("n_p0", "n_0p", "n_00", "grad_residual", "feas_residual", "comp_residual",
                                      "inactive_violations", "sign_violations", "strong")})
