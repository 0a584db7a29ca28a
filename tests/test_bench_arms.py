"""The two bench arms build the same workload independently.

`bench.py --impl reference` builds its KKT without the product library
(oracle/ref_scopf.cpp: instance generator + reference ModelBuilder +
reference SparseSym); the product arm builds it through libnclopf_b200.so.
CPU: same contingency ids, same sizes, same model coordinates, same K pattern
as the reference assembly of the product model. GPU: the product arm's K
values equal the reference arm's (eval is bit-exact except sin/cos ulps).
"""
import numpy as np
import pytest

import bench
from oracle.ref import RefModel, RefScopf, ref_condensed_kkt
from paper_2510_13333_b200.scopf import GRIDS, Scopf, contingency_ids


@pytest.mark.parametrize("grid,K", [("case9", 0), ("case118", 16), ("activsg500", 16), ("activsg500", 300)])
def test_reference_arm_instance_matches_product(grid, K):
    assert bench._grid_dims(grid) == GRIDS[grid]
    ids = bench._contingency_ids(grid, K) if K else None
    if K:
        assert ids == contingency_ids(grid, K)
    s = Scopf(grid, K)
    kind, nb, nl, ng = GRIDS[grid]
    rs = RefScopf(kind, nb, nl, ng, bench.SEED, K, ids)
    assert (rs.n, rs.m) == (s.n, s.m)
    bp, br = s.bounds(), rs.bounds()
    for k in bp:
        np.testing.assert_array_equal(bp[k], br[k])
    R1 = rs.model()
    R2 = RefModel.from_families(s.n, s.m, s.families())
    for a, b in zip(R1.jac_coords() + R1.hess_coords(), R2.jac_coords() + R2.hess_coords()):
        np.testing.assert_array_equal(a, b)
    w, lam, sig, D = bench.ipm_point(br, rs.m)
    np.testing.assert_array_equal(R1.eval_jacobian(w), R2.eval_jacobian(w))


def test_load_level_contingencies():
    """C5 (500 x 1024): screened outages x 4 load levels, paper-layout sizes
    (nvar 3,817,900, ncon 5,039,591)."""
    ids = contingency_ids("activsg500", 1024)
    nl = GRIDS["activsg500"][2]
    assert len(set(ids)) == 1024 and max(i // nl for i in ids) == 3
    assert ids[:256] == contingency_ids("activsg500", 256)
    s = Scopf("activsg500", 1024)
    assert (s.n, s.m) == (3817900, 5039591)
    # level-j contingency: same rows as level 0, balance right-hand sides scaled by 1 - 0.015 j
    a = Scopf("activsg500", 1, contingencies=[ids[0]]).bounds()
    b = Scopf("activsg500", 1, contingencies=[ids[0] + 2 * nl]).bounds()
    diff = np.nonzero(a["gl"] != b["gl"])[0]
    assert len(diff) > 0
    np.testing.assert_allclose(b["gl"][diff], 0.97 * a["gl"][diff], rtol=1e-15)
    with pytest.raises(Exception):
        Scopf("activsg500", 1, contingencies=[ids[0] + 4 * nl])


def test_reference_kkt_pattern():
    """ref_condensed_kkt = the reference SparseSym fed the product's triplet
    contract; nnz and symmetry sanity at a small size."""
    kind, nb, nl, ng = GRIDS["case118"]
    rs = RefScopf(kind, nb, nl, ng, bench.SEED, 4, bench._contingency_ids("case118", 4))
    R = rs.model()
    w, lam, sig, D = bench.ipm_point(rs.bounds(), R.m)
    K = ref_condensed_kkt(R, R.eval_hessian_lag(w, 1e-4, lam), R.eval_jacobian(w), sig, 1e-8, D)
    cp, ri, v = K.csc()
    assert K.n == R.n and cp[-1] == K.nnz()
    cols = np.repeat(np.arange(K.n), np.diff(cp))
    assert np.all(ri >= cols)  # lower CSC
    assert np.all(v[cp[:-1]] > 0)  # diagonal first in each column and positive (sig + dw + D J'J)


@pytest.mark.gpu
def test_product_kkt_equals_reference_arm_kkt(gpu):
    P = bench.build_problem("activsg500", 16)
    A = P["A"]
    kind, nb, nl, ng = GRIDS["activsg500"]
    rs = RefScopf(kind, nb, nl, ng, bench.SEED, 16, bench._contingency_ids("activsg500", 16))
    R = rs.model()
    w, lam, sig, D = bench.ipm_point(rs.bounds(), R.m)
    K = ref_condensed_kkt(R, R.eval_hessian_lag(w, 1e-4, lam), R.eval_jacobian(w), sig, 1e-8, D)
    cp, ri, v = K.csc()
    np.testing.assert_array_equal(cp, A.col_ptr())
    np.testing.assert_array_equal(ri, A.row_ind())
    va = A.values()
    assert np.max(np.abs(va - v) / np.maximum(np.abs(v), 1.0)) <= 1e-13
