"""Pin the oracle (the reference C++ compiled in place, oracle/_ref) against
the SPEC known-answer examples and invariants.

CPU only. These are the golden vectors of this path: the reference ships no
test files, so SPEC.md's [TRIVIAL]/[DERIVED] examples are the fixtures.
"""
import numpy as np
import pytest

from oracle.ref import RefError, RefFactorization, RefSparseSym, RefSymbolic, ref_symbolic_order
from tests import matgen


def ref_from_dense(K):
    r, c, v = matgen.dense_lower_triplets(K)
    return RefSparseSym(K.shape[0], r, c, v)


def test_identity_kat():
    M = ref_from_dense(np.eye(3))
    F = RefFactorization(M)
    assert F.ok() and F.inertia == (3, 0, 0)
    np.testing.assert_array_equal(F.diagonal(), [1, 1, 1])
    x, res, sweeps, conv = F.solve_refined([1, 2, 3])
    np.testing.assert_array_equal(x, [1, 2, 3])
    assert conv and sweeps == 0


def test_diag_signs_kat():
    M = ref_from_dense(np.diag([2.0, -3.0]))
    F = RefFactorization(M)
    assert F.inertia == (1, 1, 0)
    x, *_ = F.solve_refined([2, 3])
    np.testing.assert_allclose(x, [1, -1])


def test_zero_pivot_kat():  # SPEC.md:46 -> index 0 (0-based original), SURVEY §4
    M = RefSparseSym(2, [1], [0], [1.0])
    M2 = RefSparseSym(2)
    M2.add_many([0, 1, 1], [0, 0, 1], [0.0, 1.0, 0.0])
    M2.finalize()
    F = RefFactorization(M2)
    assert F.status == "zero_pivot" and F.zero_pivot_index == 0
    assert F.inertia == (0, 0, 0)


def test_threshold_relative_to_input_diag():  # SPEC.md:73, sparse_sym.cpp:286
    M = ref_from_dense(np.diag([1e13, 5.0]))
    F = RefFactorization(M)
    assert F.status == "zero_pivot" and F.zero_pivot_index == 1


def test_arrow_ordering_kat():
    n = 8
    K = np.eye(n) * 4
    K[n - 1, :] = K[:, n - 1] = 1
    K[n - 1, n - 1] = 10
    M = ref_from_dense(K)
    perm = ref_symbolic_order(M)
    np.testing.assert_array_equal(perm, np.arange(n))
    S = RefSymbolic(M)
    assert S.l_nnz == n - 1
    # apex at index 0: tie-break by index once degrees equalise
    K0 = np.eye(n) * 4
    K0[0, :] = K0[:, 0] = 1
    K0[0, 0] = 10
    perm0 = ref_symbolic_order(ref_from_dense(K0))
    np.testing.assert_array_equal(perm0, [1, 2, 3, 4, 5, 6, 0, 7])


def test_tridiagonal_zero_fill():
    n = 20
    K = np.eye(n) * 3 + np.eye(n, k=1) + np.eye(n, k=-1)
    S = RefSymbolic(ref_from_dense(K))
    assert S.l_nnz == n - 1


@pytest.mark.parametrize("seed", range(100))
def test_inertia_vs_dense_eig(seed):  # SPEC.md:68, criterion 7
    rng = np.random.default_rng(seed)
    n1, n2 = int(rng.integers(3, 20)), int(rng.integers(2, 15))
    (r, c, v), K = matgen.quasi_definite(n1, n2, 0.3, rng)
    F = RefFactorization(RefSparseSym(n1 + n2, r, c, v))
    ev = np.linalg.eigvalsh(K)
    assert F.inertia == (int((ev > 0).sum()), int((ev < 0).sum()), 0)


def test_reconstruction_and_determinism():
    rng = np.random.default_rng(7)
    (r, c, v), K = matgen.quasi_definite(30, 20, 0.2, rng)
    M = RefSparseSym(50, r, c, v)
    S = RefSymbolic(M)
    F = RefFactorization(M, S)
    lp, li, lx = F.L_csc(S.l_nnz)
    n = 50
    L = np.eye(n)
    for j in range(n):
        L[li[lp[j]:lp[j + 1]], j] = lx[lp[j]:lp[j + 1]]
    PKP = K[np.ix_(S.perm, S.perm)]
    rec = np.linalg.norm(PKP - L @ np.diag(F.diagonal()) @ L.T) / np.linalg.norm(K)
    assert rec <= 1e-10
    F2 = RefFactorization(M, S)
    assert np.array_equal(F.diagonal(), F2.diagonal())
    assert F.inertia == (30, 20, 0)


def test_refill_mismatch_and_upper_add():  # sparse_sym.cpp:13, :20-23
    M = RefSparseSym(3, [0, 1, 2], [0, 0, 2], [1.0, 2.0, 3.0])
    M.begin_refill()
    with pytest.raises(RefError) as e:
        M.add_many([2], [2], [1.0])
    assert e.value.code == -2  # logic_error
    with pytest.raises(RefError) as e2:
        RefSparseSym(3, [0], [1], [1.0])
    assert e2.value.code == -1  # invalid_argument
