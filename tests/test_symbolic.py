"""Bit-exact symbolic analysis: product (host C++ in libnclopf_b200.so) vs the
reference (oracle/_ref). CPU only — the symbolic analysis is host code.

North_star: "the symbolic analysis (permutation, etree, fill pattern) must
match bit-exactly". Covers symbolic_order (sparse_sym.cpp:139-191), analyze
(:198-260) and SparseSym::finalize's CSC/duplicate merge (:28-56)."""
import numpy as np
import pytest

from oracle.ref import RefSparseSym, RefSymbolic, ref_symbolic_order
from paper_2510_13333_b200 import sparse as ps
from paper_2510_13333_b200._lib import InvalidArgument, LogicError
from tests import matgen


def both(n, r, c, v):
    A = ps.SparseSym(n)
    A.add_many(r, c, v)
    A.finalize()
    B = RefSparseSym(n, r, c, v)
    return A, B


def assert_symbolic_equal(A, B, perm=None):
    pa = ps.symbolic_order(A)
    pb = ref_symbolic_order(B)
    np.testing.assert_array_equal(pa, pb)
    Sa = ps.analyze(A, perm)
    Sb = RefSymbolic(B, perm)
    for f in ["perm", "iperm", "parent", "up_colptr", "up_rowind", "entry_map", "l_colcount"]:
        np.testing.assert_array_equal(getattr(Sa, f), getattr(Sb, f), err_msg=f)
    assert Sa.l_nnz == Sb.l_nnz
    return Sa


@pytest.mark.parametrize("seed", range(60))
def test_random_graphs_bit_exact(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 130))
    dens = float(rng.choice([0.02, 0.05, 0.1, 0.15]))
    r, c, v = matgen.random_graph_lower(n, dens, rng, diag=bool(rng.random() < 0.8))
    r, c, v = matgen.shuffled_with_duplicates(r, c, v, rng, ndup=5)
    A, B = both(n, r, c, v)
    ca, cb = A.col_ptr(), B.csc()
    np.testing.assert_array_equal(ca, cb[0])
    np.testing.assert_array_equal(A.row_ind(), cb[1])
    np.testing.assert_array_equal(A.values(), cb[2])  # host finalize merge, same order
    assert_symbolic_equal(A, B)


@pytest.mark.parametrize("seed", range(10))
def test_kkt_like_bit_exact(seed):
    rng = np.random.default_rng(seed)
    r, c, v = matgen.kkt_like(int(rng.integers(20, 400)), int(rng.integers(10, 200)), rng)
    n = int(max(r.max(), c.max()) + 1)
    A, B = both(n, r, c, v)
    assert_symbolic_equal(A, B)


def test_given_perm_and_errors():
    rng = np.random.default_rng(3)
    r, c, v = matgen.kkt_like(30, 10, rng)
    A, B = both(40, r, c, v)
    perm = rng.permutation(40).astype(np.int32)
    assert_symbolic_equal(A, B, perm)
    with pytest.raises(InvalidArgument):
        ps.analyze(A, np.zeros(40, np.int32))  # not a bijection
    with pytest.raises(InvalidArgument):
        ps.analyze(A, np.arange(39))
    M = ps.SparseSym(3)
    with pytest.raises(InvalidArgument):
        M.add(0, 1, 1.0)  # upper triangle
    with pytest.raises(InvalidArgument):
        M.add(3, 0, 1.0)
    M.add(0, 0, 1.0)
    with pytest.raises(LogicError):
        ps.analyze(M)  # not finalized
    M.finalize()
    with pytest.raises(LogicError):
        M.finalize()
    M.begin_refill()
    with pytest.raises(LogicError):
        M.add(1, 1, 2.0)  # refill mismatch


def test_arrow_tridiag_and_empty():
    n = 8
    K = np.eye(n) * 4
    K[0, :] = K[:, 0] = 1
    K[0, 0] = 9
    A, B = both(n, *matgen.dense_lower_triplets(K))
    S = assert_symbolic_equal(A, B)
    assert S.l_nnz == n - 1
    E = ps.SparseSym(0)
    E.finalize()
    assert len(ps.symbolic_order(E)) == 0


def test_matrix_market_matches_reference():
    rng = np.random.default_rng(5)
    r, c, v = matgen.kkt_like(10, 4, rng)
    A, B = both(14, r, c, v)
    assert A.write_matrix_market() == B.write_matrix_market()


@pytest.mark.parametrize("seed", range(3))
def test_high_degree_nodes_bit_exact(seed):
    """Nodes above the ordering's bitmap threshold (degree > kBig = 256), like the
    SCOPF base-case variables that couple every contingency block."""
    rng = np.random.default_rng(77 + seed)
    n = 2600
    r, c = [], []
    for i in range(1, n):  # sparse backbone: random tree + chords
        j = int(rng.integers(0, i))
        r.append(i), c.append(j)
    for _ in range(2 * n):
        i, j = sorted(rng.integers(0, n, 2))[::-1]
        if i != j:
            r.append(int(i)), c.append(int(j))
    for hub in rng.choice(n, 4, replace=False):  # hubs of degree ~1100-1300
        for j in rng.choice(n, int(rng.integers(1100, 1300)), replace=False):
            if j != hub:
                r.append(int(max(hub, j))), c.append(int(min(hub, j)))
    r += list(range(n)); c += list(range(n))
    v = rng.standard_normal(len(r))
    A, B = both(n, np.array(r), np.array(c), v)
    assert_symbolic_equal(A, B)


@pytest.mark.parametrize("grid,K", [("case118", 16), ("activsg500", 16)])
def test_scopf_kkt_symbolic_bit_exact(grid, K):
    """The condensed SCOPF KKT pattern itself (the bench / solve matrix):
    perm, etree, permuted pattern, entry map and column counts identical to
    the reference's symbolic_order + analyze (a SCOPF pattern was
    never under test; the 500x256 record is profiles/r02_symbolic_500x256.json)."""
    from paper_2510_13333_b200.kkt import Kkt
    from paper_2510_13333_b200.scopf import Scopf
    s = Scopf(grid, K)
    A = Kkt(s.build_model()).matrix
    cp, ri = A.col_ptr(), A.row_ind()
    n = A.dim()
    cols = np.repeat(np.arange(n, dtype=np.int32), np.diff(cp))
    B = RefSparseSym(n, ri, cols, np.ones(len(ri)))
    assert_symbolic_equal(A, B)
