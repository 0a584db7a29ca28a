"""Seeded test-matrix generators (lower-triangle triplets)."""
import numpy as np


def random_graph_lower(n, density, rng, diag=True):
    rows, cols = [], []
    for j in range(n):
        for i in range(j + 1, n):
            if rng.random() < density:
                rows.append(i)
                cols.append(j)
    if diag:
        rows += list(range(n))
        cols += list(range(n))
    vals = rng.standard_normal(len(rows))
    return np.array(rows, np.int32), np.array(cols, np.int32), vals


def quasi_definite(n1, n2, density, rng):
    """[A B^T; B -C] with A SPD, C SPD: inertia (n1, n2, 0). Dense -> lower triplets."""
    A = rng.standard_normal((n1, n1)) * (rng.random((n1, n1)) < density)
    A = A @ A.T + n1 * np.eye(n1)
    Cm = rng.standard_normal((n2, n2)) * (rng.random((n2, n2)) < density)
    Cm = Cm @ Cm.T + n2 * np.eye(n2)
    B = rng.standard_normal((n2, n1)) * (rng.random((n2, n1)) < density)
    K = np.zeros((n1 + n2, n1 + n2))
    K[:n1, :n1] = A
    K[n1:, :n1] = B
    K[:n1, n1:] = B.T
    K[n1:, n1:] = -Cm
    return dense_lower_triplets(K), K


def dense_lower_triplets(K, keep_diag=True):
    n = K.shape[0]
    r, c = np.nonzero(np.tril(K))
    if keep_diag:
        d = np.arange(n)
        mask = np.ones(n, bool)
        have = set(zip(r.tolist(), c.tolist()))
        extra = [i for i in range(n) if (i, i) not in have]
        r = np.concatenate([r, np.array(extra, dtype=r.dtype)])
        c = np.concatenate([c, np.array(extra, dtype=c.dtype)])
    v = K[r, c]
    return r.astype(np.int32), c.astype(np.int32), v.astype(np.float64)


def shuffled_with_duplicates(r, c, v, rng, ndup=10):
    """Split some entries into duplicate triplets and shuffle the order."""
    r, c, v = list(r), list(c), list(v)
    for _ in range(ndup if len(r) else 0):
        k = rng.integers(len(r))
        part = rng.standard_normal()
        r.append(r[k])
        c.append(c[k])
        v.append(part)
        v[k] -= part
    perm = rng.permutation(len(r))
    return (np.array(r, np.int32)[perm], np.array(c, np.int32)[perm], np.array(v)[perm])


def kkt_like(nx, ny, rng, nnz_per_row=3, rho=100.0, delta=1.0):
    """2x2 KKT [H+dI J^T; J -rho^-1 I] with sparse random J and tridiagonal H."""
    rows, cols, vals = [], [], []
    for i in range(nx):
        rows.append(i); cols.append(i); vals.append(2.0 + delta + rng.random())
        if i + 1 < nx:
            rows.append(i + 1); cols.append(i); vals.append(-0.5 * rng.random())
    for k in range(ny):
        cs = rng.choice(nx, size=min(nnz_per_row, nx), replace=False)
        for cj in cs:
            rows.append(nx + k); cols.append(int(cj)); vals.append(rng.standard_normal())
        rows.append(nx + k); cols.append(nx + k); vals.append(-1.0 / rho)
    return np.array(rows, np.int32), np.array(cols, np.int32), np.array(vals)


def to_dense(n, r, c, v):
    K = np.zeros((n, n))
    np.add.at(K, (r, c), v)
    off = r != c
    np.add.at(K, (c[off], r[off]), v[off])
    return K
