"""Debug: factor + solve the bench KKT with the package found first on sys.path; save x."""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
sys.path.insert(1, ".")
from bench import build_problem  # noqa: E402
from paper_2510_13333_b200 import sparse as ps  # noqa: E402
import paper_2510_13333_b200 as pkg  # noqa: E402
print(pkg.__file__)
P = build_problem(sys.argv[3] if len(sys.argv) > 3 else "activsg500", int(sys.argv[4]) if len(sys.argv) > 4 else 16)
A, S = P["A"], P["S"]
F = ps.factorize(A, S)
rng = np.random.default_rng(1)
b = rng.standard_normal(A.dim())
x1 = F.solve(b)
x2 = F.solve(b)
print("repeat bitwise:", np.array_equal(x1, x2))
np.save(sys.argv[2], np.stack([x1, F.diagonal()]))
