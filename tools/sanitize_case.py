"""One factor + solve (+ one sharded emulated factor) of a small SCOPF KKT, for
compute-sanitizer (tests/test_sanitizer.py): exercises the register-front,
group, warp-single, CTA and large-front paths and the flag protocol."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2510_13333_b200 import _lib  # noqa: E402
from paper_2510_13333_b200 import sparse as ps  # noqa: E402
from paper_2510_13333_b200.kkt import Kkt  # noqa: E402
from paper_2510_13333_b200.scopf import Scopf  # noqa: E402

_lib.check(_lib.lib.ncl_init(0))
grid, K = (sys.argv[1], int(sys.argv[2])) if len(sys.argv) > 2 else ("case118", 4)
s = Scopf(grid, K)
M = s.build_model()
kk = Kkt(M)
rng = np.random.default_rng(5)
kk.assemble(0.1 * rng.standard_normal(M.nnzh), rng.standard_normal(M.nnzj), 1.0 + rng.random(s.n), 0.0,
            10.0 + rng.random(M.m))
A = kk.matrix
S = ps.analyze(A)
F = ps.factorize(A, S)
x = F.solve(rng.standard_normal(s.n))
F.refactorize(A)
x2 = F.solve(rng.standard_normal(s.n))
_lib.check(_lib.lib.ncl_synchronize())
print("ok", F.status, float(np.max(np.abs(x))), float(np.max(np.abs(x2))))
