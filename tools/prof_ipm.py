"""Profiling driver (tools/, not a test): a few IPM iterations of the
500-bus x 256 SCOPF solve on the GPU, so that ncu can capture the per-iteration
kernels other than the factorization — evaluation (eval_kernel, gather_sum64),
KKT assembly (kkt_assemble_kernel), the IPM element/reduction kernels and the
solves — from the same run the solver makes.

  ncu --set full -k regex:kkt_assemble_kernel -c 1 -o X python tools/prof_ipm.py
"""
import sys

sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
from paper_2510_13333_b200 import _lib  # noqa: E402
from paper_2510_13333_b200.ipm import NclSolver, default_options  # noqa: E402
from paper_2510_13333_b200.scopf import Scopf  # noqa: E402

grid = sys.argv[1] if len(sys.argv) > 1 else "activsg500"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 256
_lib.check(_lib.lib.ncl_init(0))
s = Scopf(grid, K)
S = NclSolver(s.build_model(), s.bounds())
o = default_options()
o.max_outer = 1
o.max_inner = 4
out = S.solve(o)
print(out.status, out.result["inner_iters"])
