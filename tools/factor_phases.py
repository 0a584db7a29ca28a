"""Phase split of the bench factorization (NCL_FACTOR_PHASES debug timer):
  NCL_FACTOR_PHASES=1 python tools/factor_phases.py [grid K reps]"""
import os
import sys

os.environ.setdefault("NCL_FACTOR_PHASES", "1")
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
import numpy as np  # noqa: E402
from bench import build_problem  # noqa: E402
from paper_2510_13333_b200 import _lib, sparse as ps  # noqa: E402

grid = sys.argv[1] if len(sys.argv) > 1 else "activsg500"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
_lib.check(_lib.lib.ncl_init(0))
P = build_problem(grid, K)
F = ps.factorize(P["A"], P["S"])
for _ in range(reps):
    F.refactorize(P["A"])
print(F.status, F.inertia)
