"""Debug: host-buffer factor+solve paths at 500x256 (pinned torch buffers)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from bench import build_problem  # noqa: E402
from paper_2510_13333_b200 import _lib  # noqa: E402
from paper_2510_13333_b200 import sparse as ps  # noqa: E402

_lib.check(_lib.lib.ncl_init(0))
P = build_problem("activsg500", 256)
A, S = P["A"], P["S"]
F = ps.factorize(A, S)
n = A.dim()
vals_h = torch.from_numpy(A.values()).pin_memory()
b_h = torch.from_numpy(np.random.default_rng(1).standard_normal(n)).pin_memory()
x_h = torch.empty(n, dtype=torch.float64).pin_memory()
for name in ("old", "new", "old", "new"):
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if name == "new":
            F.factor_solve_host(A, vals_h, b_h, x_h)
        else:
            A.set_values(vals_h, where=ps.HOST)
            F.refactorize(A)
            x_h.copy_(b_h)
            F.solve_in_place(x_h, ps.HOST)
            F._status()
        ts.append(time.perf_counter() - t0)
    print(name, "ms", 1e3 * np.median(ts), 1e3 * min(ts))
t0 = time.perf_counter(); A.set_values(vals_h, where=ps.HOST); t1 = time.perf_counter()
print("set_values H2D ms", 1e3 * (t1 - t0))
