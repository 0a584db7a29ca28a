import sys, json, time; sys.path.insert(0, '/root/repo')
from paper_2510_13333_b200 import _lib
from paper_2510_13333_b200.scopf import Scopf
from paper_2510_13333_b200.ipm import solve_scopf
from oracle.ref import RefModel, ref_ncl_solve
_lib.check(_lib.lib.ncl_init(0))
for grid, K in [("activsg500", 4), ("activsg500", 16), ("case118", 16)]:
    s = Scopf(grid, K)
    t = time.time(); g = solve_scopf(s); tg = time.time() - t
    R = RefModel.from_families(s.n, s.m, s.families())
    t = time.time(); r = ref_ncl_solve(R, s.bounds()); tr = time.time() - t
    print(json.dumps({"grid": grid, "K": K, "gpu": [g.status, g.result["outer_iters"], g.result["inner_iters"], g.result["objective"], tg],
                      "cpu": [r["status"], r["result"]["outer_iters"], r["result"]["inner_iters"], r["result"]["objective"], tr]}), flush=True)
