"""GPU NCL/IPM solve of one SCOPF config; optionally the full-precision
per-iteration trace (for tools/trace_diff.py against tools/oracle_solve.py's).

  python tools/gpu_solve.py GRID K [--trace OUT.json] [--oracle]
"""
import collections
import json
import sys
import time

sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
from paper_2510_13333_b200 import _lib  # noqa: E402
from paper_2510_13333_b200.ipm import NclSolver, default_options  # noqa: E402
from paper_2510_13333_b200.scopf import Scopf  # noqa: E402

grid, K = sys.argv[1], int(sys.argv[2])
trace_out = sys.argv[sys.argv.index("--trace") + 1] if "--trace" in sys.argv else None
_lib.check(_lib.lib.ncl_init(0))
t0 = time.time()
s = Scopf(grid, K)
M = s.build_model()
S = NclSolver(M, s.bounds())
t_build = time.time() - t0
o = default_options()
o.verbose = 1
t0 = time.time()
out = S.solve(o)
wall = time.time() - t0
r = out.result
summary = {"grid": grid, "K": K, "n": s.n, "m": s.m, "status": out.status, "build_s": t_build, "wall_s": wall,
           **{k: r[k] for k in ["outer_iters", "inner_iters", "factorizations", "objective", "r_inf", "inf_pr",
                                "inf_du", "t_total", "t_init", "t_eval", "t_factor", "t_solve", "t_linesearch",
                                "t_other"]}}
print(json.dumps(summary))
if trace_out:
    with open(trace_out, "w") as f:
        json.dump({"grid": grid, "K": K, "variant": "b200", "status": out.status, "result": r, "wall_s": wall,
                   "trace": out.trace}, f)
if "--oracle" in sys.argv:
    from oracle.ref import RefModel, ref_ncl_solve
    R = RefModel.from_families(s.n, s.m, s.families())
    t0 = time.time()
    ref = ref_ncl_solve(R, s.bounds())
    rr = ref["result"]
    print(json.dumps({"oracle": True, "status": ref["status"], "wall": time.time() - t0,
                      **{k: rr[k] for k in ["outer_iters", "inner_iters", "factorizations", "objective", "r_inf",
                                            "t_factor", "t_solve", "t_eval"]}}))
tr = [t for t in out.trace if "iter" in t]
print(json.dumps({"sweeps": dict(collections.Counter(t["sweeps"] for t in tr)),
                  "factorizations_per_iter": dict(collections.Counter(t["factorizations"] for t in tr)),
                  "ls_backtracks": dict(collections.Counter(t["ls"] for t in tr))}))
