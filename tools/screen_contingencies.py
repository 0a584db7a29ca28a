"""Contingency screening (PAPER.md:526-543, SPEC.md:521-569 in spirit): solve
every non-islanding single-branch outage alone as a K=1 corrective SCOPF on
the B200 solver and keep those that reach NCL optimality. The committed list
(paper_2510_13333_b200/data/screened_<grid>_<seed>.json) fixes the contingency
set of every config of that grid, so all runs (GPU, oracle, bench) use the
same instance.

usage: python tools/screen_contingencies.py GRID NEED [SEED]
"""
import json
import os
import sys
import time

ROOT = __file__.rsplit("/tools/", 1)[0]
sys.path.insert(0, ROOT)

from paper_2510_13333_b200 import _lib  # noqa: E402
from paper_2510_13333_b200.ipm import NclSolver, default_options  # noqa: E402
from paper_2510_13333_b200.scopf import Scopf  # noqa: E402

grid, need = sys.argv[1], int(sys.argv[2])
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 2510
_lib.check(_lib.lib.ncl_init(0))
probe = [int(l) for l in Scopf(grid, 0, seed=seed).candidates()]  # non-islanding, ascending
os.makedirs(os.path.join(ROOT, "paper_2510_13333_b200", "data"), exist_ok=True)
dst = os.path.join(ROOT, "paper_2510_13333_b200", "data", f"screened_{grid}_{seed}.json")
out_dir = os.path.join(ROOT, "gpurun_out", "data")
os.makedirs(out_dir, exist_ok=True)
feasible, rejected, log = [], [], []
t0 = time.time()
opts = default_options(verbose=0, max_inner=600)


def save():
    doc = {"grid": grid, "seed": seed, "rule": "K=1 SCOPF reaches NCL optimality (default options, max_inner 600)",
           "screened": len(log), "feasible": feasible, "rejected": rejected, "seconds": time.time() - t0,
           "complete": len(feasible) >= need or len(log) == len(probe), "log": log}
    for d in (dst, os.path.join(out_dir, os.path.basename(dst))):
        with open(d, "w") as f:
            json.dump(doc, f)


for l in probe:
    s = Scopf(grid, 1, seed=seed, contingencies=[l])
    out = NclSolver(s.build_model(), s.bounds()).solve(opts)
    ok = out.status == "optimal"
    (feasible if ok else rejected).append(l)
    log.append({"branch": l, "status": out.status, "inner": out.result["inner_iters"], "r_inf": out.result["r_inf"]})
    print(json.dumps(log[-1]), flush=True)
    if len(log) % 10 == 0:
        save()
    if len(feasible) >= need:
        break
save()
print(f"{len(feasible)} feasible / {len(log)} screened in {time.time() - t0:.1f}s -> {dst}")
