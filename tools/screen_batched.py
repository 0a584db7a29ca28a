"""Batched contingency screening of a whole grid: every
non-islanding single-branch outage's Eq. 5 system as one block of ONE B200 NCL
solve, against the committed K=1-SCOPF screening (data/screened_*.json).

  python tools/screen_batched.py GRID OUT.json [BATCH]
"""
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2510_13333_b200 import _lib  # noqa: E402
from paper_2510_13333_b200 import screening as scr  # noqa: E402
from paper_2510_13333_b200.scopf import screened  # noqa: E402

grid, out = sys.argv[1], sys.argv[2]
batch = int(sys.argv[3]) if len(sys.argv) > 3 else None
_lib.check(_lib.lib.ncl_init(0))
t0 = time.time()
rep = scr.screen_all(grid, batch=batch)
wall = time.time() - t0
feas = sorted(r.id for r in rep.records if r.objective <= scr.FEAS_TOL)
infeas = sorted(r.id for r in rep.records if r.objective > scr.FEAS_TOL)
ref = screened(grid)
doc = {"grid": grid, "batch": batch or len(rep.records), "wall_s": wall, "contingencies": len(rep.records),
       "feasible": len(feas), "infeasible": infeas,
       "statuses": sorted({r.status for r in rep.records}), "iters": sorted({r.iters for r in rep.records}),
       "ranking_top10": rep.ranking[:10],
       "objectives": {r.id: r.objective for r in rep.records},
       "k1_scopf_screen_feasible": None if ref is None else len(ref),
       "k1_scopf_rejected": None if ref is None else sorted(set(r.id for r in rep.records) - set(ref))}
json.dump(doc, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in doc.items() if k != "objectives"}))
