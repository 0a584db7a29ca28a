"""CPU oracle NCL/IPM solve of one SCOPF config (reference sparse_core/model_ad
backend). Writes a JSON summary + the full-precision per-iteration trace; used
to pin GPU parity at sizes too large for the test suite (tools/, not a test).

  python tools/oracle_solve.py GRID K OUT.json
  NCL_REF_VARIANT=fma python tools/oracle_solve.py ...   # reference built with FMA
"""
import json
import os
import sys
import time

sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
from oracle.ref import RefModel, ref_ncl_solve  # noqa: E402
from paper_2510_13333_b200.ipm import NclOptions  # noqa: E402
from paper_2510_13333_b200.scopf import Scopf  # noqa: E402
import oracle.ref as R  # noqa: E402

grid, K, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
s = Scopf(grid, K)
M = RefModel.from_families(s.n, s.m, s.families())
o = NclOptions()
R.lib().ref_ipm_default_options(R.C.byref(o))
o.verbose = 1
t0 = time.time()
ref = ref_ncl_solve(M, s.bounds(), options=o)
wall = time.time() - t0
json.dump({"grid": grid, "K": K, "variant": os.environ.get("NCL_REF_VARIANT", "") or "default",
           "lib": R.LIB.rsplit("/oracle/", 1)[-1], "wall_s": wall, "status": ref["status"], "result": ref["result"],
           "trace": ref["trace"]}, open(out, "w"))
print(json.dumps({"status": ref["status"], "wall_s": wall, **ref["result"]}))
