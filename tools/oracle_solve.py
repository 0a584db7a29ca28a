"""CPU oracle NCL/IPM solve of one SCOPF config (reference sparse_core/model_ad
backend). Writes a JSON summary + the trace; used to pin GPU parity at sizes
too large for the test suite (tools/, not a test)."""
import json, sys, time
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
from paper_2510_13333_b200.scopf import Scopf
from oracle.ref import RefModel, ref_ncl_solve
grid, K, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
s = Scopf(grid, K)
R = RefModel.from_families(s.n, s.m, s.families())
t0 = time.time()
ref = ref_ncl_solve(R, s.bounds())
json.dump({"grid": grid, "K": K, "wall_s": time.time() - t0, "status": ref["status"], "result": ref["result"],
           "trace": ref["trace"]}, open(out, "w"))
print(json.dumps({"status": ref["status"], "wall_s": time.time() - t0, **ref["result"]}))
