"""Full-size symbolic bit-exactness record (tools/, not a test: the reference
ordering takes ~30 s here): the product's symbolic_order + analyze of the
condensed SCOPF KKT pattern against the reference's, field by field, with
both timings.   python tools/symbolic_record.py activsg500 256 OUT.json"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle.ref import RefSparseSym, RefSymbolic, ref_symbolic_order  # noqa: E402
from paper_2510_13333_b200 import sparse as ps  # noqa: E402
from paper_2510_13333_b200.kkt import Kkt  # noqa: E402
from paper_2510_13333_b200.scopf import Scopf  # noqa: E402

grid, K, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
s = Scopf(grid, K)
A = Kkt(s.build_model()).matrix
n = A.dim()
cp, ri = A.col_ptr(), A.row_ind()
B = RefSparseSym(n, ri, np.repeat(np.arange(n, dtype=np.int32), np.diff(cp)), np.ones(len(ri)))
t = time.perf_counter(); pa = ps.symbolic_order(A); ta = time.perf_counter() - t
t = time.perf_counter(); pb = ref_symbolic_order(B); tb = time.perf_counter() - t
Sa, Sb = ps.analyze(A, pa), RefSymbolic(B, pb)
eq = {f: bool(np.array_equal(getattr(Sa, f), getattr(Sb, f)))
      for f in ["perm", "iperm", "parent", "up_colptr", "up_rowind", "entry_map", "l_colcount"]}
eq["l_nnz"] = int(Sa.l_nnz) == int(Sb.l_nnz)
rec = {"grid": grid, "K": K, "n": n, "nnz": int(len(ri)), "l_nnz": int(Sa.l_nnz), "equal": eq,
       "all_equal": all(eq.values()), "symbolic_order_s": {"product": ta, "reference": tb}}
json.dump(rec, open(out, "w"), indent=1)
print(json.dumps(rec))
