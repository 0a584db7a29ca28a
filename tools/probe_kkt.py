"""Quick probe: build the SCOPF KKT at a config, time setup, GPU factor+solve."""
import sys, time, ctypes as C
import numpy as np
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
from paper_2510_13333_b200 import _lib, sparse as ps
from paper_2510_13333_b200.scopf import Scopf
from paper_2510_13333_b200.kkt import Kkt

grid = sys.argv[1] if len(sys.argv) > 1 else "activsg500"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 256
ref = len(sys.argv) > 3 and sys.argv[3] == "ref"
_lib.check(_lib.lib.ncl_init(0))
t = time.time(); s = Scopf(grid, K); t_spec = time.time() - t
t = time.time(); M = s.build_model(); t_model = time.time() - t
t = time.time(); kk = Kkt(M); t_kkt = time.time() - t
rng = np.random.default_rng(0)
bd = s.bounds()
w = bd["x0"]
lam = 0.1 * rng.standard_normal(M.m)
t = time.time(); hess = M.eval_hessian_lag(w, 1e-4, lam); jac = M.eval_jacobian(w); t_eval = time.time() - t
sig = 1.0 + rng.random(M.n)
D = np.full(M.m, 100.0)
kk.assemble(hess, jac, sig, 0.0, D)
A = kk.matrix
t = time.time(); S = ps.analyze(A); t_an = time.time() - t
info = S.info()
print(f"{grid}x{K}: n={M.n} m={M.m} nnzJ={M.nnzj} nnzH={M.nnzh} nnzK={A.nnz()} | spec {t_spec:.2f}s model {t_model:.2f}s "
      f"kkt {t_kkt:.2f}s eval(host path) {t_eval:.3f}s analyze {t_an:.2f}s", flush=True)
print("  symbolic:", info, flush=True)
F = ps.factorize(A, S)
print("  status", F.status, F.inertia, flush=True)
b = rng.standard_normal(M.n)
x = np.empty_like(b)
import torch
db = torch.from_numpy(b).cuda()
dx = torch.empty_like(db)
for rep in range(3):
    _lib.lib.ncl_synchronize()
    t = time.perf_counter(); F.refactorize(A); _lib.lib.ncl_synchronize(); tf = time.perf_counter() - t
    t = time.perf_counter(); dx.copy_(db); F.solve_in_place(dx, where=1); _lib.lib.ncl_synchronize(); ts = time.perf_counter() - t
    print(f"  factor {tf*1e3:.3f} ms  solve {ts*1e3:.3f} ms", flush=True)
r = ps.solve_refined(F, A, b)
print("  refined residual", r.residual, r.sweeps, r.converged, flush=True)
if ref:
    from oracle.ref import RefSparseSym, RefFactorization, RefSymbolic
    cp, ri, v = A.col_ptr(), A.row_ind(), A.values()
    rows = ri; cols = np.repeat(np.arange(M.n), np.diff(cp))
    R = RefSparseSym(M.n, rows, cols, v)
    t = time.time(); RS = RefSymbolic(R, S.perm); print(f"  ref analyze(perm) {time.time()-t:.2f}s", flush=True)
    t = time.time(); RF = RefFactorization(R, RS); tf = time.time() - t
    t = time.time(); xr = RF.solve(b); ts = time.time() - t
    print(f"  REF factor {tf*1e3:.1f} ms solve {ts*1e3:.1f} ms inertia {RF.inertia}", flush=True)
    xg = F.solve(b)
    print("  max rel diff x", np.max(np.abs(xg - xr)) / np.max(np.abs(xr)), flush=True)
