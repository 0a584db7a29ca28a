import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2510_13333_b200 import _lib
_lib.check(_lib.lib.ncl_init(0))
from tests.test_shard import _assembled
from paper_2510_13333_b200 import sparse as ps
from paper_2510_13333_b200.dist import ShardPlan, var_groups, combine_status
s, M, kk, S = _assembled("case118", 8, 5)
A = kk.matrix
F1 = ps.factorize(A, S)
G = 2
Ss = [S, ps.analyze(A, S.perm)]
plans = [ShardPlan(Ss[r], var_groups(s), s.K + 1, G, r) for r in range(G)]
Fs = [ps.factorize(A, Ss[r]) for r in range(G)]
info = plans[0].info()
dev = torch.device("cuda")
sends = [torch.full((info.cb_chunk,), float("nan"), dtype=torch.float64, device=dev) for _ in range(G)]
for r in range(G):
    plans[r].factor_phase_a(Fs[r], A, sends[r])
print("cb send nan per rank", [int(torch.isnan(t).sum()) for t in sends])
recv = torch.cat(sends).contiguous()
ist = [plans[r].factor_phase_b(Fs[r], A, recv) for r in range(G)]
print("istat", ist)
tot = combine_status(ist)
for r in range(G):
    ShardPlan.set_status(Fs[r], tot)
b = np.random.default_rng(6).standard_normal(s.n)
xr = F1.solve(b)
# world-1 split path
P1 = ShardPlan(S, var_groups(s), s.K + 1, 1, 0)
F0 = ps.factorize(A, S)
snd = torch.zeros(max(1, P1.info().cb_chunk), dtype=torch.float64, device=dev)
P1.factor_phase_a(F0, A, snd); P1.factor_phase_b(F0, A, snd)
x0 = torch.from_numpy(b.copy()).to(dev); cv0 = torch.zeros(1, dtype=torch.float64, device=dev)
P1.solve_phase_a(F0, x0, cv0); P1.solve_phase_b(F0, x0, cv0)
print("world1 split equal", np.array_equal(x0.cpu().numpy(), xr))
xs = [torch.from_numpy(b.copy()).to(dev) for _ in range(G)]
cvs = [torch.full((info.cv_chunk,), float("nan"), dtype=torch.float64, device=dev) for _ in range(G)]
for r in range(G):
    plans[r].solve_phase_a(Fs[r], xs[r], cvs[r])
bd = plans[0].boundary()
print("boundary owners", bd.owner.tolist(), "cv_off", bd.cv_off.tolist())
for r in range(G):
    print("rank", r, "cv send", cvs[r].cpu().numpy().round(4).tolist()[:40])
rc = torch.cat(cvs).contiguous()
for r in range(G):
    plans[r].solve_phase_b(Fs[r], xs[r], rc)
    xx = xs[r].cpu().numpy()
    print("rank", r, "nan", int(np.isnan(xx).sum()), "nonzero", int((xx != 0).sum()), "match", int((xx == xr).sum()))
