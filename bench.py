"""bench.py — KKT factor+solve per IPM iteration (and, when the IPM runs,
SCOPF time-to-solve) on the ACTIVSg500-size x 256-contingency SCOPF.

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
One JSON line from rank 0. A "step" = one KKT numeric factorization + one
triangular solve (the per-IPM-iteration linear-algebra hot path) of the
condensed Newton matrix of the synthetic 500-bus x 256-contingency SCOPF
(paper layout, seed 2510), inputs resident in HBM; L2 is flushed (256 MiB
write) between timed steps. `e2e` is the same step through the C-ABI with
HOST buffers (H2D of K's values and the RHS, D2H of the solution inside the
timed region). `--impl reference` times the reference's own CPU
factorize + solve (oracle/_ref, compiled from /root/reference/proj/src) on
the same matrix — rank 0 only.

Multi-GPU (torchrun, one rank per GPU): the same KKT is factored and solved
contingency-sharded (include/nclopf_dist.h): each rank factors its block of
contingency subtrees, the subtree-root contribution blocks are all-gathered
over NVLink by the library's NCCL communicator, the separator is factored
redundantly ("scaling": "strong", time = max over ranks). The end-to-end NCL
solve (time_to_solve) runs on rank 0 only; the IPM itself is not sharded.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GRID, K_CONT, SEED = "activsg500", 256, 2510
METRIC = "SCOPF time-to-solve (s) + KKT factor+solve ms/IPM iter, 500-bus x 256 contingencies"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--grid", default=GRID)
    ap.add_argument("--K", type=int, default=K_CONT)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-solve", action="store_true", help="skip the end-to-end NCL solve (time to solve)")
    return ap.parse_args()


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for k, nm in enumerate(names):
                    if r[3 + k].lower().startswith("active"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _berr(R, x, b):
    """normwise backward error ||Kx - b||_inf / (||K||_inf ||x||_inf + ||b||_inf)
    with the reference's own SpMV and norm"""
    r = R.multiply(x) - b
    return float(np.max(np.abs(r)) / (R.norm_inf() * np.max(np.abs(x)) + np.max(np.abs(b))))


def workload(grid, K):
    """One workload string for both arms (same_config)."""
    return f"{grid}x{K} condensed KKT factor+solve (paper layout, seed {SEED})"


def ipm_point(bd, m, seed=SEED):
    """The IPM-like point the bench KKT is formed at (both arms): w = x0,
    lambda ~ 0.1 N(0, 1), bound duals 1 / distance to the bounds (zero for
    free variables), D = rho = 100 on every row."""
    w = bd["x0"]
    rng = np.random.default_rng(seed)
    lam = 0.1 * rng.standard_normal(m)
    xl, xu = bd["xl"], bd["xu"]
    sig = np.zeros(len(w))
    fl, fu = np.isfinite(xl), np.isfinite(xu)
    sig[fl] += 1.0 / np.maximum(w[fl] - xl[fl], 1e-2)
    sig[fu] += 1.0 / np.maximum(xu[fu] - w[fu], 1e-2)
    return w, lam, sig, np.full(m, 100.0)


def build_problem(grid, K):
    """Synthetic SCOPF -> model -> condensed KKT at an IPM-like point."""
    from paper_2510_13333_b200 import sparse as ps
    from paper_2510_13333_b200.kkt import Kkt
    from paper_2510_13333_b200.scopf import Scopf

    t0 = time.perf_counter()
    s = Scopf(grid, K, seed=SEED)
    M = s.build_model()
    kk = Kkt(M)
    t_build = time.perf_counter() - t0
    bd = s.bounds()
    w, lam, sig, D = ipm_point(bd, M.m)
    hess = M.eval_hessian_lag(w, 1e-4, lam)
    jac = M.eval_jacobian(w)
    kk.assemble(hess, jac, sig, 1e-8, D)
    t0 = time.perf_counter()
    S = ps.analyze(kk.matrix)
    t_an = time.perf_counter() - t0
    return dict(scopf=s, model=M, kkt=kk, A=kk.matrix, S=S, t_build=t_build, t_analyze=t_an)


def run_reference(a, world):
    """--impl reference: the reference's own CPU factorize + solve
    (oracle/_ref: /root/reference/proj/src compiled unmodified) on the same
    workload, built WITHOUT the product library: the instance generator
    compiled into the oracle, the reference ModelBuilder for H and J, the
    reference SparseSym for K, the reference symbolic_order + analyze for the
    ordering (untimed), then `steps` timed factorize + solve."""
    import json as _json

    from oracle.ref import RefFactorization, RefScopf, RefSymbolic, ref_condensed_kkt, ref_symbolic_order

    kind, nb, nl, ng = _grid_dims(a.grid)
    t0 = time.perf_counter()
    rs = RefScopf(kind, nb, nl, ng, SEED, a.K, _contingency_ids(a.grid, a.K))
    R = rs.model()
    w, lam, sig, D = ipm_point(rs.bounds(), R.m)
    K = ref_condensed_kkt(R, R.eval_hessian_lag(w, 1e-4, lam), R.eval_jacobian(w), sig, 1e-8, D)
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    perm = ref_symbolic_order(K)
    RS = RefSymbolic(K, perm)
    t_order = time.perf_counter() - t0
    n = K.n
    b = np.random.default_rng(1).standard_normal(n)
    times = []
    for it in range(a.warmup + a.steps):
        t0 = time.perf_counter()
        F = RefFactorization(K, RS)
        F.solve(b)
        dt = time.perf_counter() - t0
        if it >= a.warmup:
            times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    unit = "ms/IPM-iter (KKT factor+solve)"
    with open("/proc/self/maps") as f:
        maps = f.read()
    assert "libnclopf_b200" not in maps, "the reference arm must not load the product library"
    line = {"metric": METRIC, "impl": "reference", "value": ms, "unit": unit,
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(a.grid, a.K), "N": n, "nnzK": K.nnz(), "l_nnz": int(RS.l_nnz),
                       "status": F.status, "inertia": list(F.inertia),
                       "setup_s": {"build": t_build, "symbolic_order+analyze": t_order}},
            "cpu_baseline": {"value": ms, "unit": unit, "cores": 1, "kind": "reference", "cpu": _cpu_model(),
                             "sample": f"{a.steps} reference factorize+solve of the {a.grid}x{a.K} KKT "
                                       "(model, K and ordering built by the reference code; 1 thread: "
                                       "the reference has no threads)"},
            "e2e": {"value": ms, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(_json.dumps(line), flush=True)


def _grid_dims(grid):
    # GRIDS of paper_2510_13333_b200/scopf.py, restated so the reference arm
    # never imports the product package (which loads libnclopf_b200.so)
    return {"case9": (0, 9, 9, 3), "case118": (1, 118, 186, 54), "activsg500": (1, 500, 597, 56),
            "activsg2000": (1, 2000, 3206, 432)}[grid]


def _contingency_ids(grid, K):
    """paper_2510_13333_b200.scopf.contingency_ids without importing the
    package: screened outages, then the same outages at load levels 1..3."""
    p = os.path.join(ROOT, "paper_2510_13333_b200", "data", f"screened_{grid}_{SEED}.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        base = json.load(f)["feasible"]
    nl = _grid_dims(grid)[2]
    ids = [l + nl * j for j in range(4) for l in base]
    if len(ids) < K:
        raise ValueError(f"only {len(ids)} contingencies for {grid}")
    return ids[:K]


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical CPUs)"
    except OSError:
        pass
    return None


def main():
    a = _args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if a.impl == "reference":
        if rank == 0:
            run_reference(a, world)
        return

    import torch

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2510_13333_b200 import _lib
    from paper_2510_13333_b200 import sparse as ps

    _lib.check(_lib.lib.ncl_init(local))
    P = build_problem(a.grid, a.K)
    A, S = P["A"], P["S"]
    info = S.info()
    n, nnzk = A.dim(), A.nnz()
    F = ps.factorize(A, S)
    st = F._status()
    stream = torch.cuda.ExternalStream(_lib.lib.ncl_stream())
    dev = torch.device("cuda", local)
    b_h = torch.from_numpy(np.random.default_rng(1).standard_normal(n)).pin_memory()
    b_d = b_h.to(dev)
    x_d = torch.empty_like(b_d)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2

    plan = None
    if world > 1:
        # contingency-sharded factor/solve over the library's NCCL communicator
        from paper_2510_13333_b200.dist import ShardPlan, init_nccl, var_groups
        init_nccl(world, rank, dist)
        plan = ShardPlan(S, var_groups(P["scopf"]), a.K + 1, world, rank)

    def refactor():
        if plan is not None:
            plan.refactorize(F, A)
        else:
            F.refactorize(A)

    def solve(x, where):
        if plan is not None:
            plan.solve_in_place(F, x, where)
        else:
            F.solve_in_place(x, where=where)

    def step_device():
        refactor()
        with torch.cuda.stream(stream):
            x_d.copy_(b_d)
        solve(x_d, ps.DEVICE)

    torch.cuda.synchronize()
    for _ in range(a.warmup):
        step_device()
    torch.cuda.synchronize()

    # ---- device-resident timed region: per-step CUDA events on the library stream
    launches0 = _lib.lib.ncl_kernel_launches()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for e0, e1, e2 in ev:
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
                e0.record(stream)
            refactor()
            with torch.cuda.stream(stream):
                e1.record(stream)
                x_d.copy_(b_d)
            solve(x_d, ps.DEVICE)
            with torch.cuda.stream(stream):
                e2.record(stream)
        torch.cuda.synchronize()
    launches = _lib.lib.ncl_kernel_launches() - launches0
    fact_ms = [e0.elapsed_time(e1) for e0, e1, _ in ev]
    solve_ms = [e1.elapsed_time(e2) for _, e1, e2 in ev]
    step_ms = sum(f + s for f, s in zip(fact_ms, solve_ms)) / a.steps
    if dist:
        t = torch.tensor([step_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms = float(t.item())

    # ---- e2e through the C-ABI with host buffers
    vals_h = torch.from_numpy(A.values()).pin_memory()
    x_h = torch.empty(n, dtype=torch.float64).pin_memory()
    def e2e_step():
        if plan is None:
            # one C-ABI call: H2D of K's values and of b (the latter under the
            # factorization), factor, solve, D2H of x and of the status words
            F.factor_solve_host(A, vals_h, b_h, x_h)
        else:
            A.set_values(vals_h, where=ps.HOST)  # H2D of K's values
            refactor()
            x_h.copy_(b_h)
            solve(x_h, ps.HOST)  # H2D of b, D2H of x (synchronous)
            F._status()  # D2H of status + inertia

    for _ in range(max(2, a.warmup)):  # the same calls as the timed steps
        e2e_step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e2e = []
    for _ in range(a.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()
        e2e.append(time.perf_counter() - t0)
    e2e_ms = 1e3 * sum(e2e) / len(e2e)
    if dist:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # ---- roofline of the dominant kernel (the numeric factorization)
    peak, peak_src = _peaks()
    fact_avg_s = 1e-3 * sum(fact_ms) / len(fact_ms)
    B_fact = 8 * nnzk + 12 * info.l_nnz + 8 * n
    achieved = B_fact / fact_avg_s / 1e9
    prof_traffic = None
    # ncu DRAM bytes of one refactorization of THIS configuration
    # (tools/factor_traffic.py); null when that configuration was not captured
    tp = os.path.join(ROOT, "profiles", f"factor_traffic_{a.grid}x{a.K}.json")
    if os.path.exists(tp):
        with open(tp) as f:
            prof_traffic = json.load(f).get("bytes_per_launch")

    # ---- time to solve: the whole NCL/IPM solve of the same SCOPF on this GPU
    tts = None
    if not a.no_solve and rank == 0:
        from paper_2510_13333_b200.ipm import NclSolver, default_options

        del F  # free the bench factor before the solver allocates its own
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        sol = NclSolver(P["model"], P["scopf"].bounds())
        out = sol.solve(default_options(verbose=0))
        t_solve = time.perf_counter() - t0
        r = out.result
        its = max(1, r["inner_iters"])
        tts = {"seconds": t_solve, "gpus": 1, "status": out.status, "outer_iters": r["outer_iters"],
               "inner_iters": r["inner_iters"], "factorizations": r["factorizations"],
               "objective": r["objective"], "r_inf": r["r_inf"], "inf_pr": r["inf_pr"], "inf_du": r["inf_du"],
               "analyze_s": r["t_init"],
               "kkt_factor_solve_ms_per_iter": 1e3 * (r["t_factor"] + r["t_solve"]) / its,
               "split_s": {k: r[k] for k in ("t_init", "t_eval", "t_factor", "t_solve", "t_linesearch", "t_other")},
               "paper_gpu_s": 170.75, "paper_ref": "PAPER.md:611 (A30 + cuDSS, real ACTIVSg500)"}
        del sol

    cpu = None
    if rank == 0 and not a.no_cpu_baseline and os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libnclopf_ref.so")):
        # the reference factorize + solve of the SAME matrix (this arm's K
        # values, this arm's permutation — bit-identical to the reference
        # symbolic_order, tests/test_symbolic.py), timed, and used as the
        # parity check of the bench step itself: D (pivot order), inertia,
        # status and x of the GPU factor + solve against the reference's
        from oracle.ref import RefFactorization, RefSparseSym, RefSymbolic

        cp, ri, v = A.col_ptr(), A.row_ind(), A.values()
        R = RefSparseSym(n, ri, np.repeat(np.arange(n, dtype=np.int32), np.diff(cp)), v)
        RS = RefSymbolic(R, S.perm)
        bb = b_h.numpy().copy()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            G = RefFactorization(R, RS)
            xr = G.solve(bb)
            ts.append(time.perf_counter() - t0)
        Fp = ps.factorize(A, S)
        dg, dr = Fp.diagonal(), G.diagonal()
        xg = Fp.solve(bb)
        ia = Fp.inertia
        parity = {"status_equal": Fp.status == G.status, "inertia_equal": (ia.n_pos, ia.n_neg, ia.n_zero) == G.inertia,
                  # componentwise D error is large only at pivots that are
                  # small after cancellation (K is indefinite at this point);
                  # the normwise errors and the backward errors of both
                  # solutions say whether the two factorizations are equally
                  # accurate
                  "D_max_rel": float(np.max(np.abs(dg - dr) / np.maximum(np.abs(dr), 1e-300))),
                  "D_rel_p99": float(np.quantile(np.abs(dg - dr) / np.maximum(np.abs(dr), 1e-300), 0.99)),
                  "D_norm_rel": float(np.max(np.abs(dg - dr)) / max(1e-300, float(np.max(np.abs(dr))))),
                  "x_max_rel": float(np.max(np.abs(xg - xr)) / max(1e-300, float(np.max(np.abs(xr))))),
                  "berr_gpu": _berr(R, xg, bb), "berr_ref": _berr(R, xr, bb),
                  "perm_equal": bool(np.array_equal(RS.perm, S.perm)),
                  "l_nnz_equal": int(RS.l_nnz) == int(info.l_nnz)}
        del Fp
        cpu = {"value": 1e3 * statistics.median(ts), "unit": "ms/IPM-iter (KKT factor+solve)", "cores": 1,
               "kind": "reference", "cpu": _cpu_model(),
               "sample": f"3 reference factorize+solve of the same {a.grid}x{a.K} KKT (median), 1 thread",
               "parity_vs_gpu": parity}

    if rank == 0:
        line = {
            "metric": METRIC, "value": step_ms, "unit": "ms/IPM-iter (KKT factor+solve)", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": step_ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(a.grid, a.K),
                       "N": n, "nnzK": nnzk, "l_nnz": info.l_nnz, "supernodes": info.nsupernodes,
                       "sn_height": info.max_height, "flops": info.flops, "l2": "flushed (256 MiB write) between steps",
                       "parallelism": f"contingency-sharded x{world} (NCCL all-gather of subtree-root CBs)"
                       if world > 1 else "single",
                       "factor_ms": sum(fact_ms) / a.steps, "solve_ms": sum(solve_ms) / a.steps,
                       "status": "ok" if st[0] == 0 else "zero_pivot",
                       "inertia": [st[2].n_pos, st[2].n_neg, st[2].n_zero],
                       "setup_s": {"build": P["t_build"], "analyze": P["t_analyze"]}},
            "clocks": clk.summary(),
            "e2e": {"value": e2e_ms, "unit": "ms/IPM-iter (KKT factor+solve)",
                    "h2d_bytes_per_step": 8 * nnzk + 8 * n, "d2h_bytes_per_step": 8 * n + 20},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": prof_traffic, "peak_source": peak_src,
                         "kernel": "factor (supernodal LDL^T, maxdiag+thresh+factor_kernel)",
                         "algorithmic_bytes": B_fact},
            "cpu_baseline": cpu,
            "time_to_solve": tts,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
