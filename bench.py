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
    w = bd["x0"]
    rng = np.random.default_rng(SEED)
    lam = 0.1 * rng.standard_normal(M.m)
    hess = M.eval_hessian_lag(w, 1e-4, lam)
    jac = M.eval_jacobian(w)
    # IPM-like diagonal: bound duals 1 / distance to the bounds (zero for free variables)
    xl, xu = bd["xl"], bd["xu"]
    sig = np.zeros(M.n)
    fl, fu = np.isfinite(xl), np.isfinite(xu)
    sig[fl] += 1.0 / np.maximum(w[fl] - xl[fl], 1e-2)
    sig[fu] += 1.0 / np.maximum(xu[fu] - w[fu], 1e-2)
    D = np.full(M.m, 100.0)  # rho = 100
    kk.assemble(hess, jac, sig, 1e-8, D)
    t0 = time.perf_counter()
    S = ps.analyze(kk.matrix)
    t_an = time.perf_counter() - t0
    return dict(scopf=s, model=M, kkt=kk, A=kk.matrix, S=S, t_build=t_build, t_analyze=t_an)


def run_reference(a, world):
    """--impl reference: the reference CPU factorize+solve (oracle/_ref) on the same matrix."""
    from oracle.ref import RefFactorization, RefSparseSym, RefSymbolic

    P = build_problem(a.grid, a.K)
    A, S = P["A"], P["S"]
    n = A.dim()
    cp, ri, v = A.col_ptr(), A.row_ind(), A.values()
    cols = np.repeat(np.arange(n, dtype=np.int32), np.diff(cp))
    R = RefSparseSym(n, ri, cols, v)
    RS = RefSymbolic(R, S.perm)  # perm bit-identical to the reference symbolic_order (tests/test_symbolic.py)
    b = np.random.default_rng(1).standard_normal(n)
    times = []
    for it in range(a.warmup + a.steps):
        t0 = time.perf_counter()
        F = RefFactorization(R, RS)
        F.solve(b)
        dt = time.perf_counter() - t0
        if it >= a.warmup:
            times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    line = {"metric": METRIC, "impl": "reference", "value": ms, "unit": "ms/IPM-iter (KKT factor+solve)",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{a.grid}x{a.K} condensed KKT factor+solve", "N": n, "nnzK": A.nnz()},
            "cpu_baseline": {"value": ms, "unit": "ms/IPM-iter (KKT factor+solve)", "cores": 1,
                             "kind": "reference", "sample": f"{a.steps} factorize+solve of the {a.grid}x{a.K} KKT"},
            "e2e": {"value": ms, "unit": "ms/IPM-iter (KKT factor+solve)", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


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
    for _ in range(2):
        A.set_values(vals_h, where=ps.HOST)
        refactor()
        x_h.copy_(b_h)
        solve(x_h, ps.HOST)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e2e = []
    for _ in range(a.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        A.set_values(vals_h, where=ps.HOST)  # H2D of K's values
        refactor()
        x_h.copy_(b_h)
        solve(x_h, ps.HOST)  # H2D of b, D2H of x (synchronous)
        sp, zp, *_ = F._status()  # D2H of status + inertia
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
    tp = os.path.join(ROOT, "profiles", "factor_traffic.json")
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
        from oracle.ref import RefFactorization, RefSparseSym, RefSymbolic

        cp, ri, v = A.col_ptr(), A.row_ind(), A.values()
        R = RefSparseSym(n, ri, np.repeat(np.arange(n, dtype=np.int32), np.diff(cp)), v)
        RS = RefSymbolic(R, S.perm)
        bb = b_h.numpy().copy()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            RefFactorization(R, RS).solve(bb)
            ts.append(time.perf_counter() - t0)
        cpu = {"value": 1e3 * statistics.median(ts), "unit": "ms/IPM-iter (KKT factor+solve)", "cores": 1,
               "kind": "reference",
               "sample": f"3 reference factorize+solve of the same {a.grid}x{a.K} KKT (median), 1 thread"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": step_ms, "unit": "ms/IPM-iter (KKT factor+solve)", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": step_ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{a.grid}x{a.K} condensed KKT factor+solve (paper layout, seed {SEED})",
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
