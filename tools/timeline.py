"""Per-phase / per-height timeline of one traced factorization.

    NCL_TASK_TRACE=gpurun_out/trace.bin python bench.py --steps 2 --warmup 1 --no-solve --no-cpu-baseline
    python tools/timeline.py gpurun_out/trace.bin [grid K]

The trace (capi.cpp run_factor) holds per-task globaltimer start/end, the task
layout (tptr, nodes); heights/parents come from re-running the symbolic
analysis of the same KKT here (deterministic)."""
import sys

import numpy as np

sys.path.insert(0, ".")


def main():
    path = sys.argv[1]
    grid = sys.argv[2] if len(sys.argv) > 2 else "activsg500"
    K = int(sys.argv[3]) if len(sys.argv) > 3 else 256
    raw = open(path, "rb").read()
    ntask, nleaf, split, _ = np.frombuffer(raw[:16], np.int32)
    o = 16
    tr = np.frombuffer(raw[o:o + 16 * ntask], np.uint64).reshape(ntask, 2).astype(np.int64)
    o += 16 * ntask
    tptr = np.frombuffer(raw[o:o + 4 * (ntask + 1)], np.int32)
    o += 4 * (ntask + 1)
    nodes = np.frombuffer(raw[o:], np.int32)
    from paper_2510_13333_b200 import sparse as ps
    from paper_2510_13333_b200.kkt import Kkt
    from paper_2510_13333_b200.scopf import Scopf
    sc = Scopf(grid, K, seed=2510)
    S = ps.analyze(Kkt(sc.build_model()).matrix)
    d = ps.supernodes(S)
    h, par = d["height"], d["parent"]
    w = np.diff(d["first"])
    nr = np.diff(d["rptr"])
    valid = tr[:, 0] > 0
    t0 = tr[valid, 0].min()
    st, en = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3  # us
    st[~valid] = np.nan  # tasks run outside the persistent kernels (large fronts) carry no stamps
    en[~valid] = np.nan
    task_of = np.full(len(par), -1, np.int64)
    for t in range(ntask):
        task_of[nodes[tptr[t]:tptr[t + 1]]] = t
    # ready time of a task: max end over the tasks of its nodes' children
    ready = np.zeros(ntask)
    for s_ in range(len(par)):
        p = par[s_]
        if p >= 0 and task_of[p] != task_of[s_] and task_of[p] >= 0 and task_of[s_] >= 0:
            tp = task_of[p]
            ready[tp] = max(ready[tp], en[task_of[s_]])
    print(f"tasks {ntask} (groups {nleaf}, singles {split - nleaf}, cta {ntask - split}); end {en[valid].max():.1f} us")
    for name, a, b in (("groups", 0, nleaf), ("singles", nleaf, split), ("cta", split, ntask)):
        if b <= a:
            continue
        sl = slice(a, b)
        print(f"{name:8s} start {np.nanmin(st[sl]):8.1f} end {np.nanmax(en[sl]):8.1f} "
              f"mean dur {np.nanmean(en[sl] - st[sl]):7.2f} mean wait {np.nanmean(np.maximum(0, st[sl] - ready[sl])):7.2f}")
    print("cta part by height of the task's last node: n, start, end, mean dur, p90 dur, mean nr, mean w, mean start-ready")
    hl = np.array([h[nodes[tptr[t + 1] - 1]] for t in range(split, ntask)])
    lastn = np.array([nodes[tptr[t + 1] - 1] for t in range(split, ntask)])
    for lv in np.unique(hl):
        m = hl == lv
        idx = np.arange(split, ntask)[m]
        if not valid[idx].any():
            print(f"  h={lv:2d} {m.sum():5d} (large-front path, not stamped)")
            continue
        m = m & valid[split:]
        idx = np.arange(split, ntask)[m]
        du = en[idx] - st[idx]
        print(f"  h={lv:2d} {m.sum():5d} {st[idx].min():8.1f} {en[idx].max():8.1f} {du.mean():7.2f} "
              f"{np.percentile(du, 90):7.2f} {nr[lastn[m]].mean():6.1f} {w[lastn[m]].mean():5.1f} "
              f"{np.mean(st[idx] - ready[idx]):7.2f}")


if __name__ == "__main__":
    main()


def singles_by_size(path, grid="activsg500", K=256):
    """Singles (warp tasks outside groups): count and mean duration by nr range."""
    raw = open(path, "rb").read()
    ntask, nleaf, split, _ = np.frombuffer(raw[:16], np.int32)
    o = 16
    tr = np.frombuffer(raw[o:o + 16 * ntask], np.uint64).reshape(ntask, 2).astype(np.int64)
    o += 16 * ntask
    tptr = np.frombuffer(raw[o:o + 4 * (ntask + 1)], np.int32)
    o += 4 * (ntask + 1)
    nodes = np.frombuffer(raw[o:], np.int32)
    from paper_2510_13333_b200 import sparse as ps
    from paper_2510_13333_b200.kkt import Kkt
    from paper_2510_13333_b200.scopf import Scopf
    S = ps.analyze(Kkt(Scopf(grid, K, seed=2510).build_model()).matrix)
    d = ps.supernodes(S)
    nr = np.diff(d["rptr"])
    w = np.diff(d["first"])
    du = (tr[:, 1] - tr[:, 0]) / 1e3
    idx = np.arange(nleaf, split)
    nn = np.array([nr[nodes[tptr[t]]] for t in idx])
    ww = np.array([w[nodes[tptr[t]]] for t in idx])
    for lo, hi in ((0, 16), (16, 32), (32, 48), (48, 64), (64, 100), (100, 200)):
        m = (nn > lo) & (nn <= hi)
        if m.any():
            print(f"  nr in ({lo},{hi}]: {m.sum():6d} singles, mean w {ww[m].mean():5.1f}, mean dur {du[idx[m]].mean():6.2f} us, "
                  f"sum {du[idx[m]].sum() / 1e3:8.1f} ms-warp")


def solve_timeline(solve_path, factor_path, grid="activsg500", K=256):
    """Forward/backward solve phases from NCL_SOLVE_TRACE (task layout from the factor trace)."""
    raw = open(factor_path, "rb").read()
    ntask, nleaf, split, _ = np.frombuffer(raw[:16], np.int32)
    o = 16 + 16 * ntask
    tptr = np.frombuffer(raw[o:o + 4 * (ntask + 1)], np.int32)
    o += 4 * (ntask + 1)
    nodes = np.frombuffer(raw[o:], np.int32)
    sr = open(solve_path, "rb").read()
    n2 = np.frombuffer(sr[:16], np.int32)[0]
    assert n2 == ntask
    tr = np.frombuffer(sr[16:], np.uint64).reshape(2, ntask, 2).astype(np.int64)
    from paper_2510_13333_b200 import sparse as ps
    from paper_2510_13333_b200.kkt import Kkt
    from paper_2510_13333_b200.scopf import Scopf
    S = ps.analyze(Kkt(Scopf(grid, K, seed=2510).build_model()).matrix)
    h = ps.supernodes(S)["height"]
    t0 = tr[0][tr[0][:, 0] > 0, 0].min()
    for name, T in (("forward", tr[0]), ("backward", tr[1])):
        st, en = (T[:, 0] - t0) / 1e3, (T[:, 1] - t0) / 1e3
        print(f"{name}: start {st[T[:, 0] > 0].min():.1f} end {en[T[:, 0] > 0].max():.1f} us")
        for pn, a, b in (("groups", 0, nleaf), ("singles", nleaf, split), ("cta", split, ntask)):
            sl = slice(a, b)
            print(f"  {pn:8s} start {st[sl].min():8.1f} end {en[sl].max():8.1f} mean dur {np.mean(en[sl] - st[sl]):7.2f}")
        hl = np.array([h[nodes[tptr[t + 1] - 1]] for t in range(split, ntask)])
        for lv in np.unique(hl):
            idx = np.arange(split, ntask)[hl == lv]
            print(f"    h={lv:2d} {len(idx):5d} {st[idx].min():8.1f} {en[idx].max():8.1f} dur {np.mean(en[idx] - st[idx]):7.2f}")


def cta_phases(path, grid="activsg500", K=256):
    """CTA-path phase split per height: claim->after wait, assembly, dense+writeout, fence+publish (us)."""
    raw = open(path, "rb").read()
    ntask, nleaf, split, _ = np.frombuffer(raw[:16], np.int32)
    o = 16
    tr = np.frombuffer(raw[o:o + 16 * ntask], np.uint64).reshape(ntask, 2).astype(np.int64)
    o += 16 * ntask
    tptr = np.frombuffer(raw[o:o + 4 * (ntask + 1)], np.int32)
    o += 4 * (ntask + 1)
    nodes = np.frombuffer(raw[o:], np.int32)
    ph = np.fromfile(path + ".phase", np.uint64).reshape(-1, 4).astype(np.int64)
    from paper_2510_13333_b200 import sparse as ps
    from paper_2510_13333_b200.kkt import Kkt
    from paper_2510_13333_b200.scopf import Scopf
    S = ps.analyze(Kkt(Scopf(grid, K, seed=2510).build_model()).matrix)
    h = ps.supernodes(S)["height"]
    rows = []
    for t in range(split, ntask):
        s = nodes[tptr[t]]
        if ph[s, 0] == 0:
            continue
        rows.append((h[s], (ph[s, 0] - tr[t, 0]) / 1e3, (ph[s, 1] - ph[s, 0]) / 1e3, (ph[s, 2] - ph[s, 1]) / 1e3,
                     (ph[s, 3] - ph[s, 2]) / 1e3))
    rows = np.array(rows)
    print("height  n   wait   assembly   dense+writeout   publish  (mean us)")
    for lv in np.unique(rows[:, 0]):
        m = rows[:, 0] == lv
        print(f"  h={int(lv):2d} {m.sum():5d} {rows[m, 1].mean():7.2f} {rows[m, 2].mean():9.2f} {rows[m, 3].mean():12.2f} "
              f"{rows[m, 4].mean():9.2f}")
