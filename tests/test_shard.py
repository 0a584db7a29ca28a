"""Contingency sharding of the multifrontal factorization.

CPU: the per-rank plans partition the work (owned / shared / boundary) and the
boundary exchange (pack -> all-gather -> unpack) moves every block to the
right place — checked with world_size-2 gloo processes on the CPU.
GPU: the sharded factorization (single-GPU emulation of G ranks, and the
world=1 sharded path) is bitwise identical to the unsharded one.
"""
import os

import numpy as np
import pytest

from paper_2510_13333_b200 import sparse as ps
from paper_2510_13333_b200.dist import ShardPlan, var_groups
from paper_2510_13333_b200.kkt import Kkt
from paper_2510_13333_b200.scopf import Scopf


def _problem(grid="case118", K=8):
    s = Scopf(grid, K)
    M = s.build_model()
    kk = Kkt(M)
    S = ps.analyze(kk.matrix)
    return s, M, kk, S


def _cb_layout(S):
    d = ps.supernodes(S)
    w = np.diff(d["first"]).astype(np.int64)
    m2 = np.diff(d["rptr"]) - w
    cb_off = np.concatenate([[0], np.cumsum(m2 * (m2 + 1) // 2)])
    return d, w, m2, cb_off


@pytest.mark.parametrize("G", [1, 2, 3, 4])
def test_plans_partition_the_tree(G):
    s, M, kk, S = _problem()
    g = var_groups(s)
    plans = [ShardPlan(S, g, s.K + 1, G, r) for r in range(G)]
    d, w, m2, _ = _cb_layout(S)
    nsn = len(w)
    owners = [p.owners() for p in plans]
    for o in owners[1:]:
        np.testing.assert_array_equal(o, owners[0])  # every rank derives the same ownership
    own = owners[0]
    assert own.min() >= -1 and own.max() < G
    # a contingency's supernodes all land on the rank of its contingency block
    assert set(np.unique(own[own >= 0]).tolist()) <= set(range(G))
    infos = [p.info() for p in plans]
    assert sum(i.owned_supernodes for i in infos) == int((own >= 0).sum())
    assert all(i.shared_supernodes == int((own < 0).sum()) for i in infos)
    assert len({i.n_phase_b for i in infos}) == 1
    # report columns partition the pivots
    assert sum(i.report_cols for i in infos) == S.n
    # parents of owned supernodes are owned by the same rank or shared
    par = d["parent"]
    for sn in range(nsn):
        if own[sn] >= 0 and par[sn] >= 0:
            assert own[par[sn]] in (own[sn], -1)
    b = plans[0].boundary()
    for p in plans[1:]:
        bb = p.boundary()
        np.testing.assert_array_equal(bb.ids, b.ids)
        np.testing.assert_array_equal(bb.cb_off, b.cb_off)
    if G == 1:
        assert infos[0].n_phase_a + infos[0].n_phase_b == nsn


def _exchange_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s, M, kk, S = _problem()
        g = var_groups(s)
        plan = ShardPlan(S, g, s.K + 1, world, rank)
        info, b = plan.info(), plan.boundary()
        d, w, m2, cb_off = _cb_layout(S)
        own = plan.owners()
        truth = np.zeros(cb_off[-1])
        for sn in range(len(w)):  # the CB every rank would compute, tagged by supernode
            truth[cb_off[sn]:cb_off[sn + 1]] = sn + np.arange(cb_off[sn + 1] - cb_off[sn]) * 1e-6
        local = np.where(np.repeat(own, m2 * (m2 + 1) // 2) == rank, truth, np.nan)  # only my own blocks are valid
        send = np.zeros(info.cb_chunk)
        for sn, o, off in zip(b.ids, b.owner, b.cb_off):
            if o == rank:
                n = m2[sn] * (m2[sn] + 1) // 2
                send[off:off + n] = local[cb_off[sn]:cb_off[sn] + n]
        parts = [torch.zeros(info.cb_chunk, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(send))
        for sn, o, off in zip(b.ids, b.owner, b.cb_off):
            if o != rank:
                n = m2[sn] * (m2[sn] + 1) // 2
                local[cb_off[sn]:cb_off[sn] + n] = parts[o].numpy()[off:off + n]
        ok = all(np.array_equal(local[cb_off[sn]:cb_off[sn + 1]], truth[cb_off[sn]:cb_off[sn + 1]]) for sn in b.ids)
        q.put((rank, ok, int(info.n_boundary), int(info.cb_chunk)))
    finally:
        dist.destroy_process_group()


def test_boundary_exchange_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _ in res), res
    assert res[0][2] == res[1][2] and res[0][2] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("grid,K,G", [("case118", 8, 2), ("case118", 8, 4), ("activsg500", 8, 8)])
def test_emulated_shards_bitwise(gpu, grid, K, G):
    from paper_2510_13333_b200.dist import refactorize_emulated
    s, M, kk, S = _problem(grid, K)
    rng = np.random.default_rng(3)
    n = s.n
    kk.assemble(rng.standard_normal(M.nnzh) * 0.1, rng.standard_normal(M.nnzj), 1.0 + rng.random(n), 0.0,
                10.0 + rng.random(M.m))
    A = kk.matrix
    F1 = ps.factorize(A, S)
    D1, L1 = F1.diagonal(), F1.L_csc()[2]
    F2 = ps.factorize(A, S)
    plans = [ShardPlan(S, var_groups(s), s.K + 1, G, r) for r in range(G)]
    refactorize_emulated(F2, A, plans)
    assert np.array_equal(F2.diagonal(), D1)
    assert np.array_equal(F2.L_csc()[2], L1)
    assert F2.inertia == F1.inertia


@pytest.mark.gpu
def test_world1_shard_path_bitwise(gpu):
    s, M, kk, S = _problem("case118", 8)
    rng = np.random.default_rng(4)
    kk.assemble(rng.standard_normal(M.nnzh) * 0.1, rng.standard_normal(M.nnzj), 1.0 + rng.random(s.n), 0.0,
                10.0 + rng.random(M.m))
    A = kk.matrix
    F1 = ps.factorize(A, S)
    F2 = ps.factorize(A, S)
    plan = ShardPlan(S, var_groups(s), s.K + 1, 1, 0)
    plan.refactorize(F2, A)
    assert np.array_equal(F2.diagonal(), F1.diagonal())
    b = rng.standard_normal(s.n)
    x1 = F1.solve(b)
    x2 = b.copy()
    plan.solve_in_place(F2, x2)
    assert np.array_equal(x1, x2)


def _assembled(grid, K, seed):
    s, M, kk, S = _problem(grid, K)
    rng = np.random.default_rng(seed)
    kk.assemble(rng.standard_normal(M.nnzh) * 0.1, rng.standard_normal(M.nnzj), 1.0 + rng.random(s.n), 0.0,
                10.0 + rng.random(M.m))
    return s, M, kk, S


def _split_phase_world(s, A, S, G, rng):
    """One process drives G ranks through the split-phase API: every rank has
    its own symbolic copy (own completion flags), factor and plan; the
    all-gathers are device copies of the ranks' send chunks, laid out as
    ncclAllGather lays them out. Returns the per-rank D / x and combined istat."""
    import torch
    from paper_2510_13333_b200 import _lib
    from paper_2510_13333_b200.dist import combine_status

    def sync():  # torch's stream <-> the library's stream (ncl_stream)
        torch.cuda.synchronize()
        _lib.check(_lib.lib.ncl_synchronize())

    perm = S.perm
    Ss = [S] + [ps.analyze(A, perm) for _ in range(G - 1)]
    groups = var_groups(s)
    plans = [ShardPlan(Ss[r], groups, s.K + 1, G, r) for r in range(G)]
    Fs = [ps.factorize(A, Ss[r]) for r in range(G)]  # allocation (and a throw-away unsharded factor)
    info = plans[0].info()
    dev = torch.device("cuda")
    sends = [torch.full((max(1, info.cb_chunk),), float("nan"), dtype=torch.float64, device=dev) for _ in range(G)]
    sync()
    for r in range(G):
        plans[r].factor_phase_a(Fs[r], A, sends[r])
    sync()
    recv = torch.cat([t[:info.cb_chunk] for t in sends]).contiguous()
    sync()
    ist = [plans[r].factor_phase_b(Fs[r], A, recv) for r in range(G)]
    tot = combine_status(ist)
    for r in range(G):
        ShardPlan.set_status(Fs[r], tot)
    b = rng.standard_normal(s.n)
    xs = [torch.from_numpy(b.copy()).to(dev) for _ in range(G)]
    cvs = [torch.full((max(1, info.cv_chunk),), float("nan"), dtype=torch.float64, device=dev) for _ in range(G)]
    sync()
    for r in range(G):
        plans[r].solve_phase_a(Fs[r], xs[r], cvs[r])
    sync()
    recv_cv = torch.cat([t[:info.cv_chunk] for t in cvs]).contiguous()
    sync()
    for r in range(G):
        plans[r].solve_phase_b(Fs[r], xs[r], recv_cv)
    sync()
    x = xs[0].clone()
    for r in range(1, G):
        x += xs[r]  # the all-reduce(sum) of ncl_shard_solve: every entry has one non-zero term
    D = [plans[r].diagonal(Fs[r]) for r in range(G)]
    return plans, Fs, D, b, x.cpu().numpy(), tot


@pytest.mark.gpu
@pytest.mark.parametrize("grid,K,G", [("case118", 8, 2), ("activsg500", 16, 4), ("activsg500", 256, 8)])
def test_split_phase_exchange_bitwise(gpu, grid, K, G):
    """pack -> exchange -> unpack through the library (the NCCL all-gather
    replaced by device copies): every rank's reported D, the combined inertia
    and the summed x are bitwise the unsharded factor's / solve's."""
    s, M, kk, S = _assembled(grid, K, 5)
    A = kk.matrix
    F1 = ps.factorize(A, S)
    D1 = F1.diagonal()
    rng = np.random.default_rng(6)
    plans, Fs, D, b, x, tot = _split_phase_world(s, A, S, G, rng)
    got = np.full(s.n, np.nan)
    for r in range(G):
        m = ~np.isnan(D[r])
        assert not np.any(~np.isnan(got[m])), "a pivot reported by two ranks"
        got[m] = D[r][m]
    assert np.array_equal(got, D1)
    assert all(F.status == "ok" for F in Fs)
    assert Fs[0].inertia == F1.inertia
    assert np.array_equal(x, F1.solve(b))
    # the whole-factor getters refuse a sharded factor
    from paper_2510_13333_b200._lib import NclError
    with pytest.raises(NclError):
        Fs[1].diagonal()
    with pytest.raises(NclError):
        Fs[1].solve(b)


@pytest.mark.gpu
def test_split_phase_exchange_500x1024_g8(gpu):
    """BASELINE configs[4]: the 500-bus x 1024-contingency KKT split 8 ways
    (128 contingencies per rank), bitwise against the unsharded factor."""
    s, M, kk, S = _assembled("activsg500", 1024, 7)
    A = kk.matrix
    F1 = ps.factorize(A, S)
    D1 = F1.diagonal()
    plans, Fs, D, b, x, tot = _split_phase_world(s, A, S, 8, np.random.default_rng(8))
    got = np.where(np.isnan(D[0]), 0.0, D[0])
    for r in range(1, 8):
        got = np.where(np.isnan(D[r]), got, D[r])
    assert np.array_equal(got, D1)
    assert Fs[0].inertia == F1.inertia
    assert np.array_equal(x, F1.solve(b))


def _two_process_worker(rank, world, port, q):
    """one rank of a world-2 run on ONE GPU: the library's pack / unpack with a
    host-staged gloo all-gather as the transport (NCCL refuses two ranks on one
    device), then the gloo reductions of istat and x."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_13333_b200 import _lib
        _lib.check(_lib.lib.ncl_init(0))
        s, M, kk, S = _assembled("case118", 8, 9)
        A = kk.matrix
        F1 = ps.factorize(A, S)
        F = ps.factorize(A, ps.analyze(A, S.perm))
        plan = ShardPlan(F._symb, var_groups(s), s.K + 1, world, rank)
        info = plan.info()
        send = np.zeros(info.cb_chunk)
        plan.factor_phase_a(F, A, send)
        parts = [torch.zeros(info.cb_chunk, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(send))
        ist = plan.factor_phase_b(F, A, torch.cat(parts).numpy())
        t = torch.from_numpy(ist.astype(np.int64))
        zp = t[:1].clone()
        dist.all_reduce(zp, op=dist.ReduceOp.MIN)
        cnt = t[1:].clone()
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
        ShardPlan.set_status(F, np.concatenate([zp.numpy(), cnt.numpy()]))
        D = plan.diagonal(F)
        m = ~np.isnan(D)
        okD = bool(np.array_equal(D[m], F1.diagonal()[m]))
        b = np.random.default_rng(10).standard_normal(s.n)
        x = b.copy()
        cv = np.zeros(info.cv_chunk)
        plan.solve_phase_a(F, x, cv)
        parts = [torch.zeros(info.cv_chunk, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(cv))
        plan.solve_phase_b(F, x, torch.cat(parts).numpy())
        xt = torch.from_numpy(x)
        dist.all_reduce(xt, op=dist.ReduceOp.SUM)
        okx = bool(np.array_equal(xt.numpy(), F1.solve(b)))
        q.put((rank, okD, okx, F.inertia == F1.inertia, int(m.sum()), int(info.n_boundary)))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_split_phase_two_processes_one_gpu(gpu):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_two_process_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(len(r) == 6 for r in res), res
    assert all(r[1] and r[2] and r[3] for r in res), res
    s, M, kk, S = _problem("case118", 8)
    assert res[0][4] + res[1][4] == s.n  # the ranks' reported pivots partition the columns
    assert res[0][5] > 0
