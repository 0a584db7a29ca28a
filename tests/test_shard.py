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
