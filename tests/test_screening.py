"""Contingency screening (Eq. 5): the Eq. 5
builder's structure, select_representative's rules (the SPEC examples), and
on the GPU the batched screen (every contingency's system a block of one
NCL solve) against one-by-one solves and against the CPU oracle solving the
same systems, plus determinism."""
import numpy as np
import pytest

from paper_2510_13333_b200 import screening as scr
from paper_2510_13333_b200.scopf import Scopf


def rep(*objs, structural=()):
    r = scr.ScreeningReport()
    for i, o in enumerate(objs):
        r.records.append(scr.Record(i, "x", o, 1, i in structural))
    return r


def test_select_representative_spec_examples():
    # all feasible, K=2 -> top-2 by objective
    assert scr.select_representative(rep(1e-9, 5e-3, 1e-4, 2e-3), 2) == [1, 3]
    # an islanding contingency is excluded regardless of rank
    assert scr.select_representative(rep(1e-9, 5e-3, 1e-4, 2e-3, structural=(1,)), 2) == [3, 2]
    # objective above the hard cap is structural too
    assert 1 not in scr.select_representative(rep(1e-9, 0.5, 1e-4), 2)
    # K = feasible count -> all of them, hardest first
    assert scr.select_representative(rep(3e-3, 1e-9, 2e-3), 3) == [0, 2, 1]
    with pytest.raises(scr.NotEnoughFeasible):
        scr.select_representative(rep(1e-9, 0.5), 2)
    assert rep(1e-9, 5e-3, 1e-4).ranking == [1, 2, 0]


def test_screening_system_structure():
    """K equal, separable blocks; no objective; base set points as row constants"""
    base = Scopf("case118", 0)
    nb, ng = base.info.nb, base.info.ng
    pg0, v0 = np.linspace(0.2, 0.8, ng), np.full(nb, 1.01)
    ids = [int(i) for i in base.candidates()[:3]]
    s = Scopf.screening(base, pg0, v0, ids)
    K = 3
    assert s.K == K and s.n % K == 0 and s.m % K == 0
    nvb, mb = s.n // K, s.m // K
    assert nvb == base.n + 1 + 4 * ng  # one contingency scenario + recourse (paper layout)
    for f in s.families():
        assert not f.objective or len(f.vars) == 0, f.name  # no objective instances
        if f.objective or len(f.rows) == 0:
            continue
        blk_r = f.rows // mb
        blk_v = f.vars.reshape(len(f.rows), -1) // nvb
        assert np.all(blk_v == blk_r[:, None]), f.name  # a row only touches its own block's variables
    bd = s.bounds()
    fam = {f.name: f for f in s.families()}
    agc = fam["agc_droop_fixed_base"]
    np.testing.assert_array_equal(bd["gl"][agc.rows[:ng]], -pg0)  # -p0 on the droop rows
    np.testing.assert_array_equal(bd["gu"][agc.rows[:ng]], -pg0)


@pytest.mark.gpu
def test_batched_screen_matches_one_by_one_and_is_deterministic(gpu):
    base = Scopf("case118", 0)
    pg0, v0, out = scr.base_set_points(base)
    assert out.status == "optimal"
    ids = [int(i) for i in base.candidates()[:12]]
    obj, status, iters = scr.solve_batch(base, pg0, v0, ids)
    obj2, _, _ = scr.solve_batch(base, pg0, v0, ids)
    assert np.array_equal(obj, obj2)  # determinism
    one = np.array([scr.solve_batch(base, pg0, v0, [i])[0][0] for i in ids])
    feas = one <= scr.FEAS_TOL
    assert np.array_equal(obj <= scr.FEAS_TOL, feas)  # same feasible / infeasible split
    inf = ~feas
    if inf.any():  # the least-squares measure of infeasible blocks, independent of the batch
        np.testing.assert_allclose(obj[inf], one[inf], rtol=1e-3)
    print("screen case118", dict(zip(ids, obj.tolist())), status, iters)


@pytest.mark.gpu
def test_screen_against_cpu_oracle(gpu):
    """the same Eq. 5 systems through the CPU oracle (reference model_ad +
    sparse_core under the shared NCL/IPM control flow)"""
    from oracle.ref import RefModel, ref_ncl_solve
    base = Scopf("case118", 0)
    pg0, v0, _ = scr.base_set_points(base)
    ids = [int(i) for i in base.candidates()[:4]]
    obj, status, _ = scr.solve_batch(base, pg0, v0, ids)
    s = Scopf.screening(base, pg0, v0, ids)
    ref = ref_ncl_solve(RefModel.from_families(s.n, s.m, s.families()), s.bounds())
    r = ref["r"].reshape(len(ids), -1)
    robj = np.sum(r * r, axis=1)
    assert ref["status"] == status
    np.testing.assert_allclose(obj, robj, rtol=1e-4, atol=1e-10)


@pytest.mark.gpu
def test_zero_load_network_is_feasible_under_every_outage(gpu):
    """zero-load network -> every objective <= 1e-10"""
    from paper_2510_13333_b200 import matpower as mp
    txt = open(mp.DATA + "/case9.m").read()
    for a, b in (("90\t30", "0\t0"), ("100\t35", "0\t0"), ("125\t50", "0\t0"), ("\t10;", "\t0;")):
        txt = txt.replace(a, b)  # no load, and no minimum generation (all-zero injections are feasible)
    net = mp.PowerNetwork(txt)
    base = Scopf(network=net, K=0)
    pg0, v0, out = scr.base_set_points(base)
    ids = [int(i) for i in base.candidates()]
    obj, status, _ = scr.solve_batch(base, pg0, v0, ids)
    assert np.all(obj <= 1e-10), obj
