"""matpower_io: the parser, per-unit conversion, branch
admittances, round trip, validation errors — the SPEC's examples — and the
SCOPF of a parsed case equal to the built-in one."""
import numpy as np
import pytest

from paper_2510_13333_b200 import matpower as mp
from paper_2510_13333_b200._lib import InvalidArgument
from paper_2510_13333_b200.scopf import Scopf


def case(bus, gen, branch, gencost=None, base=100):
    rows = lambda M: "\n".join("\t" + "\t".join(str(v) for v in r) + ";" for r in M)  # noqa: E731
    t = f"function mpc = t\nmpc.version = '2';\nmpc.baseMVA = {base};\nmpc.bus = [\n{rows(bus)}\n];\n"
    t += f"mpc.gen = [\n{rows(gen)}\n];\nmpc.branch = [\n{rows(branch)}\n];\n"
    if gencost is not None:
        t += f"mpc.gencost = [\n{rows(gencost)}\n];\n"
    return t


BUS2 = [[1, 3, 0, 0, 0, 0, 1, 1, 0, 230, 1, 1.1, 0.9], [2, 1, 100, 20, 0, 0, 1, 1, 0, 230, 1, 1.1, 0.9]]
GEN1 = [[1, 0, 0, 100, -100, 1, 100, 1, 200, 0]]
BR = lambda r=0.0, x=0.1, b=0.0, tap=0, shift=0, st=1: [[1, 2, r, x, b, 100, 100, 100, tap, shift, st, -360, 360]]  # noqa: E731


def test_minimal_case_counts_and_per_unit():
    n = mp.PowerNetwork(case(BUS2, GEN1, BR(), [[2, 0, 0, 3, 0.1, 10, 0]]))
    assert n.counts() == (2, 1, 1)
    assert n.buses()["pd"][1] == 1.0  # 100 MW on 100 MVA
    y = n.branch_admittances()[0]
    assert abs(y[0] - (0 - 10j)) < 1e-12  # r=0, x=0.1, tap=1: y_series = -j10


def test_branch_admittance_examples():
    ys = 1 / (0.01 + 0.1j)
    y = mp.PowerNetwork(case(BUS2, GEN1, BR(r=0.01, x=0.1))).branch_admittances()[0]
    assert abs(ys - (0.9901 - 9.901j)) < 1e-4
    np.testing.assert_allclose(y, [ys, -ys, -ys, ys], rtol=1e-14)
    y2 = mp.PowerNetwork(case(BUS2, GEN1, BR(r=0.01, x=0.1, b=0.2))).branch_admittances()[0]
    np.testing.assert_allclose([y2[0] - y[0], y2[3] - y[3]], [0.1j, 0.1j], atol=1e-14)
    y3 = mp.PowerNetwork(case(BUS2, GEN1, BR(x=0.1, tap=2))).branch_admittances()[0]
    assert abs(y3[0] - (1 / 0.1j) / 4) < 1e-14
    # symmetry with tap = 1, shift = 0
    y4 = mp.PowerNetwork(case(BUS2, GEN1, BR(r=0.02, x=0.2, b=0.1))).branch_admittances()[0]
    assert y4[1] == y4[2]
    with pytest.raises(InvalidArgument, match="DegenerateBranch"):
        mp.PowerNetwork(case(BUS2, GEN1, BR(r=0, x=0))).branch_admittances()


def test_round_trip_and_idempotence():
    n = mp.case9()
    t = n.serialize()
    m = mp.PowerNetwork(t)
    assert m.to_json() == n.to_json()
    assert m.serialize() == t
    assert mp.case9().to_json() == n.to_json()


@pytest.mark.parametrize("text,what", [
    (case([[1, 1] + BUS2[0][2:], BUS2[1]], GEN1, BR()), "no reference bus"),
    (case([BUS2[0], [2, 3] + BUS2[1][2:]], GEN1, BR()), "more than one reference"),
    (case(BUS2, GEN1, [[1, 7, 0, 0.1, 0, 100, 100, 100, 0, 0, 1, -360, 360]]), "dangling"),
    (case(BUS2, [[1, 0, 0, 100, -100, 1, 100, 1, 10, 50]], BR()), "inverted"),
    (case(BUS2, GEN1, BR(), [[1, 0, 0, 2, 0, 0, 100, 1000]]), "piecewise"),
    (case(BUS2, GEN1, BR()).replace("0.1\t0.0\t100", "0.1x\t0.0\t100"), "line 12"),
])
def test_validation_and_parse_errors(text, what):
    with pytest.raises(InvalidArgument, match=what):
        mp.PowerNetwork(text)


def test_out_of_service_kept_in_data_excluded_from_model():
    txt = open(mp.DATA + "/case9.m").read().replace(
        "\t8\t9\t0.032\t0.161\t0.306\t250\t250\t250\t0\t0\t1", "\t8\t9\t0.032\t0.161\t0.306\t250\t250\t250\t0\t0\t0")
    n = mp.PowerNetwork(txt)
    assert n.info.nbranch == 9 and n.info.nbranch_in == 8
    assert Scopf(network=n, K=0).info.nl == 8


def test_parsed_case9_is_the_builtin_case9():
    """the SCOPF built from data/case9.m equals the typed-in case9: every
    family's program, rows, variables and parameters, and all bounds"""
    a, b = Scopf(network=mp.case9(), K=2), Scopf("case9", 2)
    assert (a.n, a.m) == (b.n, b.m)
    for fa, fb in zip(a.families(), b.families()):
        assert fa.name == fb.name
        for k in ("rows", "vars", "params"):
            assert np.array_equal(getattr(fa, k), getattr(fb, k)), (fa.name, k)
    ba, bb = a.bounds(), b.bounds()
    for k in ba:
        assert np.array_equal(ba[k], bb[k]), k


@pytest.mark.gpu
def test_parsed_case9_solves_to_the_known_optimum(gpu):
    from paper_2510_13333_b200.ipm import solve_scopf
    out = solve_scopf(Scopf(network=mp.case9(), K=0))
    assert out.status == "optimal"
    assert abs(out.result["objective"] - 5296.69) < 0.01  # MATPOWER case9 optimum
