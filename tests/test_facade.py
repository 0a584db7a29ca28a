"""Drop-in proof of the C++ boundary: tests/facade/caller.cpp
is written against the reference API only (nclopf::ModelBuilder /
ExpressionTemplate / ModelFunctions / fd_check / SparseSym / symbolic_order /
analyze / factorize / solve_refined, /root/reference/proj/include/nclopf/*.hpp).
The same source is compiled against the reference (oracle/_ref/facade_caller_ref,
oracle/Makefile) and against the B200 façade (include/nclopf_b200/nclopf/*.hpp
over libnclopf_b200.so); on the GPU both binaries run and their outputs agree:
patterns, orderings, counts, statuses and exception behaviour exactly, values
to rounding (the GPU factorization sums in another order)."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2510_13333_b200", "libnclopf_b200.so")
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "facade_caller_ref")


def build_facade(out_dir):
    exe = os.path.join(out_dir, "facade_caller")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include", "nclopf_b200"),
                    "-I" + os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "facade", "caller.cpp"), LIB,
                    "-Wl,-rpath," + os.path.dirname(LIB), "-o", exe], check=True, capture_output=True, text=True)
    return exe


def test_caller_compiles_against_the_facade(tmp_path):
    """the reference caller compiles and links unchanged against the façade"""
    exe = build_facade(str(tmp_path))
    assert os.path.exists(exe)


EXACT = ["n", "m", "nnzj", "nnzh", "caught", "caught_after_finalize", "fd_pass", "nnzK", "jac_rows", "jac_cols",
         "hess_rows", "hess_cols", "col_ptr", "row_ind", "perm", "parent", "l_colcount", "entry_map", "l_nnz",
         "status_ok", "zpi", "inertia", "refined_converged", "owning_same_perm", "kkt_inertia", "zero_pivot_status",
         "zero_pivot_index", "mm_bytes"]
CLOSE = ["obj", "grad", "cons", "jac", "hess", "jv", "jty", "max_abs_diag", "norm_inf", "frobenius", "K_times_ones",
         "values", "D", "x", "x_refined"]


@pytest.mark.gpu
def test_facade_matches_reference(gpu, tmp_path):
    if not os.path.exists(REF_BIN):
        pytest.skip("oracle/_ref/facade_caller_ref not built (make -C oracle)")
    exe = build_facade(str(tmp_path))
    ours = json.loads(subprocess.run([exe], check=True, capture_output=True, text=True).stdout)
    ref = json.loads(subprocess.run([REF_BIN], check=True, capture_output=True, text=True).stdout)
    for k in EXACT:
        assert ours[k] == ref[k], k
    for k in CLOSE:
        a, b = np.atleast_1d(ours[k]), np.atleast_1d(ref[k])
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12 * max(1.0, float(np.max(np.abs(b)))), err_msg=k)
    assert ours["refined_sweeps"] <= ref["refined_sweeps"] + 1
