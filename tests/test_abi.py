"""The C-ABI library loads and exports every symbol include/*.h declares."""
import os
import re
import subprocess

from tests.conftest import ROOT


def declared_symbols():
    names = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if not h.endswith(".h"):
            continue
        txt = open(os.path.join(ROOT, "include", h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"^\s*[A-Za-z_][\w\s\*]*?\b(ncl_\w+)\s*\(", txt, flags=re.M):
            names.add(m.group(1))
    return names


def test_library_exports_all_declared_symbols():
    from paper_2510_13333_b200 import _lib
    so = _lib.LIB_PATH
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    decl = declared_symbols()
    assert len(decl) > 40
    missing = decl - exported
    assert not missing, missing
    # and the Python binding declares argtypes for all of them
    assert not (decl - _lib.DECLARED), decl - _lib.DECLARED


def test_no_gpu_fails_loudly_without_fallback():
    import torch
    from paper_2510_13333_b200 import _lib
    if torch.cuda.is_available():
        return
    rc = _lib.lib.ncl_init(0)
    assert rc == _lib.NCL_E_CUDA
    assert b"no CUDA device" in _lib.lib.ncl_last_error()
