"""ctypes binding of the product C-ABI (include/nclopf_b200.h).

Loads the in-tree ``libnclopf_b200.so``. There is deliberately no fallback:
if the library is missing, importing fails loudly (build it with
``__graft_entry__.build()`` or ``make -C paper_2510_13333_b200``).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnclopf_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: the B200 path has no CPU fallback; build it first "
        "(python -c 'import __graft_entry__ as g; g.build()')")

lib = C.CDLL(LIB_PATH)

i32, i64, f64 = C.c_int, C.c_int64, C.c_double
P = C.c_void_p
pi32 = C.POINTER(C.c_int)
pf64 = C.POINTER(C.c_double)


class SymbInfo(C.Structure):
    _fields_ = [("n", i32), ("l_nnz", i64), ("nsupernodes", i32), ("max_height", i32),
                ("max_width", i32), ("max_rows", i32), ("l_storage", i64), ("flops", f64),
                ("cb_storage", i64), ("nsplit", i32), ("n_big", i32), ("n_tasks", i32)]


_SIGS = {
    "ncl_init": (i32, [i32]),
    "ncl_synchronize": (i32, []),
    "ncl_last_error": (C.c_char_p, []),
    "ncl_stream": (P, []),
    "ncl_device_alloc": (i32, [C.POINTER(P), i64]),
    "ncl_device_free": (i32, [P]),
    "ncl_memcpy": (i32, [P, P, i64, i32]),
    "ncl_kernel_launches": (i64, []),
    "ncl_sym_create": (i32, [i32, C.POINTER(P)]),
    "ncl_sym_destroy": (None, [P]),
    "ncl_sym_add": (i32, [P, i64, P, P, P]),
    "ncl_sym_finalize": (i32, [P]),
    "ncl_sym_begin_refill": (i32, [P]),
    "ncl_sym_refill": (i32, [P]),
    "ncl_sym_refill_values": (i32, [P, P, i32]),
    "ncl_sym_dim": (i32, [P]),
    "ncl_sym_nnz": (i32, [P]),
    "ncl_sym_num_triplets": (i64, [P]),
    "ncl_sym_finalized": (i32, [P]),
    "ncl_sym_get_csc": (i32, [P, P, P, P]),
    "ncl_sym_set_values": (i32, [P, P, i32]),
    "ncl_sym_device_values": (P, [P]),
    "ncl_sym_max_abs_diag": (i32, [P, pf64]),
    "ncl_sym_norm_inf": (i32, [P, pf64]),
    "ncl_sym_frobenius_norm": (i32, [P, pf64]),
    "ncl_sym_multiply": (i32, [P, P, P, i32]),
    "ncl_sym_same_pattern": (i32, [P, P]),
    "ncl_sym_write_matrix_market": (i32, [P, C.c_char_p, i64, C.POINTER(i64)]),
    "ncl_symbolic_order": (i32, [P, P]),
    "ncl_analyze": (i32, [P, P, C.POINTER(P)]),
    "ncl_symb_destroy": (None, [P]),
    "ncl_symb_info_get": (i32, [P, C.POINTER(SymbInfo)]),
    "ncl_symb_supernodes": (i32, [P, P, P, P, P, P]),
    "ncl_symb_get": (i32, [P, P, P, P, P, P, P, P]),
    "ncl_factorize": (i32, [P, P, f64, C.POINTER(P)]),
    "ncl_refactorize": (i32, [P, P, f64]),
    "ncl_fact_destroy": (None, [P]),
    "ncl_fact_status": (i32, [P, pi32, pi32, pi32, pi32, pi32]),
    "ncl_fact_diagonal": (i32, [P, P]),
    "ncl_fact_solve": (i32, [P, P, i32]),
    "ncl_factor_solve_host": (i32, [P, P, P, P, P, C.c_double] + [C.POINTER(C.c_int)] * 5),
    "ncl_solve_refined": (i32, [P, P, P, f64, i32, P, i32, pf64, pi32, pi32]),
    "ncl_fact_get_L": (i32, [P, P, P, P]),
}

DECLARED = set()
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)  # AttributeError here = a symbol the header declares is missing
    _fn.restype = _res
    _fn.argtypes = _args
    DECLARED.add(_name)


def register(sigs: dict) -> None:
    """Declare more C-ABI entry points (used by sibling modules)."""
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
        DECLARED.add(name)


NCL_OK, NCL_E_INVALID, NCL_E_LOGIC, NCL_E_DOMAIN, NCL_E_CUDA, NCL_E_INTERNAL, NCL_E_NOMEM = 0, -1, -2, -3, -4, -5, -6


class NclError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class InvalidArgument(NclError, ValueError):
    pass


class LogicError(NclError):
    pass


class DomainError(NclError):
    pass


class CudaError(NclError):
    pass


_EXC = {NCL_E_INVALID: InvalidArgument, NCL_E_LOGIC: LogicError, NCL_E_DOMAIN: DomainError,
        NCL_E_CUDA: CudaError}


def check(rc: int) -> None:
    if rc != NCL_OK:
        msg = lib.ncl_last_error().decode(errors="replace")
        raise _EXC.get(rc, NclError)(rc, msg)
