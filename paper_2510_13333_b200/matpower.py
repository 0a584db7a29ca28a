"""matpower_io over the C-ABI (include/nclopf_matpower.h):
MATPOWER case text -> validated per-unit network, branch admittances, the
canonical serializer / JSON dump, and Scopf(network=...) for the SCOPF of a
parsed case."""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

from ._lib import P, check, f64, i32, i64, lib, register
from .sparse import _ptr


class NetworkInfo(C.Structure):
    _fields_ = [("base_mva", f64), ("nbus", i32), ("nbranch", i32), ("ngen", i32), ("ref", i32),
                ("nbranch_in", i32), ("ngen_in", i32)]


register({
    "ncl_matpower_parse": (i32, [C.c_char_p, C.POINTER(P)]),
    "ncl_network_destroy": (None, [P]),
    "ncl_network_info_get": (i32, [P, C.POINTER(NetworkInfo)]),
    "ncl_network_buses": (i32, [P, P, P, P, P, P, P]),
    "ncl_network_branch_admittances": (i32, [P, P]),
    "ncl_network_serialize": (i32, [P, C.c_char_p, i64, C.POINTER(i64)]),
    "ncl_network_json": (i32, [P, C.c_char_p, i64, C.POINTER(i64)]),
})

DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data")


class PowerNetwork:
    """parse_case(text); errors raise InvalidArgument
    ("ParseError(line N): ..." / "ValidationError: ...")."""

    def __init__(self, text: str):
        h = C.c_void_p()
        check(lib.ncl_matpower_parse(text.encode(), C.byref(h)))
        self._h = h
        self.info = NetworkInfo()
        check(lib.ncl_network_info_get(h, C.byref(self.info)))

    @classmethod
    def from_file(cls, path: str) -> "PowerNetwork":
        with open(path) as f:
            return cls(f.read())

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.ncl_network_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def name(self) -> str:
        return self.to_json()["name"]

    def counts(self):
        return self.info.nbus, self.info.nbranch, self.info.ngen

    def buses(self) -> dict:
        nb = self.info.nbus
        out = {k: np.empty(nb, np.int32) for k in ("id", "type")} | {k: np.empty(nb) for k in ("pd", "qd", "vmin", "vmax")}
        check(lib.ncl_network_buses(self._h, *[_ptr(out[k]) for k in ("id", "type", "pd", "qd", "vmin", "vmax")]))
        return out

    def branch_admittances(self) -> np.ndarray:
        """(nbranch, 4) complex: y_ff, y_ft, y_tf, y_tt"""
        y = np.empty(8 * self.info.nbranch)
        check(lib.ncl_network_branch_admittances(self._h, _ptr(y)))
        return (y[0::2] + 1j * y[1::2]).reshape(-1, 4)

    def _text(self, fn) -> str:
        ln = C.c_int64()
        check(fn(self._h, None, 0, C.byref(ln)))
        buf = C.create_string_buffer(ln.value + 1)
        check(fn(self._h, buf, ln.value + 1, C.byref(ln)))
        return buf.value.decode()

    def serialize(self) -> str:
        return self._text(lib.ncl_network_serialize)

    def to_json(self) -> dict:
        return json.loads(self._text(lib.ncl_network_json))


def case9() -> PowerNetwork:
    return PowerNetwork.from_file(os.path.join(DATA, "case9.m"))


__all__ = ["PowerNetwork", "NetworkInfo", "case9"]
