"""ORACLE (test infrastructure only). Greedy constraint coloring, R1.

`greedy_color` calls the plain-C implementation in oracle/c/greedy_color.c
(compiled by __graft_entry__.build() or on first use); `greedy_color_py` is the
same definition in pure Python for small inputs (used to pin the C one).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "c", "greedy_color.c")
_LIB = os.path.join(_HERE, "c", "liboracle_color.so")
_lib = None


def build_c() -> str:
    if (not os.path.exists(_LIB)) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_c())
        _lib.oracle_greedy_color.restype = ctypes.c_int
        _lib.oracle_greedy_color.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
                                             ctypes.c_int64, ctypes.c_void_p]
    return _lib


def greedy_color(idx: np.ndarray, n_verts: int) -> np.ndarray:
    """Color of each constraint (row of idx), sequential greedy in row order."""
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    n, arity = idx.shape
    out = np.zeros(n, np.int32)
    if n == 0:
        return out
    nc = _load().oracle_greedy_color(n, arity, idx.ctypes.data, int(n_verts), out.ctypes.data)
    if nc < 0:
        raise RuntimeError("greedy coloring needs more than 256 colors")
    return out


def greedy_color_py(idx: np.ndarray, n_verts: int) -> np.ndarray:
    used = [0] * n_verts
    out = np.zeros(len(idx), np.int32)
    for j, row in enumerate(idx.tolist()):
        m = 0
        for v in row:
            m |= used[v]
        c = 0
        while (m >> c) & 1:
            c += 1
        out[j] = c
        for v in row:
            used[v] |= 1 << c
    return out
