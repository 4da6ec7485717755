"""CPU checks of the boundary: the C-ABI library builds for sm_100a, loads, and exports every
symbol include/dxpbd.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    h = open(os.path.join(ROOT, "include", "dxpbd.h")).read()
    return sorted(set(re.findall(r"\b(dxpbd_[a-z_]+)\s*\(", h)))


def test_header_declares_api():
    names = _declared()
    for n in ("dxpbd_create", "dxpbd_forward", "dxpbd_backward", "dxpbd_grads", "dxpbd_destroy"):
        assert n in names


def test_library_builds_loads_and_exports():
    from paper_2301_01396_b200 import build as b
    path = b.build()
    L = ctypes.CDLL(path)
    for n in _declared():
        assert hasattr(L, n), n
    from paper_2301_01396_b200 import api
    for n in _declared():
        assert n in api.EXPORTED and hasattr(api, n), n
    assert api.dxpbd_version() == 100
    assert api.dxpbd_last_error() == ""


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2301_01396_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("oracle/", ""), f


def test_sm100a_cubin():
    import subprocess
    from paper_2301_01396_b200 import build as b
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", b.build()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_out_buffer_validation():
    """dxpbd_grads / dxpbd_positions write in place: a wrong-size, wrong-dtype or non-contiguous
    `out` is rejected before the call (no silent copy, no write past the end)."""
    import numpy as np
    from paper_2301_01396_b200 import api
    good = np.zeros((4, 3), np.float32)
    assert api._out_arg(good, 12, "t").ptr == good.ctypes.data
    for bad in (np.zeros((4, 3), np.float64), np.zeros((5, 3), np.float32), np.zeros((3, 8), np.float32)[:, ::2],
                np.zeros((2, 3), np.float32)):
        with pytest.raises(ValueError):
            api._out_arg(bad, 12, "t")
    import torch
    with pytest.raises(ValueError):
        api._out_arg(torch.zeros(13), 12, "t")
    t = torch.zeros(12)
    assert api._out_arg(t, 12, "t").ptr == t.data_ptr()
