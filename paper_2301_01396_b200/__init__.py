"""B200-native DiffXPBD hot path (arXiv 2301.01396): C-ABI CUDA library + thin binding.

The product path is `paper_2301_01396_b200.api` -> libdxpbd.so (sm_100a kernels).
It never imports `oracle/` and has no CPU fallback.
"""
from . import api  # noqa: F401
from .api import (  # noqa: F401
    dxpbd_create, dxpbd_destroy, dxpbd_forward, dxpbd_positions, dxpbd_backward, dxpbd_grads,
    dxpbd_set_params, dxpbd_coloring, dxpbd_stats, dxpbd_last_error, dxpbd_version,
    dxpbd_profile, dxpbd_kernel_times,
)
