"""Seeded synthetic scene generators shared by the oracle tests, the CUDA-path
tests and bench.py.

This package holds NO arithmetic of the method (no constraint values, no
projections, no derivatives): only mesh topology, material/compliance draws,
masses, collider definitions, forces and targets, all seeded. See DESIGN.md
"Input recipe".
"""
from .scenes import (  # noqa: F401
    Scene,
    cloth_grid,
    cloth_tube,
    tet_block,
    body_capsules,
    tiny_cloth,
    medium_cloth,
    volumetric_block,
    garment,
    large_cloth,
    CONFIGS,
    make_config,
    as_float32_exact,
)
