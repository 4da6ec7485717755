"""GPU parity for the tetrahedral Neo-Hookean blocks (configs[2] regime: 1.03 cm spacing,
dt = 1/1200 s, E ~ U(1e4, 1e6) Pa, nu ~ U(0.3, 0.45)): positions within 1e-4 and material /
initial-state gradients within 1e-3 relative L2 vs the fp64 oracle.

With C_D = ||F|| - sqrt 3 and C_H = det F - 1 (reading R6) the rest state is a fixed point and the
block is well conditioned at the config's stiffness (oracle pins in tests/test_oracle_forward.py),
so parity is asserted over whole frames (20 substeps): at 40^3 (full size) forward, at 16^3
(multi-tile) forward + adjoint."""
import numpy as np
import pytest

from synth import volumetric_block
from tests.gpu_helpers import f32, gpu_run, oracle_run, rel_l2
from tests.test_gpu_cloth import _compare

pytestmark = pytest.mark.gpu


def _block(n, substeps, iterations=1, soft=False, frames=1):
    """configs[2] regime at reduced vertex count; `substeps` substeps of dt = 1/1200 s per frame."""
    s = volumetric_block(n=n, frames=frames, substeps=substeps, iterations=iterations, side=0.4 * (n - 1) / 39)
    s = s.replace(frame_dt=substeps / 1200.0)
    if soft:
        rng = np.random.default_rng(7)
        E = rng.uniform(1e4, 1e5, size=len(s.tet_a))
        nu = rng.uniform(0.3, 0.45, size=len(s.tet_a))
        s = s.replace(tet_a=np.sqrt(E / (2 * (1 + nu))), tet_b=np.sqrt(E * nu / ((1 + nu) * (1 - 2 * nu))))
    return f32(s)


@pytest.mark.parametrize("iters", [1, 2])
def test_volumetric_stiff_frame(iters):
    """configs[2] stiffness, one full frame (20 substeps), 6^3 vertices."""
    s = _block(6, 20, iters)
    g = gpu_run(s, ("material",))
    o = oracle_run(s)
    assert np.abs(o["x"][-1] - o["x"][0]).max() > 1e-4   # the block actually sags
    _compare(g, o, ("material", "v0", "x0"))


def test_volumetric_two_frames():
    """Two frames of 20 substeps at the config's stiffness, keyframe at the end (8^3)."""
    s = _block(8, 20, frames=2)
    g = gpu_run(s, ("material",))
    o = oracle_run(s)
    _compare(g, o, ("material", "v0", "x0"))


def test_volumetric_mid_size_frame_backward():
    """16^3 vertices (16875 tets, several PCG tiles), config stiffness, one frame x 20 substeps,
    forward + adjoint: positions and material gradients element-wise diagnostics."""
    s = _block(16, 20)
    g = gpu_run(s, ("material",))
    o = oracle_run(s)
    _compare(g, o, ("material", "v0", "x0"))
    d = np.abs(np.asarray(g["material"], float) - o["material"])
    assert d.max() <= 1e-2 * np.abs(o["material"]).max(), d.max()


def test_volumetric_no_pd():
    s = _block(5, 2)
    g = gpu_run(s, ("material",), pd=0)
    o = oracle_run(s, pd=False)
    _compare(g, o, ("material", "v0", "x0"))


def test_tet_coloring_bit_exact():
    from oracle import greedy_color
    from paper_2301_01396_b200 import api
    s = f32(volumetric_block(n=9, frames=1))
    g = gpu_run(s, frames=1, backward=False)
    np.testing.assert_array_equal(api.dxpbd_coloring(g["scene"], 1), greedy_color(s.tet_idx, s.num_vertices))


def test_volumetric_full_size_forward_frame():
    """configs[2] at full size (40^3 vertices, ~300k tets), one full frame (20 substeps) at its dt."""
    s = _block(40, 20)
    g = gpu_run(s, backward=False)
    o = oracle_run(s, backward=False)
    assert np.abs(o["x"][-1] - o["x"][0]).max() > 1e-4
    assert rel_l2(g["x"][-1], o["x"][-1]) < 1e-4


def test_volumetric_sphere_contacts():
    """Tets plus a sphere pressed into the top corner (the tet-only PCG path with contact blocks
    Qc): positions, material and sphere gradients vs the oracle."""
    s = _block(6, 3)
    h = float(s.x0[:, 1].max())
    s = s.replace(spheres=np.array([[h, h + 0.012, h, 0.025]], np.float32).astype(np.float64))
    g = gpu_run(s, ("material", "sphere"))
    o = oracle_run(s)
    assert np.abs(o["x"][-1] - o["x"][0]).max() > 1e-3   # the contacts push vertices
    _compare(g, o, ("material", "sphere", "v0", "x0"))


def test_tet_pcg_paths_agree(monkeypatch):
    """The 2-launch tet PCG iteration (k_cg_tetv + k_cg_update_tet) against the 4-launch one
    (tile matvec, k_cg_tet, k_fold_q4, update): same arithmetic per vertex, only the p.q block
    sums are grouped differently."""
    s = _block(16, 2, soft=True)
    h = float(s.x0[:, 1].max())
    s = s.replace(spheres=np.array([[h, h + 0.02, h, 0.06]], np.float32).astype(np.float64))
    a = gpu_run(s, ("material", "sphere"))
    monkeypatch.setenv("DXPBD_TETV", "0")
    b = gpu_run(s, ("material", "sphere"))
    assert rel_l2(a["x"][-1], b["x"][-1]) < 1e-6
    for k in ("material", "sphere", "x0"):
        assert rel_l2(a[k], b[k]) < 1e-4, k
    assert a["stats"]["cg_iters_total"] == b["stats"]["cg_iters_total"]


def test_tet_overlap_schedule_matches_serial(monkeypatch):
    """Replay of substep n-1 on the low-priority stream during the PCG of substep n, with the tet
    blocks and material controls double-buffered, against DXPBD_OVERLAP=0.  The tet matvec and
    rhs gather their corner contributions per vertex in a fixed order (no float atomics), so the
    two schedules agree bit for bit."""
    s = _block(8, 4, soft=True, frames=2)
    a = gpu_run(s, ("material",))
    monkeypatch.setenv("DXPBD_OVERLAP", "0")
    b = gpu_run(s, ("material",))
    assert a["loss"] == b["loss"]
    for k in ("material", "x0", "v0"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    assert a["stats"]["cg_iters_total"] == b["stats"]["cg_iters_total"]


def test_tet_gradients_deterministic():
    """configs[2]-shaped block at 16^3 over one frame, run twice: the material, x0 and v0
    gradients are bit-identical (corner contributions gathered per vertex in a fixed order instead
    of float atomics; VERDICT r1 "non-determinism on the tet path")."""
    s = _block(16, 20, soft=False, frames=1)
    a = gpu_run(s, ("material",))
    b = gpu_run(s, ("material",))
    assert a["loss"] == b["loss"]
    for k in ("material", "x0", "v0"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
