"""GPU edge cases and full-size checks of the C-ABI path against the oracle (or against
properties that hold at any size where the oracle cannot run: zero goal => zero gradients,
linearity of the adjoint in dphi/dq)."""
import numpy as np
import pytest

from synth import Scene, tiny_cloth, large_cloth, garment, medium_cloth
from synth.scenes import _base
from tests.gpu_helpers import f32, gpu_run, oracle_run, random_network, rel_l2
from tests.test_gpu_cloth import _compare

pytestmark = pytest.mark.gpu


def _api():
    from paper_2301_01396_b200 import api
    return api


def test_contacts_only_no_constraints():
    """E = 0: a free particle cloud falling onto a sphere (contact path alone)."""
    rng = np.random.default_rng(3)
    x = rng.uniform(-0.2, 0.2, size=(300, 3)) + np.array([0, 0.32, 0])
    d = _base("pts", 300, x_rest=x, inv_mass=np.full(300, 1000.0), spheres=np.array([[0, 0, 0, 0.3]]))
    s = f32(Scene(**d, frame_dt=1 / 60, substeps=5, iterations=1, frames=3, thickness=0.005,
                  collision_compliance=1e-9, key_frames=np.array([3], np.int32), targets=(x - 0.05)[None]))
    g = gpu_run(s, ("sphere",))
    o = oracle_run(s)
    _compare(g, o, ("sphere", "x0", "v0"))


def test_irregular_network_pull_layout_tails():
    """An irregular mesh of mean degree 16 (several tiles, large halos): the pull layout needs more than
    kTileV overflow entries per tile and more than 8 secondaries per vertex (the kernels' in-loop tail
    paths), checked on the host-only layout; positions and gradients against the oracle."""
    api = _api()
    s = f32(random_network())
    L = api.dxpbd_pull_layout(**api.scene_kwargs(s))
    assert L["tiles"] >= 2
    assert int(L["tdesc"][:, 3].max()) > L["tile_v"]                 # overflow entries beyond one per thread
    assert int((L["tdesc"][:, 2] >> 8).max()) > 4                   # secondary pairs beyond the 4 held in registers
    g = gpu_run(s, ("compliance",))
    assert g["stats"]["pull"]
    o = oracle_run(s)
    _compare(g, o, ("compliance", "x0", "v0"))


def test_zero_keyframes_and_keyframe_at_frame0():
    api = _api()
    s = f32(tiny_cloth(n=8, frames=2))
    sc = api.dxpbd_create(**api.scene_kwargs(s), max_frames=2, grad_flags=api.flags("compliance", "v0"))
    api.dxpbd_forward(sc, s.x0, s.v0, None, 2)
    loss = api.dxpbd_backward(sc, [], np.zeros((0, s.num_vertices, 3), np.float32))
    assert loss == 0.0
    assert np.abs(api.dxpbd_grads(sc, "compliance")).max() == 0.0
    assert np.abs(api.dxpbd_grads(sc, "v0")).max() == 0.0
    # keyframe at frame 0 only: dphi/dx0 = W (x0 - x*), every other gradient 0
    tgt = s.x0 + 0.01
    loss = api.dxpbd_backward(sc, [0], tgt[None])
    gx = api.dxpbd_grads(sc, "x0")
    free = s.inv_mass > 0
    np.testing.assert_allclose(gx[free], (s.x0 - tgt)[free], rtol=1e-6, atol=1e-9)
    assert np.abs(api.dxpbd_grads(sc, "v0")).max() == 0.0
    assert loss == pytest.approx(0.5 * (0.01 ** 2) * 3 * s.num_vertices, rel=1e-5)


def test_all_pinned_and_zero_frames():
    api = _api()
    s = f32(tiny_cloth(n=4, frames=1))
    s = s.replace(inv_mass=np.zeros_like(s.inv_mass))
    g = gpu_run(s, ("compliance", "v0"))
    np.testing.assert_array_equal(g["x"][-1], g["x"][0])
    assert np.abs(g["compliance"]).max() == 0.0 and np.abs(g["v0"]).max() == 0.0
    s2 = f32(tiny_cloth(n=4, frames=1))
    sc = api.dxpbd_create(**api.scene_kwargs(s2), max_frames=1)
    api.dxpbd_forward(sc, s2.x0, s2.v0, None, 0)
    np.testing.assert_array_equal(api.dxpbd_positions(sc, 0), s2.x0.astype(np.float32))


def test_errors_are_reported():
    api = _api()
    s = f32(tiny_cloth(n=4, frames=1))
    sc = api.dxpbd_create(**api.scene_kwargs(s), max_frames=1)
    with pytest.raises(api.DxpbdError):
        api.dxpbd_backward(sc, [1], s.targets)          # backward before forward
    with pytest.raises(api.DxpbdError):
        api.dxpbd_forward(sc, s.x0, s.v0, None, 5)      # exceeds max_frames
    bad = s.dist_idx.copy()
    bad[0, 0] = s.num_vertices + 3
    kw = api.scene_kwargs(s)
    kw["dist_idx"] = bad
    with pytest.raises(api.DxpbdError):
        api.dxpbd_create(**kw, max_frames=1)


def test_large_cloth_full_size_one_substep():
    """configs[4] at full size (2944^2, 26M DoF), one substep with its forces: all positions."""
    s = f32(large_cloth(frames=1, substeps=1, key_frames=(1,)).replace(frame_dt=1 / 600))
    g = gpu_run(s, backward=False)
    o = oracle_run(s, backward=False)
    assert rel_l2(g["x"][-1], o["x"][-1]) < 1e-4
    # the step itself, to the float32 output quantum (|x| ~ 5 m -> ulp 4.8e-7 m)
    step_err = np.abs((g["x"][-1] - g["x"][0]) - (o["x"][-1] - o["x"][0])).max()
    assert step_err < 1e-6, step_err


def test_large_cloth_full_size_adjoint_properties():
    """configs[4] at full size, 2 frames: the adjoint is linear in dphi/dq (g(x* - 2d) - g0 =
    2 (g(x* - d) - g0) to PCG tolerance) and a goal at the simulated state (up to the float32
    output quantum, ~1e-7 m) gives gradients 1e-4 smaller than a 1e-3 m residual."""
    api = _api()
    s = f32(large_cloth(frames=2, key_frames=(2,)))
    sc = api.dxpbd_create(**api.scene_kwargs(s), max_frames=2, grad_flags=api.flags("forces"))
    api.dxpbd_forward(sc, s.x0, s.v0, s.forces, 2)
    x2 = api.dxpbd_positions(sc, 2)
    api.dxpbd_backward(sc, [2], x2[None])
    g0 = api.dxpbd_grads(sc, "forces")
    d = np.random.default_rng(0).standard_normal(x2.shape).astype(np.float32) * 1e-3
    api.dxpbd_backward(sc, [2], (x2 - d)[None])
    g1 = api.dxpbd_grads(sc, "forces")
    api.dxpbd_backward(sc, [2], (x2 - 2 * d)[None])
    g2 = api.dxpbd_grads(sc, "forces")
    assert np.isfinite(g1).all() and np.abs(g1).max() > 0
    assert np.abs(g0).max() < 1e-3 * np.abs(g1).max()
    assert rel_l2(g2 - g0, 2 * (g1 - g0)) < 1e-4


def test_garment_full_size_ten_frames_forward():
    """configs[3] at full size (512x512 tube, 12 capsules) over 10 frames x 10 substeps: positions
    against the fp64 oracle at frames 2, 5 and 10, with thousands of vertex-capsule contacts active
    by frame 10 (observed 2e-8, 2e-8, 7e-6; about 3 minutes of oracle time)."""
    from tests.garment_case import contacts
    s = f32(garment(frames=10))
    g = gpu_run(s, backward=False)
    o = oracle_run(s, backward=False)
    errs = {f: rel_l2(g["x"][f], o["x"][f]) for f in (2, 5, 10)}
    assert contacts(s, o["x"][10]) > 1000
    assert max(errs.values()) < 1e-4, errs


def test_medium_cloth_full_size_backward_short():
    """configs[1] at full size (256^2, sphere), one substep at its dt: gradients of compliance and x0."""
    s = f32(medium_cloth(frames=1, substeps=1).replace(frame_dt=1 / 600))
    g = gpu_run(s, ("compliance", "x0"))
    o = oracle_run(s)
    _compare(g, o, ("compliance", "x0", "v0"))


def test_medium_cloth_full_size_full_length_forward():
    """configs[1] at its full size and horizon (256^2 cloth dropped on the sphere, 60 frames x 10
    substeps) against the fp64 oracle at every 10th frame (about 3 minutes of oracle time).  The
    workload is well conditioned until the cloth has met the sphere: positions within 1e-4 up to
    frame 20 (observed 2e-8 / 4e-6).  Afterwards wrinkling amplifies round-off -- the oracle
    itself moves by 4e-3 .. 2e-2 under a 1e-9 m perturbation of x0 (tests/medium_sensitivity.py,
    tests/golden/medium_cloth_sensitivity.json) -- so later frames are only required to stay below
    that self-sensitivity; contacts must be active at the end."""
    import json
    import os
    s = f32(medium_cloth())
    assert s.frames == 60 and len(s.x0) == 256 * 256
    sens = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "medium_cloth_sensitivity.json")))["rel_l2"]
    g = gpu_run(s, backward=False)
    o = oracle_run(s, backward=False)
    errs = {f: rel_l2(g["x"][f], o["x"][f]) for f in range(10, 61, 10)}
    xe = o["x"][60]
    near = np.linalg.norm(xe - s.spheres[0, :3], axis=1) - s.spheres[0, 3] < s.thickness + 1e-3
    assert near.sum() > 1000, near.sum()             # the cloth lies on the sphere
    assert errs[10] < 1e-4 and errs[20] < 1e-4, errs
    for f in (30, 40, 50, 60):
        assert errs[f] < max(1e-4, sens[str(f)]), (f, errs)


def test_large_cloth_full_size_substeps_bench_config():
    """configs[4] in the bench's launch configuration (2944^2, dt = 1/600, forces, the same kernels
    and launch shapes bench.py times), three consecutive substeps forward (velocities carried
    between substeps): all positions vs the oracle.  (A full 10-substep frame agrees as well but
    takes the fp64 oracle ~6 min.)"""
    s = f32(large_cloth(frames=1, substeps=3, key_frames=(1,)).replace(frame_dt=3 / 600))
    g = gpu_run(s, backward=False)
    o = oracle_run(s, backward=False)
    assert rel_l2(g["x"][-1], o["x"][-1]) < 1e-4
    step_err = np.abs((g["x"][-1] - g["x"][0]) - (o["x"][-1] - o["x"][0])).max()
    assert step_err < 1e-5, step_err


def test_schedule_switches_do_not_change_results(monkeypatch):
    """The performance schedules (replay / PCG stream overlap with double-buffered blocks, deferred
    u += alpha p, derivative blocks cached by the forward) reorder work but not arithmetic: results
    equal the plain schedule bit for bit."""
    api = _api()
    s = f32(large_cloth(n=96, frames=2, substeps=3, side=10.0 * 95 / 2943.0, key_frames=(2,)).replace(frame_dt=3 / 600))

    def run():
        sc = api.dxpbd_create(**api.scene_kwargs(s), max_frames=2, grad_flags=api.flags("forces", "x0", "v0"))
        api.dxpbd_forward(sc, s.x0, s.v0, s.forces, 2)
        loss = api.dxpbd_backward(sc, s.key_frames, s.targets)
        return loss, [api.dxpbd_grads(sc, k) for k in ("forces", "x0", "v0")]

    la, ga = run()
    for k, v in (("DXPBD_OVERLAP", "0"), ("DXPBD_DEFER_U", "0"), ("DXPBD_QCACHE", "0")):
        monkeypatch.setenv(k, v)
    lb, gb = run()
    assert la == lb
    for a, b in zip(ga, gb):
        np.testing.assert_array_equal(a, b)


def test_contact_overlap_schedule_matches_serial(monkeypatch):
    """Cloth with a sphere collider: replay of substep n-1 overlapped with the PCG of substep n
    (contact blocks and collider controls double-buffered) against DXPBD_OVERLAP=0.  The cloth
    path is deterministic, so the adjoint state gradients are bit-identical; the collider
    gradient is a double-atomic sum over vertices (order may differ), so it is compared to 1e-12."""
    api = _api()
    s = f32(medium_cloth(n=48, frames=3))

    def run():
        sc = api.dxpbd_create(**api.scene_kwargs(s), max_frames=3, grad_flags=api.flags("sphere", "x0", "v0"))
        api.dxpbd_forward(sc, s.x0, s.v0, s.forces, 3)
        loss = api.dxpbd_backward(sc, s.key_frames, s.targets)
        return loss, {k: api.dxpbd_grads(sc, k) for k in ("sphere", "x0", "v0")}

    la, ga = run()
    monkeypatch.setenv("DXPBD_OVERLAP", "0")
    lb, gb = run()
    assert la == lb
    for k in ("x0", "v0"):
        np.testing.assert_array_equal(ga[k], gb[k])
    np.testing.assert_allclose(ga["sphere"], gb["sphere"], rtol=1e-12, atol=0)


@pytest.mark.parametrize("switch", ["DXPBD_QCACHE", "DXPBD_OVERLAP"])
def test_garment_block_cache_and_overlap_match_serial(monkeypatch, switch):
    """Garment (12 capsules, shape gradients, some pinned vertices): the forward caches the
    distance blocks, contact blocks and collider controls of the last substeps (all of them at
    this size) and the backward reads them instead of replaying.  Against the cache off / the
    serial schedule: positions and state gradients bit-identical, shape gradient (double-atomic
    sums) to 1e-12."""
    api = _api()
    from tests.garment_case import garment_case
    s = garment_case(64, 48, warm_frames=10, frames=3)

    def run():
        sc = api.dxpbd_create(**api.scene_kwargs(s), max_frames=3, grad_flags=api.flags("shape", "x0", "v0"))
        api.dxpbd_forward(sc, s.x0, s.v0, s.forces, 3)
        loss = api.dxpbd_backward(sc, s.key_frames, s.targets)
        st = api.dxpbd_stats(sc)
        return loss, {k: api.dxpbd_grads(sc, k) for k in ("shape", "x0", "v0")}, st

    la, ga, sa = run()
    monkeypatch.setenv(switch, "0")
    lb, gb, sb = run()
    if switch == "DXPBD_QCACHE":
        assert sa["cached_substeps"] > 0 and sb["cached_substeps"] == 0
    assert np.isfinite(la) and abs(la - lb) <= 1e-12 * abs(lb)
    for k in ("x0", "v0"):
        np.testing.assert_array_equal(ga[k], gb[k])
    np.testing.assert_allclose(ga["shape"], gb["shape"], rtol=1e-12, atol=1e-30)


def _run_all(s, grads, frames):
    api = _api()
    sc = api.dxpbd_create(**api.scene_kwargs(s), max_frames=frames, grad_flags=api.flags(*grads))
    api.dxpbd_forward(sc, s.x0, s.v0, None if s.forces is None else s.forces[:frames], frames)
    xs = [api.dxpbd_positions(sc, f) for f in range(frames + 1)]
    kf = [k for k in np.asarray(s.key_frames).tolist() if k <= frames]
    loss = api.dxpbd_backward(sc, kf, s.targets[: len(kf)])
    return xs, loss, {k: api.dxpbd_grads(sc, k) for k in grads}, api.dxpbd_stats(sc)


def _wave_cases():
    from tests.garment_case import garment_case
    return [
        ("large96", lambda: f32(large_cloth(n=96, frames=2, substeps=3, side=10.0 * 95 / 2943.0, key_frames=(2,))
                                .replace(frame_dt=3 / 600)), ("forces", "x0", "v0")),
        ("tiny", lambda: f32(tiny_cloth(frames=3)), ("compliance", "v0", "x0")),
        ("sphere", lambda: f32(medium_cloth(n=48, frames=3)), ("compliance", "x0", "v0")),
        ("garment", lambda: garment_case(64, 48, warm_frames=10, frames=2), ("x0", "v0")),
    ]


@pytest.mark.parametrize("case", range(4))
def test_wave_sweep_bit_identical(monkeypatch, case):
    """The wavefront sweep (prediction + every distance color of a substep in one launch, wave.cuh)
    reproduces the per-color launches bit for bit: positions of every frame, the loss and every
    gradient (its replay variant writes the same blocks), for several wave-tile sizes and for a
    persistent and a one-item-per-CTA grid."""
    name, mk, grads = _wave_cases()[case]
    s = mk()
    frames = s.frames
    monkeypatch.setenv("DXPBD_WAVE", "0")
    xa, la, ga, sa = _run_all(s, grads, frames)
    assert sa["wave_tiles"] == 0
    monkeypatch.setenv("DXPBD_WAVE", "1")
    for g, gf, gr in ((2, 0, -1), (1, -1, 0), (4, 7, 3)):
        monkeypatch.setenv("DXPBD_WAVE_G", str(g))
        monkeypatch.setenv("DXPBD_WAVE_GRID_FWD", str(gf))
        monkeypatch.setenv("DXPBD_WAVE_GRID_REP", str(gr))
        xb, lb, gb, sb = _run_all(s, grads, frames)
        assert sb["wave_tiles"] > 0, name
        for f in range(frames + 1):
            np.testing.assert_array_equal(xa[f], xb[f], err_msg=f"{name} g={g} frame {f}")
        assert la == lb, (name, g)
        for k in grads:
            np.testing.assert_array_equal(ga[k], gb[k], err_msg=f"{name} g={g} {k}")


@pytest.mark.parametrize("case", range(4))
def test_fused_predict_bit_identical(monkeypatch, case):
    """Prediction fused into the first distance color (k_dist_first: forward, block-caching forward
    and replay; large scenes, or any scene with the sweep graphs off) reproduces the separate
    prediction pass bit for bit: positions of every frame, loss and every gradient, with and
    without the forward's block cache."""
    name, mk, grads = _wave_cases()[case]
    s = mk()
    frames = s.frames
    monkeypatch.setenv("DXPBD_SWEEP_GRAPH", "0")
    monkeypatch.setenv("DXPBD_FUSE_PREDICT", "0")
    xa, la, ga, _ = _run_all(s, grads, frames)
    monkeypatch.setenv("DXPBD_FUSE_PREDICT", "1")
    for qcache in ("1", "0"):
        monkeypatch.setenv("DXPBD_QCACHE", qcache)
        xb, lb, gb, _ = _run_all(s, grads, frames)
        for f in range(frames + 1):
            np.testing.assert_array_equal(xa[f], xb[f], err_msg=f"{name} qcache={qcache} frame {f}")
        assert la == lb, (name, qcache)
        for k in grads:
            np.testing.assert_array_equal(ga[k], gb[k], err_msg=f"{name} qcache={qcache} {k}")


@pytest.mark.parametrize("case", range(4))
def test_pull_matvec_matches_push(monkeypatch, case):
    """The pull-style PCG kernels (pull.cuh: one vertex per thread, persistent and one tile per CTA)
    solve the same systems as the push kernels (k_cg_matvec_tma / k_rhs_tma): identical positions,
    loss and gradients up to the summation order of the solves (1e-5), same iteration counts +- 1."""
    name, mk, grads = _wave_cases()[case]
    s = mk()
    frames = s.frames
    monkeypatch.setenv("DXPBD_PULL", "0")
    xa, la, ga, sa = _run_all(s, grads, frames)
    assert not sa["pull"]
    monkeypatch.setenv("DXPBD_PULL", "1")
    for persist in ("1", "0"):
        monkeypatch.setenv("DXPBD_PULL_PERSIST", persist)
        xb, lb, gb, sb = _run_all(s, grads, frames)
        if case == 0:
            assert sb["pull"], name
        for f in range(frames + 1):
            np.testing.assert_array_equal(xa[f], xb[f], err_msg=f"{name} frame {f}")
        assert abs(la - lb) <= 1e-6 * abs(la), name
        assert abs(sa["cg_iters_total"] - sb["cg_iters_total"]) <= sa["solves"], name
        for k in grads:
            assert rel_l2(gb[k], ga[k]) < 1e-5, (name, persist, k, rel_l2(gb[k], ga[k]))


def _pcg_cases():
    from synth import volumetric_block
    return [
        ("tma_cloth", lambda: f32(large_cloth(n=64, frames=2, substeps=3, side=10.0 * 63 / 2943.0, key_frames=(2,))
                                  .replace(frame_dt=3 / 600)), ("forces", "x0", "v0")),
        ("sphere", lambda: f32(medium_cloth(n=32, frames=3)), ("compliance", "sphere", "x0")),
        ("tets", lambda: f32(volumetric_block(n=6, frames=2, substeps=4)), ("material", "x0")),
        ("k3_generic", lambda: f32(tiny_cloth(n=12, frames=2, iterations=3)), ("compliance", "v0")),
    ]


@pytest.mark.parametrize("case", range(4))
def test_pcg_graph_matches_host_polls(monkeypatch, case):
    """The PCG iteration loop as a CUDA graph (conditional WHILE node, convergence decided by the
    update kernel's last block) against the host-polled loop: same kernels, same convergence test,
    so positions, loss, gradients and the iteration statistics are identical."""
    name, mk, grads = _pcg_cases()[case]
    s = mk()
    monkeypatch.setenv("DXPBD_PCG_GRAPH", "0")
    xa, la, ga, sa = _run_all(s, grads, s.frames)
    monkeypatch.setenv("DXPBD_PCG_GRAPH", "1")
    xb, lb, gb, sb = _run_all(s, grads, s.frames)
    det = name != "tets"   # the tet matvec accumulates with float atomics (run-to-run summation order)
    for f in range(s.frames + 1):
        np.testing.assert_array_equal(xa[f], xb[f])
    assert la == lb, name
    for k in grads:
        if not det or k in ("sphere", "shape"):   # atomics: summation order may differ
            assert rel_l2(gb[k], ga[k]) < 1e-4, (name, k, rel_l2(gb[k], ga[k]))
        else:
            np.testing.assert_array_equal(ga[k], gb[k], err_msg=f"{name} {k}")
    assert sa["solves"] == sb["solves"]
    if det:
        for key in ("cg_iters_total", "cg_iters_max"):
            assert sa[key] == sb[key], (name, key, sa[key], sb[key])
        assert abs(sa["worst_relres"] - sb["worst_relres"]) <= 1e-12 + 1e-9 * sa["worst_relres"]
    else:
        assert abs(sa["cg_iters_total"] - sb["cg_iters_total"]) <= 0.05 * sa["cg_iters_total"]


def test_pcg_graph_reports_nonconvergence(monkeypatch):
    """A solve that cannot reach the tolerance within cg_max_iter fails the backward with an error in
    graph mode too (detected on the device, reported at the end of the call)."""
    api = _api()
    s = f32(tiny_cloth(n=12, frames=2))
    for mode in ("0", "1"):
        monkeypatch.setenv("DXPBD_PCG_GRAPH", mode)
        sc = api.dxpbd_create(**api.scene_kwargs(s), max_frames=2, cg_tol=1e-12, cg_max_iter=2)
        api.dxpbd_forward(sc, s.x0, s.v0, None, 2)
        with pytest.raises(api.DxpbdError, match="converge"):
            api.dxpbd_backward(sc, [2], s.targets)


def _batch_compare(scenes, grads, frames, per_collider=None):
    """Run each scene alone and all of them as one batch handle; positions per scene bit-identical
    (same colors, same per-vertex collider order, same fp64 arithmetic), gradients per scene within
    the gradient bar (the batch solves one block-diagonal system with one global residual test)."""
    api = _api()
    solo = [_run_all(s, grads, frames) for s in scenes]
    kw = api.batch_scene_kwargs(scenes)
    sc = api.dxpbd_create(**kw, max_frames=frames, grad_flags=api.flags(*grads))
    x0, v0, forces, kf, tg = api.batch_inputs(scenes, frames)
    api.dxpbd_forward(sc, x0, v0, forces, frames)
    xb = [api.dxpbd_positions(sc, f) for f in range(frames + 1)]
    kf = [k for k in kf.tolist() if k <= frames]
    loss = api.dxpbd_backward(sc, kf, tg[: len(kf)])
    assert abs(loss - sum(r[1] for r in solo)) <= 1e-5 * abs(loss)
    for f in range(frames + 1):
        for b, xs in enumerate(api.batch_split(xb[f], scenes)):
            np.testing.assert_array_equal(xs, solo[b][0][f], err_msg=f"scene {b} frame {f}")
    for k in grads:
        g = api.dxpbd_grads(sc, k)
        if k in ("x0", "v0"):
            parts = api.batch_split(g, scenes)
        elif k == "compliance":
            parts = np.split(g, np.cumsum([len(s.dist_idx) for s in scenes])[:-1])
        else:   # per collider / coefficient families
            parts = np.split(np.ravel(g), np.cumsum(per_collider)[:-1])
        for b, gp in enumerate(parts):
            ref = np.asarray(solo[b][2][k]).ravel()
            # the batch's one global residual test vs each scene's own: differences of the order of the
            # PCG tolerance; bar = the north_star gradient bar
            assert rel_l2(np.ravel(gp), ref) < 1e-3, (k, b, rel_l2(np.ravel(gp), ref))


def test_batch_of_cloth_sphere_scenes_matches_individual():
    """configs[1]-shaped batch: three cloths of different sizes, each dropped on its own sphere."""
    scenes = []
    for b, n in enumerate((20, 24, 16)):
        s = f32(medium_cloth(n=n, frames=4, seed=11 + b))
        sph = np.asarray(s.spheres, np.float64).copy()
        sph[:, 3] *= 1.0 + 0.1 * b                      # a different sphere per scene
        scenes.append(f32(s.replace(spheres=sph)))
    _batch_compare(scenes, ("compliance", "x0", "sphere"), 4, per_collider=[4, 4, 4])


def test_batch_of_garments_shape_gradients_match_individual():
    """configs[3]-shaped batch: two garments on their own 12-capsule bodies with their own shape
    vectors (block-diagonal shape bases), shape gradients per scene."""
    from tests.garment_case import garment_case
    a = garment_case(48, 32, warm_frames=20, frames=3, seed=3)
    b = garment_case(48, 32, warm_frames=20, frames=3, seed=5)
    _batch_compare([a, b], ("shape", "x0"), 3, per_collider=[len(a.shape_beta), len(b.shape_beta)])


def test_batch_rejects_coupled_scenes():
    api = _api()
    s = f32(tiny_cloth(n=4, frames=1))
    kw = api.batch_scene_kwargs([s, s])
    kw["dist_idx"] = kw["dist_idx"].copy()
    kw["dist_idx"][0, 1] = s.num_vertices + 1          # a constraint across scenes 0 and 1
    with pytest.raises(api.DxpbdError, match="scenes"):
        api.dxpbd_create(**kw, max_frames=1)
