"""GPU checks of the vertex-partitioned domain decomposition (dxpbd_group_*):
P partitions with per-color halo exchange reproduce the single scene — positions bit for bit
(a color is vertex-disjoint, every partition runs the same per-constraint arithmetic), loss and
gradients up to the summation order of the all-reduced PCG scalars — and the oracle within the
parity tolerances."""
import numpy as np
import pytest

from synth import large_cloth, medium_cloth
from tests.gpu_helpers import f32, oracle_run, rel_l2

pytestmark = pytest.mark.gpu

GRADS = ("forces", "x0", "v0")


def _api():
    from paper_2301_01396_b200 import api
    return api


def _scene(n=96, frames=3, substeps=4):
    s = large_cloth(n=n, frames=frames, substeps=substeps, side=10.0 * (n - 1) / 2943.0, key_frames=(frames,))
    return f32(s.replace(frame_dt=substeps / 600.0))


def _single(s):
    api = _api()
    sc = api.dxpbd_create(**api.scene_kwargs(s), max_frames=s.frames, grad_flags=api.flags(*GRADS), cg_max_iter=1000)
    api.dxpbd_forward(sc, s.x0, s.v0, s.forces, s.frames)
    x = [api.dxpbd_positions(sc, f) for f in range(s.frames + 1)]
    loss = api.dxpbd_backward(sc, s.key_frames, s.targets)
    return dict(x=x, loss=loss, **{g: api.dxpbd_grads(sc, g) for g in GRADS}, stats=api.dxpbd_stats(sc))


def _group(s, P):
    api = _api()
    g = api.dxpbd_group_create(**api.scene_kwargs(s), num_parts=P, max_frames=s.frames,
                               grad_flags=api.flags(*GRADS), cg_max_iter=1000)
    api.dxpbd_group_forward(g, s.x0, s.v0, s.forces, s.frames)
    x = [api.dxpbd_group_positions(g, f) for f in range(s.frames + 1)]
    loss = api.dxpbd_group_backward(g, s.key_frames, s.targets)
    return dict(x=x, loss=loss, **{k: api.dxpbd_group_grads(g, k) for k in GRADS}, stats=api.dxpbd_group_stats(g))


@pytest.mark.parametrize("P", [2, 3, 5])
def test_group_equals_single_scene(P):
    s = _scene()
    a = _single(s)
    b = _group(s, P)
    for f in range(s.frames + 1):
        np.testing.assert_array_equal(b["x"][f], a["x"][f])      # per-color exchange: bit for bit
    assert b["loss"] == pytest.approx(a["loss"], rel=1e-6)
    for k in GRADS:
        assert rel_l2(b[k], a[k]) < 1e-5, (k, rel_l2(b[k], a[k]))
    assert abs(b["stats"]["cg_iters_total"] - a["stats"]["cg_iters_total"]) <= 0.05 * a["stats"]["cg_iters_total"] + 2


def test_group_without_exchange_differs(monkeypatch):
    """Negative control: with the halo exchanges switched off the partitions drift apart, so the
    equality above is produced by the exchange lists, not by shared state."""
    s = _scene(n=64, frames=1, substeps=3)
    a = _single(s)
    monkeypatch.setenv("DXPBD_GROUP_NO_EXCHANGE", "1")
    api = _api()
    g = api.dxpbd_group_create(**api.scene_kwargs(s), num_parts=2, max_frames=1)
    api.dxpbd_group_forward(g, s.x0, s.v0, s.forces, 1)
    assert np.abs(api.dxpbd_group_positions(g, 1) - a["x"][1]).max() > 0


def test_group_matches_oracle():
    s = _scene(n=40, frames=2, substeps=3)
    b = _group(s, 2)
    o = oracle_run(s)
    for f in range(s.frames + 1):
        assert rel_l2(b["x"][f], o["x"][f]) < 1e-4
    for k in GRADS:
        assert rel_l2(b[k], o[k]) < 1e-3, (k, rel_l2(b[k], o[k]))


def test_group_with_sphere_collider():
    """configs[1]-style cloth on a sphere: contacts run redundantly per partition."""
    api = _api()
    s = f32(medium_cloth(n=64, frames=2).replace(substeps=5, frame_dt=5 / 600.0))
    sc = api.dxpbd_create(**api.scene_kwargs(s), max_frames=2)
    api.dxpbd_forward(sc, s.x0, s.v0, None, 2)
    g = api.dxpbd_group_create(**api.scene_kwargs(s), num_parts=3, max_frames=2)
    api.dxpbd_group_forward(g, s.x0, s.v0, None, 2)
    for f in range(3):
        np.testing.assert_array_equal(api.dxpbd_group_positions(g, f), api.dxpbd_positions(sc, f))


def test_group_rejects_unsupported():
    api = _api()
    s = _scene(n=32, frames=1, substeps=1)
    with pytest.raises(api.DxpbdError):
        api.dxpbd_group_create(**api.scene_kwargs(s), num_parts=2, grad_flags=api.flags("compliance"))
    with pytest.raises(api.DxpbdError):
        api.dxpbd_group_create(**{**api.scene_kwargs(s), "iterations": 2}, num_parts=2)


def test_group_full_size_forward_bit_exact():
    """configs[4] at full size (2944^2), 1 frame: 4 partitions reproduce the single scene bit for bit."""
    api = _api()
    s = f32(large_cloth(frames=1, key_frames=(1,)))
    sc = api.dxpbd_create(**api.scene_kwargs(s), max_frames=1)
    api.dxpbd_forward(sc, s.x0, s.v0, s.forces, 1)
    a = api.dxpbd_positions(sc, 1)
    del sc
    g = api.dxpbd_group_create(**api.scene_kwargs(s), num_parts=4, max_frames=1)
    api.dxpbd_group_forward(g, s.x0, s.v0, s.forces, 1)
    np.testing.assert_array_equal(api.dxpbd_group_positions(g, 1), a)


def test_distributed_group_world1_equals_single():
    """The NCCL transport path (dxpbd_group_create_dist) with a one-rank communicator: the same
    schedule as the in-process group with NCCL all-reduces; equals the single scene exactly."""
    api = _api()
    s = _scene(n=64, frames=2, substeps=3)
    a = _single(s)
    uid = api.dxpbd_nccl_unique_id()
    g = api.dxpbd_group_create_dist(**api.scene_kwargs(s), rank=0, world=1, nccl_id=uid, max_frames=s.frames,
                                    grad_flags=api.flags(*GRADS), cg_max_iter=1000)
    api.dxpbd_group_forward(g, s.x0, s.v0, s.forces, s.frames)
    for f in range(s.frames + 1):
        np.testing.assert_array_equal(api.dxpbd_group_positions(g, f), a["x"][f])
    loss = api.dxpbd_group_backward(g, s.key_frames, s.targets)
    assert loss == pytest.approx(a["loss"], rel=1e-6)
    for k in GRADS:
        assert rel_l2(api.dxpbd_group_grads(g, k), a[k]) < 1e-5


def test_group_trajectory_memory_falls_with_P():
    """Each partition stores its trajectory only for the vertices it holds (owned tiles + tile halos)
    plus 3 rolling full-V states: at a 256^2 crop of configs[4] the per-partition trajectory bytes
    fall roughly as 1/P (stats field 12 against the single scene's field 13), and the group still
    reproduces the single scene's positions bit for bit."""
    api = _api()
    s = _scene(n=256, frames=2, substeps=5)
    a = _single(s)
    prev = None
    for P in (2, 4, 8):
        g = api.dxpbd_group_create(**api.scene_kwargs(s), num_parts=P, max_frames=s.frames,
                                   grad_flags=api.flags(*GRADS), cg_max_iter=1000)
        st = api.dxpbd_group_stats(g)
        frac = st["traj_bytes_part"] / st["traj_bytes_single"]
        print(P, frac, st["held_max"])
        assert frac < 1.0 / P + 0.15 + 3.0 / (s.frames * s.substeps + 1), (P, frac)
        if prev is not None:
            assert frac < prev
        prev = frac
        if P == 4:
            api.dxpbd_group_forward(g, s.x0, s.v0, s.forces, s.frames)
            for f in range(s.frames + 1):
                np.testing.assert_array_equal(api.dxpbd_group_positions(g, f), a["x"][f])
        del g
