"""Shared helpers of the GPU parity tests: run a synth.Scene through the C-ABI (CUDA path)
and through the oracle on the same float32-rounded inputs."""
import numpy as np

from synth import as_float32_exact


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def gpu_run(scene, grads=(), frames=None, pd=1, cg_tol=1e-6, cg_max_iter=1000, device_inputs=True,
            backward=True):
    import torch
    from paper_2301_01396_b200 import api
    s = scene
    frames = s.frames if frames is None else frames
    sc = api.dxpbd_create(**api.scene_kwargs(s), max_frames=frames, grad_flags=api.flags(*grads),
                          pd_projection=pd, cg_tol=cg_tol, cg_max_iter=cg_max_iter)
    dev = "cuda" if device_inputs else "cpu"
    t = lambda a: torch.as_tensor(np.asarray(a, np.float32), device=dev)  # noqa: E731
    forces = None if s.forces is None else t(s.forces[:frames])
    api.dxpbd_forward(sc, t(s.x0), t(s.v0), forces, frames)
    out = dict(scene=sc, x=[api.dxpbd_positions(sc, f) for f in range(frames + 1)])
    if backward:
        kf = [k for k in np.asarray(s.key_frames).tolist() if k <= frames]
        tg = s.targets[: len(kf)]
        w = None if s.weights is None else t(s.weights)
        out["loss"] = api.dxpbd_backward(sc, kf, t(tg), w)
        for g in grads:
            out[g] = api.dxpbd_grads(sc, g)
        for g in ("x0", "v0"):
            out[g] = api.dxpbd_grads(sc, g)
        out["stats"] = api.dxpbd_stats(sc)
    return out


def oracle_run(scene, frames=None, pd=True, backward=True, solver="direct"):
    from oracle import OracleModel
    s = scene
    frames = s.frames if frames is None else frames
    m = OracleModel(s, pd_projection=pd, solver=solver)
    xs = m.simulate(s.x0, s.v0, s.forces, frames)
    out = dict(model=m, x=[xs[f * s.substeps] for f in range(frames + 1)])
    if backward:
        kf = np.array([k for k in np.asarray(s.key_frames).tolist() if k <= frames], np.int32)
        phi, gr = m.backward(xs, s.v0, s.forces, key_frames=kf, targets=s.targets[: len(kf)],
                             weights=s.weights)
        out["loss"] = phi
        out.update(gr)
    return out


def f32(scene):
    return as_float32_exact(scene)


def random_network(V=1100, k=8, seed=5):
    """An irregular spring network (not a lattice): every vertex tied to k random others among its 60
    nearest neighbours in a unit cube (mean degree 2k), a few pinned vertices."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.0, 1.0, size=(V, 3))
    pairs = set()
    for i in range(V):
        near = np.argsort(((x - x[i]) ** 2).sum(1))[1:61]
        for j in rng.choice(near, size=k, replace=False):
            pairs.add((min(i, int(j)), max(i, int(j))))
    idx = np.array(sorted(pairs), np.int32)
    w = np.full(V, 1000.0)
    w[rng.choice(V, size=12, replace=False)] = 0.0
    from synth import Scene
    from synth.scenes import _base
    d = _base("network", V, x_rest=x, x0=x + 0.004 * rng.standard_normal(x.shape) * (w > 0)[:, None], inv_mass=w,
              dist_idx=idx, dist_compliance=10.0 ** rng.uniform(-8, -6, len(idx)))
    tgt = x + 0.02 * rng.standard_normal(x.shape)
    return Scene(**d, frame_dt=1 / 60, substeps=4, iterations=1, frames=2, key_frames=np.array([2], np.int32),
                 targets=tgt[None])
