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
