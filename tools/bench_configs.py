"""Full-length forward + adjoint of every BASELINE config (configs[0..4]) once on cuda:0 through the
C-ABI, with each config's gradient families; prints one JSON line per config (ms per step, per
substep, PCG iterations).  Not the driver's bench (bench.py times configs[4]); this records that
the other four configs run at their full size and length.  Synthetic seeded inputs (synth/)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2301_01396_b200 import api  # noqa: E402
from synth import as_float32_exact, garment, large_cloth, medium_cloth, tiny_cloth, volumetric_block  # noqa: E402

CASES = [
    ("configs[0] tiny_cloth 16x16, 30 frames x 10 substeps", lambda: tiny_cloth(), ("compliance", "v0")),
    ("configs[1] medium_cloth 256x256 + sphere, 60 frames x 10", lambda: medium_cloth(), ("compliance", "x0")),
    ("configs[2] volumetric_block 40^3 (~300k tets), 50 frames x 20", lambda: volumetric_block(), ("material",)),
    ("configs[3] garment 512x512 tube + 12 capsules, 120 frames x 10", lambda: garment(), ("shape",)),
    ("configs[4] large_cloth 2944x2944, 30 frames x 10", lambda: large_cloth(), ("forces",)),
]


def garment_targets(s, t):
    """configs[3] target: the drape produced by the ground-truth shape vector (BASELINE configs[3]),
    simulated by the library itself (a performance input only; parity tests build it with the
    oracle, tests/garment_case.py)."""
    gt = s.replace(shape_beta=np.asarray(s.meta["shape_beta_gt"], np.float32).astype(np.float64))
    sc = api.dxpbd_create(**api.scene_kwargs(gt), max_frames=s.frames)
    api.dxpbd_forward(sc, t(s.x0), t(s.v0), None, s.frames)
    x = api.dxpbd_positions(sc, s.frames)
    del sc
    return x[None]


def capsule_contacts(s, x, tol=1e-3):
    """(vertex, capsule) pairs within tol of the collision thickness, and the mean vertex height."""
    r = s.cap_r0 + s.cap_rbasis @ s.shape_beta
    L = s.cap_L0 + s.cap_lbasis @ s.shape_beta
    n = 0
    for k in range(len(r)):
        c, a = s.cap_center[k], s.cap_axis[k]
        tt = np.clip((x - c) @ a, -L[k] / 2, L[k] / 2)
        n += int((np.linalg.norm(x - (c + tt[:, None] * a), axis=1) - r[k] < s.thickness + tol).sum())
    return n


def run(name, make, grads):
    s = as_float32_exact(make())
    dev = "cuda:0"
    t = lambda a: None if a is None else torch.as_tensor(np.asarray(a, np.float32), device=dev)  # noqa: E731
    extra = {}
    if s.name == "garment":
        s = s.replace(targets=garment_targets(s, t))
    t0 = time.perf_counter()
    sc = api.dxpbd_create(**api.scene_kwargs(s), max_frames=s.frames, grad_flags=api.flags(*grads), cg_max_iter=2000)
    t_create = time.perf_counter() - t0
    x0, v0, f, tg = t(s.x0), t(s.v0), t(s.forces), t(s.targets)
    w = t(s.weights) if s.weights is not None else None
    fwds, tots = [], []
    for _ in range(REPEAT):   # the first pass includes one-time work (graph instantiation, lazy buffers)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        ev[0].record()
        api.dxpbd_forward(sc, x0, v0, f, s.frames)
        ev[1].record()
        loss = api.dxpbd_backward(sc, s.key_frames, tg, w)
        for g in grads:
            api.dxpbd_grads(sc, g)
        ev[2].record()
        torch.cuda.synchronize()
        fwds.append(ev[0].elapsed_time(ev[1]))
        tots.append(ev[0].elapsed_time(ev[2]))
    st = api.dxpbd_stats(sc)
    if s.name == "garment":
        xl = api.dxpbd_positions(sc, s.frames).astype(np.float64)
        extra = dict(mean_height_last_frame=float(xl[:, 1].mean()), min_height_last_frame=float(xl[:, 1].min()),
                     capsule_contacts_last_frame=capsule_contacts(s, xl),
                     rms_miss_to_target=float(np.sqrt(2 * loss / s.num_vertices)),
                     shape_grad=api.dxpbd_grads(sc, "shape").tolist())
    N = s.frames * s.substeps
    k = int(np.argmin(tots))   # best of REPEAT full-length passes
    fwd, tot = fwds[k], tots[k]
    line = dict(config=name, vertices=s.num_vertices, constraints=len(s.dist_idx), tets=len(s.tet_idx),
                colliders=len(s.spheres) + len(s.cap_center), frames=s.frames, substeps=s.substeps, grads=list(grads),
                ms_forward=fwd, ms_forward_adjoint=tot, ms_per_substep_fwd=fwd / N, ms_per_substep_fwd_adjoint=tot / N,
                cg_iters_per_substep=st["cg_iters_total"] / max(st["solves"], 1), cg_iters_max=st["cg_iters_max"],
                worst_relres=st["worst_relres"], tma_path=st["tma"], loss=loss, create_s=t_create,
                passes=REPEAT, ms_forward_adjoint_all=tots, **extra)
    print(json.dumps(line), flush=True)
    del sc


def run_batch(name, make, grads, B):
    """B independent seeded copies of a config in ONE handle (include/dxpbd.h vertex_scene): one
    launch sequence serves every scene, so launch-bound small configs gain throughput ~B."""
    scenes = [as_float32_exact(make(seed)) for seed in range(1, B + 1)]
    dev = "cuda:0"
    t = lambda a: None if a is None else torch.as_tensor(np.asarray(a, np.float32), device=dev)  # noqa: E731
    kw = api.batch_scene_kwargs(scenes)
    s0 = scenes[0]
    t0 = time.perf_counter()
    sc = api.dxpbd_create(**kw, max_frames=s0.frames, grad_flags=api.flags(*grads), cg_max_iter=2000)
    t_create = time.perf_counter() - t0
    x0, v0, f, kf, tg = api.batch_inputs(scenes, s0.frames)
    x0, v0, f, tg = t(x0), t(v0), t(f), t(tg)
    fwds, tots = [], []
    for _ in range(REPEAT):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        ev[0].record()
        api.dxpbd_forward(sc, x0, v0, f, s0.frames)
        ev[1].record()
        loss = api.dxpbd_backward(sc, kf, tg)
        for g in grads:
            api.dxpbd_grads(sc, g)
        ev[2].record()
        torch.cuda.synchronize()
        fwds.append(ev[0].elapsed_time(ev[1]))
        tots.append(ev[0].elapsed_time(ev[2]))
    st = api.dxpbd_stats(sc)
    k = int(np.argmin(tots))
    N = s0.frames * s0.substeps
    E = sum(len(s.dist_idx) for s in scenes)
    line = dict(config=name, batch=B, vertices=sum(s.num_vertices for s in scenes), constraints=E,
                frames=s0.frames, substeps=s0.substeps, grads=list(grads), ms_forward=fwds[k],
                ms_forward_adjoint=tots[k], ms_per_substep_fwd=fwds[k] / N, ms_per_substep_fwd_adjoint=tots[k] / N,
                ms_per_scene_substep_fwd_adjoint=tots[k] / N / B,
                constraint_solves_per_s=E * N / (tots[k] * 1e-3),
                cg_iters_per_substep=st["cg_iters_total"] / max(st["solves"], 1), worst_relres=st["worst_relres"],
                tma_path=st["tma"], loss=loss, create_s=t_create, passes=REPEAT, ms_forward_adjoint_all=tots)
    print(json.dumps(line), flush=True)
    del sc


BATCHES = {
    "b0": ("configs[0] tiny_cloth 16x16 x64 batch", lambda seed: tiny_cloth(seed=seed), ("compliance", "v0"), 64),
    "b1": ("configs[1] medium_cloth 256x256 + sphere x8 batch", lambda seed: medium_cloth(seed=seed), ("compliance", "x0"), 8),
}

REPEAT = 3

if __name__ == "__main__":
    which = sys.argv[1:] or [str(i) for i in range(len(CASES))]
    for w in which:
        if w in BATCHES:
            run_batch(*BATCHES[w])
        else:
            run(*CASES[int(w)])
