"""configs[3] garment cases for the parity tests, built with the oracle only (no input comes from
the CUDA path).  The garment hangs from its pinned neckline over the 12-capsule body
(synth.garment); a case starts from the oracle's draped state after `warm_frames` frames (so the
collision constraints are active from the first substep) and its keyframe target is the oracle's
drape under the seeded ground-truth shape vector beta_gt (BASELINE configs[3]: "distance to the
drape produced by a seeded ground-truth coefficient vector")."""
import numpy as np

from oracle import OracleModel
from synth import as_float32_exact, garment


def _f32(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def garment_case(n_around: int, n_along: int, warm_frames: int, frames: int, seed: int = 3):
    s = as_float32_exact(garment(n_around=n_around, n_along=n_along, frames=frames, seed=seed))
    m = OracleModel(s)
    x, v = s.x0.copy(), s.v0.copy()
    for _ in range(warm_frames * s.substeps):
        x, v, _ = m.step(x, v)
    s = s.replace(x0=_f32(x), v0=_f32(v))
    sg = s.replace(shape_beta=_f32(s.meta["shape_beta_gt"]))
    xs = OracleModel(sg).simulate(sg.x0, sg.v0, None, frames)
    return s.replace(key_frames=np.array([frames], np.int32), targets=_f32(xs[frames * s.substeps])[None])


def contacts(s, x, tol=1e-4) -> int:
    """Number of (free vertex, capsule) pairs within `tol` of contact (C < tol) at positions x."""
    m = OracleModel(s)
    free = np.nonzero(m.free)[0]
    return int(sum((m.ev_capsule(x, k, free)["C"][:, 0] < tol).sum() for k in range(len(m.cap_c))))
