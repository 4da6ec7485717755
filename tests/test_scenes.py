"""Workload sanity of the seeded scenes (synth/): the configs[3] garment starts clear of the body
and, simulated by the oracle, drapes over it (rests on the shoulders, collisions active) instead
of falling off."""
import numpy as np

from oracle import OracleModel
from synth import as_float32_exact, garment


def _gaps(s, x, beta):
    r = s.cap_r0 + s.cap_rbasis @ beta
    L = s.cap_L0 + s.cap_lbasis @ beta
    out = []
    for k in range(len(r)):
        c, a = s.cap_center[k], s.cap_axis[k]
        t = np.clip((x - c) @ a, -L[k] / 2, L[k] / 2)
        out.append(np.linalg.norm(x - (c + t[:, None] * a), axis=1) - r[k])
    return np.array(out)


def test_garment_starts_clear_of_the_body():
    s = garment(n_around=64, n_along=48, frames=1)
    for beta in (s.shape_beta, s.meta["shape_beta_gt"]):
        assert _gaps(s, s.x0, beta).min() > s.thickness + 0.005
    assert np.all(s.inv_mass[:64] == 0) and np.all(s.inv_mass[64:] > 0)   # neckline ring pinned


def test_garment_drapes_on_the_body():
    s = as_float32_exact(garment(n_around=64, n_along=48, frames=30))
    m = OracleModel(s)
    x, v = s.x0.copy(), s.v0.copy()
    for _ in range(s.frames * s.substeps):
        x, v, _ = m.step(x, v)
    y_body = (0.1, 1.8)
    assert y_body[0] < x[:, 1].mean() < y_body[1]
    assert x[:, 1].min() > 0.5                         # nothing slid off the body
    assert np.abs(v).max() < 5.0
    free = s.inv_mass > 0
    assert (_gaps(s, x[free], s.shape_beta) < s.thickness + 1e-3).sum() >= 10   # resting on it
