"""Pins of the oracle forward substep (Sec.3.1) and its coloring."""
import json
import os

import numpy as np
import pytest

from oracle import OracleModel, greedy_color, greedy_color_py
from synth import Scene, tiny_cloth, cloth_grid, tet_block, volumetric_block
from synth.scenes import _base

GOLD = os.path.join(os.path.dirname(__file__), "golden")
rng = np.random.default_rng(77)


def scene_from(x, w, edges=None, comp=None, frame_dt=0.01, substeps=1, iterations=1, gravity=(0, 0, 0),
               frames=1, **kw):
    V = len(x)
    d = dict(x_rest=np.asarray(x, float), inv_mass=np.asarray(w, float))
    if edges is not None:
        d["dist_idx"] = np.asarray(edges, np.int32)
        d["dist_compliance"] = np.asarray(comp, float)
    d.update(kw)
    b = _base("test", V, **d)
    b["gravity"] = np.asarray(gravity, float)
    return Scene(**b, frame_dt=frame_dt, substeps=substeps, iterations=iterations, frames=frames)


def test_two_particle_projection_golden():
    g = json.load(open(os.path.join(GOLD, "distance_projection.json")))
    for case in g["cases"]:
        dt = 0.1
        alpha = case["alpha_tilde"] * dt * dt
        s = scene_from([[0, 0, 0], [2.0, 0, 0]], [case["w_a"], case["w_b"]], [[0, 1]], [alpha],
                       frame_dt=dt)
        # rest length 1: overwrite x_rest-derived value
        m = OracleModel(s)
        m.rest = np.array([1.0])
        x1, _, rec = m.step(s.x0, np.zeros((2, 3)), record=True)
        np.testing.assert_allclose(x1[0], case["x_a_new"], atol=1e-15)
        np.testing.assert_allclose(x1[1], case["x_b_new"], atol=1e-15)
        assert rec["lam.dist"][0] == pytest.approx(case["dlambda"])


def test_pendulum_length_and_compliance():
    """Single distance constraint to a pinned vertex: alpha=0 keeps |x_b - x_a| = L exactly after every
    substep; alpha>0 stretches it by about m g alpha (spring elongation under gravity)."""
    L = 0.5
    x = [[0, 0, 0], [L, 0, 0]]
    s = scene_from(x, [0.0, 1.0], [[0, 1]], [0.0], frame_dt=1 / 60, substeps=10, gravity=(0, -9.81, 0),
                   frames=30)
    m = OracleModel(s)
    xs = m.simulate(s.x0, s.v0)
    for xn in xs[1:]:
        assert abs(np.linalg.norm(xn[1] - xn[0]) - L) < 1e-14
    # compliant spring hanging at rest: XPBD equilibrium elongation = m g alpha (alpha = 1/k)
    alpha = 1e-3
    s2 = scene_from([[0, 0, 0], [0, -L, 0]], [0.0, 1.0], [[0, 1]], [alpha], frame_dt=1 / 60,
                    substeps=10, iterations=1, gravity=(0, -9.81, 0), frames=600)
    m2 = OracleModel(s2)
    xs2 = m2.simulate(s2.x0, s2.v0)
    # damped by the implicit integrator; the end state is the static equilibrium
    assert abs(np.linalg.norm(xs2[-1][1]) - (L + 9.81 * alpha)) < 1e-6


def test_free_fall_closed_form():
    s = scene_from([[0.1, 0.2, 0.3]], [2.0], frame_dt=0.1, substeps=4, gravity=(0, -9.81, 0.5),
                   frames=3)
    m = OracleModel(s)
    v0 = np.array([[1.0, 2.0, -1.0]])
    xs = m.simulate(s.x0, v0)
    dt = s.dt
    for N, xn in enumerate(xs):
        exp = s.x0 + N * dt * v0 + dt * dt * np.array(s.gravity) * N * (N + 1) / 2
        np.testing.assert_allclose(xn, exp, atol=1e-13)


def test_predict_examples():
    s = scene_from([[0, 0, 0.0]], [1.0], frame_dt=0.1)
    m = OracleModel(s)
    np.testing.assert_allclose(m.predict(np.zeros((1, 3)), np.zeros((1, 3)), np.array([[0, -10.0, 0]])),
                               [[0, -0.1, 0]], atol=1e-15)
    s = scene_from([[0, 0, 0.0]], [1.0], frame_dt=0.5)
    m = OracleModel(s)
    np.testing.assert_allclose(m.predict(np.zeros((1, 3)), np.array([[1.0, 0, 0]]), np.zeros((1, 3))),
                               [[0.5, 0, 0]], atol=1e-15)
    s = scene_from([[1.0, 2, 3]], [0.0], frame_dt=0.5, gravity=(0, -9.81, 0))
    m = OracleModel(s)
    np.testing.assert_allclose(m.predict(s.x0, np.array([[1.0, 0, 0]]), np.ones((1, 3))), s.x0)


def test_pinned_never_move():
    s = tiny_cloth(n=6, frames=4)
    m = OracleModel(s)
    xs = m.simulate(s.x0, s.v0)
    pins = ~m.free
    for xn in xs:
        np.testing.assert_array_equal(xn[pins], s.x0[pins])


@pytest.mark.parametrize("with_tets", [False, True])
def test_momentum_conservation(with_tets):
    """No gravity, no pins: internal constraint impulses cancel (Eq. position update with M^-1)."""
    if with_tets:
        t = tet_block(3, 0.3, 1000.0, seed=5)
        w = t["inv_mass"].copy()
        w[w == 0] = w.max()
        s = scene_from(t["x_rest"], w, tet_idx=t["tet_idx"], tet_a=t["tet_a"], tet_b=t["tet_b"],
                       frame_dt=1 / 60, substeps=5, iterations=3, frames=2)
    else:
        c = cloth_grid(5, 4, 1.0, 0.8, 0.0, 1e-3, seed=3)
        w = 1.0 / rng.uniform(0.5, 2.0, size=20) * 1e3
        s = scene_from(c["x_rest"], w, c["dist_idx"], c["dist_compliance"] * 1e4, frame_dt=1 / 60,
                       substeps=5, iterations=3, frames=2)
    m = OracleModel(s)
    x0 = s.x_rest + 0.05 * rng.normal(size=s.x_rest.shape)
    v0 = rng.normal(size=s.x_rest.shape)
    mass = 1.0 / w
    p0 = (mass[:, None] * v0).sum(0)
    x, v = x0, v0
    for _ in range(6):
        x, v, _ = m.step(x, v)
        p = (mass[:, None] * v).sum(0)
        assert np.abs(p - p0).max() < 1e-10 * max(1.0, np.abs(p0).max())


def test_residual_decreases_with_iterations():
    """alpha = 0, a stretched swatch: ||C|| after K GS sweeps is non-increasing in K."""
    c = cloth_grid(6, 6, 1.0, 1.0, 0.0, 1e-3, seed=0)
    s0 = scene_from(c["x_rest"], c["inv_mass"], c["dist_idx"], np.zeros(len(c["dist_idx"])),
                    frame_dt=1 / 60)
    x_str = s0.x_rest * np.array([1.2, 1.0, 1.1]) + 0.01 * rng.normal(size=s0.x_rest.shape)
    res = []
    for K in (1, 2, 4, 8, 16):
        s = s0.replace(iterations=K)
        m = OracleModel(s)
        x1, _, _ = m.step(x_str, np.zeros_like(x_str))
        d = np.linalg.norm(x1[m.dist_idx[:, 0]] - x1[m.dist_idx[:, 1]], axis=1) - m.rest
        res.append(np.linalg.norm(d))
    assert all(b <= a + 1e-15 for a, b in zip(res, res[1:])), res
    assert res[-1] < 0.5 * res[0]


def test_collision_projection_to_thickness():
    """One vertex inside a sphere, alpha = 0: one projection moves it to gap = h (Eq. xpbd, scalar)."""
    s = scene_from([[0.0, 0.28, 0.0]], [1000.0], frame_dt=1 / 600, spheres=np.array([[0, 0, 0, 0.3]]),
                   thickness=0.005, collision_compliance=0.0)
    m = OracleModel(s)
    x1, _, _ = m.step(s.x0, np.zeros((1, 3)))
    assert np.linalg.norm(x1[0]) == pytest.approx(0.305, abs=1e-14)
    # above the surface by more than h: untouched (unilateral)
    s2 = s.replace(x_rest=np.array([[0.0, 0.4, 0]]), x0=np.array([[0.0, 0.4, 0]]))
    m2 = OracleModel(s2)
    x2, _, _ = m2.step(s2.x0, np.zeros((1, 3)))
    np.testing.assert_allclose(x2, s2.x0, atol=0)


def test_tet_hydrostatic_converges_to_volume_preservation():
    """Stiff hydrostatic row (huge lambda, K = 60 iterations): det F -> 1 (C_H = det F - 1,
    PAPER.md l.229, R6)."""
    t = tet_block(2, 1.0, 1000.0, seed=1)
    w = np.full(8, 1.0)
    s = scene_from(t["x_rest"], w, tet_idx=t["tet_idx"][:1], tet_a=np.array([1e-3]),
                   tet_b=np.array([1e6]), frame_dt=1 / 60, iterations=60)
    m = OracleModel(s)
    x = s.x_rest * 1.1
    x1, _, _ = m.step(x, np.zeros_like(x))
    from oracle import constraints as cf
    F = cf.tet_F(x1[m.tet_idx], m.Dminv)
    assert np.linalg.det(F[0]) == pytest.approx(1.0, abs=1e-6)


def _block(n=6, **kw):
    from synth import as_float32_exact
    return as_float32_exact(volumetric_block(n=n, frames=1, substeps=20, **kw))


def test_tet_rest_state_is_fixed_point():
    """Zero gravity, start at rest: every constraint is zero (R6), so dlam = 0 and the block must
    stay exactly at rest (config stiffness E in 1e4..1e6 Pa, 1 iteration / substep, 100 substeps)."""
    s = _block(6).replace(gravity=np.zeros(3))
    m = OracleModel(s)
    x, v = s.x0.copy(), s.v0.copy()
    for _ in range(100):
        x, v, _ = m.step(x, v)
    assert np.abs(x - s.x0).max() < 1e-12
    assert np.abs(v).max() < 1e-10


def test_tet_block_bounded_under_gravity():
    """Bottom face pinned, gravity on: the block sags and oscillates but stays bounded (no
    blow-up): after 400 substeps (20 frames) the top layer is above the floor, below its rest
    height + 1 cm, and no vertex moves faster than 10 m/s (free fall over the run: 3.3 m/s)."""
    s = _block(6)
    m = OracleModel(s)
    x, v = s.x0.copy(), s.v0.copy()
    vmax = 0.0
    for _ in range(400):
        x, v, _ = m.step(x, v)
        vmax = max(vmax, float(np.abs(v).max()))
    top = s.x0[:, 1] > s.x0[:, 1].max() - 1e-9
    assert vmax < 10.0
    assert np.all(x[top, 1] > 0.0) and np.all(x[top, 1] < s.x0[top, 1] + 0.01)
    assert np.all(np.isfinite(x))


def test_tet_self_sensitivity_one_frame():
    """A 1e-9 m perturbation of x0 changes the state after one full frame (20 substeps) by at
    most 1e-6 m (well-conditioned integrator at the config's stiffness)."""
    s = _block(6)
    m = OracleModel(s)
    rng_ = np.random.default_rng(3)
    dx = 1e-9 * rng_.standard_normal(s.x0.shape) * m.free[:, None]
    xa, va = s.x0.copy(), s.v0.copy()
    xb, vb = s.x0 + dx, s.v0.copy()
    for _ in range(20):
        xa, va, _ = m.step(xa, va)
        xb, vb, _ = m.step(xb, vb)
    assert np.abs(xa - xb).max() < 1e-6


# ------------------------------------------------------------------ coloring
@pytest.mark.parametrize("trial", range(6))
def test_greedy_coloring_c_vs_python_and_minimality(trial):
    V = int(rng.integers(5, 40))
    k = int(rng.integers(2, 5))
    n = int(rng.integers(1, 80))
    idx = np.array([rng.choice(V, size=k, replace=False) for _ in range(n)], np.int32)
    c = greedy_color(idx, V)
    cp = greedy_color_py(idx, V)
    np.testing.assert_array_equal(c, cp)
    # validity + greedy minimality (brute force)
    for j in range(n):
        for i in range(j):
            if c[i] == c[j]:
                assert not set(idx[i]) & set(idx[j])
        earlier = {c[i] for i in range(j) if set(idx[i]) & set(idx[j])}
        assert c[j] == min(set(range(len(earlier) + 1)) - earlier)


def test_grid_coloring_counts():
    s = tiny_cloth(n=16)
    c = greedy_color(s.dist_idx, s.num_vertices)
    assert c.max() + 1 == 12     # 2 structural-u, 2 structural-v, 4 shear, 2+2 bending
    b = volumetric_block(n=5)
    ct = greedy_color(b.tet_idx, b.num_vertices)
    assert ct.max() + 1 <= 64
