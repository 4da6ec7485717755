"""Pins of oracle/constraints.py and oracle.xpbd.psd_project against closed forms,
central finite differences and invariances."""
import json
import os

import numpy as np
import pytest

from oracle import constraints as cf
from oracle.xpbd import psd_project

rng = np.random.default_rng(1234)
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def fd_jac(f, x, h=1e-6):
    x = np.asarray(x, float)
    f0 = np.asarray(f(x))
    J = np.zeros(f0.shape + x.shape)
    for i in np.ndindex(x.shape):
        e = np.zeros_like(x)
        e[i] = h
        J[(Ellipsis,) + i] = (np.asarray(f(x + e)) - np.asarray(f(x - e))) / (2 * h)
    return J


def rel(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


# ------------------------------------------------------------------ distance
def test_distance_closed_form():
    g = json.load(open(os.path.join(GOLD, "distance_projection.json")))
    xs = np.array([[[0.0, 0, 0], [2.0, 0, 0]]])
    C, gr, H, l = cf.distance(xs, np.array([1.0]))
    assert C[0] == pytest.approx(g["C"])
    np.testing.assert_allclose(gr[0], g["grad"], atol=0)


@pytest.mark.parametrize("trial", range(5))
def test_distance_fd(trial):
    xs = rng.normal(size=(1, 2, 3))
    L = np.array([0.7])
    f = lambda y: cf.distance(y.reshape(1, 2, 3), L)[0][0]
    g = lambda y: cf.distance(y.reshape(1, 2, 3), L)[1][0]
    x = xs.ravel()
    C, gr, H, _ = cf.distance(xs, L)
    assert rel(gr[0], fd_jac(f, x)) < 1e-8
    assert rel(H[0], fd_jac(g, x)) < 1e-7
    assert np.abs(H[0] - H[0].T).max() < 1e-12
    # translation invariance
    assert abs(f(x + np.tile([0.3, -1, 2], 2)) - C[0]) < 1e-12
    assert np.abs(gr[0][:3] + gr[0][3:]).max() < 1e-15


# ------------------------------------------------------------------ colliders
@pytest.mark.parametrize("trial", range(4))
def test_sphere_fd(trial):
    c = rng.normal(size=3)
    r, h = 0.4, 0.01
    x = c + rng.normal(size=(1, 3)) * 0.5
    C, g, H, dCdu, dgdu, _ = cf.sphere(x, c, r, h)
    f = lambda y: cf.sphere(y.reshape(1, 3), c, r, h)[0][0]
    gg = lambda y: cf.sphere(y.reshape(1, 3), c, r, h)[1][0]
    assert rel(g[0], fd_jac(f, x.ravel())) < 1e-8
    assert rel(H[0], fd_jac(gg, x.ravel())) < 1e-7
    u = np.concatenate([c, [r]])
    fu = lambda u: cf.sphere(x, u[:3], u[3], h)[0][0]
    gu = lambda u: cf.sphere(x, u[:3], u[3], h)[1][0]
    assert rel(dCdu[0], fd_jac(fu, u)) < 1e-8
    assert rel(dgdu[0], fd_jac(gu, u).T) < 1e-7


def test_sphere_gap_examples():
    c = np.zeros(3)
    C, *_ = cf.sphere(np.array([[0, 1.005, 0.0]]), c, 1.0, 0.0)
    assert C[0] == pytest.approx(0.005)
    C, g, *_ = cf.sphere(np.array([[0, 1.0, 0.0]]), c, 1.0, 0.0)
    assert C[0] == 0.0 and np.allclose(g[0], [0, 1, 0])


@pytest.mark.parametrize("where", ["interior", "top", "bottom"])
def test_capsule_fd(where):
    c = np.array([0.1, 0.2, -0.3])
    a = rng.normal(size=3)
    a /= np.linalg.norm(a)
    r, L, h = 0.2, 0.6, 0.005
    perp = np.cross(a, [1.0, 0, 0])
    perp /= np.linalg.norm(perp)
    sv = {"interior": 0.1, "top": 0.5, "bottom": -0.45}[where]
    x = (c + sv * a + 0.35 * perp)[None]
    C, g, H, dCdu, dgdu, _ = cf.capsule(x, c, a, r, L, h)
    f = lambda y: cf.capsule(y.reshape(1, 3), c, a, r, L, h)[0][0]
    gg = lambda y: cf.capsule(y.reshape(1, 3), c, a, r, L, h)[1][0]
    assert rel(g[0], fd_jac(f, x.ravel())) < 1e-8
    assert rel(H[0], fd_jac(gg, x.ravel())) < 1e-6
    assert np.abs(H[0] - H[0].T).max() < 1e-12
    u = np.array([r, L])
    fu = lambda u: cf.capsule(x, c, a, u[0], u[1], h)[0][0]
    gu = lambda u: cf.capsule(x, c, a, u[0], u[1], h)[1][0]
    assert rel(dCdu[0], fd_jac(fu, u)) < 1e-8
    np.testing.assert_allclose(dgdu[0], fd_jac(gu, u).T, atol=1e-8)


# ------------------------------------------------------------------ tets
def _unit_tet():
    x = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]])
    return x, np.array([[0, 1, 2, 3]])


def test_tet_rest_values():
    """PAPER.md l.229 (reading R6): C_D = ||F||_F - sqrt 3 and C_H = det F - 1 both vanish at
    rest (F = I), so U = 1/2 C^T alpha^-1 C (Eq. xpbdUenergy l.76) is zero there."""
    x, t = _unit_tet()
    Dminv, vol = cf.tet_rest(x, t)
    assert vol[0] == pytest.approx(1 / 6)
    G = cf.tet_G(Dminv)
    C, g, H = cf.tet(x[t], Dminv, G, "D")
    assert C[0] == pytest.approx(0.0, abs=1e-12)
    # grad C_D at F = I: dC/dF = I/sqrt3 -> vertex 1 gets column 0 of F: (1, 0, 0)/sqrt3
    np.testing.assert_allclose(g[0].reshape(4, 3)[1], [1 / np.sqrt(3), 0, 0], atol=1e-12)
    C, g, H = cf.tet(x[t], Dminv, G, "H")
    assert C[0] == pytest.approx(0.0, abs=1e-12)
    # grad C_H at F = I: cof(I) = I
    np.testing.assert_allclose(g[0].reshape(4, 3)[2], [0, 1, 0], atol=1e-12)
    # F = 2I: C_D = sqrt(12) - sqrt(3) = sqrt(3), det = 8
    C, *_ = cf.tet(2 * x[t], Dminv, G, "D")
    assert C[0] == pytest.approx(np.sqrt(3), abs=1e-12)
    C, *_ = cf.tet(2 * x[t], Dminv, G, "H")
    assert C[0] == pytest.approx(7.0, abs=1e-12)
    # pure shear F = [[1, 0.5, 0], [0, 1, 0], [0, 0, 1]]: det = 1, ||F||^2 = 3.25
    xs = x.copy()
    xs[2] = [0.5, 1.0, 0.0]
    C, *_ = cf.tet(xs[t], Dminv, G, "H")
    assert C[0] == pytest.approx(0.0, abs=1e-12)
    C, *_ = cf.tet(xs[t], Dminv, G, "D")
    assert C[0] == pytest.approx(np.sqrt(3.25) - np.sqrt(3), abs=1e-12)


def test_regular_tet_volume():
    x = np.array([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1.0]]) / np.sqrt(8)  # edge 1
    _, vol = cf.tet_rest(x, np.array([[0, 1, 2, 3]]))
    assert vol[0] == pytest.approx(np.sqrt(2) / 12)


@pytest.mark.parametrize("kind", ["D", "H"])
@pytest.mark.parametrize("trial", range(3))
def test_tet_fd_and_invariances(kind, trial):
    xr = rng.normal(size=(4, 3))
    t = np.array([[0, 1, 2, 3]])
    Dminv, vol = cf.tet_rest(xr, t)
    G = cf.tet_G(Dminv)
    xs = xr + 0.2 * rng.normal(size=(4, 3))
    f = lambda y: cf.tet(y.reshape(1, 4, 3), Dminv, G, kind)[0][0]
    gg = lambda y: cf.tet(y.reshape(1, 4, 3), Dminv, G, kind)[1][0]
    C, g, H = cf.tet(xs[None], Dminv, G, kind)
    assert rel(g[0], fd_jac(f, xs.ravel())) < 1e-7
    assert rel(H[0], fd_jac(gg, xs.ravel())) < 1e-6
    assert np.abs(H[0] - H[0].T).max() < 1e-10 * np.abs(H[0]).max()
    # translation invariance: C unchanged, stencil row sums of grad and Hessian vanish
    assert abs(f(xs.ravel() + np.tile([1.0, -2, 0.5], 4)) - C[0]) < 1e-10
    assert np.abs(g[0].reshape(4, 3).sum(0)).max() < 1e-12
    assert np.abs(H[0].reshape(4, 3, 12).sum(0)).max() < 1e-10
    # rotation invariance
    Rm, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    if np.linalg.det(Rm) < 0:
        Rm[:, 0] *= -1
    assert abs(f((xs @ Rm.T).ravel()) - C[0]) < 1e-9


# ------------------------------------------------------------------ PD projection
def test_psd_examples():
    A = np.diag([2.0, 1, 1])
    np.testing.assert_allclose(psd_project(A), A, atol=1e-14)
    np.testing.assert_allclose(psd_project(np.array([[0.0, 1], [1, 0]])), [[0.5, 0.5], [0.5, 0.5]],
                               atol=1e-14)
    np.testing.assert_allclose(psd_project(np.zeros((3, 3))), 0, atol=0)
    for _ in range(20):
        B = rng.normal(size=(6, 6))
        B = B + B.T
        P = psd_project(B)
        assert np.linalg.eigvalsh(P).min() >= -1e-10
        # projection is idempotent and the nearest PSD matrix in Frobenius norm
        np.testing.assert_allclose(psd_project(P), P, atol=1e-10)
        for _k in range(5):
            Z = rng.normal(size=(6, 3))
            S = Z @ Z.T
            assert np.linalg.norm(B - P) <= np.linalg.norm(B - S) + 1e-12
