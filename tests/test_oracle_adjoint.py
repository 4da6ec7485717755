"""Pins of the oracle's derivative accumulation (Sec.4.3/4.4), PD projection use,
filtered solve (Sec.4.2.1) and adjoint recursion (Eqs. rawAdjoint/adjointXPBD/gradientRule)."""
import copy

import numpy as np
import pytest

from oracle import OracleModel
from oracle import constraints as cf
from synth import Scene, cloth_grid, tiny_cloth
from synth.scenes import _base

rng = np.random.default_rng(2024)


def mk(x, w, frame_dt=0.01, substeps=1, iterations=1, gravity=(0, 0, 0), frames=1, **kw):
    d = dict(x_rest=np.asarray(x, float), inv_mass=np.asarray(w, float))
    d.update(kw)
    b = _base("t", len(x), **d)
    b["gravity"] = np.asarray(gravity, float)
    return Scene(**b, frame_dt=frame_dt, substeps=substeps, iterations=iterations, frames=frames)


def fd(f, u, h):
    u = np.asarray(u, float)
    out = []
    for i in range(u.size):
        e = np.zeros_like(u)
        e.flat[i] = h
        out.append((np.asarray(f(u + e)) - np.asarray(f(u - e))) / (2 * h))
    return np.stack(out, -1)


def rel(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


# ----------------------------------------------------------------------------------------------
# P1: fixed-iterate multiplier iteration.  With the stencil positions held fixed, K applications
# of Eq. xpbd give lambda_K(x,u) = Sum_k dlambda_k, and the Sec.4.3 accumulation must equal
#   D = d/dx [lambda_K(x) grad C(x)^T]   and   e = d/du [lambda_K(x,u) grad C(x,u)^T]
# exactly.  This pins every term of d dlam/dx, db/dx (running sum), dJ/dx dlam, and d dlam/du.
# ----------------------------------------------------------------------------------------------
def _family_setup(fam):
    if fam == "dist":
        x = rng.normal(size=(2, 3))
        w = rng.uniform(0.5, 2.0, size=2)
        s = mk(x * 0.8, w, dist_idx=np.array([[0, 1]]), dist_compliance=np.array([3e-4]))
        m = OracleModel(s)
        st, rows = np.array([[0, 1]]), np.array([0])

        def ev(m, x):
            return m.ev_dist(x, rows)

        def at(m):
            return m.at_dist[rows][:, None]

        def get_u(m):
            return m.alpha.copy()

        def set_u(m, u):
            m.set_compliance(u)
        key = "dist"
    elif fam == "tet":
        xr = rng.normal(size=(4, 3))
        w = rng.uniform(0.5, 2.0, size=4)
        s = mk(xr, w, tet_idx=np.array([[0, 1, 2, 3]]), tet_a=np.array([0.9]), tet_b=np.array([1.7]))
        m = OracleModel(s)
        x = xr + 0.15 * rng.normal(size=(4, 3))
        st, rows = np.array([[0, 1, 2, 3]]), np.array([0])

        def ev(m, x):
            return m.ev_tet(x, rows)

        def at(m):
            return np.stack([m.at_D[rows], m.at_H[rows]], 1)

        def get_u(m):
            return np.array([m.ta[0], m.tb[0]])

        def set_u(m, u):
            m.set_material(u[:1], u[1:])
        key = fam
    elif fam == "sph":
        x = np.array([[0.1, 0.25, -0.05]])
        w = np.array([1.3])
        s = mk(x, w, spheres=np.array([[0.0, 0.0, 0.0, 0.3]]), thickness=0.01, collision_compliance=2e-4)
        m = OracleModel(s)
        st, rows = np.array([[0]]), np.array([0])

        def ev(m, x):
            return m.ev_sphere(x, 0, np.array([0]))

        def at(m):
            return np.array([[m.at_coll]])

        def get_u(m):
            return m.spheres[0].copy()

        def set_u(m, u):
            m.spheres = u[None].copy()
        key = "sph"
    else:  # capsule, endpoint region so that L matters
        x = np.array([[0.15, 0.32, 0.02]])
        w = np.array([0.7])
        s = mk(x, w, cap_center=np.array([[0.0, 0.0, 0.0]]), cap_axis=np.array([[0.0, 1.0, 0.0]]),
               cap_r0=np.array([0.2]), cap_L0=np.array([0.5]), cap_rbasis=np.zeros((1, 0)),
               cap_lbasis=np.zeros((1, 0)), thickness=0.01, collision_compliance=2e-4)
        m = OracleModel(s)
        st, rows = np.array([[0]]), np.array([0])

        def ev(m, x):
            return m.ev_capsule(x, 0, np.array([0]))

        def at(m):
            return np.array([[m.at_coll]])

        def get_u(m):
            return np.array([m.cap_r[0], m.cap_L[0]])

        def set_u(m, u):
            m.cap_r, m.cap_L = u[:1].copy(), u[1:].copy()
        key = "cap"
    return m, x, st, rows, ev, at, get_u, set_u, key


def _accumulate(m, x, st, rows, ev, at, key, K):
    rec = m.new_record()
    lam = np.zeros((max(len(rec[key + ".S"]), 1), at(m).shape[1]))
    for _ in range(K):
        m._project(x.copy(), st, ev(m, x), at(m), lam, rec, key, rows)   # x held fixed
    return rec, lam


def _lamK_g(m, x, ev, at, K, st):
    """Plain multiplier iteration at fixed x, written from Eq. xpbd; returns lambda_K * grad C."""
    e = ev(m, x)
    C, g = e["C"][0], e["g"][0]                        # (m,), (m,3k)
    wst = np.repeat(m.w[st[0]], 3)
    a = at(m)[0]
    J = (g * wst) @ g.T + np.diag(a)
    lam = np.zeros(len(C))
    for _ in range(K):
        lam = lam + np.linalg.solve(J, -C - a * lam)
    return g.T @ lam


@pytest.mark.parametrize("fam", ["dist", "tet", "sph", "cap"])
@pytest.mark.parametrize("K", [1, 3])
def test_fixed_iterate_accumulation_matches_fd(fam, K):
    m, x, st, rows, ev, at, get_u, set_u, key = _family_setup(fam)
    rec, lam = _accumulate(m, x, st, rows, ev, at, key, K)
    D = rec[key + ".D"][0]
    Dfd = fd(lambda y: _lamK_g(m, y.reshape(x.shape), ev, at, K, st), x.ravel(), 1e-6)
    sl = st[0]
    Dfd = Dfd.reshape(len(sl) * 3, x.shape[0] * 3) if x.shape[0] == len(sl) else Dfd
    assert rel(D, Dfd) < 1e-6, (fam, K)
    # controls
    u0 = get_u(m)

    def fu(u):
        mm = copy.deepcopy(m)
        set_u(mm, u)
        return _lamK_g(mm, x, ev, at, K, st)

    efd = fd(fu, u0, 1e-7 * max(1.0, np.abs(u0).max()))
    e = rec[key + ".e"][0]          # (nu, 3k)
    assert rel(e.T, efd) < 1e-5, (fam, K)
    assert np.abs(lam[0]).max() > 0


@pytest.mark.parametrize("fam", ["dist", "tet", "sph", "cap"])
def test_converged_block_symmetry_rowsum(fam):
    """PAPER.md Sec.4.3.1: at convergence M dDx/dx is symmetric and stencil rows sum to zero."""
    m, x, st, rows, ev, at, get_u, set_u, key = _family_setup(fam)
    if fam == "tet":
        # soften so the running sum converges within K iterations
        m.at_D = m.at_D * 0 + 5.0
        m.at_H = m.at_H * 0 + 7.0
    elif fam == "dist":
        m.at_dist = m.at_dist * 0 + 2.0
    else:
        m.at_coll = 2.0
    rec, lam = _accumulate(m, x, st, rows, ev, at, key, 400)
    D = rec[key + ".D"][0]
    assert np.abs(D - D.T).max() < 1e-9 * np.abs(D).max()
    if D.shape[0] > 3:
        assert np.abs(D.reshape(-1, 3, D.shape[1]).sum(0)).max() < 1e-9 * np.abs(D).max()
    # converged value: lambda H - g g^T / at
    e = ev(m, x)
    a = at(m)[0]
    g = e["g"][0]
    Dc = np.einsum("a,aij->ij", lam[0], e["H"][0]) - g.T @ np.diag(1.0 / a) @ g
    np.testing.assert_allclose(D, Dc, rtol=1e-8, atol=1e-10 * np.abs(D).max())


# ----------------------------------------------------------------------------------------------
# P5: 1-D chain (motion along the chain axis only, unequal masses).  grad C is constant, so the
# converged XPBD step is the exact implicit step and the paper's adjoint is the exact derivative:
# central FD of the whole simulation must match to ~1e-6 (pins Eq. adjointXPBD with the M
# handling of R4, the recursion of Eq. rawAdjoint and every gradient of Eq. gradientRule).
# ----------------------------------------------------------------------------------------------
def _chain_scene(K=300, steps=4):
    x = np.array([[0.0, 0, 0], [1.0, 0, 0], [2.1, 0, 0], [2.9, 0, 0]])
    w = 1.0 / np.array([1.0, 2.0, 0.5, 1.5])
    dt = 0.05
    e = np.array([[0, 1], [1, 2], [2, 3]])
    comp = np.array([1.0, 0.6, 1.7]) * dt * dt        # at ~ 1: soft enough to converge fast
    s = mk(x, w, frame_dt=dt, substeps=1, iterations=K, frames=steps, dist_idx=e,
           dist_compliance=comp)
    x0 = x + np.array([[0.05, 0, 0], [-0.02, 0, 0], [0.1, 0, 0], [0.0, 0, 0]])
    v0 = np.array([[0.3, 0, 0], [-0.1, 0, 0], [0.2, 0, 0], [-0.4, 0, 0]])
    forces = np.zeros((steps, 4, 3))
    forces[:, :, 0] = rng.normal(size=(steps, 4)) * 0.5
    tgt = x0 + np.array([[0.1, 0, 0]]) * np.arange(4)[:, None]
    return s.replace(x0=x0, v0=v0, forces=forces, key_frames=np.array([2, steps], np.int32),
                     targets=np.stack([tgt, tgt + np.array([0.05, 0, 0])]))


def _phi(s, m=None):
    m = OracleModel(s, pd_projection=False) if m is None else m
    xs = m.simulate(s.x0, s.v0, s.forces, s.frames)
    return m.loss(xs, s.key_frames, s.targets)[0]


def test_chain_adjoint_matches_fd():
    s = _chain_scene()
    m = OracleModel(s, pd_projection=False)
    xs = m.simulate(s.x0, s.v0, s.forces)
    phi, gr = m.backward(xs, s.v0, s.forces)
    h = 1e-6
    gx = fd(lambda u: _phi(s.replace(x0=s.x0 + np.pad(u[:, None], ((0, 0), (0, 2))))), np.zeros(4), h)
    gv = fd(lambda u: _phi(s.replace(v0=s.v0 + np.pad(u[:, None], ((0, 0), (0, 2))))), np.zeros(4), h)
    assert rel(gr["x0"][:, 0], gx) < 1e-6
    assert rel(gr["v0"][:, 0], gv) < 1e-6
    for fr in range(s.frames):
        def ff(u, fr=fr):
            F = s.forces.copy()
            F[fr, :, 0] += u
            return _phi(s.replace(forces=F))
        assert rel(gr["forces"][fr, :, 0], fd(ff, np.zeros(4), h)) < 1e-6
    ga = fd(lambda u: _phi(s.replace(dist_compliance=u)), s.dist_compliance, 1e-9)
    assert rel(gr["compliance"], ga) < 1e-5
    # transverse components are exactly zero (no transverse excitation)
    assert np.abs(gr["v0"][:, 1:]).max() < 1e-14


def test_chain_literal_left_multiply_differs_with_unequal_masses():
    """R4: solving (M - D) xhat = M rhs (literal "left multiply by M") is not the adjoint when
    masses differ; our (M - D) y = rhs, xhat = M y is (the FD test above)."""
    s = _chain_scene()
    m = OracleModel(s, pd_projection=False)
    xs = m.simulate(s.x0, s.v0, s.forces)
    _, gr, steps = m.backward(xs, s.v0, s.forces, keep=True)
    st = steps[0]
    y = st["y"]
    A = m.system_matrix(st["Q"]).toarray()
    xhat_literal = np.linalg.solve(A, np.repeat(m.m, 3) * st["r"].ravel())
    assert rel(xhat_literal, (m.m[:, None] * y).ravel()) > 1e-3


# ----------------------------------------------------------------------------------------------
# closed forms, linearity, filtering
# ----------------------------------------------------------------------------------------------
def test_free_particle_gradients_closed_form():
    """Single free particle, mass m, N substeps, loss 1/2 |x_N - x*|^2:
    dphi/dx0 = e, dphi/dv0 = N dt e, dphi/df_frame = dt^2/m * (substeps of the frame) e."""
    mass = 2.5
    s = mk([[0.0, 1.0, 0.0]], [1 / mass], frame_dt=0.1, substeps=3, frames=2, gravity=(0, -9.81, 0))
    tgt = np.array([[0.3, 0.2, -0.1]])
    s = s.replace(v0=np.array([[1.0, 0.5, 0.0]]), forces=np.ones((2, 1, 3)),
                  key_frames=np.array([2], np.int32), targets=tgt[None])
    m = OracleModel(s)
    xs, phi, gr = m.run()
    e = xs[-1] - tgt
    N, dt = 6, s.dt
    np.testing.assert_allclose(gr["x0"], e, rtol=1e-12)
    np.testing.assert_allclose(gr["v0"], N * dt * e, rtol=1e-12)
    # force of frame 0 acts on substeps 0..2: x_N depends on f0 with weight dt^2/m * sum(N - n) ...
    w0 = sum(N - n for n in range(0, 3)) * dt * dt / mass
    w1 = sum(N - n for n in range(3, 6)) * dt * dt / mass
    np.testing.assert_allclose(gr["forces"][0], w0 * e, rtol=1e-12)
    np.testing.assert_allclose(gr["forces"][1], w1 * e, rtol=1e-12)
    assert phi == pytest.approx(0.5 * (e ** 2).sum())


def test_single_step_force_gradient():
    s = mk([[0.0, 0.0, 0.0]], [1.0], frame_dt=0.1, frames=1)
    tgt = np.array([[0.2, -0.1, 0.3]])
    s = s.replace(forces=np.zeros((1, 1, 3)), key_frames=np.array([1], np.int32), targets=tgt[None])
    xs, phi, gr = OracleModel(s).run()
    np.testing.assert_allclose(gr["forces"][0], 0.01 * (xs[1] - tgt), rtol=1e-13)


def test_zero_goal_zero_gradient_and_linearity():
    s = tiny_cloth(n=5, frames=2, substeps=2)
    m = OracleModel(s)
    xs = m.simulate(s.x0, s.v0)
    # targets equal to the simulated states: all gradients exactly zero
    phi0, g0 = m.backward(xs, s.v0, key_frames=np.array([2]), targets=xs[-1][None])
    assert phi0 == 0.0
    for k in ("x0", "v0", "compliance", "forces"):
        assert np.abs(g0[k]).max() == 0.0
    # linearity in dphi/dq: doubling the residual doubles every gradient
    d = 0.05 * rng.normal(size=xs[-1].shape)
    _, g1 = m.backward(xs, s.v0, key_frames=np.array([2]), targets=(xs[-1] - d)[None])
    _, g2 = m.backward(xs, s.v0, key_frames=np.array([2]), targets=(xs[-1] - 2 * d)[None])
    for k in ("x0", "v0", "compliance", "forces"):
        np.testing.assert_allclose(g2[k], 2 * g1[k], rtol=1e-9, atol=1e-14 * np.abs(g2[k]).max())


def test_filtered_solve():
    s = tiny_cloth(n=4, frames=1, substeps=1)
    m = OracleModel(s)
    xs = m.simulate(s.x0, s.v0)
    _, _, rec = m.step(xs[0], s.v0, record=True)
    Q = m.blocks(rec)
    r = rng.normal(size=(m.V, 3))
    y = m.solve(Q, r)
    assert np.all(y[~m.free] == 0.0)
    A = m.system_matrix(Q).toarray()
    fdof = np.repeat(m.free, 3)
    res = A[np.ix_(fdof, fdof)] @ y.ravel()[fdof] - r.ravel()[fdof]
    assert np.abs(res).max() < 1e-10 * np.abs(r).max()
    # r nonzero only on pinned vertices -> y = 0
    r2 = np.zeros_like(r)
    r2[~m.free] = 1.0
    assert np.abs(m.solve(Q, r2)).max() == 0.0
    # A = M only (no constraint blocks): y = M^-1 r
    Z = {k: v * 0 for k, v in Q.items()}
    np.testing.assert_allclose(m.solve(Z, r)[m.free], (m.w[:, None] * r)[m.free], rtol=1e-13)


def test_cg_solver_matches_direct():
    """solver="cg" (l.201 "PCG ... preferred") reaches the direct solve's solution: the same filtered
    system residual bound and the same gradients, on cloth with forces and keyframes."""
    from synth import large_cloth
    s = large_cloth(n=12, frames=2, substeps=3, side=0.05, key_frames=(1, 2))
    ga = []
    for solver in ("direct", "cg"):
        m = OracleModel(s, solver=solver)
        xs = m.simulate(s.x0, s.v0, s.forces, 2)
        phi, g = m.backward(xs, s.v0, s.forces, key_frames=np.array([1, 2]), targets=s.targets)
        ga.append(g)
        if solver == "cg":
            _, _, rec = m.step(xs[0], s.v0, s.forces[0], record=True)
            Q = m.blocks(rec)
            r = rng.normal(size=(m.V, 3))
            y = m.solve(Q, r)
            assert np.all(y[~m.free] == 0.0)
            A = m.system_matrix(Q)
            fdof = np.repeat(m.free, 3)
            res = A[fdof][:, fdof] @ y.ravel()[fdof] - r.ravel()[fdof]
            assert np.linalg.norm(res) <= 1e-12 * np.linalg.norm(r.ravel()[fdof])
    for k in ("forces", "x0", "v0", "compliance"):
        np.testing.assert_allclose(ga[1][k], ga[0][k], rtol=0, atol=1e-10 * np.abs(ga[0][k]).max())


def test_projected_system_is_spd():
    s = tiny_cloth(n=6, frames=1, substeps=1)
    m = OracleModel(s)
    x = s.x0 + 0.01 * rng.normal(size=s.x0.shape)   # mixed tension / compression
    _, _, rec = m.step(x, s.v0, record=True)
    Q = m.blocks(rec)
    assert all(np.linalg.eigvalsh(q).min() >= -1e-10 for q in Q["dist"])
    fdof = np.repeat(m.free, 3)
    A = m.system_matrix(Q).toarray()[np.ix_(fdof, fdof)]
    assert np.abs(A - A.T).max() < 1e-12 * np.abs(A).max()
    assert np.linalg.eigvalsh(A).min() > 0


def test_cloth_3d_fd_sanity():
    """Full 3-D cloth with curvature: the paper's adjoint is an approximation of the exact
    derivative of the discrete XPBD map (R3); in a soft, converged regime it agrees
    with central FD to a few percent and always points in the FD direction."""
    c = cloth_grid(3, 3, 0.4, 0.4, 0.0, 1e-2, seed=4, pins=(0, 2))
    dt = 1 / 60
    s = mk(c["x_rest"], c["inv_mass"], frame_dt=dt, substeps=2, iterations=80, frames=3,
           gravity=(0, -9.81, 0), dist_idx=c["dist_idx"],
           dist_compliance=np.full(len(c["dist_idx"]), 0.3 * dt * dt / 2))
    tgt = c["x_rest"] + np.array([0.0, -0.05, 0.02])
    s = s.replace(key_frames=np.array([3], np.int32), targets=tgt[None])
    m = OracleModel(s, pd_projection=False)
    xs = m.simulate(s.x0, s.v0)
    _, gr = m.backward(xs, s.v0)
    gv = fd(lambda u: _phi(s.replace(v0=u.reshape(-1, 3)), OracleModel(s, pd_projection=False)),
            s.v0.ravel(), 1e-6)
    cos = gv @ gr["v0"].ravel() / (np.linalg.norm(gv) * np.linalg.norm(gr["v0"]))
    assert cos > 0.99
    assert rel(gr["v0"].ravel(), gv) < 0.1


# ----------------------------------------------------------------------------------------------
# Collider parameters through a full simulation (Sec.5.3 chain rule, R7).  A particle
# pressed by gravity onto the top of a sphere / the top cap of a vertical capsule moves along the
# contact normal only, so (as for the chain) the converged adjoint is exact.
# ----------------------------------------------------------------------------------------------
def _contact_scene(kind):
    dt = 1 / 60
    base = dict(frame_dt=dt, substeps=2, iterations=200, frames=3, gravity=(0, -9.81, 0),
                thickness=0.01, collision_compliance=0.5 * dt * dt / 4)
    if kind == "sphere":
        s = mk([[0.0, 0.31, 0.0]], [2.0], spheres=np.array([[0.0, 0.0, 0.0, 0.3]]), **base)
    else:
        Rb = np.array([[0.3, -0.2]])
        Lb = np.array([[0.5, 0.25]])
        s = mk([[0.0, 0.51, 0.0]], [2.0], cap_center=np.array([[0.0, 0.1, 0.0]]),
               cap_axis=np.array([[0.0, 1.0, 0.0]]), cap_r0=np.array([0.1]), cap_L0=np.array([0.6]),
               cap_rbasis=Rb, cap_lbasis=Lb, shape_beta=np.array([0.1, -0.2]), **base)
    tgt = np.array([[0.0, 0.2, 0.0]])
    return s.replace(v0=np.array([[0.0, -0.2, 0.0]]), key_frames=np.array([3], np.int32),
                     targets=tgt[None])


def test_sphere_params_fd():
    s = _contact_scene("sphere")
    m = OracleModel(s, pd_projection=False)
    xs, phi, gr = m.run()
    assert (xs[-1][0, 1] < 0.31)
    g = fd(lambda u: _phi(s.replace(spheres=u[None])), s.spheres[0], 1e-7)
    assert rel(gr["sphere"][0, [1, 3]], g[[1, 3]]) < 1e-6
    assert abs(gr["sphere"][0, 0]) < 1e-12 and abs(gr["sphere"][0, 2]) < 1e-12


def test_capsule_shape_coeff_fd():
    s = _contact_scene("capsule")
    m = OracleModel(s, pd_projection=False)
    xs, phi, gr = m.run()
    g = fd(lambda u: _phi(s.replace(shape_beta=u)), s.shape_beta, 1e-7)
    assert rel(gr["shape"], g) < 1e-6


def test_tet_material_fd_sanity():
    """Small soft block, converged iterations: material gradient points along FD (R3 approximation)."""
    from synth import tet_block
    t = tet_block(3, 0.2, 1000.0, seed=9, E_range=(2e3, 5e3))
    dt = 1 / 60
    s = mk(t["x_rest"], t["inv_mass"], frame_dt=dt, substeps=1, iterations=30, frames=2,
           gravity=(0, -9.81, 0), tet_idx=t["tet_idx"], tet_a=t["tet_a"], tet_b=t["tet_b"])
    tgt = t["x_rest"] + np.array([0.0, -0.01, 0.003])
    s = s.replace(key_frames=np.array([2], np.int32), targets=tgt[None])
    m = OracleModel(s, pd_projection=False)
    xs, phi, gr = m.run()
    ab = np.concatenate([s.tet_a, s.tet_b])
    T = len(s.tet_a)
    sel = rng.choice(2 * T, size=8, replace=False)

    def f(u):
        v = ab.copy()
        v[sel] = u
        return _phi(s.replace(tet_a=v[:T], tet_b=v[T:]))
    g = fd(f, ab[sel], 1e-4)
    ga = np.concatenate([gr["material"][:, 0], gr["material"][:, 1]])[sel]
    cos = g @ ga / (np.linalg.norm(g) * np.linalg.norm(ga))
    assert cos > 0.98, cos


# ----------------------------------------------------------------------------------------------
# Tet PD projection in deformation-gradient coordinates (Sec.4.3.2 l.201, reading R5):
# Q = G^T psd(-sym D~) G with D~ = Gp^T D Gp.  Pinned without re-deriving the formula: the
# result must be PSD, keep the translation null space, equal -sym(D) when that is already PSD,
# and its F-space image must be the Frobenius-nearest PSD matrix to -S (checked against random
# PSD candidates).
# ----------------------------------------------------------------------------------------------
def _tet_blocks_case(S):
    from synth import tet_block
    t = tet_block(2, 0.3, 1000.0, seed=4)
    s = mk(t["x_rest"], t["inv_mass"] + 1.0, tet_idx=t["tet_idx"][:3], tet_a=t["tet_a"][:3],
           tet_b=t["tet_b"][:3])
    m = OracleModel(s, pd_projection=True)
    rec = m.new_record()
    rec["tet.D"] = np.einsum("nai,nab,nbj->nij", m.G, S, m.G)    # D = G^T S G (a function of F)
    return m, m.blocks(rec)["tet"]


def test_tet_fspace_pd_projection_psd_input_unchanged():
    Z = rng.normal(size=(3, 9, 9))
    S = -(Z @ np.swapaxes(Z, 1, 2))                      # -S PSD
    m, Q = _tet_blocks_case(S)
    D = np.einsum("nai,nab,nbj->nij", m.G, S, m.G)
    np.testing.assert_allclose(Q, -0.5 * (D + np.swapaxes(D, 1, 2)), atol=1e-9 * np.abs(D).max())


def test_tet_fspace_pd_projection_properties():
    B = rng.normal(size=(3, 9, 9))
    S = B + np.swapaxes(B, 1, 2)                         # indefinite
    m, Q = _tet_blocks_case(S)
    for j in range(3):
        ev = np.linalg.eigvalsh(Q[j])
        assert ev.min() >= -1e-9 * np.abs(ev).max()
        assert np.sum(ev > 1e-9 * np.abs(ev).max()) <= 9           # rank <= 9 (image of G^T)
        tr = np.tile(rng.normal(size=3), 4)                        # rigid translation
        assert np.abs(Q[j] @ tr).max() < 1e-9 * np.abs(Q[j]).max()
        # F-space image: G Q G^T = (G G^T) P (G G^T) with P the projected matrix; recover P
        GGt = m.G[j] @ m.G[j].T
        P = np.linalg.solve(GGt, np.linalg.solve(GGt, m.G[j] @ Q[j] @ m.G[j].T).T).T
        assert np.abs(P - P.T).max() < 1e-9 * np.abs(P).max()
        assert np.linalg.eigvalsh(P).min() >= -1e-9 * np.abs(P).max()
        # Frobenius-nearest PSD matrix to -S[j]
        dP = np.linalg.norm(-S[j] - P)
        for _ in range(50):
            Z = rng.normal(size=(9, int(rng.integers(1, 10))))
            assert dP <= np.linalg.norm(-S[j] - Z @ Z.T) + 1e-12
        for _ in range(50):                                        # nor any nearby PSD matrix P + e v v^T
            v = rng.normal(size=9)
            assert dP <= np.linalg.norm(-S[j] - P - 1e-2 * np.outer(v, v)) + 1e-12
