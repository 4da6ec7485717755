"""ORACLE (test infrastructure only). DiffXPBD forward substep and adjoint pass,
fp64, written from PAPER.md step by step.  Reading numbers R1..R12 refer to
DESIGN.md "Readings of the paper".

Forward (Sec.3.1, Eqs. xpbd / xpbdUpdateRule, l.79-96):
    x~ = x_n + dt (v_n + dt M^-1 f_ext)                    (gravity enters as f_ext = M g)
    lambda = 0; K iterations of Gauss-Seidel over constraints j (colored order, R1):
        dlam_j = (-C_j - at_j lam_j) / (grad C_j M^-1 grad C_j^T + at_j),  at = alpha / dt^2
        lam_j += dlam_j ;  x += M^-1 grad C_j^T dlam_j
    x_{n+1} = x ;  v_{n+1} = (x_{n+1} - x_n) / dt

Derivative blocks, accumulated per constraint and iteration at the iterate used
for the position update (Sec.4.3, l.166-194, "M^-1 omitted"):
    d dlam/dx = -J^-1 (dJ/dx dlam - db/dx),   db/dx = -grad C - at * Sum(prev d dlam/dx)
    dJ/dx dlam = 2 dlam H M^-1 grad C^T
    D_j += dlam H + grad C^T (d dlam/dx)            (D = M d(Delta x)/dx)
Controls u (Sec.4.4, l.203-205, same derivation with u in place of x):
    d dlam/du = J^-1 (-dC/du - dat/du lam - at Sum(prev d dlam/du) - dJ/du dlam)
    e_j += dlam d(grad C)/du + grad C^T d dlam/du    (M d(Delta x)/du)
Positive-definite projection once per step (Sec.4.3.2, l.200-201; R5): Q_j = psd(-sym D_j).

Adjoint (PAPER.md Eqs. rawAdjoint / adjointXPBD l.135-159, Supplement l.489-501;
index mapping and the symmetric form in R3/R4): with r = xbar_{n+1} + vbar_{n+1}/dt,
    (M + Sum_j Q_j)_free y = r_free        (filtered, Sec.4.2.1; pinned y = 0)
    z = M y     (paper's x^_n)
    xbar_n = z - vbar_{n+1}/dt + dphi/dx_n ;  vbar_n = dt z
Gradients (Eq. gradientRule l.110-112): dphi/du += e_j . y_stencil ;
    dphi/df_frame += dt^2 y  (R8) ; dphi/dx_0 = xbar_0 ; dphi/dv_0 = vbar_0.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import constraints as cf
from .coloring import greedy_color

_EPS_LEN = 1e-9


def psd_project(A: np.ndarray) -> np.ndarray:
    """Symmetric positive semi-definite projection by eigenvalue clamping
    (Sec.4.3.2 l.201 "project all derivative blocks to positive
    definiteness" [nocedal]; clamp floor 0, R5).  A (...,n,n) symmetric."""
    lam, V = np.linalg.eigh(A)
    lam = np.maximum(lam, 0.0)
    return np.einsum("...ij,...j,...kj->...ik", V, lam, V)


def _rows1(ev):
    """Single-row constraint: add the row axis m = 1 expected by OracleModel._project."""
    ev["C"] = ev["C"][:, None]
    ev["g"] = ev["g"][:, None, :]
    ev["H"] = ev["H"][:, None]
    ev["dCdu"] = ev["dCdu"][:, :, None]
    ev["dgdu"] = ev["dgdu"][:, :, None, :]
    ev["datdu"] = ev["datdu"][:, :, None]
    return ev


def sym(A):
    return 0.5 * (A + np.swapaxes(A, -1, -2))


class OracleModel:
    """fp64 oracle of one scene (synth.Scene)."""

    def __init__(self, scene, pd_projection: bool = True, solver: str = "direct"):
        s = scene
        self.s = s
        assert solver in ("direct", "cg")
        self.solver = solver
        self.V = s.num_vertices
        self.w = np.asarray(s.inv_mass, float)
        self.free = self.w > 0
        self.m = np.where(self.free, 1.0 / np.where(self.free, self.w, 1.0), 0.0)
        self.dt = s.frame_dt / s.substeps
        self.pd = pd_projection
        dt2 = self.dt * self.dt
        # distance constraints
        self.dist_idx = np.asarray(s.dist_idx, np.int64)
        self.E = len(self.dist_idx)
        xr = np.asarray(s.x_rest, float)
        if self.E:
            self.rest = np.linalg.norm(xr[self.dist_idx[:, 0]] - xr[self.dist_idx[:, 1]], axis=1)
        else:
            self.rest = np.zeros(0)
        self.set_compliance(np.asarray(s.dist_compliance, float))
        self.dist_color = greedy_color(self.dist_idx, self.V)
        self.dist_groups = [np.nonzero(self.dist_color == c)[0]
                            for c in range(int(self.dist_color.max()) + 1 if self.E else 0)]
        # tetrahedra (Sec.5.2; R6)
        self.tet_idx = np.asarray(s.tet_idx, np.int64)
        self.T = len(self.tet_idx)
        if self.T:
            self.Dminv, self.vol = cf.tet_rest(xr, self.tet_idx)
            self.G = cf.tet_G(self.Dminv)
            self.Gp = np.linalg.pinv(self.G)           # (T,12,9), G Gp = I_9
        self.set_material(np.asarray(s.tet_a, float), np.asarray(s.tet_b, float))
        self.tet_color = greedy_color(self.tet_idx, self.V)
        self.tet_groups = [np.nonzero(self.tet_color == c)[0]
                           for c in range(int(self.tet_color.max()) + 1 if self.T else 0)]
        # colliders (Sec.4.5, Sec.5.3; R7)
        self.spheres = np.asarray(s.spheres, float).reshape(-1, 4)
        self.cap_c = np.asarray(s.cap_center, float).reshape(-1, 3)
        self.cap_a = np.asarray(s.cap_axis, float).reshape(-1, 3)
        self.set_shape(np.asarray(s.shape_beta, float))
        self.h = float(s.thickness)
        self.at_coll = float(s.collision_compliance) / dt2
        self.gravity = np.asarray(s.gravity, float)

    # ------------------------------------------------------------ parameters
    def set_compliance(self, alpha):
        self.alpha = np.asarray(alpha, float)
        self.at_dist = self.alpha / self.dt ** 2

    def set_material(self, a, b):
        """mu = a^2, lambda = b^2; alpha_D = 1/(mu V), alpha_H = 1/(lambda V)."""
        self.ta, self.tb = np.asarray(a, float), np.asarray(b, float)
        if self.T:
            dt2 = self.dt ** 2
            self.at_D = 1.0 / (self.ta ** 2 * self.vol * dt2)
            self.at_H = 1.0 / (self.tb ** 2 * self.vol * dt2)

    def set_shape(self, beta):
        s = self.s
        self.beta = np.asarray(beta, float)
        nc = len(self.cap_c)
        if nc:
            self.cap_r = np.asarray(s.cap_r0, float) + np.asarray(s.cap_rbasis, float).reshape(nc, -1) @ self.beta
            self.cap_L = np.asarray(s.cap_L0, float) + np.asarray(s.cap_lbasis, float).reshape(nc, -1) @ self.beta
        else:
            self.cap_r = np.zeros(0)
            self.cap_L = np.zeros(0)

    @property
    def num_colliders(self):
        return len(self.spheres) + len(self.cap_c)

    # ------------------------------------------------------------ forward
    def predict(self, x, v, f):
        """x~ = x_n + dt (v_n + dt M^-1 f_ext), f_ext = M g + f  (Eq. xpbdUpdateRule l.91; R2)."""
        dt = self.dt
        xt = x + dt * v + dt * dt * (self.gravity[None] + self.w[:, None] * f)
        xt[~self.free] = x[~self.free]
        return xt

    def _project(self, x, st, ev, at, lam, rec, key, rows, active=None):
        """One Gauss-Seidel projection of a batch of vertex-disjoint block constraints with m rows
        each (Eqs. xpbd l.81 and l.85 in their matrix form; m = 1 except tets, m = 2, R6), plus the
        Sec.4.3/4.4 derivative accumulation in matrix form:
            J = grad C M^-1 grad C^T + diag(at),  b = -C - at*lam,  dlam = J^-1 b
            dJ/dx dlam = H_a Dx + Sum_b dlam_b H_b M^-1 g_a^T   (row a),  Dx = M^-1 grad C^T dlam
            d dlam/dx = J^-1 (db/dx - dJ/dx dlam),  db/dx = -grad C - at * Sum(prev d dlam/dx)
            D += Sum_a dlam_a H_a + Sum_a g_a^T (d dlam_a/dx)
        st: (N,k) vertex ids; ev: C (N,m), g (N,m,3k), H (N,m,3k,3k) (record only),
        dCdu (N,nu,m), dgdu (N,nu,m,3k), datdu (N,nu,m);  at: (N,m);  lam: indexed by rows."""
        C, g = ev["C"], ev["g"]
        N, k = st.shape
        m = C.shape[1]
        wst = np.repeat(self.w[st], 3, axis=1)                       # (N,3k) diagonal of M^-1
        ok = (self.w[st].sum(1) > 0) & (ev["len"] > _EPS_LEN)
        if active is not None:
            ok &= active
        gw = g * wst[:, None, :]                                       # g M^-1
        J = np.einsum("nai,nbi->nab", gw, g) + at[:, :, None] * np.eye(m)[None]
        detJ = np.linalg.det(J)
        ok &= np.abs(detJ) > 0
        Js = np.where(ok[:, None, None], J, np.eye(m)[None])
        Jinv = np.linalg.inv(Js)
        lam_r = lam[rows].reshape(N, m)
        b = -C - at * lam_r
        dl = np.where(ok[:, None], np.einsum("nab,nb->na", Jinv, b), 0.0)
        if rec is not None:
            H = ev["H"]
            S = rec[key + ".S"][rows].reshape(N, m, -1)
            Dx = np.einsum("nai,na->ni", gw, dl)                         # M^-1 grad C^T dlam
            Jx = (np.einsum("naij,nj->nai", H, Dx)
                  + np.einsum("nb,nbij,naj->nai", dl, H, gw))
            s = np.einsum("nab,nbi->nai", Jinv, -g - at[:, :, None] * S - Jx)
            s = np.where(ok[:, None, None], s, 0.0)
            rec[key + ".D"][rows] += (np.einsum("na,naij->nij", dl, H)
                                      + np.einsum("nai,naj->nij", g, s))
            rec[key + ".S"][rows] = (S + s).reshape(rec[key + ".S"][rows].shape)
            if "dCdu" in ev:
                dCdu, dgdu, datdu = ev["dCdu"], ev["dgdu"], ev["datdu"]   # (N,nu,m) ...
                Tu = rec[key + ".T"][rows].reshape(N, -1, m)
                dJ = (datdu[:, :, :, None] * np.eye(m)[None, None]
                      + np.einsum("nuai,nbi->nuab", dgdu * wst[:, None, None, :], g)
                      + np.einsum("nai,nubi->nuab", gw, dgdu))
                rhs = (-dCdu - datdu * lam_r[:, None, :] - at[:, None, :] * Tu
                       - np.einsum("nuab,nb->nua", dJ, dl))
                t = np.einsum("nab,nub->nua", Jinv, rhs)
                t = np.where(ok[:, None, None], t, 0.0)
                rec[key + ".e"][rows] += (np.einsum("na,nuai->nui", dl, dgdu)
                                          + np.einsum("nua,nai->nui", t, g))
                rec[key + ".T"][rows] = (Tu + t).reshape(rec[key + ".T"][rows].shape)
        lam[rows] = (lam_r + dl).reshape(lam[rows].shape)
        dx = np.einsum("nai,na->ni", gw, dl).reshape(N, k, 3)
        x[st] = x[st] + dx

    # per-family evaluators: C, grad C, Hessian and control partials at the current iterate
    def ev_dist(self, x, grp):
        """distance (cloth stretch/shear/bend); control u = own compliance alpha_j, dat/du = 1/dt^2."""
        n = len(grp)
        C, g, H, l = cf.distance(x[self.dist_idx[grp]], self.rest[grp])
        return _rows1(dict(C=C, g=g, H=H, len=l, dCdu=np.zeros((n, 1)), dgdu=np.zeros((n, 1, 6)),
                           datdu=np.full((n, 1), 1.0 / self.dt ** 2)))

    def ev_tet(self, x, grp, need_H=True):
        """Neo-Hookean block (Sec.5.2 l.229, R6): rows (C_D, C_H) = (||F|| - sqrt3,
        det F - 1) solved together; controls u = (a, b), mu = a^2, lambda = b^2,
        alpha_D = 1/(mu V), alpha_H = 1/(lambda V).  C does not depend on u (dC/du = 0)."""
        n = len(grp)
        a, b, V = self.ta[grp], self.tb[grp], self.vol[grp]
        dt2 = self.dt ** 2
        st = self.tet_idx[grp]
        CD, gD, HD = cf.tet(x[st], self.Dminv[grp], self.G[grp], "D", need_H=need_H)
        CH, gH, HH = cf.tet(x[st], self.Dminv[grp], self.G[grp], "H", need_H=need_H)
        z = np.zeros(n)
        datdu = np.stack([np.stack([-2.0 / (a ** 3 * V * dt2), z], 1),        # d/da (rows D, H)
                          np.stack([z, -2.0 / (b ** 3 * V * dt2)], 1)], 1)     # d/db
        dCdu = np.zeros((n, 2, 2))
        return dict(C=np.stack([CD, CH], 1), g=np.stack([gD, gH], 1),
                    H=np.stack([HD, HH], 1) if need_H else None,
                    len=np.ones(n), dCdu=dCdu, dgdu=np.zeros((n, 2, 2, 12)), datdu=datdu)

    def ev_sphere(self, x, ci, verts):
        c, r = self.spheres[ci, :3], self.spheres[ci, 3]
        C, g, H, dCdu, dgdu, dist = cf.sphere(x[verts], c, r, self.h)
        return _rows1(dict(C=C, g=g, H=H, len=dist, dCdu=dCdu, dgdu=dgdu,
                           datdu=np.zeros((len(verts), 4))))

    def ev_capsule(self, x, ki, verts):
        C, g, H, dCdu, dgdu, dist = cf.capsule(x[verts], self.cap_c[ki], self.cap_a[ki],
                                               self.cap_r[ki], self.cap_L[ki], self.h)
        return _rows1(dict(C=C, g=g, H=H, len=dist, dCdu=dCdu, dgdu=dgdu,
                           datdu=np.zeros((len(verts), 2))))

    def new_record(self):
        nsph, ncap, V, E, T = len(self.spheres), len(self.cap_c), self.V, self.E, self.T
        return {
            "dist.S": np.zeros((E, 6)), "dist.D": np.zeros((E, 6, 6)),
            "dist.T": np.zeros((E, 1)), "dist.e": np.zeros((E, 1, 6)),
            "tet.S": np.zeros((T, 2, 12)), "tet.D": np.zeros((T, 12, 12)),
            "tet.T": np.zeros((T, 2, 2)), "tet.e": np.zeros((T, 2, 12)),
            "sph.S": np.zeros((nsph * V, 3)), "sph.D": np.zeros((nsph * V, 3, 3)),
            "sph.T": np.zeros((nsph * V, 4)), "sph.e": np.zeros((nsph * V, 4, 3)),
            "cap.S": np.zeros((ncap * V, 3)), "cap.D": np.zeros((ncap * V, 3, 3)),
            "cap.T": np.zeros((ncap * V, 2)), "cap.e": np.zeros((ncap * V, 2, 3)),
        }

    def step(self, x_n, v_n, f=None, record: bool = False):
        """One XPBD substep (Eqs. xpbd, position update, xpbdUpdateRule).  With record=True
        also returns the Sec.4.3/4.4 derivative data of the step (replay, R9)."""
        s = self.s
        if f is None:
            f = np.zeros_like(x_n)
        x = self.predict(x_n, v_n, f)
        nsph, ncap = len(self.spheres), len(self.cap_c)
        lam_d = np.zeros(self.E)
        lam_t = np.zeros((self.T, 2))
        lam_s = np.zeros(nsph * self.V)
        lam_k = np.zeros(ncap * self.V)
        rec = self.new_record() if record else None
        freev = np.nonzero(self.free)[0]
        for _it in range(s.iterations):
            # 1) distance constraints, color by color (R1)
            for grp in self.dist_groups:
                self._project(x, self.dist_idx[grp], self.ev_dist(x, grp), self.at_dist[grp][:, None],
                              lam_d, rec, "dist", grp)
            # 2) tetrahedra, color by color; (C_D, C_H) as one 2-row block per tet (R6)
            for grp in self.tet_groups:
                at = np.stack([self.at_D[grp], self.at_H[grp]], 1)
                self._project(x, self.tet_idx[grp], self.ev_tet(x, grp, need_H=rec is not None), at, lam_t, rec,
                              "tet", grp)
            # 3) collisions: per free vertex, colliders in order (spheres, capsules), C<0 only (R7)
            for ci in range(nsph):
                ev = self.ev_sphere(x, ci, freev)
                self._project(x, freev[:, None], ev, np.full((len(freev), 1), self.at_coll), lam_s, rec,
                              "sph", ci * self.V + freev, active=ev["C"][:, 0] < 0)
            for ki in range(ncap):
                ev = self.ev_capsule(x, ki, freev)
                self._project(x, freev[:, None], ev, np.full((len(freev), 1), self.at_coll), lam_k, rec,
                              "cap", ki * self.V + freev, active=ev["C"][:, 0] < 0)
        v_next = (x - x_n) / self.dt
        if record:
            rec["lam.dist"] = lam_d
            rec["lam.tet"] = lam_t
        return x, v_next, rec

    def simulate(self, x0, v0, forces=None, frames=None):
        """Forward over `frames` frames; returns states x_0..x_N (N = frames*substeps)."""
        frames = self.s.frames if frames is None else frames
        xs = [np.array(x0, float)]
        x, v = xs[0].copy(), np.array(v0, float)
        for n in range(frames * self.s.substeps):
            f = None if forces is None else forces[n // self.s.substeps]
            x, v, _ = self.step(x, v, f)
            xs.append(x.copy())
        return xs

    # ------------------------------------------------------------ backward
    def blocks(self, rec):
        """Per-constraint system blocks Q_j = psd(-sym D_j) (Sec.4.3.2; R5).
        Tets are projected in deformation-gradient coordinates: D~ = Gp^T D Gp (R5)."""
        proj = psd_project if self.pd else (lambda A: A)
        out = {}
        out["dist"] = proj(-sym(rec["dist.D"])) if self.E else np.zeros((0, 6, 6))
        if self.T:
            Dt = np.einsum("nia,nij,njb->nab", self.Gp, rec["tet.D"], self.Gp)
            out["tet"] = np.einsum("nai,nab,nbj->nij", self.G, proj(-sym(Dt)), self.G)
        else:
            out["tet"] = np.zeros((0, 12, 12))
        out["sph"] = proj(-sym(rec["sph.D"]))
        out["cap"] = proj(-sym(rec["cap.D"]))
        return out

    def system_matrix(self, Q):
        """A = M + Sum_j P_j^T Q_j P_j over all 3V DoFs (Eq. adjointXPBD left-multiplied, R4)."""
        V = self.V
        rows, cols, vals = [np.arange(3 * V)], [np.arange(3 * V)], [np.repeat(self.m, 3)]

        def add(st, B):
            if len(st) == 0:
                return
            k = st.shape[1]
            dof = (3 * st[:, :, None] + np.arange(3)[None, None]).reshape(len(st), 3 * k)
            rows.append(np.repeat(dof, 3 * k, axis=1).ravel())
            cols.append(np.tile(dof, (1, 3 * k)).ravel())
            vals.append(B.reshape(len(st), -1).ravel())

        add(self.dist_idx, Q["dist"])
        add(self.tet_idx, Q["tet"])
        allv = np.arange(V)
        for ci in range(len(self.spheres)):
            add(allv[:, None], Q["sph"][ci * V:(ci + 1) * V])
        for ki in range(len(self.cap_c)):
            add(allv[:, None], Q["cap"][ki * V:(ki + 1) * V])
        A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(3 * V, 3 * V)).tocsr()
        return A

    def solve(self, Q, r):
        """Filtered solve (Sec.4.2.1): free DoFs only, pinned components of y are exactly 0.
        Direct sparse solve = the exact solution CG converges to (l.201 "a direct solver can be used").
        solver="cg": the paper's preferred alternative (l.201 "PCG ... preferred"), plain conjugate
        gradients on the same SPD system run to a relative residual of 1e-13 (for large test scenes,
        where the direct factorisation takes minutes; pinned against "direct" in the CPU tests)."""
        A = self.system_matrix(Q)
        fd = np.repeat(self.free, 3)
        y = np.zeros(3 * self.V)
        rf = r.reshape(-1)[fd]
        if np.any(rf != 0):
            Aff = A[fd][:, fd].tocsc()
            if self.solver == "direct":
                y[fd] = spla.spsolve(Aff, rf)
            else:
                yf, info = spla.cg(Aff.tocsr(), rf, rtol=1e-13, atol=0.0, maxiter=20 * len(rf))
                assert info == 0, info
                y[fd] = yf
        return y.reshape(self.V, 3)

    def loss(self, xs, key_frames, targets, weights=None):
        """phi = 1/2 Sum_k ||W (x_{n_k} - x*_k)||^2 (Sec.4.1 l.129, beta = 0, W diagonal;
        R10).  Returns phi and {state index: dphi/dx}."""
        sub = self.s.substeps
        W = np.ones(self.V) if weights is None else np.asarray(weights, float)
        phi = 0.0
        d = {}
        for k, fr in enumerate(np.asarray(key_frames).tolist()):
            n = int(fr) * sub
            diff = xs[n] - targets[k]
            phi += 0.5 * float((W[:, None] * diff * diff).sum())
            d[n] = d.get(n, 0.0) + W[:, None] * diff
        return phi, d

    def backward(self, xs, v0, forces=None, key_frames=None, targets=None, weights=None,
                 keep=False):
        """Adjoint pass over the stored trajectory xs (x_0..x_N), Eqs. rawAdjoint/adjointXPBD/
        gradientRule with the step replay of R9.  Returns (phi, grads dict[, per-step data])."""
        s = self.s
        dt, sub = self.dt, s.substeps
        N = len(xs) - 1
        key_frames = s.key_frames if key_frames is None else key_frames
        targets = s.targets if targets is None else targets
        phi, dphi = self.loss(xs, key_frames, targets, weights)
        V = self.V
        zero = np.zeros((V, 3))
        ax = np.array(dphi.get(N, zero), float)
        av = zero.copy()
        ax[~self.free] = 0.0
        nframes = (N + sub - 1) // sub
        gr = dict(
            compliance=np.zeros(self.E), forces=np.zeros((nframes, V, 3)),
            material=np.zeros((self.T, 2)), sphere=np.zeros((len(self.spheres), 4)),
            cap_rL=np.zeros((len(self.cap_c), 2)),
        )
        steps = []
        nsph = len(self.spheres)
        for n in reversed(range(N)):
            r = ax + av / dt
            r[~self.free] = 0.0
            if np.any(r != 0):
                v_n = np.asarray(v0, float) if n == 0 else (xs[n] - xs[n - 1]) / dt
                f = None if forces is None else forces[n // sub]
                _, _, rec = self.step(xs[n], v_n, f, record=True)
                Q = self.blocks(rec)
                y = self.solve(Q, r)
                # control gradients: dphi/du += e . y_stencil (Eq. gradientRule)
                if self.E:
                    ys = y[self.dist_idx].reshape(self.E, 6)
                    gr["compliance"] += np.einsum("nj,nj->n", rec["dist.e"][:, 0], ys)
                if self.T:
                    ys = y[self.tet_idx].reshape(self.T, 12)
                    gr["material"] += np.einsum("nuj,nj->nu", rec["tet.e"], ys)
                for ci in range(nsph):
                    e = rec["sph.e"][ci * V:(ci + 1) * V]
                    gr["sphere"][ci] += np.einsum("vuj,vj->u", e, y)
                for ki in range(len(self.cap_c)):
                    e = rec["cap.e"][ki * V:(ki + 1) * V]
                    gr["cap_rL"][ki] += np.einsum("vuj,vj->u", e, y)
                if keep:
                    steps.append(dict(n=n, y=y, r=r, Q=Q, rec=rec))
            else:
                y = zero.copy()
            z = self.m[:, None] * y
            gr["forces"][n // sub] += dt * dt * y
            ax = z - av / dt + dphi.get(n, zero)
            av = dt * z
            ax[~self.free] = 0.0
            av[~self.free] = 0.0
        gr["x0"] = ax
        gr["v0"] = av
        if len(self.cap_c):
            nc = len(self.cap_c)
            gr["shape"] = (np.asarray(s.cap_rbasis, float).reshape(nc, -1).T @ gr["cap_rL"][:, 0]
                           + np.asarray(s.cap_lbasis, float).reshape(nc, -1).T @ gr["cap_rL"][:, 1])
        else:
            gr["shape"] = np.zeros(len(self.beta))
        if keep:
            return phi, gr, steps
        return phi, gr

    def run(self, with_grads=True, **kw):
        """Convenience: forward over the scene's frames from its x0, v0, forces; then backward."""
        s = self.s
        xs = self.simulate(s.x0, s.v0, s.forces, s.frames)
        if not with_grads:
            return xs
        phi, gr = self.backward(xs, s.v0, s.forces, **kw)
        return xs, phi, gr
