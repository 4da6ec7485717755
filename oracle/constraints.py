"""ORACLE (test infrastructure only). Constraint functions C(x), gradients
grad C, Hessians d(grad C)/dx and control partials, fp64, vectorised over a
batch of constraints.  Stencil vectors are flattened vertex-major:
[x_0 (3), x_1 (3), ...].

Families (BASELINE.json north_star):
  * distance   C = |x_a - x_b| - L          (cloth stretch/shear/bend; Eq.1 C(x))
  * sphere     C = |x - c| - r - h          ("stiff springs ... thickness")
  * capsule    C = |x - cp(x)| - r - h      (same; cp = closest point on the segment)
  * tet_dev    C_D = sqrt(tr(F^T F)) - sqrt(3)   (offset so that C_D(I) = 0: DESIGN.md R6)
  * tet_hyd    C_H = det(F) - 1                  (PAPER.md l.229 as printed; R6)
  Both vanish at the rest state F = I, so U = 1/2 C^T alpha^-1 C (Eq. xpbdUenergy l.76) is zero
  there and the rest state is a fixed point of the XPBD substep (reading R6).
"""
from __future__ import annotations

import numpy as np

I3 = np.eye(3)


def _outer(a, b):
    return a[..., :, None] * b[..., None, :]


# ---------------------------------------------------------------- distance
def distance(xs: np.ndarray, rest: np.ndarray):
    """xs (N,2,3). Returns C (N,), g (N,6), H (N,6,6)."""
    d = xs[:, 0] - xs[:, 1]
    l = np.linalg.norm(d, axis=1)
    n = d / l[:, None]
    C = l - rest
    g = np.concatenate([n, -n], 1)
    K = (I3[None] - _outer(n, n)) / l[:, None, None]
    H = np.zeros((len(xs), 6, 6))
    H[:, :3, :3] = K
    H[:, 3:, 3:] = K
    H[:, :3, 3:] = -K
    H[:, 3:, :3] = -K
    return C, g, H, l


# ---------------------------------------------------------------- sphere
def sphere(x: np.ndarray, center: np.ndarray, radius: float, h: float):
    """x (N,3). Controls u = (c_x, c_y, c_z, r).
    Returns C, g (N,3), H (N,3,3), dC/du (N,4), dg/du (N,4,3), dist."""
    d = x - center[None]
    dist = np.linalg.norm(d, axis=1)
    n = d / dist[:, None]
    C = dist - radius - h
    P = (I3[None] - _outer(n, n)) / dist[:, None, None]
    dCdu = np.concatenate([-n, -np.ones((len(x), 1))], 1)
    dgdu = np.zeros((len(x), 4, 3))
    dgdu[:, :3, :] = -P          # d n / d c_k  (P symmetric)
    return C, n, P, dCdu, dgdu, dist


# ---------------------------------------------------------------- capsule
def capsule(x: np.ndarray, center: np.ndarray, axis: np.ndarray, radius: float, length: float,
            h: float):
    """Segment center +- (length/2) axis, radius r.  Controls u = (r, L).
    interior iff -L/2 < s < L/2 (s = (x-c).axis); otherwise the endpoint is the witness."""
    s = (x - center[None]) @ axis
    half = 0.5 * length
    interior = (s > -half) & (s < half)
    tcl = np.clip(s, -half, half)
    cp = center[None] + tcl[:, None] * axis[None]
    d = x - cp
    dist = np.linalg.norm(d, axis=1)
    n = d / dist[:, None]
    C = dist - radius - h
    aa = _outer(axis, axis)
    H = (I3[None] - _outer(n, n) - interior[:, None, None] * aa[None]) / dist[:, None, None]
    dcp_dL = np.where(interior, 0.0, np.where(s >= half, 0.5, -0.5))[:, None] * axis[None]
    dCdu = np.stack([-np.ones(len(x)), -np.einsum("ni,ni->n", n, dcp_dL)], 1)
    dgdu = np.zeros((len(x), 2, 3))
    Pn = I3[None] - _outer(n, n)
    dgdu[:, 1, :] = -np.einsum("nij,nj->ni", Pn, dcp_dL) / dist[:, None]
    return C, n, H, dCdu, dgdu, dist


# ---------------------------------------------------------------- tetrahedra
def tet_rest(x_rest: np.ndarray, tets: np.ndarray):
    """Dm^{-1} (T,3,3) with Dm columns x_i - x_0 (i=1..3); rest volume |det Dm|/6."""
    p = x_rest[tets]
    Dm = (p[:, 1:] - p[:, :1]).transpose(0, 2, 1)
    return np.linalg.inv(Dm), np.abs(np.linalg.det(Dm)) / 6.0


def tet_G(Dminv: np.ndarray) -> np.ndarray:
    """G (T,9,12): vec(F) = G x_stencil, vec column-major (index 3*col+row)."""
    T = len(Dminv)
    G = np.zeros((T, 9, 12))
    for col in range(3):
        for row in range(3):
            for k in range(1, 4):
                G[:, 3 * col + row, 3 * k + row] = Dminv[:, k - 1, col]
            G[:, 3 * col + row, row] = -Dminv[:, :, col].sum(1)
    return G


def _skew(v):
    S = np.zeros(v.shape[:-1] + (3, 3))
    S[..., 0, 1] = -v[..., 2]
    S[..., 0, 2] = v[..., 1]
    S[..., 1, 0] = v[..., 2]
    S[..., 1, 2] = -v[..., 0]
    S[..., 2, 0] = -v[..., 1]
    S[..., 2, 1] = v[..., 0]
    return S


def tet_F(xs: np.ndarray, Dminv: np.ndarray):
    Ds = (xs[:, 1:] - xs[:, :1]).transpose(0, 2, 1)
    return Ds @ Dminv


SQRT3 = np.sqrt(3.0)


def tet_dev_F(F: np.ndarray):
    """C_D = ||F||_F - sqrt(3); returns C, dC/dvecF (T,9), d2C/dvecF2 (T,9,9)."""
    f = F.transpose(0, 2, 1).reshape(len(F), 9)
    nrm = np.linalg.norm(f, axis=1)
    C = nrm - SQRT3
    P = f / nrm[:, None]
    HF = (np.eye(9)[None] - _outer(P, P)) / nrm[:, None, None]
    return C, P, HF


def tet_hyd_F(F: np.ndarray):
    """C_H = det F - 1; dC/dF = cof(F) = [f1 x f2, f2 x f0, f0 x f1]."""
    f0, f1, f2 = F[:, :, 0], F[:, :, 1], F[:, :, 2]
    c0, c1, c2 = np.cross(f1, f2), np.cross(f2, f0), np.cross(f0, f1)
    det = np.einsum("ni,ni->n", f0, c0)
    C = det - 1.0
    P = np.concatenate([c0, c1, c2], 1)
    HF = np.zeros((len(F), 9, 9))
    # block (i,j) = d cof_i / d f_j ; d(a x b)/da = -[b]x, d(a x b)/db = [a]x
    HF[:, 0:3, 3:6] = -_skew(f2)
    HF[:, 0:3, 6:9] = _skew(f1)
    HF[:, 3:6, 6:9] = -_skew(f0)
    HF[:, 3:6, 0:3] = _skew(f2)
    HF[:, 6:9, 0:3] = -_skew(f1)
    HF[:, 6:9, 3:6] = _skew(f0)
    return C, P, HF


def tet(xs: np.ndarray, Dminv: np.ndarray, G: np.ndarray, kind: str, need_H=True):
    """Returns C, g (T,12) = G^T dC/dvecF, H (T,12,12) = G^T H_F G (None if not need_H)."""
    F = tet_F(xs, Dminv)
    if kind == "D":
        C, P, HF = tet_dev_F(F)
    else:
        C, P, HF = tet_hyd_F(F)
    g = np.einsum("nij,ni->nj", G, P)
    H = np.einsum("nai,nab,nbj->nij", G, HF, G) if need_H else None
    return C, g, H
