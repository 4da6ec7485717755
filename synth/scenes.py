"""Seeded synthetic scenes shaped like the workloads of BASELINE.json `configs`
(the paper's own meshes and scans are not available).

Everything here is plain input preparation: vertex grids, constraint index
lists (topology only -- rest lengths, colorings and every other method
quantity are computed independently by the oracle and by the CUDA library),
seeded compliances / materials / forces / targets, lumped masses and analytic
collider definitions. Arrays are float64; `as_float32_exact` rounds a scene
through float32 so that the fp64 oracle and the fp32 CUDA path start from
bit-identical inputs.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field
from typing import Optional

import numpy as np


@dataclass
class Scene:
    name: str
    x_rest: np.ndarray                  # (V,3) rest positions [m]
    x0: np.ndarray                      # (V,3) initial positions [m]
    v0: np.ndarray                      # (V,3) initial velocities [m/s]
    inv_mass: np.ndarray                # (V,)  1/kg, 0 = pinned (infinite mass)
    dist_idx: np.ndarray                # (E,2) int32 distance-constraint stencils
    dist_compliance: np.ndarray         # (E,)  alpha [m/N]
    tet_idx: np.ndarray                 # (T,4) int32 tetrahedra (positive orientation)
    tet_a: np.ndarray                   # (T,)  a, mu = a^2
    tet_b: np.ndarray                   # (T,)  b, lambda = b^2
    spheres: np.ndarray                 # (S,4) center xyz, radius
    cap_center: np.ndarray              # (K,3) capsule centers
    cap_axis: np.ndarray                # (K,3) unit axes
    cap_r0: np.ndarray                  # (K,)  radius at zero shape coefficients
    cap_L0: np.ndarray                  # (K,)  segment length at zero shape coefficients
    cap_rbasis: np.ndarray              # (K,NS) d radius / d beta
    cap_lbasis: np.ndarray              # (K,NS) d length / d beta
    shape_beta: np.ndarray              # (NS,) shape coefficients
    gravity: np.ndarray                 # (3,)
    frame_dt: float
    substeps: int
    iterations: int
    frames: int
    thickness: float = 0.0
    collision_compliance: float = 0.0
    forces: Optional[np.ndarray] = None     # (frames,V,3) per-frame external force [N]
    key_frames: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    targets: Optional[np.ndarray] = None    # (nk,V,3) keyframe targets
    weights: Optional[np.ndarray] = None    # (V,) per-vertex goal weights (W_n diagonal)
    meta: dict = field(default_factory=dict)

    @property
    def num_vertices(self) -> int:
        return int(self.x_rest.shape[0])

    @property
    def dt(self) -> float:
        return self.frame_dt / self.substeps

    @property
    def num_steps(self) -> int:
        return self.frames * self.substeps

    def replace(self, **kw) -> "Scene":
        return dataclasses.replace(self, **kw)


def _empty_colliders(ns: int = 0):
    return dict(
        spheres=np.zeros((0, 4)),
        cap_center=np.zeros((0, 3)), cap_axis=np.zeros((0, 3)),
        cap_r0=np.zeros(0), cap_L0=np.zeros(0),
        cap_rbasis=np.zeros((0, ns)), cap_lbasis=np.zeros((0, ns)),
        shape_beta=np.zeros(ns),
    )


def as_float32_exact(s: Scene) -> Scene:
    """Round every floating array of the scene through float32 (kept as float64)."""
    kw = {}
    for f in dataclasses.fields(s):
        v = getattr(s, f.name)
        if isinstance(v, np.ndarray) and v.dtype.kind == "f":
            kw[f.name] = v.astype(np.float32).astype(np.float64)
        elif isinstance(v, float) and f.name not in ("frame_dt",):
            kw[f.name] = float(np.float32(v))
    kw["frame_dt"] = float(np.float32(s.frame_dt))
    return dataclasses.replace(s, **kw)


# --------------------------------------------------------------------------
# Cloth topology: structural + shear + bending distance constraints on a grid
# (BASELINE.json north_star "cloth stretch/shear/bending distance constraints").
# Order: structural-u, structural-v, shear-a, shear-b, bend-u, bend-v; row-major.
# --------------------------------------------------------------------------
def _grid_edges(nu: int, nv: int, wrap_u: bool) -> np.ndarray:
    vid = np.arange(nu * nv, dtype=np.int64).reshape(nv, nu)
    groups = []

    def pairs(di, dj):
        # (i, j) -- (i+di, j+dj), dj >= 0; column index wraps when wrap_u
        rows = np.arange(nv - di)
        cols = np.arange(nu) if wrap_u else np.arange(nu - dj)
        I, Jc = np.meshgrid(rows, cols, indexing="ij")
        return np.stack([vid[I, Jc].ravel(), vid[I + di, (Jc + dj) % nu].ravel()], 1)

    groups.append(pairs(0, 1))      # structural along u
    groups.append(pairs(1, 0))      # structural along v
    groups.append(pairs(1, 1))      # shear a
    # shear b: (i, j+1)-(i+1, j)
    if wrap_u:
        I, Jc = np.meshgrid(np.arange(nv - 1), np.arange(nu), indexing="ij")
        groups.append(np.stack([vid[I, (Jc + 1) % nu].ravel(), vid[I + 1, Jc].ravel()], 1))
    else:
        I, Jc = np.meshgrid(np.arange(nv - 1), np.arange(nu - 1), indexing="ij")
        groups.append(np.stack([vid[I, Jc + 1].ravel(), vid[I + 1, Jc].ravel()], 1))
    if nu >= 3 or wrap_u:
        groups.append(pairs(0, 2))  # bending along u
    if nv >= 3:
        groups.append(pairs(2, 0))  # bending along v
    e = np.concatenate([g for g in groups if len(g)], 0).astype(np.int32)
    return e


def cloth_grid(nu: int, nv: int, side_u: float, side_v: float, height: float,
               mass: float, seed: int, pins=(), center=(0.0, 0.0)) -> dict:
    """Square cloth in the x-z plane at y=height; vertex id = i*nu + j."""
    j = np.arange(nu)
    i = np.arange(nv)
    J, I = np.meshgrid(j, i)
    x = np.zeros((nv, nu, 3))
    x[..., 0] = center[0] - 0.5 * side_u + J * (side_u / max(nu - 1, 1))
    x[..., 1] = height
    x[..., 2] = center[1] - 0.5 * side_v + I * (side_v / max(nv - 1, 1))
    x = x.reshape(-1, 3)
    inv_mass = np.full(nu * nv, 1.0 / mass)
    for p in pins:
        inv_mass[p] = 0.0
    edges = _grid_edges(nu, nv, wrap_u=False)
    rng = np.random.default_rng(seed)
    comp = np.exp(rng.uniform(np.log(1e-8), np.log(1e-6), size=len(edges)))
    return dict(x_rest=x, inv_mass=inv_mass, dist_idx=edges, dist_compliance=comp)


def cloth_tube(n_around: int, n_along: int, radius: float, length: float, top: float,
               mass: float, seed: int) -> dict:
    """Cylindrical cloth tube, axis y, top ring at y=top; wraps around u."""
    th = 2 * np.pi * np.arange(n_around) / n_around
    ys = top - length * np.arange(n_along) / max(n_along - 1, 1)
    TH, Y = np.meshgrid(th, ys)
    x = np.stack([radius * np.cos(TH), Y, radius * np.sin(TH)], -1).reshape(-1, 3)
    inv_mass = np.full(len(x), 1.0 / mass)
    edges = _grid_edges(n_around, n_along, wrap_u=True)
    rng = np.random.default_rng(seed)
    comp = np.exp(rng.uniform(np.log(1e-8), np.log(1e-6), size=len(edges)))
    return dict(x_rest=x, inv_mass=inv_mass, dist_idx=edges, dist_compliance=comp)


# 5-tet split of a unit cube (corner (a,b,c) -> bit a*4+b*2+c); mirrored on odd cells
_CUBE5 = np.array([[0, 4, 2, 1], [6, 2, 4, 7], [5, 4, 1, 7], [3, 1, 2, 7], [4, 2, 1, 7]])


def tet_block(n: int, side: float, density: float, seed: int,
              E_range=(1e4, 1e6), nu_range=(0.3, 0.45)) -> dict:
    """n^3 vertex block (y up), (n-1)^3 cubes x 5 tets; bottom face pinned."""
    h = side / (n - 1)
    g = np.arange(n)
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    x = np.stack([X, Y, Z], -1).reshape(-1, 3) * h
    vid = lambda ix, iy, iz: (ix * n + iy) * n + iz  # noqa: E731
    tets = []
    c = np.arange(n - 1)
    CX, CY, CZ = np.meshgrid(c, c, c, indexing="ij")
    CX, CY, CZ = CX.ravel(), CY.ravel(), CZ.ravel()
    odd = (CX + CY + CZ) % 2 == 1
    for t in _CUBE5:
        cols = []
        for corner in t:
            a, b, cc = (corner >> 2) & 1, (corner >> 1) & 1, corner & 1
            ax = np.where(odd, 1 - a, a)
            cols.append(vid(CX + ax, CY + b, CZ + cc))
        tets.append(np.stack(cols, 1))
    # interleave: cube-major order (cube k -> its 5 tets)
    tets = np.stack(tets, 1).reshape(-1, 4)
    # orient positively
    p = x[tets]
    vol6 = np.einsum("ij,ij->i", np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), p[:, 3] - p[:, 0])
    neg = vol6 < 0
    tets[neg] = tets[neg][:, [0, 2, 1, 3]]
    vol = np.abs(vol6) / 6.0
    mass = np.zeros(len(x))
    np.add.at(mass, tets.ravel(), np.repeat(density * vol / 4.0, 4))
    inv_mass = 1.0 / mass
    inv_mass[x[:, 1] < 0.5 * h] = 0.0
    rng = np.random.default_rng(seed)
    E = rng.uniform(*E_range, size=len(tets))
    nu = rng.uniform(*nu_range, size=len(tets))
    mu = E / (2 * (1 + nu))
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    return dict(x_rest=x, inv_mass=inv_mass, tet_idx=tets.astype(np.int32),
                tet_a=np.sqrt(mu), tet_b=np.sqrt(lam))


def body_capsules(num_shape: int, seed: int) -> dict:
    """12-capsule analytic body (y up). radius/length linear in shape coefficients."""
    # center, axis, r0, L0
    caps = [
        ((0.0, 1.45, 0.0), (1, 0, 0), 0.060, 0.36),   # shoulders
        ((0.0, 1.15, 0.0), (0, 1, 0), 0.140, 0.40),   # torso
        ((0.0, 1.56, 0.0), (0, 1, 0), 0.050, 0.08),   # neck
        ((0.0, 1.70, 0.0), (0, 1, 0), 0.100, 0.06),   # head
        ((0.26, 1.25, 0.0), (0, 1, 0), 0.045, 0.26),  # upper arm R
        ((-0.26, 1.25, 0.0), (0, 1, 0), 0.045, 0.26), # upper arm L
        ((0.27, 0.98, 0.0), (0, 1, 0), 0.040, 0.24),  # forearm R
        ((-0.27, 0.98, 0.0), (0, 1, 0), 0.040, 0.24), # forearm L
        ((0.10, 0.65, 0.0), (0, 1, 0), 0.070, 0.36),  # thigh R
        ((-0.10, 0.65, 0.0), (0, 1, 0), 0.070, 0.36), # thigh L
        ((0.10, 0.25, 0.0), (0, 1, 0), 0.050, 0.36),  # shin R
        ((-0.10, 0.25, 0.0), (0, 1, 0), 0.050, 0.36), # shin L
    ]
    rng = np.random.default_rng(seed)
    K = len(caps)
    return dict(
        cap_center=np.array([c[0] for c in caps], float),
        cap_axis=np.array([c[1] for c in caps], float),
        cap_r0=np.array([c[2] for c in caps], float),
        cap_L0=np.array([c[3] for c in caps], float),
        cap_rbasis=rng.normal(0.0, 0.004, size=(K, num_shape)),
        cap_lbasis=rng.normal(0.0, 0.01, size=(K, num_shape)),
    )


def _smooth_field(rng, pts: np.ndarray, amp: float, nmodes: int = 4) -> np.ndarray:
    """Seeded low-frequency displacement field (sum of random sinusoids)."""
    out = np.zeros_like(pts)
    for _ in range(nmodes):
        k = rng.normal(0, 2.0, size=3)
        ph = rng.uniform(0, 2 * np.pi)
        d = rng.normal(0, 1.0, size=3)
        out += np.sin(pts @ k + ph)[:, None] * d[None, :]
    return amp * out / nmodes


def _base(name, V, ns=0, **kw) -> dict:
    d = dict(name=name, x0=None, v0=np.zeros((V, 3)),
             dist_idx=np.zeros((0, 2), np.int32), dist_compliance=np.zeros(0),
             tet_idx=np.zeros((0, 4), np.int32), tet_a=np.zeros(0), tet_b=np.zeros(0),
             gravity=np.array([0.0, -9.81, 0.0]))
    d.update(_empty_colliders(ns))
    d.update(kw)
    if d["x0"] is None:
        d["x0"] = d["x_rest"].copy()
    return d


def tiny_cloth(n: int = 16, frames: int = 30, substeps: int = 10, iterations: int = 1,
               seed: int = 0) -> Scene:
    """configs[0]: 16x16, 1 m, 1 g/vertex, two top corners pinned, 30 frames x 10 substeps x 1 it."""
    c = cloth_grid(n, n, 1.0, 1.0, 0.0, 1e-3, seed, pins=(0, n - 1))
    V = n * n
    rng = np.random.default_rng(seed + 1000)
    x = c["x_rest"]
    # seeded target drape: sag away from the pinned row plus a smooth perturbation
    s = (x[:, 2] - x[:, 2].min())
    tgt = x.copy()
    tgt[:, 1] -= 0.6 * s
    tgt[:, 2] -= 0.6 * s * s
    tgt += _smooth_field(rng, x, 0.02)
    d = _base("tiny_cloth", V, **c)
    return Scene(**d, frame_dt=1 / 60, substeps=substeps, iterations=iterations, frames=frames,
                 key_frames=np.array([frames], np.int32), targets=tgt[None])


def medium_cloth(n: int = 256, frames: int = 60, substeps: int = 10, iterations: int = 1,
                 seed: int = 1) -> Scene:
    """configs[1]: 256x256 (~197k DoF) dropped onto a fixed sphere r=0.3, collisions."""
    c = cloth_grid(n, n, 1.0, 1.0, 0.35, 1e-3, seed)
    V = n * n
    rng = np.random.default_rng(seed + 1000)
    x = c["x_rest"]
    rr = np.sqrt(x[:, 0] ** 2 + x[:, 2] ** 2)
    tgt = x.copy()
    tgt[:, 1] = np.where(rr < 0.3, np.sqrt(np.maximum(0.31 ** 2 - rr ** 2, 0.0)), -0.8 * (rr - 0.3))
    tgt += _smooth_field(rng, x, 0.01)
    d = _base("medium_cloth", V, **c)
    d["spheres"] = np.array([[0.0, 0.0, 0.0, 0.3]])
    return Scene(**d, frame_dt=1 / 60, substeps=substeps, iterations=iterations, frames=frames,
                 thickness=0.005, collision_compliance=1e-9,
                 key_frames=np.array([frames], np.int32), targets=tgt[None])


def volumetric_block(n: int = 40, frames: int = 50, substeps: int = 20, iterations: int = 1,
                     seed: int = 2, side: float = 0.4) -> Scene:
    """configs[2]: n^3 grid x 5 tets/cube, stable Neo-Hookean, bottom face fixed."""
    t = tet_block(n, side, 1000.0, seed)
    V = n ** 3
    rng = np.random.default_rng(seed + 1000)
    x = t["x_rest"]
    tgt = x.copy()
    tgt[:, 1] -= 0.05 * (x[:, 1] / side) ** 2
    tgt += _smooth_field(rng, x, 0.004)
    d = _base("volumetric_block", V, **t)
    return Scene(**d, frame_dt=1 / 60, substeps=substeps, iterations=iterations, frames=frames,
                 key_frames=np.array([frames], np.int32), targets=tgt[None])


def _capsule_dims(body: dict, beta: np.ndarray):
    """Capsule radii / segment lengths at shape coefficients beta (input geometry only: used to
    place the garment clear of the body)."""
    return body["cap_r0"] + body["cap_rbasis"] @ beta, body["cap_L0"] + body["cap_lbasis"] @ beta


def garment_profile(body: dict, betas, h: float, n_along: int):
    """Rest profile (radius, height) of the garment tube, a surface of revolution about the body's
    y axis: a neckline ring around the neck capsule, a shallow cone over the shoulder capsule and
    the upper arms, then a cylinder outside the arms down to hip height.  Placed 8 mm (+ thickness)
    clear of the body for every shape vector in `betas`.  Rows are spaced uniformly in arc length."""
    rs, Ls = zip(*[_capsule_dims(body, np.asarray(b, float)) for b in betas])
    r, L = np.max(rs, 0), np.max(Ls, 0)
    clear = h + 0.008
    neck, sh = 2, 0                     # body_capsules order: shoulders, torso, neck, head, arms ...
    y_sh = body["cap_center"][sh][1]
    R0 = r[neck] + h + 0.03             # neckline radius
    y_top = y_sh + r[sh] + 0.05
    half = 0.5 * L[sh]
    slope = (0.05 - clear) / max(half - R0, 1e-3)     # cone passes the shoulder segment end `clear` above
    arms = [4, 5, 6, 7]
    R1 = max(abs(body["cap_center"][k][0]) + r[k] for k in arms) + 0.03
    y_c = y_top - slope * (R1 - R0)
    y_bot = 0.85
    # polyline (rho, y): neckline -> cone end -> hem
    P = np.array([[R0, y_top], [R1, y_c], [R1, y_bot]])
    seg = np.linalg.norm(np.diff(P, axis=0), axis=1)
    s = np.linspace(0.0, seg.sum(), n_along)
    rho = np.interp(s, np.concatenate([[0], np.cumsum(seg)]), P[:, 0])
    y = np.interp(s, np.concatenate([[0], np.cumsum(seg)]), P[:, 1])
    return rho, y


def garment(n_around: int = 512, n_along: int = 512, frames: int = 120, substeps: int = 10,
            iterations: int = 1, seed: int = 3, num_shape: int = 10) -> Scene:
    """configs[3]: cloth tube over a 12-capsule body; capsule r, L linear in 10 coefficients.

    The tube's top (neckline) ring is pinned around the neck; the garment hangs from it over the
    shoulder capsule and the arms (the drape).  Targets: the drape produced by the seeded ground
    truth coefficients `meta["shape_beta_gt"]` -- a simulation result, so it is not made here
    (targets = None): the parity tests compute it with the oracle, the performance runs with the
    library."""
    body = body_capsules(num_shape, seed)
    rng = np.random.default_rng(seed + 1000)
    beta = rng.normal(0.0, 1.0, size=num_shape)
    beta_gt = rng.normal(0.0, 1.0, size=num_shape)
    h = 0.005
    rho, y = garment_profile(body, (beta, beta_gt), h, n_along)
    th = 2 * np.pi * np.arange(n_around) / n_around
    TH = np.broadcast_to(th[None, :], (n_along, n_around))
    x = np.stack([rho[:, None] * np.cos(TH), np.broadcast_to(y[:, None], TH.shape),
                  rho[:, None] * np.sin(TH)], -1).reshape(-1, 3)
    V = n_around * n_along
    inv_mass = np.full(V, 1.0 / 1e-3)
    inv_mass[:n_around] = 0.0                       # neckline ring (row 0) pinned
    edges = _grid_edges(n_around, n_along, wrap_u=True)
    crng = np.random.default_rng(seed)
    comp = np.exp(crng.uniform(np.log(1e-8), np.log(1e-6), size=len(edges)))
    d = _base("garment", V, ns=num_shape, x_rest=x, inv_mass=inv_mass, dist_idx=edges, dist_compliance=comp)
    d.update(body)
    d["shape_beta"] = beta
    return Scene(**d, frame_dt=1 / 60, substeps=substeps, iterations=iterations, frames=frames,
                 thickness=h, collision_compliance=1e-9,
                 key_frames=np.array([frames], np.int32), targets=None,
                 meta=dict(shape_beta_gt=beta_gt))


def large_cloth(n: int = 2944, frames: int = 30, substeps: int = 10, iterations: int = 1,
                seed: int = 4, side: float = 10.0, with_forces: bool = True,
                key_frames=(10, 20, 30)) -> Scene:
    """configs[4]: n^2 grid (2944^2 ~ 26M DoF), per-frame per-vertex forces N(0, 0.1 N)."""
    c = cloth_grid(n, n, side, side, 0.0, 1e-3, seed, pins=(0, n - 1))
    V = n * n
    rng = np.random.default_rng(seed + 1000)
    forces = None
    if with_forces:
        forces = rng.standard_normal(size=(frames, V, 3), dtype=np.float32).astype(np.float64) * 0.1
    x = c["x_rest"]
    kf = np.array([k for k in key_frames if k <= frames], np.int32)
    s = (x[:, 2] - x[:, 2].min()) / side
    tg = []
    for q, k in enumerate(kf):
        t = x.copy()
        t[:, 1] -= (0.2 + 0.2 * q) * side * s
        t[:, 2] -= (0.1 + 0.1 * q) * side * s * s
        tg.append(t)
    d = _base("large_cloth", V, **c)
    return Scene(**d, frame_dt=1 / 60, substeps=substeps, iterations=iterations, frames=frames,
                 forces=forces, key_frames=kf, targets=np.stack(tg) if len(tg) else None)


CONFIGS = {
    "tiny_cloth": tiny_cloth,
    "medium_cloth": medium_cloth,
    "volumetric_block": volumetric_block,
    "garment": garment,
    "large_cloth": large_cloth,
}


def make_config(name: str, **kw) -> Scene:
    return CONFIGS[name](**kw)
