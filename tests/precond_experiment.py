"""Preconditioner check on the oracle's assembled adjoint matrix (not collected by pytest; run
`python tests/precond_experiment.py`).  configs[4] regime at 96^2 vertices: PCG iterations to a
1e-6 relative residual from zero for a random and a smooth right-hand side with the mass
(the CUDA path's), the scalar diagonal and the 3x3 vertex-block Jacobi preconditioners.
Recorded in DESIGN.md ("Preconditioner"); test infrastructure, it imports oracle/."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tests/", 1)[0])
from oracle import OracleModel  # noqa: E402
from synth import as_float32_exact, large_cloth  # noqa: E402


def pcg(A, b, pinv, tol=1e-6):
    x = np.zeros_like(b)
    r = b.copy()
    z = pinv(r)
    p = z.copy()
    rz = r @ z
    bb = b @ b
    for it in range(5000):
        q = A @ p
        a = rz / (p @ q)
        x += a * p
        r -= a * q
        if r @ r <= tol * tol * bb:
            return it + 1
        z = pinv(r)
        rz2 = r @ z
        p = z + (rz2 / rz) * p
        rz = rz2
    return -1


def main():
    s = as_float32_exact(large_cloth(n=96, frames=2, substeps=3, side=10.0 * 95 / 2943.0,
                                     key_frames=(2,)).replace(frame_dt=3 / 600))
    m = OracleModel(s)
    xs = m.simulate(s.x0, s.v0, s.forces, 2)
    n = len(xs) - 2
    v_n = (xs[n] - xs[n - 1]) / m.dt
    f = None if s.forces is None else s.forces[n // s.substeps]
    _, _, rec = m.step(xs[n], v_n, f, record=True)
    A = m.system_matrix(m.blocks(rec)).tocsr()
    fd = np.repeat(m.free, 3)
    Aff = A[fd][:, fd].tocsr()
    nb = Aff.shape[0] // 3
    b_rand = np.random.default_rng(0).normal(size=3 * nb)
    b_smooth = Aff @ np.ones(3 * nb)
    mass = np.repeat(m.m[m.free], 3)
    d = Aff.diagonal()
    co = Aff.tocoo()
    sel = co.row // 3 == co.col // 3
    blocks = np.zeros((nb, 3, 3))
    np.add.at(blocks, (co.row[sel] // 3, co.row[sel] % 3, co.col[sel] % 3), co.data[sel])
    binv = np.linalg.inv(blocks)
    pre = {"mass": lambda r: r / mass, "diagonal": lambda r: r / d,
           "block3": lambda r: np.einsum("vij,vj->vi", binv, r.reshape(-1, 3)).ravel()}
    for k, P in pre.items():
        print(f"{k:9s} random rhs {pcg(Aff, b_rand, P):3d} it, smooth rhs {pcg(Aff, b_smooth, P):3d} it")
    print(f"diag(A)/mass: median {np.median(d / mass):.2f}, max {d.max() / mass.min():.2f}")


if __name__ == "__main__":
    main()
