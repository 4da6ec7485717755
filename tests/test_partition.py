"""Vertex-partitioned domain decomposition (paper_2301_01396_b200.partition) on CPU: plan
invariants, and a world_size-2 gloo execution of the partitioned colored Gauss-Seidel substep and
of the partitioned PCG matvec that must reproduce the global (single-device) computation.  The
per-rank compute is the oracle's (test infrastructure), the plan and the exchanges are the
product's host logic."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _scene():
    from synth import large_cloth, as_float32_exact
    return as_float32_exact(large_cloth(n=24, frames=1, substeps=2, iterations=2, side=1.0, key_frames=(1,)))


def test_plan_invariants():
    from oracle import greedy_color
    from paper_2301_01396_b200.partition import plan, morton_order
    s = _scene()
    col = greedy_color(s.dist_idx, s.num_vertices)
    for world in (1, 2, 3, 4):
        P = plan(s.x_rest, s.dist_idx, col, world)
        owned = np.concatenate([p.owned for p in P])
        assert sorted(owned.tolist()) == list(range(s.num_vertices))
        cons = np.concatenate([c for p in P for c in p.cons])
        assert sorted(cons.tolist()) == list(range(len(s.dist_idx)))      # each constraint exactly once
        for p in P:
            assert not set(p.ghosts.tolist()) & set(p.owned.tolist())
            for (c, dst), v in p.send.items():
                np.testing.assert_array_equal(P[dst].recv[(c, p.rank)], v)
    perm = morton_order(s.x_rest)
    assert sorted(perm.tolist()) == list(range(s.num_vertices))


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _exchange(dist, P, key_send, key_recv, x, world):
    """Point-to-point exchange of vertex rows: send x[ids] for every (key, dst) and overwrite
    x[ids] with what (key, src) sends; neighbours only."""
    import torch
    reqs = []
    for dst in range(world):
        ids = key_send(dst)
        if ids is not None:
            reqs.append(dist.isend(torch.as_tensor(x[ids]), dst))
    for src in range(world):
        ids = key_recv(src)
        if ids is not None:
            buf = torch.empty((len(ids), 3), dtype=torch.float64)
            dist.recv(buf, src)
            x[ids] = buf.numpy()
    for r in reqs:
        r.wait()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle import OracleModel
    from paper_2301_01396_b200.partition import plan
    dist.init_process_group("gloo", init_method="env://")
    s = _scene()
    m = OracleModel(s)
    P = plan(s.x_rest, s.dist_idx, m.dist_color, world)[rank]
    held = np.concatenate([P.owned, P.ghosts])
    # ---- partitioned forward substeps (R1 sweep, exchange after every color)
    x = s.x0.copy()
    v = s.v0.copy()
    dt = m.dt
    for n in range(s.num_steps):
        xn = x.copy()
        x = m.predict(xn, v, s.forces[0])
        lam = np.zeros(m.E)
        for _it in range(s.iterations):
            for c, grp in enumerate(P.cons):
                if len(grp):
                    m._project(x, m.dist_idx[grp], m.ev_dist(x, grp), m.at_dist[grp][:, None], lam, None, "dist", grp)
                _exchange(dist, P, lambda d, c=c: P.send.get((c, d)), lambda r_, c=c: P.recv.get((c, r_)), x, world)
        v = (x - xn) / dt
    # ---- partitioned PCG matvec of the global replayed system: q = (M + Sum Q_j) p
    xs_g = m.simulate(s.x0, s.v0, s.forces, 1)
    _, _, rec = m.step(xs_g[0], s.v0, s.forces[0], record=True)
    Qb = m.blocks(rec)["dist"]                       # (E,6,6) per-constraint blocks
    p = np.random.default_rng(5).standard_normal(x.shape)
    pl = np.zeros_like(p)
    pl[P.owned] = p[P.owned]                         # only owned values are known locally
    _exchange(dist, P, lambda d: P.halo_send.get(d), lambda r_: P.halo_recv.get(r_), pl, world)
    ql = np.zeros_like(p)
    ql[P.owned] = (m.m[:, None] * pl)[P.owned]
    mine = np.concatenate(P.cons)
    st = m.dist_idx[mine]
    dq = np.einsum("nij,nj->ni", Qb[mine], pl[st].reshape(len(mine), 6)).reshape(len(mine), 2, 3)
    contrib = np.zeros_like(p)
    np.add.at(contrib, st[:, 0], dq[:, 0])
    np.add.at(contrib, st[:, 1], dq[:, 1])
    # contributions to ghost vertices go to their owners (accumulate)
    import torch as _t
    reqs = []
    for dst, ids in P.halo_recv.items():             # my ghosts are owned by dst
        reqs.append(dist.isend(_t.as_tensor(contrib[ids]), dst))
    for src, ids in P.halo_send.items():             # src mirrors my owned vertices
        buf = _t.empty((len(ids), 3), dtype=_t.float64)
        dist.recv(buf, src)
        contrib[ids] += buf.numpy()
    for r_ in reqs:
        r_.wait()
    ql[P.owned] += contrib[P.owned]
    ql[~m.free] = 0.0
    dist.barrier()
    q.put(dict(rank=rank, held=held, x=x[held], owned=P.owned, q=ql[P.owned]))
    dist.destroy_process_group()


def test_partitioned_sweep_and_matvec_world2():
    import torch.multiprocessing as mp
    from oracle import OracleModel
    s = _scene()
    m = OracleModel(s)
    xs = m.simulate(s.x0, s.v0, s.forces, 1)       # global reference sweep
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, qu)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [qu.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for r in res:
        # every vertex a rank holds (owned and ghost) equals the global sweep bit for bit
        np.testing.assert_array_equal(r["x"], xs[-1][r["held"]])
    # global matvec
    _, _, rec = m.step(xs[0], s.v0, s.forces[0], record=True)
    A = m.system_matrix(m.blocks(rec)).toarray()
    p = np.random.default_rng(5).standard_normal((m.V, 3))
    qg = (A @ p.ravel()).reshape(m.V, 3)
    qg[~m.free] = 0.0
    for r in res:
        np.testing.assert_allclose(r["q"], qg[r["owned"]], rtol=1e-12, atol=1e-12 * np.abs(qg).max())
