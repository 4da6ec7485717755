"""Vertex-partitioned domain decomposition on CPU with the PRODUCT's planner: the host-only C call
`dxpbd_partition_plan` (the same `partition_plan` / `dist_topology` code that `dxpbd_group_create`
and `dxpbd_group_create_dist` build their exchange lists from, include/dxpbd.h).  Plan invariants,
and a world_size-2 gloo execution of the partitioned colored Gauss-Seidel substep and of the
partitioned PCG matvec driven by those lists, which must reproduce the global (single-device)
computation.  The per-rank compute is the oracle's (test infrastructure); the plan and the
exchange pattern are the product's."""
import os
import socket
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _scene():
    from synth import large_cloth, as_float32_exact
    # 48 x 48 = 2304 vertices = 4.5 Morton tiles of 512: a ragged last tile
    return as_float32_exact(large_cloth(n=48, frames=1, substeps=2, iterations=1, side=1.0, key_frames=(1,)))


def _plan(s, world, rank):
    from paper_2301_01396_b200 import api
    return api.dxpbd_partition_plan(**api.scene_kwargs(s), num_parts=world, rank=rank, max_frames=1)


def _internal(s, pl):
    """Constraint endpoints in internal (Morton) ids, oriented a < b, and the owning rank of each
    internal vertex (tile ranges [t0, t1) of every rank)."""
    vinv = np.empty_like(pl["vperm"])
    vinv[pl["vperm"]] = np.arange(len(pl["vperm"]))
    ab = np.sort(vinv[np.asarray(s.dist_idx)], axis=1)
    return vinv, ab


def test_plan_invariants():
    from oracle import greedy_color
    s = _scene()
    col = greedy_color(s.dist_idx, s.num_vertices)
    V, tv = s.num_vertices, 512
    for world in (1, 2, 3, 4):
        plans = [_plan(s, world, r) for r in range(world)]
        pl0 = plans[0]
        assert sorted(pl0["vperm"].tolist()) == list(range(V))                  # a permutation
        assert pl0["colors"] == col.max() + 1                                    # the same greedy colors (R1)
        assert [p["t0"] for p in plans] == sorted(p["t0"] for p in plans)
        assert plans[0]["t0"] == 0 and plans[-1]["t1"] == pl0["tiles"]
        for a, b in zip(plans, plans[1:]):
            assert a["t1"] == b["t0"]                                            # contiguous tile ranges
        vinv, ab = _internal(s, pl0)
        owner = np.empty(V, np.int64)
        for r, p in enumerate(plans):
            owner[p["t0"] * tv: min(p["t1"] * tv, V)] = r
        # tile halos: the other endpoints of cross-tile constraints
        halo = {}
        cross = ab[:, 0] // tv != ab[:, 1] // tv
        for a_, b_ in ab[cross]:
            halo.setdefault(a_ // tv, set()).add(b_)
            halo.setdefault(b_ // tv, set()).add(a_)
        for r, p in enumerate(plans):
            held = set(np.nonzero(owner == r)[0].tolist())
            myh = set()
            for t in range(p["t0"], p["t1"]):
                myh |= {v for v in halo.get(t, ()) if owner[v] != r}
            held |= myh
            for q, other in enumerate(plans):
                for k in list(range(p["colors"])) + ["halo", "blocks"]:
                    # what r sends to q is exactly what q expects from r
                    np.testing.assert_array_equal(p["send"][k][q], other["recv"][k][r])
                if q == r:
                    continue
                # per color: every endpoint of r's constraints of that color held by q is sent to q
                for c in range(p["colors"]):
                    mine = (col == c) & (owner[ab[:, 0]] == r)
                    need = {v for v in ab[mine].ravel().tolist() if owner[v] == q or v in _held_halo(plans[q], owner, halo, q)}
                    assert set(p["send"][c][q].tolist()) == need
                # halo: r's own vertices in q's tile halos
                assert set(p["send"]["halo"][q].tolist()) == {v for v in _held_halo(plans[q], owner, halo, q) if owner[v] == r}
                # blocks: one b-tile copy per constraint owned by r whose b lies in q
                nb = int(((owner[ab[:, 0]] == r) & (owner[ab[:, 1]] == q) & cross).sum())
                assert len(p["send"]["blocks"][q]) == nb
            assert set().union(*[set(p["recv"]["halo"][q].tolist()) for q in range(world)]) == myh


def _held_halo(p, owner, halo, q):
    out = set()
    for t in range(p["t0"], p["t1"]):
        out |= {v for v in halo.get(t, ()) if owner[v] != q}
    return out


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _exchange(dist, send, recv, x, world, rank):
    """Point-to-point exchange of vertex rows (user ids): send x[ids] to every peer with a list and
    overwrite x[ids] with what each peer sends."""
    import torch
    reqs = []
    for dst in range(world):
        ids = send.get(dst)
        if dst != rank and ids is not None and len(ids):
            reqs.append(dist.isend(torch.as_tensor(x[ids]), dst))
    for src in range(world):
        ids = recv.get(src)
        if src != rank and ids is not None and len(ids):
            buf = torch.empty((len(ids), 3), dtype=torch.float64)
            dist.recv(buf, src)
            x[ids] = buf.numpy()
    for r in reqs:
        r.wait()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from oracle import OracleModel
    dist.init_process_group("gloo", init_method="env://")
    s = _scene()
    m = OracleModel(s)
    pl = _plan(s, world, rank)
    vp = pl["vperm"]                                  # internal -> user
    vinv, ab = _internal(s, pl)
    tv = pl["tile_v"]
    v0, v1 = pl["t0"] * tv, min(pl["t1"] * tv, s.num_vertices)
    owned = vp[v0:v1]                                 # user ids of the owned vertices
    mine = np.nonzero((ab[:, 0] >= v0) & (ab[:, 0] < v1))[0]          # constraints owned (lower endpoint)
    user = lambda lists: {k: vp[v] for k, v in lists.items()}          # noqa: E731
    # ---- partitioned forward substeps (R1 sweep, exchange along the plan's lists after every color)
    x = s.x0.copy()
    v = s.v0.copy()
    for _n in range(s.num_steps):
        xn = x.copy()
        x = m.predict(xn, v, s.forces[0])
        lam = np.zeros(m.E)
        for c in range(pl["colors"]):
            grp = mine[m.dist_color[mine] == c]
            if len(grp):
                m._project(x, m.dist_idx[grp], m.ev_dist(x, grp), m.at_dist[grp][:, None], lam, None, "dist", grp)
            _exchange(dist, user(pl["send"][c]), user(pl["recv"][c]), x, world, rank)
        v = (x - xn) / m.dt
    # ---- partitioned PCG matvec of the global replayed system, q = (M + Sum Q_j) p, over owned rows:
    # every constraint touching an owned vertex, with the neighbours' p from the plan's halo lists
    xs_g = m.simulate(s.x0, s.v0, s.forces, 1)
    _, _, rec = m.step(xs_g[0], s.v0, s.forces[0], record=True)
    Qb = m.blocks(rec)["dist"]
    p = np.random.default_rng(5).standard_normal(x.shape)
    pl_p = np.zeros_like(p)
    pl_p[owned] = p[owned]                            # only owned values are known locally
    _exchange(dist, user(pl["send"]["halo"]), user(pl["recv"]["halo"]), pl_p, world, rank)
    is_owned = np.zeros(s.num_vertices, bool)
    is_owned[owned] = True
    touch = np.nonzero(is_owned[m.dist_idx[:, 0]] | is_owned[m.dist_idx[:, 1]])[0]
    st = m.dist_idx[touch]
    dq = np.einsum("nij,nj->ni", Qb[touch], pl_p[st].reshape(len(touch), 6)).reshape(len(touch), 2, 3)
    ql = np.zeros_like(p)
    ql[owned] = (m.m[:, None] * pl_p)[owned]
    contrib = np.zeros_like(p)
    np.add.at(contrib, st[:, 0], dq[:, 0])
    np.add.at(contrib, st[:, 1], dq[:, 1])
    ql[owned] += contrib[owned]
    ql[~m.free] = 0.0
    held = np.nonzero(is_owned | np.isin(np.arange(s.num_vertices), vp[np.concatenate(
        [pl["recv"]["halo"][r] for r in range(world)])]))[0]
    dist.barrier()
    q.put(dict(rank=rank, x=x[owned], owned=owned, q=ql[owned], held=held, xh=x[held]))
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
        # owned vertices and every halo vertex a rank holds equal the global sweep bit for bit
        np.testing.assert_array_equal(r["x"], xs[-1][r["owned"]])
        np.testing.assert_array_equal(r["xh"], xs[-1][r["held"]])
    _, _, rec = m.step(xs[0], s.v0, s.forces[0], record=True)
    A = m.system_matrix(m.blocks(rec)).toarray()
    p = np.random.default_rng(5).standard_normal((m.V, 3))
    qg = (A @ p.ravel()).reshape(m.V, 3)
    qg[~m.free] = 0.0
    for r in res:
        np.testing.assert_allclose(r["q"], qg[r["owned"]], rtol=1e-12, atol=1e-12 * np.abs(qg).max())
