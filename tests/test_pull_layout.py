"""CPU checks of the pull layout of the adjoint PCG's tile kernels (csrc/pull.cuh), through the
host-only C call dxpbd_pull_layout: a numpy emulation of the kernel's two passes over the
library's own index stream must reproduce A_dist p = Sum_j P_j^T Q_j P_j p (PAPER.md Eq.
adjointXPBD l.150-161 with the blocks of Sec.4.3 l.166-194) computed directly from the
constraints, and the layout must keep the structural promises the kernels rely on."""
import numpy as np
import pytest

from synth import garment, large_cloth, medium_cloth, tiny_cloth
from tests.gpu_helpers import random_network


def _layout(s):
    from paper_2301_01396_b200 import api
    return api.dxpbd_pull_layout(**api.scene_kwargs(s))


def _cases():
    return [
        ("tiny16", lambda: tiny_cloth()),
        ("cloth96", lambda: large_cloth(n=96, frames=1, side=10.0 * 95 / 2943.0, key_frames=(1,))),
        ("cloth_ragged", lambda: large_cloth(n=75, frames=1, side=10.0 * 74 / 2943.0, key_frames=(1,))),
        ("sphere48", lambda: medium_cloth(n=48, frames=1)),
        ("garment_tube", lambda: garment(n_around=64, n_along=48, frames=1)),
        ("random_network", lambda: random_network()),   # irregular, degree 16: overflow > kTileV, > 8 secondaries
    ]


def _emulate(L, Q_user, p):
    """q = A_dist p with the kernel's data flow: per tile, vector slots (own, halo), primary pass
    (y = Q (p_i - p_o) into the entry's slot, added to the own vertex), overflow entries, secondary
    pass (signed sum of the listed y slots)."""
    TV, hcap, nt = L["tile_v"], L["hcap"], L["tiles"]
    V = len(L["vperm"])
    E = len(L["perm"])
    Qs = np.full((L["block_slots"] + 1, 3, 3), np.nan)          # blocks in layout order; padding stays NaN
    for q in range(E):
        Qs[L["tpos"][q]] = Q_user[L["perm"][q]]
        if L["fpos"][q] >= 0:
            Qs[L["fpos"][q]] = Q_user[L["perm"][q]]
    out = np.zeros((V, 3))
    written = np.zeros(L["block_slots"] + 1, bool)
    for t in range(nt):
        qbase, ibase, z, nover = (int(v) for v in L["tdesc"][t])
        K0, KS2 = z & 0xff, (z >> 8) & 0xff
        K02 = (K0 + 1) // 2
        ix = L["idx"][ibase:]
        prim = ix[: K02 * TV].reshape(K02, TV)
        sec = ix[K02 * TV: (K02 + KS2) * TV].reshape(KS2, TV)
        over = ix[(K02 + KS2) * TV: (K02 + KS2) * TV + nover]
        sp = np.zeros((TV + hcap, 3))
        nv = min(TV, V - t * TV)
        sp[:nv] = p[t * TV: t * TV + nv]
        for h in range(hcap):
            if L["hpad"][t, h] >= 0:
                sp[TV + h] = p[L["hpad"][t, h]]
        yb = np.full((L["ycap"], 3), np.nan)
        acc = np.zeros((TV, 3))
        for i in range(TV):
            for k in range(K0):
                en = (int(prim[k // 2, i]) >> (16 * (k & 1))) & 0xffff
                o = en & 0x7ff
                if o == 0x7ff:
                    continue
                pos = k * TV + (i & ~31) + (en >> 11)
                assert not written[qbase + pos], "two entries share a block slot"
                written[qbase + pos] = True
                y = Qs[qbase + pos] @ (sp[i] - sp[o])
                acc[i] += y
                yb[pos] = y
        for e in range(nover):
            own, oth = int(over[e]) & 0xffff, int(over[e]) >> 16
            pos = K0 * TV + e
            assert not written[qbase + pos]
            written[qbase + pos] = True
            yb[pos] = Qs[qbase + pos] @ (sp[own] - sp[oth])
        for i in range(TV):
            for k in range(2 * KS2):
                en = (int(sec[k // 2, i]) >> (16 * (k & 1))) & 0xffff
                if en == 0xffff:
                    continue
                y = yb[en & 0x7fff]
                acc[i] += y if en & 0x8000 else -y
        out[t * TV: t * TV + nv] = acc[:nv]
    return out, written


@pytest.mark.parametrize("case", range(6))
def test_pull_layout_reproduces_the_constraint_sum(case):
    name, mk = _cases()[case]
    s = mk()
    L = _layout(s)
    V, E = len(s.x0), len(s.dist_idx)
    rng = np.random.default_rng(11 + case)
    B = rng.standard_normal((E, 3, 3))
    Q = B @ B.transpose(0, 2, 1)                                   # symmetric blocks, user constraint order
    p_user = rng.standard_normal((V, 3))
    vperm = L["vperm"]
    p = p_user[vperm]                                              # internal order
    got, written = _emulate(L, Q, p)
    # direct sum over the constraints (user order), mapped to internal order
    want_user = np.zeros((V, 3))
    a, b = s.dist_idx[:, 0], s.dist_idx[:, 1]
    y = np.einsum("eij,ej->ei", Q, p_user[a] - p_user[b])
    np.add.at(want_user, a, y)
    np.add.at(want_user, b, -y)
    np.testing.assert_allclose(got, want_user[vperm], rtol=1e-11, atol=1e-11, err_msg=name)
    # every constraint has one slot in its a-tile and, when it crosses tiles, one in its b-tile; every
    # written slot is a constraint's
    TV = L["tile_v"]
    ab = L["sorted_ab"]
    cross = ab[:, 0] // TV != ab[:, 1] // TV
    assert np.array_equal(L["fpos"] >= 0, cross), name
    slots = np.concatenate([L["tpos"], L["fpos"][cross]])
    assert len(np.unique(slots)) == len(slots) == int(written.sum()), name
    assert np.array_equal(np.sort(ab[:, 0]) >= 0, np.ones(E, bool)) and (ab[:, 0] < ab[:, 1]).all()
    # sorted constraints are the user's, re-indexed
    inv = np.empty(V, np.int64)
    inv[vperm] = np.arange(V)
    ua = np.sort(inv[s.dist_idx[L["perm"]]], axis=1)
    assert np.array_equal(ua, ab), name


@pytest.mark.parametrize("case", (1, 2))
def test_pull_layout_structure_on_cloth_grids(case):
    """On a cloth lattice the layout keeps what the kernel's speed relies on: six dense slabs nearly
    full (little padding), overflow entries = cross-tile copies only, conflict-free direct accesses
    (distinct 16-byte bank groups within each quarter-warp), and the replay's per-color writes in
    runs of whole 32-byte sectors."""
    name, mk = _cases()[case]
    s = mk()
    L = _layout(s)
    TV = L["tile_v"]
    V, E = len(s.x0), len(s.dist_idx)
    ab = L["sorted_ab"]
    ncross = int((ab[:, 0] // TV != ab[:, 1] // TV).sum())
    assert L["block_slots"] <= 1.35 * (E + ncross), (name, L["block_slots"], E, ncross)
    bad = tot = 0
    for t in range(L["tiles"]):
        qbase, ibase, z, nover = (int(v) for v in L["tdesc"][t])
        K0 = z & 0xff
        assert K0 <= L["dense_slabs_max"]
        prim = L["idx"][ibase: ibase + ((K0 + 1) // 2) * TV].reshape((K0 + 1) // 2, TV)
        for k in range(K0):
            en = (prim[k // 2] >> (16 * (k & 1))) & 0xffff
            lanes = (en >> 11).astype(int)
            for w0 in range(0, TV, 32):                            # a warp's lanes are a permutation
                assert sorted(lanes[w0: w0 + 32]) == list(range(32)), (name, t, k)
            on = (en & 0x7ff) != 0x7ff
            for q0 in range(0, TV, 8):                             # quarter-warp: distinct bank groups
                b = lanes[q0: q0 + 8][on[q0: q0 + 8]] & 7
                tot += len(b)
                bad += len(b) - len(np.unique(b))
    assert bad <= 0.02 * tot, (name, bad, tot)
    # replay writes: a color launch writes the slots of its constraints; a slot's 32-byte sector mate
    # (slot ^ 1) should be written by the same launch, or by nobody (padding), for nearly all slots
    from oracle.coloring import greedy_color
    color = greedy_color(np.asarray(s.dist_idx, np.int32), V)[L["perm"]]   # per sorted constraint (R1)
    owner = np.full(L["block_slots"] + 2, -1, np.int64)
    cross = L["fpos"] >= 0
    owner[L["tpos"]] = color
    owner[L["fpos"][cross]] = color[cross]
    used = np.flatnonzero(owner[:-2] >= 0)
    mate = owner[used ^ 1]
    split = int(((mate >= 0) & (mate != owner[used])).sum())
    assert split <= 0.15 * len(used), (name, split, len(used))


def test_pull_layout_rejects_bad_input():
    from paper_2301_01396_b200 import api
    s = tiny_cloth()
    kw = api.scene_kwargs(s)
    kw["dist_idx"] = np.asarray(kw["dist_idx"]).copy()
    kw["dist_idx"][0, 0] = 10 ** 6
    with pytest.raises(api.DxpbdError):
        api.dxpbd_pull_layout(**kw)
