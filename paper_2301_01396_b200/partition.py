"""Vertex-partitioned domain decomposition plan for one large mesh ("next" row).

Host-side plan only (numpy, create-time): which rank owns which vertices and constraints, which
vertices each rank mirrors (ghosts), and what must be exchanged after every color of the
Gauss-Seidel sweep so that the partitioned sweep reproduces the single-GPU sweep exactly:

* vertices are ordered by Morton code of the rest positions (the library's internal order) and
  split into `world` contiguous ranges (rank r owns range r);
* a distance constraint (a, b) is projected by the owner of its endpoint with the smaller Morton
  position; the other endpoint is a ghost on that rank if another rank owns it;
* within one color every vertex is written by at most one constraint (R1), so after color c the
  writer of each vertex knows its final value; it sends it to every other rank that holds the
  vertex (owner and ghost holders).  One point-to-point exchange per color, neighbours only.

The PCG matvec needs the ghost values of the search direction once per iteration (same ghost
sets) and two scalar all-reduces.  The plan is verified against the global sweep by
tests/test_partition.py (gloo, world size 2).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def _spread3(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64) & np.uint64(0x1FFFFF)
    x = (x | (x << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
    x = (x | (x << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
    x = (x | (x << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
    x = (x | (x << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
    x = (x | (x << np.uint64(2))) & np.uint64(0x1249249249249249)
    return x


def morton_order(x_rest: np.ndarray) -> np.ndarray:
    """Permutation internal -> user vertex (Z-order of the rest positions in their bounding box,
    ties by user index): the same ordering rule as the library's create step."""
    x = np.asarray(x_rest, np.float32)
    lo = x.min(0)
    ext = float((x.max(0) - lo).max())
    sc = 2097151.0 / ext if ext > 0 else 0.0
    q = np.floor((x - lo).astype(np.float64) * sc + 0.5).astype(np.uint64)   # llround of (x - lo) * sc
    key = _spread3(q[:, 0]) | (_spread3(q[:, 1]) << np.uint64(1)) | (_spread3(q[:, 2]) << np.uint64(2))
    return np.lexsort((np.arange(len(x)), key)).astype(np.int64)


@dataclass
class RankPlan:
    rank: int
    owned: np.ndarray                    # user vertex ids owned by this rank
    cons: list                           # per color: constraint ids (user order) projected here
    ghosts: np.ndarray                   # user vertex ids mirrored from other ranks
    send: dict = field(default_factory=dict)   # (color, dst) -> user vertex ids written here, held by dst
    recv: dict = field(default_factory=dict)   # (color, src) -> user vertex ids written by src, held here
    halo_send: dict = field(default_factory=dict)  # dst -> owned vertex ids that dst mirrors (PCG)
    halo_recv: dict = field(default_factory=dict)  # src -> ghost vertex ids owned by src (PCG)


def plan(x_rest: np.ndarray, dist_idx: np.ndarray, colors: np.ndarray, world: int) -> list:
    """Partition plan of a distance-constraint mesh over `world` ranks.  `colors` is the greedy
    coloring of the constraints (R1)."""
    V = len(x_rest)
    perm = morton_order(x_rest)
    pos = np.empty(V, np.int64)
    pos[perm] = np.arange(V)
    bounds = np.linspace(0, V, world + 1).round().astype(np.int64)
    owner = np.searchsorted(bounds, pos, side="right") - 1
    e = np.asarray(dist_idx, np.int64)
    lo_end = np.where(pos[e[:, 0]] <= pos[e[:, 1]], e[:, 0], e[:, 1])
    cowner = owner[lo_end]
    ncol = int(colors.max()) + 1 if len(colors) else 0
    plans = []
    for r in range(world):
        mine = np.nonzero(cowner == r)[0]
        verts = np.unique(e[mine].ravel())
        ghosts = verts[owner[verts] != r]
        plans.append(RankPlan(rank=r, owned=perm[bounds[r]:bounds[r + 1]],
                              cons=[mine[colors[mine] == c] for c in range(ncol)], ghosts=ghosts))
    held_by = [[] for _ in range(V)]
    for r in range(world):
        for v in plans[r].owned.tolist():
            held_by[v].append(r)
        for v in plans[r].ghosts.tolist():
            held_by[v].append(r)
    for r, P in enumerate(plans):
        for c in range(ncol):
            written = np.unique(e[P.cons[c]].ravel())
            for dst in range(world):
                if dst == r:
                    continue
                sel = [v for v in written.tolist() if dst in held_by[v]]
                if sel:
                    P.send[(c, dst)] = np.asarray(sel, np.int64)
                    plans[dst].recv[(c, r)] = np.asarray(sel, np.int64)
        for src in range(world):
            if src == r:
                continue
            g = P.ghosts[owner[P.ghosts] == src]
            if len(g):
                P.halo_recv[src] = g
                plans[src].halo_send[r] = g
    return plans
