import sys, numpy as np
sys.path.insert(0, '.')
from synth import as_float32_exact, volumetric_block
from tests.gpu_helpers import gpu_run, oracle_run, rel_l2
from oracle import OracleModel, greedy_color
n = 6
base = as_float32_exact(volumetric_block(n=n, frames=1, substeps=1, side=0.4 * (n - 1) / 39).replace(frame_dt=1 / 1200))
col = greedy_color(base.tet_idx, base.num_vertices)
for name, sel in [("c0", col == 0), ("c0-1", col <= 1), ("first2tets", np.arange(len(col)) < 2),
                  ("first10", np.arange(len(col)) < 10), ("all", col >= 0)]:
    s = base.replace(tet_idx=base.tet_idx[sel], tet_a=base.tet_a[sel], tet_b=base.tet_b[sel])
    g = gpu_run(s, backward=False); o = oracle_run(s, backward=False)
    dd = np.abs(g["x"][1] - o["x"][1]).max(1)
    print(name, sel.sum(), "rel", rel_l2(g["x"][1], o["x"][1]), "max", dd.max(), "disp", np.abs(o["x"][1]-o["x"][0]).max())
# single tet from the block with odd orientation
for t in range(5):
    s = base.replace(tet_idx=base.tet_idx[t:t+1], tet_a=base.tet_a[t:t+1], tet_b=base.tet_b[t:t+1])
    x0 = s.x0.copy(); x0[s.tet_idx[0]] *= 1.05
    s = s.replace(x0=x0)
    g = gpu_run(s, backward=False); o = oracle_run(s, backward=False)
    print("tet", t, s.tet_idx[0], "rel", rel_l2(g["x"][1], o["x"][1]))
