import sys, numpy as np
sys.path.insert(0, '.')
from synth import as_float32_exact, volumetric_block
from tests.gpu_helpers import gpu_run, oracle_run, rel_l2
from oracle import OracleModel
np.set_printoptions(precision=5, suppress=True, linewidth=150)
n = 6
s = as_float32_exact(volumetric_block(n=n, frames=1, substeps=1, side=0.4 * (n - 1) / 39).replace(frame_dt=1 / 1200))
g = gpu_run(s, backward=False); o = oracle_run(s, backward=False)
dd = np.abs(g["x"][1] - o["x"][1]).max(1)
print("rel", rel_l2(g["x"][1], o["x"][1]), "n bad verts", (dd > 1e-9).sum(), "of", len(dd))
m = OracleModel(s)
# which tets touch bad vertices, per color
bad = set(np.nonzero(dd > 1e-9)[0].tolist())
print("bad verts", sorted(bad)[:20])
for c, grp in enumerate(m.tet_groups):
    touched = [t for t in grp if set(s.tet_idx[t].tolist()) & bad]
    print("color", c, "ntets", len(grp), "touching bad", len(touched))
# oracle with colors processed in reverse order inside the iteration? no: check per-color partial sweeps
x = m.predict(s.x0, s.v0, np.zeros_like(s.x0))
print("pred diff vs gpu?", np.abs(x - o["x"][0]).max())
