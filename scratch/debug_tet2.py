import sys, numpy as np
sys.path.insert(0, '.')
from synth import Scene, as_float32_exact, volumetric_block
from synth.scenes import _base
from tests.gpu_helpers import gpu_run, oracle_run, rel_l2
np.set_printoptions(precision=5, suppress=True, linewidth=150)
x = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0], [1, 1, 1.0]]) * 0.1
d = dict(x_rest=x, inv_mass=np.array([0.0, 1.0, 2.0, 1.5, 1.0]), tet_idx=np.array([[0, 1, 2, 3], [1, 2, 3, 4]], np.int32),
         tet_a=np.array([30.0, 20.0]), tet_b=np.array([60.0, 50.0]))
b = _base("t", 5, **d)
b["x0"] = x * np.array([1.2, 0.9, 1.1])
b["gravity"] = np.zeros(3)
s = as_float32_exact(Scene(**b, frame_dt=1 / 60, substeps=1, iterations=1, frames=1,
                           key_frames=np.array([1], np.int32), targets=x[None]))
g = gpu_run(s, backward=False); o = oracle_run(s, backward=False)
print("2tet rel", rel_l2(g["x"][1], o["x"][1])); print(g["x"][1] - o["x"][1])
for n, sub, fr in [(3, 1, 1), (5, 1, 1), (5, 4, 1)]:
    s = as_float32_exact(volumetric_block(n=n, frames=fr, substeps=sub, side=0.1))
    g = gpu_run(s, backward=False); o = oracle_run(s, backward=False)
    dd = np.abs(g["x"][1] - o["x"][1]).max(1)
    print(n, sub, "rel", rel_l2(g["x"][1], o["x"][1]), "worst verts", np.argsort(-dd)[:6], dd.max())
    print(" ntets", len(s.tet_idx), "disp", np.abs(o["x"][1] - o["x"][0]).max())
