import sys, numpy as np
sys.path.insert(0, '.')
from synth import Scene, as_float32_exact
from synth.scenes import _base
from oracle import OracleModel
from tests.gpu_helpers import gpu_run, oracle_run, rel_l2
np.set_printoptions(precision=6, suppress=True)
x = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0]]) * 0.1
for case in ["stretched", "rest_gravity"]:
    d = dict(x_rest=x, inv_mass=np.array([0.0, 1.0, 2.0, 1.5]), tet_idx=np.array([[0, 1, 2, 3]], np.int32),
             tet_a=np.array([30.0]), tet_b=np.array([60.0]))
    b = _base("t", 4, **d)
    if case == "stretched":
        b["x0"] = x * np.array([1.2, 0.9, 1.1])
        b["gravity"] = np.zeros(3)
    s = as_float32_exact(Scene(**b, frame_dt=1 / 60, substeps=1, iterations=1, frames=1,
                               key_frames=np.array([1], np.int32), targets=x[None]))
    g = gpu_run(s, ("material",))
    o = oracle_run(s)
    print(case, "gpu\n", g["x"][1], "\noracle\n", o["x"][1], "\nrel", rel_l2(g["x"][1], o["x"][1]))
    print(" mat grad gpu", g["material"], "oracle", o["material"])
