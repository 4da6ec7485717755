"""Long-horizon parity of the configs[4] workload shape at reduced size: the full 30 frames x 10
substeps with keyframes at frames 10 / 20 / 30 and per-frame forces, gradients of forces, x0, v0,
GPU (C-ABI, default schedules) vs the fp64 oracle.  One JSON line; recorded in
profiles/r01_long_parity.json (the GPU test suite covers the same path at shorter horizons)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tests/", 1)[0])
from synth import as_float32_exact, large_cloth  # noqa: E402
from tests.gpu_helpers import gpu_run, oracle_run, rel_l2  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 96
s = as_float32_exact(large_cloth(n=n, frames=30, substeps=10, side=10.0 * (n - 1) / 2943.0, key_frames=(10, 20, 30)))
grads = ("forces", "x0", "v0")
t0 = time.perf_counter()
g = gpu_run(s, grads)
t1 = time.perf_counter()
o = oracle_run(s)
t2 = time.perf_counter()
out = dict(workload=f"large_cloth {n}x{n}, 30 frames x 10 substeps, keyframes 10/20/30, forces",
           positions_rel_l2={f: rel_l2(g["x"][f], o["x"][f]) for f in (10, 20, 30)},
           loss_gpu=g["loss"], loss_oracle=o["loss"],
           grads_rel_l2={k: rel_l2(g[k], o[k]) for k in grads},
           gpu_s=t1 - t0, oracle_s=t2 - t1)
print(json.dumps(out), flush=True)

# Oracle self-sensitivity (run on CPU, no GPU needed): perturb x0 by 1e-9 m on free vertices and
# compare the fp64 oracle with itself (rel L2 per frame).
if len(sys.argv) > 2 and sys.argv[2] == "--sensitivity":
    from oracle import OracleModel
    m = OracleModel(s)
    xa = m.simulate(s.x0, s.v0, s.forces, 30)
    x0b = s.x0 + 1e-9 * np.random.default_rng(0).standard_normal(s.x0.shape) * (s.inv_mass > 0)[:, None]
    xb = m.simulate(x0b, s.v0, s.forces, 30)
    print(json.dumps({"oracle_self_sensitivity_1e-9m": {f: rel_l2(xb[f * 10], xa[f * 10]) for f in (1, 5, 10, 15, 20, 25, 30)}}))
