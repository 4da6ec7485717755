"""Oracle self-sensitivity of configs[1] (256^2 cloth dropped on the sphere, 60 frames x 10 substeps):
the fp64 oracle against itself after a 1e-9 m perturbation of x0, relative L2 of the positions at
every 10th frame.  CPU only, calls only oracle/ and synth/ (about 6 minutes); writes
tests/golden/medium_cloth_sensitivity.json, which test_medium_cloth_full_size_full_length_forward
uses as the bound beyond the horizon on which the workload is well conditioned (after the cloth
meets the sphere, around frame 15, wrinkling amplifies round-off: DESIGN.md "Precision")."""
import json
import os
import sys

import numpy as np

ROOT = __file__.rsplit("/tests/", 1)[0]
sys.path.insert(0, ROOT)
from oracle import OracleModel  # noqa: E402
from synth import as_float32_exact, medium_cloth  # noqa: E402

s = as_float32_exact(medium_cloth())
m = OracleModel(s)
xa = m.simulate(s.x0, s.v0, None, s.frames)
xb = m.simulate(s.x0 + 1e-9 * np.random.default_rng(0).standard_normal(s.x0.shape), s.v0, None, s.frames)
out = {"workload": "medium_cloth 256x256 + sphere, 60 frames x 10 substeps (BASELINE configs[1])",
       "perturbation_m": 1e-9,
       "rel_l2": {str(f): float(np.linalg.norm(xa[f * s.substeps] - xb[f * s.substeps]) / np.linalg.norm(xa[f * s.substeps]))
                  for f in range(10, s.frames + 1, 10)}}
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "medium_cloth_sensitivity.json"), "w"), indent=1)
print(json.dumps(out))
