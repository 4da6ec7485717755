"""Kernel-class profile of configs[2] (volumetric block, 2 frames) through dxpbd_profile /
dxpbd_kernel_times; used to find the tet replay bottleneck."""
import sys, numpy as np, torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2301_01396_b200 import api
from synth import as_float32_exact, volumetric_block
s = as_float32_exact(volumetric_block(frames=2))
sc = api.dxpbd_create(**api.scene_kwargs(s), max_frames=2, grad_flags=api.flags("material"), cg_max_iter=2000)
t = lambda a: torch.as_tensor(np.asarray(a, np.float32), device="cuda:0")
api.dxpbd_forward(sc, t(s.x0), t(s.v0), None, 2); api.dxpbd_backward(sc, s.key_frames, t(s.targets))
api.dxpbd_profile(sc, True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); api.dxpbd_forward(sc, t(s.x0), t(s.v0), None, 2); api.dxpbd_backward(sc, s.key_frames, t(s.targets)); e1.record()
torch.cuda.synchronize()
print("total ms", e0.elapsed_time(e1), "substeps", 40)
kt = api.dxpbd_kernel_times(sc)
for k, (ms, n) in sorted(kt.items(), key=lambda x: -x[1][0]): print(f"{k:16s} {ms:9.2f} ms {int(n):6d} launches {1000*ms/max(n,1):8.1f} us/launch")
print(api.dxpbd_stats(sc))
