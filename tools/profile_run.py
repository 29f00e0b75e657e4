"""Small driver for ncu captures: one config, a few labels, a few iterations of hgf_aggregate_wta."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1803_00005_b200 as P  # noqa: E402
import synth  # noqa: E402
from paper_1803_00005_b200 import HGF  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--labels", type=int, default=16)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--lib", default=None, help="alternate libhgf.so (timing experiments)")
a = ap.parse_args()
if a.lib:
    P.lib_path = os.path.abspath(a.lib)
c = synth.config(a.config)
L = min(a.labels, c["L"])
scene = synth.make_stereo_scene(c["W"], c["H"], c["L"], c["seed"])
g = torch.from_numpy(scene.left).cuda()
v = synth.stereo_cost_volume_torch(scene, c["L"], "cuda", 0, L)
h = HGF(c["W"], c["H"], c["m"], c["d"], c["r"], c["lam"])
lab = torch.empty((c["H"], c["W"]), dtype=torch.int32, device="cuda")
for _ in range(a.iters):
    h.aggregate_wta(g, v, lab)
torch.cuda.synchronize()
print("ok", a.config, L, lab.float().mean().item())
