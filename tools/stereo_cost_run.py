"""ncu driver for the stereo cost construction (hgf_stereo_wta at C4 size, one 128-label chunk)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1803_00005_b200 import HGF  # noqa: E402

c = synth.config("C4")
L = 128
scene = synth.make_stereo_scene(c["W"], c["H"], L, c["seed"])
h = HGF(c["W"], c["H"], c["m"], c["d"], c["r"], c["lam"])
out = h.stereo_wta(torch.from_numpy(scene.left).cuda(), torch.from_numpy(scene.right).cuda(), L, labels=True)
torch.cuda.synchronize()
print("ok", float(out["labels"].float().mean()))
