"""One hgf_filter call at BASELINE config 5 (1920x1080 single slice) for ncu captures: m, d, r from argv."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1803_00005_b200 import HGF  # noqa: E402

m, d, r = (int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (3, 2, 9)
W, H = 1920, 1080
scene = synth.make_stereo_scene(W, H, 64, seed=5)
Y = synth.stereo_cost_volume_torch(scene, 64, "cuda", 20, 21)[0].contiguous()
I = torch.from_numpy(synth.smooth_guides(W, H, m, seed=5)).cuda()
h = HGF(W, H, m, d, r, 0.05)
dst = torch.empty((H, W), dtype=torch.float32, device="cuda")
h.filter(I, Y, dst)
torch.cuda.synchronize()
print(h.kernel_path)
h.close()
