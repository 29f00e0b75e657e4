"""Small driver for ncu captures of the single-slice hgf_filter path (BASELINE config 5 shapes)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1803_00005_b200 import HGF  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=10)
ap.add_argument("--d", type=int, default=2)
ap.add_argument("--r", type=int, default=8)
ap.add_argument("--iters", type=int, default=1)
a = ap.parse_args()
W, H = 1920, 1080
scene = synth.make_stereo_scene(W, H, 64, seed=5)
Y = synth.stereo_cost_volume_torch(scene, 64, "cuda", 20, 21)[0].contiguous()
I = torch.from_numpy(synth.smooth_guides(W, H, a.m, seed=5)).cuda()
h = HGF(W, H, a.m, a.d, a.r, 0.05)
dst = torch.empty((H, W), dtype=torch.float32, device="cuda")
for _ in range(a.iters):
    h.filter(I, Y, dst)
torch.cuda.synchronize()
print("ok")
