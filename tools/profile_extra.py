"""Small driver for ncu captures of the secondary kernels: hgf_stereo_wta (k_stereo_grad / k_stereo_cost),
hgf_segment (k_seg_hist / k_seg_cost), k_stats3 (n = 20) and the opt-in k_coef4."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1803_00005_b200 import HGF  # noqa: E402

W, H, L = 1920, 1080, 64
scene = synth.make_stereo_scene(W, H, L, seed=3)
left, right = torch.from_numpy(scene.left).cuda(), torch.from_numpy(scene.right).cuda()
h = HGF(W, H, 3, 2, 9, 0.05)
h.stereo_wta(left, right, L)
fg = torch.zeros(H, W, dtype=torch.uint8, device="cuda")
bg = torch.zeros(H, W, dtype=torch.uint8, device="cuda")
fg[100:200, 100:300] = 1
bg[800:900, 1500:1700] = 1
h.segment(left, fg, bg)
h.close()
os.environ["HGF_COEF4"] = "1"
vol = synth.stereo_cost_volume_torch(scene, L, "cuda")
h = HGF(W, H, 3, 2, 9, 0.05)
h.aggregate_wta(left, vol)
h.close()
os.environ.pop("HGF_COEF4")
I = torch.from_numpy(synth.smooth_guides(W, H, 20, seed=5)).cuda()
h = HGF(W, H, 20, 1, 8, 0.05)
h.filter(I, vol[0].contiguous())
torch.cuda.synchronize()
h.close()
print("ok")
