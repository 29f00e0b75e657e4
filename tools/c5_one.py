import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_1803_00005_b200 import HGF
W, H = 1920, 1080
scene = synth.make_stereo_scene(W, H, 64, seed=5)
Y = synth.stereo_cost_volume_torch(scene, 64, "cuda", 20, 21)[0].contiguous()
for (m, d, r) in ((3, 3, 4), (10, 2, 8)):
    I = torch.from_numpy(synth.smooth_guides(W, H, m, seed=5)).cuda()
    h = HGF(W, H, m, d, r, 0.05)
    dst = torch.empty((H, W), dtype=torch.float32, device="cuda")
    h.filter(I, Y, dst); h.filter(I, Y, dst)
    torch.cuda.synchronize()
    h.close()
