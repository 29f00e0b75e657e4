"""Small end-to-end case for compute-sanitizer runs (memcheck / racecheck): statistics (k_stats4, n = 6 and
n = 9, two row bands), the interleaved slice path and hgf_filter on ragged sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1803_00005_b200 import HGF  # noqa: E402

for (W, H, m, d, L, r) in ((77, 53, 3, 2, 5, 9), (45, 70, 3, 3, 4, 9), (150, 300, 3, 2, 3, 4)):
    scene = synth.make_stereo_scene(W, H, L, seed=7)
    g = torch.from_numpy(scene.left).cuda()
    v = synth.stereo_cost_volume_torch(scene, L, "cuda", 0, L)
    h = HGF(W, H, m, d, r, 0.05)
    lab = torch.empty((H, W), dtype=torch.int32, device="cuda")
    h.aggregate_wta(g, v, lab)
    dst = torch.empty((H, W), dtype=torch.float32, device="cuda")
    h.filter(g, v[0].contiguous(), dst)
    torch.cuda.synchronize()
    h.close()
print("ok")
