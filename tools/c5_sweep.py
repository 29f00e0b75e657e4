"""BASELINE config 5: 1920x1080 single-slice hgf_filter over guide channels n = m d (degree 1..3) and radius
r = 4..16; device ms per call (CUDA events, 3 warm-ups, median of 5) and which coefficient kernel ran."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1803_00005_b200 import HGF  # noqa: E402

W, H = 1920, 1080
scene = synth.make_stereo_scene(W, H, 64, seed=5)
Y = synth.stereo_cost_volume_torch(scene, 64, "cuda", 20, 21)[0].contiguous()
rows = []
for d, ms_ in ((1, (1, 2, 3, 4, 6, 8, 10, 12, 16, 20)), (2, (1, 2, 3, 4, 5, 6, 8, 10)), (3, (1, 2, 3, 4, 5, 6))):
    for m in ms_:
        I = torch.from_numpy(synth.smooth_guides(W, H, m, seed=5)).cuda()
        for r in (4, 8, 9, 12, 16):
            h = HGF(W, H, m, d, r, 0.05)
            dst = torch.empty((H, W), dtype=torch.float32, device="cuda")
            for _ in range(3):
                h.filter(I, Y, dst)
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                h.filter(I, Y, dst)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            h.set_profiling(True)
            h.filter(I, Y, dst)
            prof = {k: round(v[0], 3) for k, v in h.profile_read().items() if v[1]}
            path = h.kernel_path
            h.close()
            ts.sort()
            rows.append({"m": m, "d": d, "n": m * d, "r": r, "ms": round(ts[2], 3), "stage_ms": prof,
                         "kernels": path})
            print(json.dumps(rows[-1]), flush=True)
