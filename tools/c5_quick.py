import json, os, sys
sys.path.insert(0, "/root/repo")
import torch, synth
from paper_1803_00005_b200 import HGF
W, H = 1920, 1080
scene = synth.make_stereo_scene(W, H, 64, seed=5)
Y = synth.stereo_cost_volume_torch(scene, 64, "cuda", 20, 21)[0].contiguous()
for (m, d) in ((1, 1), (3, 1), (3, 2), (2, 3), (6, 1)):
    I = torch.from_numpy(synth.smooth_guides(W, H, m, seed=5)).cuda()
    for r in (4, 9):
        h = HGF(W, H, m, d, r, 0.05)
        dst = torch.empty((H, W), dtype=torch.float32, device="cuda")
        for _ in range(3): h.filter(I, Y, dst)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); h.filter(I, Y, dst); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        h.set_profiling(True); h.filter(I, Y, dst)
        prof = {k: round(v[0], 3) for k, v in h.profile_read().items() if v[1]}
        print(json.dumps({"env": os.environ.get("TAG"), "m": m, "d": d, "r": r, "ms": round(sorted(ts)[2], 3), "stage": prof, "path": h.kernel_path}), flush=True)
        h.close()
