"""Per-rank device time of a label shard at C4 (the work one GPU of an N-GPU label-sharded run does):
guidance + replicated statistics (hgf_prepare_rows over all rows) + the slice kernels on L/N labels through
the fused-merge entry point (world = 1 here, so the atomics stay local).  Gives the measured t(N) the
scaling model in DESIGN.md §10 uses; CUDA events, median of 10."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1803_00005_b200 import HGF, PeerMerge, shard_range  # noqa: E402

c = synth.config("C4")
W, H, L = c["W"], c["H"], c["L"]
scene = synth.make_stereo_scene(W, H, L, c["seed"])
g = torch.from_numpy(scene.left).cuda()
h = HGF(W, H, c["m"], c["d"], c["r"], c["lam"])
lab = torch.empty((H, W), dtype=torch.int32, device="cuda")
pm = PeerMerge(h)
full_ms = None
for n in (1, 2, 4, 8):
    l0, l1 = shard_range(L, n, 0)
    vol = synth.stereo_cost_volume_torch(scene, L, "cuda", l0, l1)

    def step():
        h.prepare_rows(g, 0, H)
        pm.aggregate(vol, lab, label_offset=l0)

    for _ in range(3):
        step()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    t = ts[5]
    full_ms = full_ms or t
    print(f"N={n}: shard labels {l0}..{l1 - 1}: {t:.3f} ms per step on one GPU; "
          f"modelled efficiency t(1)/(N t(N)) = {full_ms / (n * t):.3f} (excludes NVLink atomics + 4-byte all-reduce)",
          flush=True)
    del vol
pm.close()
h.close()
