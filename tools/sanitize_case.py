"""Small end-to-end case for compute-sanitizer runs (memcheck / racecheck / synccheck): the default slice path
(k_stats4 -> k_coef5 -> k_agg3) on ragged sizes incl. W % 4 != 0 (repacked chunk) and three strips x two label
batches, the degree-3 planar path (k_coef2 -> k_agg3), hgf_filter, the row-band statistics + fused merge entry
point, and the opt-in k_agg5."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1803_00005_b200 import HGF  # noqa: E402

for (W, H, m, d, L, r, agg5) in ((77, 53, 3, 2, 5, 9, 0), (45, 70, 3, 3, 4, 9, 0), (300, 140, 3, 2, 40, 9, 0),
                                 (300, 140, 3, 2, 40, 9, 1), (150, 300, 3, 2, 3, 4, 0)):
    os.environ["HGF_AGG5"] = str(agg5)
    scene = synth.make_stereo_scene(W, H, L, seed=7)
    g = torch.from_numpy(scene.left).cuda()
    v = synth.stereo_cost_volume_torch(scene, L, "cuda", 0, L)
    h = HGF(W, H, m, d, r, 0.05)
    lab = torch.empty((H, W), dtype=torch.int32, device="cuda")
    h.aggregate_wta(g, v, lab)
    dst = torch.empty((H, W), dtype=torch.float32, device="cuda")
    h.filter(g, v[0].contiguous(), dst)
    if h.kernel_path.startswith("coef5"):
        owners = torch.empty((H, W), dtype=torch.int64, device="cuda")
        h.fill_keys(owners)
        ptrs = torch.tensor([owners.data_ptr()], dtype=torch.int64, device="cuda")
        h.prepare_rows(g, 0, H)
        h.aggregate_wta_peer(v, ptrs, 1, H)
    torch.cuda.synchronize()
    print(W, H, m, d, L, r, h.kernel_path, flush=True)
    h.close()
print("ok")
