"""Run one aggregate_wta_ex case and report the CUDA status (debug helper).

usage: python tools/debug_case.py W H n_guide degree L radius
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1803_00005_b200 import HGF  # noqa: E402

W, H, m, d, L, r = (int(x) for x in sys.argv[1:7])
I, V = synth.iid_volume(W, H, L, m, seed=1)
h = HGF(W, H, m, d, r, 0.05)
try:
    out = h.aggregate_wta_ex(torch.from_numpy(I).cuda(), torch.from_numpy(V).cuda(), labels=True, filtered=True)
    torch.cuda.synchronize()
    print("OK", sys.argv[1:7], float(out["filtered"].abs().max()))
except Exception as e:  # noqa: BLE001
    print("FAIL", sys.argv[1:7], str(e).splitlines()[0])
