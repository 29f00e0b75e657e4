"""Device time of the label-independent pass alone (hgf_prepare_rows over all rows: guidance + statistics)
at a bench config, CUDA events, median of 20; --lib selects an alternate libhgf.so (A/B timing builds)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1803_00005_b200 as P  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--lib", default=None)
ap.add_argument("--mode", default="hgf")
a = ap.parse_args()
if a.lib:
    P.lib_path = os.path.abspath(a.lib)
import torch  # noqa: E402

c = synth.config(a.config)
scene = synth.make_stereo_scene(c["W"], c["H"], c["L"], c["seed"])
g = torch.from_numpy(scene.left).cuda()
h = P.HGF(c["W"], c["H"], c["m"], c["d"], c["r"], c["lam"], mode=a.mode)
for _ in range(3):
    h.prepare_rows(g, 0, c["H"])
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h.prepare_rows(g, 0, c["H"])
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"{a.lib or 'default'} {a.config} {a.mode}: prepare_rows {ts[10]:.3f} ms (min {ts[0]:.3f})")
