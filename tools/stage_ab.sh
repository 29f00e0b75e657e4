#!/bin/bash
# Per-stage device times (hgf profiling counters) of one config under alternative builds of libhgf.so:
# the in-tree library, then each LIB argument (.so or .so.gz) copied over it, then the in-tree one again.
# usage: bash tools/stage_ab.sh LIB...   (config: $STAGE_CFG = "W H m d r L", default C5 1920 1080 3 2 9 1)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
P=paper_1803_00005_b200
cp $P/libhgf.so /tmp/libhgf_base.so
run() {
  python - "$1" <<'PY'
import os, sys
sys.path.insert(0, ".")
import torch, synth
from paper_1803_00005_b200 import HGF
W, H, m, d, r, L = (int(v) for v in os.environ.get("STAGE_CFG", "1920 1080 3 2 9 1").split())
scene = synth.make_stereo_scene(W, H, max(L, 2), seed=5)
I = torch.from_numpy(synth.smooth_guides(W, H, m, seed=5)).cuda()
V = synth.stereo_cost_volume_torch(scene, max(L, 2), "cuda", 0, L).contiguous()
h = HGF(W, H, m, d, r, 0.05)
lab = torch.empty((H, W), dtype=torch.int32, device="cuda")
dst = torch.empty((H, W), dtype=torch.float32, device="cuda")
call = (lambda: h.filter(I, V[0], dst)) if L == 1 else (lambda: h.aggregate_wta(I, V, lab))
for _ in range(3): call()
h.set_profiling(True)
acc = {}
for _ in range(5):
    call()
    for k, v in h.profile_read().items():
        if v[1]: acc[k] = acc.get(k, 0) + v[0] / 5
print(sys.argv[1], {k: round(v, 4) for k, v in acc.items()}, h.kernel_path, flush=True)
PY
}
run base
for lib in "$@"; do
  case "$lib" in *.gz) gunzip -c "$lib" > $P/libhgf.so ;; *) cp "$lib" $P/libhgf.so ;; esac
  run "$(basename "$lib")"
done
cp /tmp/libhgf_base.so $P/libhgf.so
run base2
