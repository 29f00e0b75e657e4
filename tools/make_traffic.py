"""ncu launch list (dram bytes, duration, shared wavefronts per launch) of one C4 hgf_aggregate_wta call ->
profiles/ncu_traffic.json (per kernel class: the kernel, bytes per launch, labels per launch, commit) and a
readable summary.  usage: python tools/make_traffic.py gpurun_out/r02_traffic.csv <commit> [labels_per_launch]"""
import csv
import json
import sys
from collections import OrderedDict

src, commit = sys.argv[1], sys.argv[2]
lpl = int(sys.argv[3]) if len(sys.argv) > 3 else 128
rows = list(csv.reader(open(src)))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[start]
ki, mi, vi, idi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
launch = OrderedDict()
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    launch.setdefault(int(r[idi]), {"kernel": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
cls = {"k_poly": "guidance", "k_stats": "stats", "k_coef": "coef", "k_agg": "agg", "k_fill": "keys", "k_keys": "keys",
       "k_unpack": "keys"}
out = {"_commit": commit, "_source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none, one C4 call (tools/profile_run.py "
       "--config C4 --labels 256); bytes_per_launch = read + write, averaged over the class's launches", "C4": {}}
agg = {}
total_ms = 0.0
for i, L in launch.items():
    name = L["kernel"]
    short = name.split("(")[0].replace("void ", "").split("::")[-1]
    c = next((v for k, v in cls.items() if k in name), None)
    if c is None:
        continue
    b = L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)
    ms = L.get("gpu__time_duration.sum", 0) / 1e6
    total_ms += ms
    a = agg.setdefault(c, {"kernel": short, "n": 0, "bytes": 0.0, "ms": 0.0, "wf": 0.0})
    a["n"] += 1
    a["bytes"] += b
    a["ms"] += ms
    a["wf"] += L.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 0)
    print(f"{i:3d} {short[:34]:34s} {ms:8.3f} ms  dram {b / 1e9:7.2f} GB  smem_wf {L.get('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 0) / 1e9:6.3f} G")
print(f"total {total_ms:.3f} ms (ncu launch list: cold-cache, serialised; compare shares, not absolutes)")
for c, a in agg.items():
    out["C4"][c] = {"kernel": a["kernel"], "bytes_per_launch": a["bytes"] / a["n"], "launches": a["n"],
                    "ms_per_launch_ncu": a["ms"] / a["n"], "smem_wavefronts_per_launch": a["wf"] / a["n"],
                    "share_of_call": a["ms"] / total_ms,
                    "labels_per_launch": lpl if c in ("coef", "agg") else None}
    print(f"{c:9s} {a['kernel'][:30]:30s} launches {a['n']}  {a['bytes'] / a['n'] / 1e9:7.2f} GB/launch  "
          f"share {a['ms'] / total_ms:.3f}")
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
