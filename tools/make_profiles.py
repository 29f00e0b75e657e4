"""Turn the ncu launch list (gpu__time_duration + dram bytes per launch) of a bench.py run into
profiles/<round>_launches_summary.md and profiles/ncu_traffic.json (used by bench.py's roofline "traffic").

usage: python tools/make_profiles.py gpurun_out/r01_launches.csv C4 r01
"""
import csv
import json
import os
import sys

UNITS = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3,
         "second": 1e3}
BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9}
CLASS = {"k_coef": "coef", "k_agg": "agg", "k_stats": "stats", "k_poly_guidance": "guidance",
         "k_unpack_keys": "keys"}


def main():
    path, cfg, rnd = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui, mi, ii = (hdr.index(c) for c in ("Kernel Name", "Metric Value", "Metric Unit", "Metric Name", "ID"))
    per = {}
    for r in rows[1:]:
        per.setdefault(r[ii], {"k": r[ki]})[r[mi]] = (float(r[vi].replace(",", "")), r[ui])
    agg = {}
    for d in per.values():
        name = d["k"].split("(")[0].replace("void ", "").strip()
        t, tu = d.get("gpu__time_duration.sum", (0.0, "ns"))
        rd, ru = d.get("dram__bytes_read.sum", (0.0, "byte"))
        wr, wu = d.get("dram__bytes_write.sum", (0.0, "byte"))
        a = agg.setdefault(name, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += t * UNITS.get(tu, 1e-6)
        a[2] += rd * BYTES.get(ru, 1.0)
        a[3] += wr * BYTES.get(wu, 1.0)
    # only this library's kernels: the launch list also holds torch's synthetic-input kernels, which run
    # before the timed region
    other = {k: v for k, v in agg.items() if not any(pre in k for pre in CLASS)}
    agg = {k: v for k, v in agg.items() if any(pre in k for pre in CLASS)}
    total = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list — bench.py ({cfg}), round {rnd}", "",
             "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none`"
             " on `python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e` (cold-cache, serialised launches:"
             " compare shares, not absolute times).", "",
             "| kernel | launches | total ms | share | DRAM read GB | DRAM write GB | DRAM GB/launch |",
             "|---|---|---|---|---|---|---|"]
    traffic = {}
    for name, (n, ms, rd, wr) in sorted(agg.items(), key=lambda t: -t[1][1]):
        lines.append(f"| `{name}` | {n} | {ms:.3f} | {100 * ms / total:.1f}% | {rd / 1e9:.2f} | {wr / 1e9:.2f} |"
                     f" {(rd + wr) / n / 1e9:.3f} |")
        for pre, cls in CLASS.items():
            if pre in name:
                traffic[cls] = (rd + wr) / n
    lines.append("")
    lines.append(f"Not shown: {sum(v[0] for v in other.values())} torch launches ({sum(v[1] for v in other.values()):.1f} ms)"
                 " that build the synthetic cost volume before the timed region.")
    os.makedirs("profiles", exist_ok=True)
    open(f"profiles/{rnd}_launches_summary.md", "w").write("\n".join(lines) + "\n")
    tpath = "profiles/ncu_traffic.json"
    tj = json.load(open(tpath)) if os.path.exists(tpath) else {}
    tj[cfg] = traffic
    json.dump(tj, open(tpath, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
