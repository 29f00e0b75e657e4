"""Top SASS lines of one kernel in an ncu report by stall samples and by excess shared wavefronts.
usage: python tools/ncu_source_top.py REPORT KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]


def iv(r, c):
    try:
        return int(float(r[hdr.index(c)] or 0))
    except ValueError:
        return 0


S, NI, WF, EX = ("Warp Stall Sampling (All Samples)", "Warp Stall Sampling (Not-issued Samples)",
                 "L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive")
tot = sum(iv(r, S) for r in data)
print(f"{len(data)} SASS lines, {tot} stall samples; wavefronts shared {sum(iv(r, WF) for r in data)}, "
      f"excessive {sum(iv(r, EX) for r in data)}")
print("--- by stall samples: samples not_issued wavefronts excessive | sass")
for r in sorted(data, key=lambda r: -iv(r, S))[:n]:
    print(f"{iv(r, S):7d} {iv(r, NI):7d} {iv(r, WF):11d} {iv(r, EX):11d} | {r[hdr.index('Source')].strip()[:70]}")
print("--- by excessive shared wavefronts")
for r in sorted(data, key=lambda r: -iv(r, EX))[:12]:
    print(f"{iv(r, EX):11d} {iv(r, WF):11d} | {r[hdr.index('Address')]} {r[hdr.index('Source')].strip()[:70]}")
