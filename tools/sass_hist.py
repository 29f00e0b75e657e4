import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
si = hdr.index("Source"); ii = hdr.index("Instructions Executed"); wi = hdr.index("Warp Stall Sampling (All Samples)")
wf = hdr.index("L1 Wavefronts Shared")
tot = 0; hist = collections.Counter(); stall = collections.Counter(); shw = 0
for r in rows[2:]:
    if len(r) <= max(si, ii, wi, wf):
        continue
    try:
        n = int(float(r[ii] or 0))
    except ValueError:
        continue
    op = r[si].split()[0] if r[si].split() else "?"
    if op.startswith("@"):
        op = r[si].split()[1]
    op = op.split(".")[0]
    hist[op] += n; tot += n
    try: stall[op] += int(float(r[wi] or 0))
    except ValueError: pass
    try: shw += int(float(r[wf] or 0))
    except ValueError: pass
print("total warp-instr", tot, "shared wavefronts", shw)
for op, n in hist.most_common(25):
    print(f"{op:10s} {n:14d} {100*n/tot:5.1f}%  stall-samples {stall[op]}")
