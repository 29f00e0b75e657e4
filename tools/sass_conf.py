import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
si = hdr.index("Source"); ii = hdr.index("Instructions Executed")
wf = hdr.index("L1 Wavefronts Shared"); wfi = hdr.index("L1 Wavefronts Shared Ideal"); ex = hdr.index("L1 Wavefronts Shared Excessive")
agg = {}
for r in rows[2:]:
    if len(r) <= max(si, ii, wf, wfi, ex): continue
    try:
        w = float(r[wf] or 0); wi = float(r[wfi] or 0); n = float(r[ii] or 0)
    except ValueError:
        continue
    if w == 0: continue
    op = r[si].strip()[:60]
    agg.setdefault(op.split()[0] if not op.startswith('@') else op.split()[1], [0,0,0])
    a = agg[op.split()[0] if not op.startswith('@') else op.split()[1]]
    a[0]+=n; a[1]+=w; a[2]+=wi
for k,(n,w,wi) in sorted(agg.items(), key=lambda t:-t[1][1]):
    print(f"{k:12s} instr {n:12.0f} wavefronts {w:12.0f} ideal {wi:12.0f}  ratio {w/max(wi,1):.2f}")
