"""Aggregate an `ncu --page source --csv --print-source sass` dump: executed
warp instructions and stall samples per opcode, normalised per element."""
import csv, sys, collections
path, elems = sys.argv[1], float(sys.argv[2])
rows = list(csv.reader(open(path)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ex = collections.Counter(); st = collections.Counter(); tot = 0; stot = 0
for r in rows[2:]:
    if len(r) < len(hdr): continue
    op = r[ix["Source"]].strip().split()
    if not op: continue
    o = op[0]
    if o.startswith("@"): o = op[1]
    o = o.split(".")[0]
    n = int(r[ix["Instructions Executed"]] or 0); s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ex[o] += n; st[o] += s; tot += n; stot += s
print(f"total warp inst {tot}  thread-inst/elem {tot*32/elems:.2f}  samples {stot}")
for o, n in ex.most_common(45):
    print(f"{o:10s} {n*32/elems:6.2f}/elem  stall {100*st[o]/max(stot,1):5.1f}%")
