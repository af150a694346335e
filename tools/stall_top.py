"""Top instructions by one stall reason from an ncu source-page CSV."""
import csv, sys
path, col = sys.argv[1], sys.argv[2]
k = int(sys.argv[3]) if len(sys.argv) > 3 else 15
rows = list(csv.reader(open(path))); hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
L = []
for r in rows[2:]:
    if len(r) < len(hdr): continue
    L.append((int(r[ix[col]] or 0), int(r[ix["Instructions Executed"]] or 0), r[ix["Address"]][-5:], r[ix["Source"]].strip()))
tot = sum(x[0] for x in L)
print(col, "total", tot)
for s, n, a, src in sorted(L, reverse=True)[:k]:
    print(f"{100*s/max(tot,1):5.1f}% {n:9d} {a} {src}")
