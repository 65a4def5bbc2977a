"""Summarises an `ncu --page source --csv --print-source sass` dump: stall
reasons overall and the hottest instruction regions (scratch analysis)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if r and r[0].startswith("0x")]
# keep the first kernel instance only
seen, uniq = set(), []
for r in data:
    if r[0] in seen:
        break
    seen.add(r[0])
    uniq.append(r)
data = uniq
iS = hdr.index("Source")
iW = hdr.index("Warp Stall Sampling (All Samples)")
f = lambda x: float(x) if x not in ("", "-") else 0.0
tot = sum(f(r[iW]) for r in data)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {h: sum(f(r[hdr.index(h)]) for r in data) for h in reasons}
print("instructions", len(data), "samples", tot)
for h, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
    print(f"  {h:25s} {v / tot * 100:5.1f}%")
bins = int(sys.argv[2]) if len(sys.argv) > 2 else 20
n = len(data)
for b in range(bins):
    seg = data[b * n // bins:(b + 1) * n // bins]
    s = sum(f(r[iW]) for r in seg)
    ops = {}
    rs = {}
    for r in seg:
        toks = r[iS].strip().split()
        op = (toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")).split(".")[0]
        ops[op] = ops.get(op, 0) + 1
        for h in reasons:
            rs[h] = rs.get(h, 0) + f(r[hdr.index(h)])
    top = sorted(ops.items(), key=lambda x: -x[1])[:4]
    topr = sorted(rs.items(), key=lambda x: -x[1])[:2]
    print(f"bin{b:2d} {s / tot * 100:5.1f}% {top} {[(k[6:], round(v / max(s, 1) * 100)) for k, v in topr]}")
