"""Per-kernel mean durations from an ncu --metrics gpu__time_duration.sum --csv log."""
import csv
import sys
from collections import defaultdict

for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hdr = None
    acc = defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                acc[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"]))
    print(f)
    for k, v in acc.items():
        print(f"   {k[:60]:60s} n={len(v):3d} mean {sum(v) / len(v) / 1000:8.1f} us")
