"""DRAM bytes per launch of each config's dominant kernel from ncu metric CSVs
(`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv`):
python scripts/traffic.py out.json cfgN=<csv>:<kernel-substring> ..."""
import csv
import json
import sys
from collections import defaultdict

out = {"_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, mean over the "
                "captured launches (ncu --clock-control none, cold L2 per launch); bench.py reports it as roofline.traffic"}
for arg in sys.argv[2:]:
    name, rest = arg.split("=", 1)
    path, kern = rest.rsplit(":", 1)
    acc = defaultdict(float)
    n = defaultdict(int)
    hdr = None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if kern not in d["Kernel Name"]:
            continue
        m, v, u = d["Metric Name"], float(d["Metric Value"].replace(",", "")), d.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        if m.startswith("dram__bytes"):
            acc[d["ID"]] += v * scale
    if acc:
        out[name] = int(sum(acc.values()) / len(acc))
        out[name + "_kernel"] = kern
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out, indent=1))
