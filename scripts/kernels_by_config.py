"""Aggregates per-config ncu metric CSVs (gpu__time_duration, dram bytes, FP64 instruction
counts; `ncu --csv` of `bench.py --config cfgN`) into one JSON of per-kernel means:
python scripts/kernels_by_config.py <head> out.json cfg1=<csv> cfg2=<csv> ..."""
import csv
import json
import sys
from collections import defaultdict

head, out_path = sys.argv[1], sys.argv[2]
out = {"head": head, "kernels": {}}
for arg in sys.argv[3:]:
    name, path = arg.split("=", 1)
    per = defaultdict(lambda: defaultdict(float))
    kname = {}
    hdr = None
    for r in csv.reader(open(path, errors="replace")):
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"].replace(",", ""))
        u = d.get("Metric Unit", "")
        v *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e3, "ms": 1e6, "s": 1e9}.get(u, 1)
        per[d["ID"]][d["Metric Name"]] += v
        kname[d["ID"]] = d["Kernel Name"][:90]
    agg = defaultdict(lambda: defaultdict(list))
    for i, m in per.items():
        k = kname[i]
        agg[k]["ns"].append(m.get("gpu__time_duration.sum", 0.0))
        agg[k]["dram"].append(m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0))
        for op in ("dadd", "dmul", "dfma"):
            agg[k][op].append(m.get(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum", 0.0))
    res = {}
    for k, a in agg.items():
        if k.startswith("void at::") or "elementwise" in k or "fill" in k.lower():
            continue  # torch's own kernels (L2 flush, input set-up)
        n = len(a["ns"])
        res[k] = {"n": n, **{key: sum(v) / n for key, v in a.items()}}
    out["kernels"][name] = res
json.dump(out, open(out_path, "w"), indent=1)
for cfg, ks in out["kernels"].items():
    print(cfg, {k[:40]: round(v["ns"] / 1e3, 1) for k, v in ks.items()})
