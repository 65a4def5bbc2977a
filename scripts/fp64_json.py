"""Updates profiles/ncu_fp64.json entries from ncu FP64-instruction CSVs
(`ncu --metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_{dadd,dmul,dfma}_pred_on.sum --csv`):
python scripts/fp64_json.py profiles/ncu_fp64.json cfgN=<csv>:<kernel-substring> ...
Per launch (mean over the captured launches of the kernel)."""
import csv
import json
import sys
from collections import defaultdict

path = sys.argv[1]
out = json.load(open(path))
for arg in sys.argv[2:]:
    name, rest = arg.split("=", 1)
    csv_path, kern = rest.rsplit(":", 1)
    per = defaultdict(dict)
    names = {}
    hdr = None
    for r in csv.reader(open(csv_path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if kern not in d["Kernel Name"]:
            continue
        names[d["ID"]] = d["Kernel Name"]
        per[d["ID"]][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    if not per:
        print(name, "no launches of", kern)
        continue
    n = len(per)
    mean = lambda key: sum(v.get(key, 0.0) for v in per.values()) / n
    dadd = mean("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum")
    dmul = mean("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum")
    dfma = mean("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum")
    out[name] = {"kernel": next(iter(names.values())).split("(")[0], "pipe_ops": dadd + dmul + dfma,
                 "flops": dadd + dmul + 2 * dfma, "ncu_ns": mean("gpu__time_duration.sum")}
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))
