"""Prints one summary line per bench JSON log (used after gpurun calls)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        lines = [x for x in open(f) if x.startswith("{")]
    except OSError:
        print(f, "missing")
        continue
    if not lines:
        print(f, "NO JSON:", open(f).read()[-600:])
        continue
    d = json.loads(lines[-1])
    r = d.get("roofline", {})
    print(f"{f}: {d['ms_per_step']:.4f} ms/step  {d['value']:.3e} {d['unit']}  fused {r.get('kernel_ms', 0):.4f} ms "
          f"frac {r.get('frac') or 0:.3f}  pipeline {d.get('pipeline', {}).get('frac', 0):.3f}  "
          f"e2e {d.get('e2e', {}).get('value', 0):.3e}")
