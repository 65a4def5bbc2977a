"""Per-kernel SASS census of libfsx.so (the instructions that prove the
TMA / bulk-copy / tensor-memory / DSMEM paths and the FP64 work of each hot
kernel): python scripts/sass_census.py [lib] > profiles/<round>_sass_census.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2105_06676_b200/libfsx.so"
ops = ["UTMALDG", "UTMASTG", "UBLKCP", "UTCCP", "LDTM", "STAS", "SYNCS", "DFMA", "DMUL", "DADD", "LDS", "STS",
       "LDG", "STG"]
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
demangle = lambda n: subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
counts = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = demangle(m.group(1))
        counts[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m:
        op = m.group(1)
        for o in ops:
            if op == o or op.startswith(o + "."):
                counts[cur][o] += 1
hot = ("k_fused8192", "k_cols_tma<", "k_r2c_bulk", "k_c2r_bulk", "k_rowpair<", "k_axis_tma", "k_cols_tma_f32")
print("kernel".ljust(70), " ".join(o.rjust(7) for o in ops))
for name, c in counts.items():
    short = name.replace("fsx::", "")
    if not any(h in short for h in hot):
        continue
    print(short[:70].ljust(70), " ".join(str(c[o]).rjust(7) for o in ops))
tot = collections.Counter()
for c in counts.values():
    tot.update(c)
print("ALL KERNELS".ljust(70), " ".join(str(tot[o]).rjust(7) for o in ops))
