"""Per-source-line and per-opcode stall samples of one kernel in an ncu report:
    ncu_sass_hot.py REP KERNEL_SUBSTR [TOP]"""
import csv
import subprocess
import sys
from collections import Counter

rep, ksub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
ids = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", "gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(ids.splitlines()))
h = rows[0]
kid = None
for r in rows[2:]:
    if ksub in r[h.index("Kernel Name")]:
        kid = r[h.index("ID")]
        break
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-id", f"::regex:{ksub}:1" if kid is None else f":::{int(kid) + 1}"],
                     capture_output=True, text=True).stdout
def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(out.splitlines()))
hdr_i = next(i for i, r in enumerate(rows) if "Address" in r or "# Address" in r)
h = rows[hdr_i]
data = rows[hdr_i + 1:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
iSrc = h.index("Source")
tot = sum(num(r[iS]) for r in data if len(r) > max(iS, iE))
ops, samp = Counter(), Counter()
for r in data:
    if len(r) <= max(iS, iE, iSrc):
        continue
    src = r[iSrc].strip()
    op = src.split()[0] if src else ""
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ops[op] += num(r[iE])
    samp[op] += num(r[iS])
print("samples", tot, "instructions", sum(ops.values()))
for k, v in ops.most_common(top):
    print(f"  {k:10s} inst {v:14.0f}  samples {samp[k]:8.0f}")
