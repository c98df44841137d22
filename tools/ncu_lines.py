"""Per-CUDA-source-line instruction counts and stall samples of one kernel
(sums the SASS rows under each source line):
    ncu_lines.py REP KERNEL_ID(1-based, launch order in the report) [TOP]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kid = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-id", f":::{kid}"], capture_output=True, text=True).stdout


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


agg = defaultdict(lambda: [0.0, 0.0, ""])
path, cur, hdr = "", None, None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) <= max(iS, iE):
        continue
    if r[0]:
        cur = (path, int(r[0]))
        agg[cur][2] = r[1].strip()[:70]
        continue
    if cur is not None:
        agg[cur][0] += num(r[iS])
        agg[cur][1] += num(r[iE])
tot = sum(v[0] for v in agg.values())
print("total samples", tot, "instructions", sum(v[1] for v in agg.values()))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]:7.0f} {v[1]:11.0f}  {k[0]}:{k[1]:<5d} {v[2]}")
