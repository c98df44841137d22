"""Stall samples / instructions of a CUDA line range (as the source page maps them):
    ncu_linerange.py REP KERNEL_ID FILE LO HI"""
import csv
import subprocess
import sys

rep, kid, fname, lo, hi = sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda",
                      "--kernel-id", f":::{kid}"], capture_output=True, text=True).stdout
path = ""
hdr = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        path = r[1]
        continue
    if r[0] == "Line No" or r[0] == "#":
        hdr = r
        continue
    if hdr is None or not path.endswith(fname) or not r[0].isdigit():
        continue
    ln = int(r[0])
    if lo <= ln <= hi:
        d = dict(zip(hdr, r))
        print(f"{ln:5d} {d.get('Warp Stall Sampling (All Samples)', ''):>8} {d.get('Instructions Executed', ''):>12}  {r[1][:90]}")
