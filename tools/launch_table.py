"""Per-kernel launch table from an ncu --metrics gpu__time_duration.sum CSV.
usage: python tools/launch_table.py launches.csv [--step-kernels regex]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
seq = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("emie_cu::", "").replace("<unnamed>::", "")
    t = float(d["Metric Value"])
    unit = d.get("Metric Unit", "")
    if unit in ("nsecond", "ns"):
        t /= 1000.0
    elif unit in ("msecond", "ms"):
        t *= 1000.0
    seq.append((name, t))
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += t
print(f"{'kernel':60s} {'launches':>8s} {'total us':>10s} {'avg us':>10s}")
for k, (n, t) in agg.items():
    print(f"{k[:60]:60s} {n:8d} {t:10.1f} {t / n:10.1f}")
