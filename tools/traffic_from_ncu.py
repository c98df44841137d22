"""Write profiles/traffic.json from an ncu --set full report: per kernel, the
dram__bytes_read.sum / dram__bytes_write.sum of its first captured launch.
    python tools/traffic_from_ncu.py REP.ncu-rep "cfg3 nrhs=2" [out.json]"""
import csv
import json
import re
import subprocess
import sys
from pathlib import Path


def short(name):
    name = re.sub(r"\(.*$", "", name)                       # drop the parameter list
    name = re.sub(r"(emie_cu::)?(<unnamed>|unnamed>|\(anonymous namespace\))::|emie_cu::", "", name)
    name = re.sub(r"^void ", "", name)
    return name.replace("(int)", "").strip()


rep, config = sys.argv[1], sys.argv[2]
out = Path(sys.argv[3]) if len(sys.argv) > 3 else Path(__file__).resolve().parent.parent / "profiles" / "traffic.json"
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base",
                      "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h = rows[0]
res = json.loads(out.read_text()) if out.exists() else {}
seen = set()
for r in rows[2:]:
    k = short(r[h.index("Kernel Name")])
    if k in seen:
        continue
    seen.add(k)
    res[k] = {"config": config, "dram_bytes_read": float(r[h.index("dram__bytes_read.sum")]),
              "dram_bytes_write": float(r[h.index("dram__bytes_write.sum")]),
              "ncu_time_ns": float(r[h.index("gpu__time_duration.sum")]), "report": Path(rep).name}
out.write_text(json.dumps(res, indent=1, sort_keys=True) + "\n")
print(json.dumps(res, indent=1))
