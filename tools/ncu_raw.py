"""Print selected raw ncu metrics of one kernel: ncu_raw.py REP KERNEL_REGEX [METRIC_SUBSTR ...]"""
import csv
import re
import subprocess
import sys

rep, kre = sys.argv[1], re.compile(sys.argv[2])
keys = sys.argv[3:] or ["bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "wavefronts_mem_shared_op_ld.sum",
                        "pipe_tensor_subpipe_dmma_cycles_active.avg.pct", "dram__throughput.avg.pct",
                        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for row in rows[2:]:
    name = row[h.index("Kernel Name")] if "Kernel Name" in h else " ".join(row)
    if not kre.search(name):
        continue
    print("==", name[:90])
    for k, v in zip(h, row):
        if any(s in k for s in keys) and v not in ("", "0"):
            print("  ", k, v)
