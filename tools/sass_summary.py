"""Per-kernel SASS opcode counts of the in-tree libemie_cu.so (cuobjdump -sass):
the evidence that the hot kernels issue DMMA / TMA (UTMALDG, UBLKCP, UTMASTG)
and how their instruction mix splits. python tools/sass_summary.py > profiles/rNN_sass_summary.txt"""
import collections
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parent.parent / "paper_1512_06126_b200" / "libemie_cu.so"
WANT = re.compile(r"stream_tma_kernel|contract_mma_kernel|contract_rows_kernel|assemble_kernel|chunk_image_kernel|"
                  r"filter_design_kernel|filter_samples_kernel|dcgs|cgs|mirror_fill|system_kernel")
KEY = ["DMMA", "DFMA", "DMUL", "DADD", "UTMALDG", "UTMASTG", "UBLKCP", "UTMAPF", "SYNCS", "LDS", "STS", "LDG", "STG",
       "LDGSTS", "BAR", "SHFL"]

out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
kern, counts = None, {}
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m and kern:
        counts[kern][m.group(1)] += 1


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return r if len(r) == len(names) else names


names = [k for k in counts if WANT.search(k)]
print(f"# SASS opcode counts per kernel (static, cuobjdump -sass {LIB.name}); columns: total and selected opcodes")
print("# DMMA = FP64 tensor-core MMA (mma.sync m8n8k4 f64); UTMALDG/UTMASTG = TMA tensor load/store; "
      "UBLKCP = bulk copy (cp.async.bulk); SYNCS = mbarrier ops")
for n, d in sorted(zip(names, demangle(names)), key=lambda x: x[1]):
    c = counts[n]
    short = re.sub(r"emie_cu::\(anonymous namespace\)::", "", d)[:110]
    sel = " ".join(f"{k}={c[k]}" for k in KEY if c[k])
    print(f"{short}\n    total={sum(c.values())} {sel}")
