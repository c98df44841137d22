#!/bin/bash
# registers / spills per kernel of one csrc/*.cu file: tools/ptxas_report.sh lateral.cu
cd "$(dirname "$0")/../paper_1512_06126_b200/csrc" || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I ../../include -Xptxas -v -c "$1" -o /tmp/ptxas_report.o 2>&1 | python3 -c "
import sys, re
name = None
for l in sys.stdin:
    m = re.search(r\"Compiling entry function '(\S+)'\", l)
    if m: name = re.sub(r'_ZN7emie_cu\d+_GLOBAL__N__\w+?_cu_\w{8}', '', m.group(1))[:48]
    m = re.search(r'(\d+) bytes stack frame, (\d+) bytes spill stores', l)
    if m: sp = m.group(2)
    m = re.search(r'Used (\d+) registers', l)
    if m: print(name, m.group(1), 'regs, spill', sp)
    if 'error' in l: print(l.rstrip())
"
