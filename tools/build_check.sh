#!/bin/bash
# build in-tree; exit 1 (with the compiler output) when any nvcc step fails
out=$(python -c "from paper_1512_06126_b200 import build as b; b.build()" 2>&1)
if echo "$out" | grep -qi "error"; then echo "$out" | grep -i -A3 error | head -30; exit 1; fi
echo build ok
