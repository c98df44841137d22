#!/bin/bash
# A/B the contraction stage of bench.py across experiment builds:
#   tools/ab_contraction.sh [label=libdir ...]   (libdir holding libemie_cu.so; "default" = the in-tree build)
mkdir -p gpurun_out
run() {
  python bench.py --steps 20 --warmup 5 --no-solve --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), d['stage_ms'])"
}
run default
EMIE_CU_NO_OCTANT=1 run quadrant
for a in "$@"; do
  EMIE_CU_LIBRARY=${a#*=}/libemie_cu.so run ${a%%=*}
done
