#!/bin/bash
# time the Green's build of experiment builds: tools/greens_variants.sh exp/v1 exp/v2 ...
python tools/time_greens.py --config 3 --reps 2 2>&1 | tail -1 | sed 's/^/default /'
for d in "$@"; do
  EMIE_CU_LIBRARY=$d/libemie_cu.so python tools/time_greens.py --config 3 --reps 2 2>&1 | tail -1 | sed "s|^|$d |"
done
