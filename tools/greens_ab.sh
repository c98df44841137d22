#!/bin/bash
# Green's build A/B: parity tests, phase clocks (instrumented variant in exp/phase), timing
timeout 600 python -m pytest tests/test_gpu_greens.py -x -q 2>&1 | tail -2
[ -f exp/phase/libemie_cu.so ] && EMIE_CU_LIBRARY=exp/phase/libemie_cu.so python tools/time_greens.py --config 3 --reps 1 2>&1 | tail -8
python tools/time_greens.py --config 3 --reps 3
