# Green's pair phase: distance-ordered pairs, flushed (pair, lambda) items skipped -- stage timers + Green's tests
cd $GRAFT_REPO_ROOT
for c in 2 3 4; do echo "== cfg$c"; timeout 300 python tools/time_greens.py --config $c --reps 3 2>&1 | tail -2; done
timeout 900 python -m pytest tests/test_gpu_greens.py tests/test_gpu_greens_parity.py tests/test_gpu_vfunctions.py tests/test_gpu_e2e_parity.py -x -q 2>&1 | tail -5
