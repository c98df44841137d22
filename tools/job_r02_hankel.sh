# drop-in hankel suite + Green's tests after the unfused kernel_output geometry
cd $GRAFT_REPO_ROOT
timeout 600 oracle/_ref/dropin_test_hankel 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_greens.py tests/test_gpu_greens_parity.py tests/test_gpu_e2e_parity.py tests/test_gpu_dropin.py -x -q 2>&1 | tail -4
timeout 300 python tools/time_greens.py --config 3 --reps 2 2>&1 | tail -1
