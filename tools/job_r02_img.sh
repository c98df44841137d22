cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python tools/time_greens.py --config 3 --reps 2 > gpurun_out/img_def.log 2>&1
timeout 300 python tools/time_greens.py --config 4 --reps 2 >> gpurun_out/img_def.log 2>&1
timeout 900 python -m pytest -x -q tests/test_gpu_greens_parity.py tests/test_gpu_greens.py tests/test_gpu_vfunctions.py > gpurun_out/img_tests.log 2>&1
tail -3 gpurun_out/img_tests.log
cat gpurun_out/img_def.log
