python tools/time_greens.py --config 3 --reps 3 > gpurun_out/time_greens_skip.log 2>&1
python tools/time_greens.py --config 4 --reps 2 >> gpurun_out/time_greens_skip.log 2>&1
oracle/_ref/dropin_test_greens -tc="fetch reconstructs" > gpurun_out/dropin_fetch.log 2>&1; echo "fetch rc=$?" >> gpurun_out/dropin_fetch.log
python -m pytest tests/test_gpu_receivers.py tests/test_gpu_pipeline.py tests/test_gpu_greens_parity.py tests/test_gpu_e2e_parity.py -q -x -s > gpurun_out/gpu_new.log 2>&1
tail -5 gpurun_out/time_greens_skip.log; tail -3 gpurun_out/dropin_fetch.log; tail -25 gpurun_out/gpu_new.log
