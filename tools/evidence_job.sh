set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench_line.json 2> gpurun_out/bench.err
timeout 600 python bench.py --config 4 --no-cpu-baseline --no-solve > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:contract_rows -c 1 -o gpurun_out/cfg4_rows python tools/profile_apply.py --config 4 --applies 1 > gpurun_out/ncu_cfg4.log 2>&1
timeout 300 python tools/parity_report.py > gpurun_out/parity.log 2>&1
