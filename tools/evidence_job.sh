#!/bin/bash
# Round evidence on one B200: GPU tests, smoke, bench lines (cfg3 default, cfg4, strong N=1),
# launch list of the bench, ncu full captures (apply step kernels, Green's kernel, cfg4 contraction), parity.
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_line.json 2> gpurun_out/bench.err
timeout 600 python bench.py --config 4 --no-cpu-baseline --no-solve > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 600 python bench.py --strong --steps 20 --warmup 5 > gpurun_out/bench_strong.json 2> gpurun_out/bench_strong.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"stream_tma_kernel|contract_mma_kernel" -c 5 -o gpurun_out/apply_final python tools/profile_apply.py --config 3 --applies 1 > gpurun_out/ncu_apply.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:assemble_kernel -c 1 -o gpurun_out/greens3_final python tools/profile_greens.py --config 3 > gpurun_out/ncu_greens.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:contract_rows -c 1 -o gpurun_out/cfg4_rows_final python tools/profile_apply.py --config 4 --applies 1 > gpurun_out/ncu_cfg4.log 2>&1
timeout 300 python tools/parity_report.py > gpurun_out/parity.log 2>&1
