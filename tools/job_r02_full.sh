# round-2 evidence run: smoke, the whole -m gpu tier, bench (repo + reference arm), launch list
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python -m pytest tests -m gpu -q > gpurun_out/gputests_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests_full.log
python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
python bench.py --impl reference > gpurun_out/bench_r02_reference.json 2> gpurun_out/bench_r02_reference.err
python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 --no-solve > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 --no-solve > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/smoke.log; tail -3 gpurun_out/gputests_full.log; tail -c 300 gpurun_out/bench_r02.json; tail -c 300 gpurun_out/bench_r02_reference.json
python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/bench_r02_cfg4.json 2> gpurun_out/bench_r02_cfg4.err
tail -c 300 gpurun_out/bench_r02_cfg4.json
