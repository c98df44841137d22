# round-2 final evidence on one B200: smoke, the whole -m gpu tier, bench lines (repo arm, reference arm,
# config 4), launch list of the bench, ncu full captures (apply step, Green's build), drop-in suites
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests_full.log
timeout 900 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_r02_reference.json 2> gpurun_out/bench_r02_reference.err
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/bench_r02_cfg4.json 2> gpurun_out/bench_r02_cfg4.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-solve > gpurun_out/plain_launch.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-solve > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stream_tma|contract_mma" -s 5 -c 5 \
    -o gpurun_out/r02_apply python tools/profile_apply.py --applies 3 > gpurun_out/ncu_apply.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"chunk_image|assemble_kernel|filter_design|filter_samples" -c 4 \
    -o gpurun_out/r02_greens python tools/profile_greens.py --config 3 > gpurun_out/ncu_greens.log 2>&1
timeout 1200 bash tools/run_dropin_suites.sh > /dev/null 2>&1
tail -1 gpurun_out/smoke.log; tail -2 gpurun_out/gputests_full.log; tail -c 400 gpurun_out/bench_r02.json; echo; tail -c 300 gpurun_out/bench_r02_reference.json; echo; tail -c 200 gpurun_out/bench_r02_cfg4.json; echo; ls gpurun_out/*.ncu-rep; grep -c "rc=0" gpurun_out/dropin_suites.log; grep -v "rc=0" gpurun_out/dropin_suites.log | head
