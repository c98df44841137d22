# config 4 (256x256x64) on one B200 with the six-block row layout: ncu full capture of the streamed
# row-block contraction (DRAM traffic against the 13.0 GB + 3.2 GB algorithmic bytes), launch list of
# the cfg4 bench step, ncu full capture of the cfg4 spectra build (y pass, mirror fill)
cd $GRAFT_REPO_ROOT
timeout 600 python tools/profile_apply.py --config 4 --applies 1 > gpurun_out/cfg4_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:contract_rows -c 1 \
    -o gpurun_out/r02_cfg4_rows python tools/profile_apply.py --config 4 --applies 1 > gpurun_out/ncu_cfg4.log 2>&1
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-solve > gpurun_out/cfg4_plain_launch.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg4.csv \
    python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-solve > gpurun_out/ncu_launch_cfg4.log 2>&1
tail -3 gpurun_out/ncu_cfg4.log; tail -c 300 gpurun_out/cfg4_plain_launch.log; ls -la gpurun_out/*.ncu-rep gpurun_out/r02_launches_cfg4.csv
