cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python tools/profile_solve.py --iters 80 > gpurun_out/solve_plain.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"cgs|finalize|scale|stream_tma|contract" -s 2000 -c 400 --csv --log-file gpurun_out/solve_launch.csv python tools/profile_solve.py --iters 80 > gpurun_out/solve_ncu.log 2>&1
cat gpurun_out/solve_plain.log
