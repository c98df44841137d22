cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest -x -q tests/test_gpu_sharded.py > gpurun_out/oct_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/oct_tests.log
for lay in octant quadrant; do
timeout 300 python bench.py --strong --shard-layout $lay --steps 50 --warmup 5 --e2e-steps 10 --check > gpurun_out/strong_n1_$lay.json 2> gpurun_out/strong_n1_$lay.err
done
bash tools/two_proc_strong.sh > gpurun_out/two_proc.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/strong_launch_octant.csv python bench.py --strong --steps 3 --warmup 2 --e2e-steps 0 > gpurun_out/strong_ncu_octant.log 2>&1
tail -3 gpurun_out/oct_tests.log
for f in gpurun_out/strong_n1_*.json gpurun_out/two_proc_*.json; do echo $f; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d.get('value'), d.get('config',{}).get('shard_layout'), d.get('check'), d.get('e2e',{}).get('value'))"; done
