# staged peer epilogue (bulk copies per (column, owner)): sharded-apply tests, strong N=1 bench, two-process check
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_octant.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --strong --steps 20 --warmup 5 > gpurun_out/strong_n1.json 2> gpurun_out/strong_n1.err; tail -c 600 gpurun_out/strong_n1.json; echo
timeout 600 python bench.py --strong --config 4 --steps 5 --warmup 2 --e2e-steps 0 > gpurun_out/strong_n1_cfg4.json 2> gpurun_out/strong_n1_cfg4.err; python -c "import json; d=json.load(open('gpurun_out/strong_n1_cfg4.json')); print('cfg4 strong', d['value'], d['ms_per_step'])"
bash tools/two_proc_strong.sh > gpurun_out/two_proc.log 2>&1; grep -h "rc=" gpurun_out/two_proc.log; for f in gpurun_out/two_proc_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d.get('value'), d.get('check', d.get('parity')))" 2>/dev/null || tail -c 300 $f; done
