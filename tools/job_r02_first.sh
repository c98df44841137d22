cd $GRAFT_REPO_ROOT
for i in 1 2; do
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-solve > gpurun_out/first_$i.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/first_$i.json').read().strip().splitlines()[-1]); print({k:d.get(k) for k in ('greens_build_s','library_init_s','greens_build_warm_s','greens_stage_ms')})"
done
timeout 300 python tools/cold_build.py 2>&1 | tail -5
