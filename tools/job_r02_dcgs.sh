cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest -q tests/test_gpu_solve.py tests/test_gpu_e2e_parity.py tests/test_gpu_dropin.py 2>&1 | tail -3
for i in 1 2; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/dcgs_b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/dcgs_b.json').read().strip().splitlines()[-1]); s=d['solve']; print(s['seconds'], s['iterations'], s['ms_per_iteration'], s.get('ortho_effective'))"
done
