for i in 1 2; do for ov in 1 0; do
EMIE_CU_GREENS_OVERLAP=$ov timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-solve 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('overlap=$ov', d['greens_build_s'], d['greens_build_warm_s'], d['greens_stage_ms'])"
done; done
