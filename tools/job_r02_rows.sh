cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest -x -q tests -m gpu -k "64 or 48 or deep or cfg4 or config4 or rows or sizes" > gpurun_out/rows_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rows_tests.log
tail -3 gpurun_out/rows_tests.log
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/bench_rows_cfg4.json 2> gpurun_out/bench_rows_cfg4.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_rows_cfg4.json').read().strip().splitlines()[-1]); print(d['value'], d['stage_ms'], d.get('layout'), d.get('greens_build_warm_s'))"
