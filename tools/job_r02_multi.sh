cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
EMIE_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/multi_weak2.json 2> gpurun_out/multi_weak2.err; echo "weak rc=$?"
tail -c 600 gpurun_out/multi_weak2.json
EMIE_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > gpurun_out/multi_ref2.json 2> gpurun_out/multi_ref2.err; echo "ref rc=$?"
tail -c 400 gpurun_out/multi_ref2.json
tail -5 gpurun_out/multi_weak2.err
