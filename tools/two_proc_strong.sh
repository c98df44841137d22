set -x
export EMIE_BENCH_BACKEND=gloo
for cfg in 2 3; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 2951$cfg bench.py --gpus 2 --strong --peer-sync host --check --config $cfg --steps 5 --warmup 2 --e2e-steps 2 > gpurun_out/two_proc_peer_cfg$cfg.json 2> gpurun_out/two_proc_peer_cfg$cfg.err
echo rc=$?
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29520 bench.py --gpus 2 --strong --exchange nccl --check --config 2 --steps 3 --warmup 1 --e2e-steps 1 > gpurun_out/two_proc_a2a_cfg2.json 2> gpurun_out/two_proc_a2a_cfg2.err
echo rc=$?
tail -c 400 gpurun_out/two_proc_*.json
