exec > gpurun_out/c5.log 2>&1
for c in c5 c5w4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29575 bench.py --gpus 4 --config $c --steps 100 --warmup 5 --no-e2e --no-clocks 2>&1 | grep -E '^\{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['overlap_with_pp_p2p'], (d['nccl_comparison'] or {}).get('ms_per_step'))"
done
