exec > gpurun_out/s24.log 2>&1
for bps in 0 1; do for c in c5w4 c5; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29580 bench.py --gpus 4 --config $c --steps 200 --warmup 10 --no-e2e --no-nccl --blocks-per-sm $bps 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c bps $bps step', d['ms_per_step'], 'frac', d['roofline']['step_frac_of_tstar'], 'overlap', json.dumps(d['overlap_with_pp_p2p']))"
done; done
