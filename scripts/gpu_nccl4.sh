exec > gpurun_out/nccl4.log 2>&1
for c in c2w4 c3w4 c4w4 c5w4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 4 --config $c --steps 50 --warmup 5 --no-e2e 2>&1 | tail -3 | grep -E '^\{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', 'hb ms', d['ms_per_step'], 'tstar', d['roofline']['step_tstar_ms_measured_peaks'], 'frac', d['roofline']['step_frac_of_tstar'], 'nccl', d['nccl_comparison'])" || echo "$c failed"
done
