exec > gpurun_out/ovh3.log 2>&1
for sc in 4096 1; do for c in c2w4 c4w4 c5w4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29570 bench.py --gpus 4 --config $c --scale $sc --steps 300 --warmup 10 --no-e2e --no-clocks --no-nccl $EXTRA 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['per_kernel']; print('$c scale $sc $EXTRA', 'step', d['ms_per_step'], 'tstar', d['roofline']['step_tstar_ms_measured_peaks'], 'fwd', k['fwd']['ms'], k['fwd']['tstar_ms'], 'bwd', k['bwd']['ms'], k['bwd']['tstar_ms'])"
done; done
