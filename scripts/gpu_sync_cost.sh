exec > gpurun_out/sync_cost.log 2>&1
for dbg in 0 1; do for c in c2w4 c4w4; do for sc in 4096 1; do
HB_DEBUG_NO_SYNC=$dbg timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29570 bench.py --gpus 4 --config $c --scale $sc --steps 300 --warmup 10 --no-e2e --no-clocks --no-nccl --fwd-mode 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nosync=$dbg $c scale $sc', 'step', d['ms_per_step'], 'tstar', d['roofline']['step_tstar_ms_measured_peaks'])"
done; done; done
for sc in 4096 1; do timeout 300 python bench.py --config c2 --scale $sc --steps 300 --warmup 10 --no-e2e --no-clocks --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=1 c2 scale $sc', 'step', d['ms_per_step'])"; done
