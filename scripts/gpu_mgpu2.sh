exec > gpurun_out/mgpu${N}.log 2>&1
nvidia-smi topo -m
N=${N:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 tests/mgpu_worker.py c2 c5 c4 c3 c1; echo parity=$?
for c in c2 c3 c4 c5; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --config $c --steps 50 --warmup 5 --no-e2e | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['per_kernel']; print('$c', d['value'], d['ms_per_step'], 'fwd', k['fwd'], 'bwd', k['bwd'], d['roofline']['step_tstar_ms_measured_peaks'])"
done
