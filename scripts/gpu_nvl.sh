exec > gpurun_out/nvl.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 scripts/nvl_probe.py
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 tests/mgpu_worker.py c2 c4; echo parity=$?
HB_PUSH=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516 tests/mgpu_worker.py c2 c4 c5; echo parity_push=$?
for push in "" "--push"; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 2 --config c4 --steps 50 --warmup 5 --no-e2e $push | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['per_kernel']; print('c4 $push', d['ms_per_step'], 'fwd', k['fwd'], d['roofline']['step_tstar_ms_measured_peaks'])"
done
