exec > gpurun_out/s18.log 2>&1
timeout 300 python -m pytest tests/test_projector.py -x -q 2>&1 | tail -3
for n in 2 4; do
HB_PROJ=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n tests/mgpu_worker.py c1 c2 c3 c5 c2x4 c3x4 2>&1 | grep -E '"parity"|Error|error' | head -20
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29590 tests/mgpu_worker.py c2 c4 c5 2>&1 | grep -cE '"parity": true'
