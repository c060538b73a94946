exec > gpurun_out/s19.log 2>&1
timeout 300 python -m pytest tests/test_projector.py -x -q 2>&1 | tail -3
HB_PROJ=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29594 tests/mgpu_worker.py c1 c2 c3 c5 c2x4 c3x4 2>&1 | grep -cE '"parity": true'
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29593 scripts/fused_probe_mgpu.py c2 c2x4 c3x4 2>&1 | grep "^{"
CUDA_VISIBLE_DEVICES=0 timeout 300 python scripts/fused_probe.py
CUDA_VISIBLE_DEVICES=0 timeout 300 python scripts/proj_probe.py
