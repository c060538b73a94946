# full multi-GPU parity matrix + fresh state at N=4 and N=2
exec > gpurun_out/s23.log 2>&1
for p in 0 3 1; do for m in 0 2; do for st in 0 1; do
HB_STRICT=$st HB_PARTITION=$p HB_FWD_MODE=$m timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2959$m tests/mgpu_worker.py c2 c3 c4 c5 c1 c2x4 c3x4 c4w4 2>&1 | grep -cE '"parity": true' | tr '\n' ' '; echo " ok-configs(of 8) partition=$p fwd_mode=$m strict=$st"
done; done; done
HB_PROJ=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29594 tests/mgpu_worker.py c1 c2 c3 c5 c2x4 c3x4 2>&1 | grep -cE '"parity": true' | tr '\n' ' '; echo " ok-configs(of 6) fused projector"
timeout 900 python -m pytest tests/test_multigpu.py -q 2>&1 | tail -2
N=4 CONFIGS="c2 c3 c4 c5 c2x4 c3x4 c4w4 c5w4" TAG=_s23 bash scripts/gpu_state.sh
N=2 CONFIGS="c2 c3 c4 c5" TAG=_s23 CUDA_VISIBLE_DEVICES=0,1 bash scripts/gpu_state.sh
