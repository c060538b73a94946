# correctness + state at N=4 (and N=1 quick)
exec > gpurun_out/full4.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
for p in 0 3 1; do for m in 0 1 2; do
HB_PARTITION=$p HB_FWD_MODE=$m timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2959$m tests/mgpu_worker.py c2 c3 c4 c5 c1 2>&1 | grep -cE '"parity": true' | tr '\n' ' '; echo " ok-configs partition=$p fwd_mode=$m"
done; done
N=4 CONFIGS="c2w4 c3w4 c4w4 c5w4" TAG=w4 bash scripts/gpu_state.sh
N=4 bash scripts/gpu_state.sh
