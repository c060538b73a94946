exec > gpurun_out/mgpu_modes_n${N}.log 2>&1
for p in 4 3 1; do for m in 1 2; do
HB_PARTITION=$p HB_FWD_MODE=$m timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$m tests/mgpu_worker.py c2 c3 c4 c5 2>&1 | grep -E '^\{|Error|error' | tr '\n' ' ' ; echo " partition=$p mode=$m rc=$?"
done; done
OPTS="--partition=4 --partition=3 --fwd-mode=1 --fwd-mode=2 --partition=1" bash scripts/gpu_sweep.sh
cat gpurun_out/sweep_n${N}.log
