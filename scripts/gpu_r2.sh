exec > gpurun_out/r2_n${N}.log 2>&1
for p in 4 3; do
HB_PARTITION=$p timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29551 tests/mgpu_worker.py c2 c3 c4 c5 2>&1 | grep -E '^\{|Error|error' | cut -c1-60 | tr '\n' ' ' ; echo " partition=$p rc=$?"
done
OPTS="--partition=1 --partition=3 --partition=4" bash scripts/gpu_sweep.sh
cat gpurun_out/sweep_n${N}.log
