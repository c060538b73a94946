exec > gpurun_out/mgpu_parity_n${N}.log 2>&1
for m in 1 2; do
HB_FWD_MODE=$m timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$m tests/mgpu_worker.py c2 c3 c4 c5 c1 2>&1 | grep -E '^\{|Error|error' ; echo mode=$m parity=$?
done
