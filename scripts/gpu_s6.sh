exec > gpurun_out/s6.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python scripts/ovh_probe.py c2
for p in 0 3 1; do for m in 0 2; do
HB_PARTITION=$p HB_FWD_MODE=$m timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2959$m tests/mgpu_worker.py c2 c3 c4 c5 c1 2>&1 | grep -cE '"parity": true' | tr '\n' ' '; echo " ok-configs partition=$p fwd_mode=$m"
done; done
MODES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 scripts/sweep_probe.py c2w4:1,4,64 c4w4:1,4 c2:1,4 c4:1,4 c3:1 c5:1 2>&1 | grep "^{"
