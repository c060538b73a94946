exec > gpurun_out/s20.log 2>&1
run() { echo "== $*"; env "$@" MODES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 scripts/sweep_probe.py c2w4:4096,4 c4w4:4096,4,1 2>&1 | grep "^{"; }
run X=1
run BPS=1
run HB_DEBUG_NO_SYNC=1
run HB_DEBUG_NO_SYNC=1 BPS=1
