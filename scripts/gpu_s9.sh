exec > gpurun_out/s9.log 2>&1
run() { echo "== $*"; env "$@" MODES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 scripts/sweep_probe.py c2x4:1,8 c3x4:1 c4w4:1 2>&1 | grep "^{"; }
run X=1
run HB_TMA_CHUNK_KB=16
run HB_REMOTE_PCT=50
run HB_REMOTE_PCT=95
run HB_RED_CHUNK=8192
run HB_RED_CHUNK=131072
