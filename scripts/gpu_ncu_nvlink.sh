# NVLink bytes per boundary kernel from ncu on ONE rank of an N=2 run, with a
# single-pass metric set (no kernel replay, so no save/restore of IPC-imported
# peer buffers) and the cross-GPU barrier ON. Rank 1 runs unprofiled. Bounded by
# `timeout` so a stuck profiler cannot hold the box (see DESIGN §7 item 3).
# Usage (gpurun --gpus 2): bash scripts/gpu_ncu_nvlink.sh c2w4
exec > gpurun_out/ncu_nvlink.log 2>&1
cfg=${1:-c2w4}
port=29977
A="bench.py --gpus 2 --config $cfg --steps 3 --warmup 3 --no-e2e --no-nccl --no-cpu --no-clocks --no-overlap --matrix"
RANK=1 LOCAL_RANK=1 WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=$port timeout 240 python $A "" > gpurun_out/ncu_nvlink_r1.log 2>&1 &
peer=$!
RANK=0 LOCAL_RANK=0 WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=$port timeout 240 \
  ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum --clock-control none \
      -k regex:segments -s 2 -c 2 --csv --log-file gpurun_out/ncu_nvlink_${cfg}.csv python $A "" > gpurun_out/ncu_nvlink_r0.log 2>&1
echo "rank0 rc=$?"
wait $peer; echo "rank1 rc=$?"
