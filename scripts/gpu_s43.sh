# session 3: NVLink evidence from ncu on ONE rank of a 4-process run. The cross-GPU
# barrier is switched off (HB_DEBUG_NO_SYNC=1, diagnostics only) so rank 0's kernel
# replays never wait on peers; ranks 1-3 run unprofiled and park in the bench's barriers.
exec > gpurun_out/s43.log 2>&1
M=gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
port=29990
for cfg in c2x4 c3x4 c4w4; do
  port=$((port+1))
  A="bench.py --gpus 4 --config $cfg --steps 3 --warmup 3 --no-e2e --no-nccl --no-cpu --no-clocks --no-overlap --matrix ''"
  pids=""
  for r in 1 2 3; do
    HB_DEBUG_NO_SYNC=1 RANK=$r LOCAL_RANK=$r WORLD_SIZE=4 MASTER_ADDR=127.0.0.1 MASTER_PORT=$port timeout 600 python bench.py --gpus 4 --config $cfg --steps 3 --warmup 3 --no-e2e --no-nccl --no-cpu --no-clocks --no-overlap --matrix "" > gpurun_out/s43_${cfg}_r$r.log 2>&1 &
    pids="$pids $!"
  done
  HB_DEBUG_NO_SYNC=1 RANK=0 LOCAL_RANK=0 WORLD_SIZE=4 MASTER_ADDR=127.0.0.1 MASTER_PORT=$port timeout 600 ncu --metrics $M --clock-control none -k regex:segments -s 2 -c 2 --csv --log-file gpurun_out/s43_${cfg}_nvlink.csv python bench.py --gpus 4 --config $cfg --steps 3 --warmup 3 --no-e2e --no-nccl --no-cpu --no-clocks --no-overlap --matrix "" > gpurun_out/s43_${cfg}_r0.log 2>&1
  echo "$cfg rank0 rc=$?"
  for p in $pids; do wait $p; echo "  peer rc=$?"; done
done
