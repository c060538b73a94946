# session 3: what the cross-GPU launch protocol costs now (HB_DEBUG_NO_SYNC=1 drops it: UNSAFE, diagnostics only)
exec > gpurun_out/s39.log 2>&1
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --config c2x4 --matrix c4w4,c4,c3x4 --no-e2e --no-nccl --no-overlap --steps 300 --matrix-steps 300"
p=29900
for rep in 1 2; do
  p=$((p+1)); $T --master-port $p $B > gpurun_out/s39_sync_$rep.json 2> gpurun_out/s39_sync_$rep.err; echo "sync $rep rc=$?"
  p=$((p+1)); HB_DEBUG_NO_SYNC=1 $T --master-port $p $B > gpurun_out/s39_nosync_$rep.json 2> gpurun_out/s39_nosync_$rep.err; echo "nosync $rep rc=$?"
done
p=$((p+1)); HB_TRACE=1 $T --master-port $p scripts/trace_probe.py c4w4 c4 > gpurun_out/s39_trace_sync.jsonl 2> gpurun_out/s39_trace_sync.err; echo "trace rc=$?"
p=$((p+1)); HB_DEBUG_NO_SYNC=1 HB_TRACE=1 $T --master-port $p scripts/trace_probe.py c4w4 c4 > gpurun_out/s39_trace_nosync.jsonl 2> gpurun_out/s39_trace_nosync.err; echo "trace nosync rc=$?"
