# session 3: A/B at N=4 on one box: base (HEAD) vs per-peer waits + claim prefetch, with knobs
exec > gpurun_out/s33.log 2>&1
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --config c2x4 --matrix c3x4,c4w4,c4,c3 --no-e2e --no-nccl --no-overlap --steps 300 --matrix-steps 300"
for rep in 1 2; do
  HB_LIB_PATH=$PWD/ab/libhetbridge_base.so $T --master-port 2963$rep $B > gpurun_out/s33_base_$rep.json 2> gpurun_out/s33_base_$rep.err; echo "base $rep rc=$?"
  $T --master-port 2964$rep $B > gpurun_out/s33_new_$rep.json 2> gpurun_out/s33_new_$rep.err; echo "new $rep rc=$?"
  HB_WAIT_ALL_PEERS=1 $T --master-port 2965$rep $B > gpurun_out/s33_waitall_$rep.json 2> gpurun_out/s33_waitall_$rep.err; echo "waitall $rep rc=$?"
  HB_CLAIM_PREFETCH=0 $T --master-port 2966$rep $B > gpurun_out/s33_nopf_$rep.json 2> gpurun_out/s33_nopf_$rep.err; echo "nopf $rep rc=$?"
done
HB_TRACE=1 $T --master-port 29671 scripts/trace_probe.py c4w4 c2x4 c2w4:4096 > gpurun_out/s33_trace_n4.jsonl 2> gpurun_out/s33_trace_n4.err; echo "trace4 rc=$?"
