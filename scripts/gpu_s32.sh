# session 3: per-peer waits + dual-queue claims + read-only tail wait: parity at N=1..4, trace + bench at N=4
exec > gpurun_out/s32.log 2>&1
s=$(date +%s); timeout 1200 python -m pytest tests/ -m gpu -x -q > gpurun_out/s32_pytest_gpu.log 2>&1; echo "pytest rc=$? secs=$(( $(date +%s) - s ))"
tail -3 gpurun_out/s32_pytest_gpu.log
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node"
HB_TRACE=1 $T 4 --master-addr 127.0.0.1 --master-port 29621 scripts/trace_probe.py c4w4 c4 c2x4 c3x4 c2w4:4096 > gpurun_out/s32_trace_n4.jsonl 2> gpurun_out/s32_trace_n4.err; echo "trace4 rc=$?"
s=$(date +%s); $T 4 --master-addr 127.0.0.1 --master-port 29622 bench.py --gpus 4 > gpurun_out/s32_bench_n4.json 2> gpurun_out/s32_bench_n4.err; echo "bench4 rc=$? secs=$(( $(date +%s) - s ))"
for c in c2x4 c3x4 c4w4; do $T 4 --master-addr 127.0.0.1 --master-port 29623 bench.py --gpus 4 --config $c --matrix "" --no-e2e --no-nccl > gpurun_out/s32_bench_n4_$c.json 2> gpurun_out/s32_bench_n4_$c.err; echo "bench4 $c rc=$?"; done
