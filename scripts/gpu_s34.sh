# session 3: cycle graphs, reduce path restored; parity N=1..4; bench N=4 + N=1; NCCL NVLS all-gather probe
exec > gpurun_out/s34.log 2>&1
s=$(date +%s); timeout 1200 python -m pytest tests/ -m gpu -x -q > gpurun_out/s34_pytest_gpu.log 2>&1; echo "pytest rc=$? secs=$(( $(date +%s) - s ))"
tail -3 gpurun_out/s34_pytest_gpu.log
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node"
s=$(date +%s); $T 4 --master-addr 127.0.0.1 --master-port 29681 bench.py --gpus 4 > gpurun_out/s34_bench_n4.json 2> gpurun_out/s34_bench_n4.err; echo "bench4 rc=$? secs=$(( $(date +%s) - s ))"
$T 4 --master-addr 127.0.0.1 --master-port 29682 bench.py --gpus 4 --config c2x4 --matrix c3x4,c4w4,c4,c3 --no-e2e --no-nccl --no-overlap --steps 300 --matrix-steps 300 > gpurun_out/s34_ab_n4.json 2> gpurun_out/s34_ab_n4.err; echo "ab rc=$?"
for nv in 1 0; do NCCL_NVLS_ENABLE=$nv $T 4 --master-addr 127.0.0.1 --master-port 2969$nv scripts/nccl_ag_probe.py >> gpurun_out/s34_nccl_ag.jsonl 2>> gpurun_out/s34_nccl_ag.err; echo "nccl nvls=$nv rc=$?"; done
for nv in 1 0; do NCCL_NVLS_ENABLE=$nv $T 2 --master-addr 127.0.0.1 --master-port 2970$nv scripts/nccl_ag_probe.py >> gpurun_out/s34_nccl_ag.jsonl 2>> gpurun_out/s34_nccl_ag.err; echo "nccl2 nvls=$nv rc=$?"; done
NCCL_DEBUG=INFO NCCL_NVLS_ENABLE=1 $T 4 --master-addr 127.0.0.1 --master-port 29711 scripts/nccl_ag_probe.py > gpurun_out/s34_nccl_info.log 2>&1; grep -i "nvls\|multicast\|CollNet" gpurun_out/s34_nccl_info.log | head -20
s=$(date +%s); timeout 300 python bench.py > gpurun_out/s34_bench_n1.json 2> gpurun_out/s34_bench_n1.err; echo "bench1 rc=$? secs=$(( $(date +%s) - s ))"
