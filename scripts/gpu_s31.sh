# session 3: N=4 trace probe (per-CTA timelines), bench matrix at N=4, multicast support
exec > gpurun_out/s31.log 2>&1
nvidia-smi topo -m | head -8
python scripts/mc_probe.py
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node"
HB_TRACE=1 $T 4 --master-addr 127.0.0.1 --master-port 29611 scripts/trace_probe.py c4w4 c4 c2x4 c3x4 c2w4:4096 c4w4:64 > gpurun_out/s31_trace_n4.jsonl 2> gpurun_out/s31_trace_n4.err; echo "trace4 rc=$?"
HB_TRACE=1 timeout 300 python scripts/trace_probe.py c4 c2 c2w4:4096 > gpurun_out/s31_trace_n1.jsonl 2> gpurun_out/s31_trace_n1.err; echo "trace1 rc=$?"
s=$(date +%s); $T 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 > gpurun_out/s31_bench_n4.json 2> gpurun_out/s31_bench_n4.err; echo "bench4 rc=$? secs=$(( $(date +%s) - s ))"
s=$(date +%s); timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/s31_bench_n1.json 2> gpurun_out/s31_bench_n1.err; echo "bench1 rc=$? secs=$(( $(date +%s) - s ))"
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,NVLS $T 4 --master-addr 127.0.0.1 --master-port 29613 -c "import torch,torch.distributed as d,os;r=int(os.environ['RANK']);torch.cuda.set_device(r);d.init_process_group('nccl');x=torch.ones(1<<24,device='cuda');d.all_reduce(x);torch.cuda.synchronize();d.destroy_process_group()" > gpurun_out/s31_nccl.log 2>&1; echo "nccl rc=$?"
grep -i "nvls\|multicast" gpurun_out/s31_nccl.log | head -10
