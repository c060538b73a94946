# session 3: GPU tests (fan-out return cases) on 2 GPUs, driver-style bench at N=2 (both arms) and N=1
exec > gpurun_out/s40.log 2>&1
s=$(date +%s); timeout 1200 python -m pytest tests/ -m gpu -x -q > gpurun_out/s40_pytest_gpu.log 2>&1; echo "pytest rc=$? secs=$(( $(date +%s) - s ))"
tail -3 gpurun_out/s40_pytest_gpu.log
s=$(date +%s); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29951 bench.py --gpus 2 > gpurun_out/s40_bench_n2.json 2> gpurun_out/s40_bench_n2.err; echo "bench2 rc=$? secs=$(( $(date +%s) - s ))"
s=$(date +%s); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29952 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/s40_ref_n2.json 2> gpurun_out/s40_ref_n2.err; echo "ref2 rc=$? secs=$(( $(date +%s) - s ))"
s=$(date +%s); timeout 600 python bench.py > gpurun_out/s40_bench_n1.json 2> gpurun_out/s40_bench_n1.err; echo "bench1 rc=$? secs=$(( $(date +%s) - s ))"
python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
