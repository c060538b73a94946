# session 3: verify HEAD on a fresh box (driver's round-end sequence at N=1)
exec > gpurun_out/s30.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
s=$(date +%s); python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$? secs=$(( $(date +%s) - s ))"
s=$(date +%s); timeout 1200 python -m pytest tests/ -m gpu -x -q > gpurun_out/s30_pytest_gpu.log 2>&1; echo "pytest rc=$? secs=$(( $(date +%s) - s ))"
tail -5 gpurun_out/s30_pytest_gpu.log
s=$(date +%s); timeout 600 python bench.py > gpurun_out/s30_bench_n1.json 2> gpurun_out/s30_bench_n1.err; echo "bench rc=$? secs=$(( $(date +%s) - s ))"
s=$(date +%s); timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s30_ref_n1.json 2> gpurun_out/s30_ref_n1.err; echo "ref rc=$? secs=$(( $(date +%s) - s ))"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'copy_segments|reduce_segments' -c 40 --csv --log-file gpurun_out/s30_launches.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-clocks > gpurun_out/s30_ncu.log 2>&1; echo "ncu rc=$?"
