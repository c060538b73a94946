set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu.log
for c in c2 c3 c4 c5 c1; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?; done
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
cat gpurun_out/bench_*.json
