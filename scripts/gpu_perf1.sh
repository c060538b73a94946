exec > gpurun_out/perf1.log 2>&1
python scripts/perf_probe.py
for opt in "--no-clocks" "" "--no-clocks --blocks-per-sm 2 --threads 256" "--no-clocks --blocks-per-sm 8 --threads 256" "--no-clocks --blocks-per-sm 1 --threads 512" "--no-clocks --blocks-per-sm 16 --threads 128"; do
  timeout 300 python bench.py --config c2 --steps 30 --warmup 5 --no-cpu --no-e2e $opt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$opt', d['ms_per_step'], d['roofline']['per_kernel'], d['clocks'])"
done
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
