exec > gpurun_out/perf2.log 2>&1
python scripts/perf_probe.py
for c in c2 c3 c4 c5; do
for opt in "--no-clocks" "" "--no-clocks --threads 256" "--no-clocks --blocks-per-sm 1"; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu --no-e2e $opt | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['per_kernel']; print('$c', '$opt', d['ms_per_step'], 'fwd', k['fwd']['ms'], k['fwd']['frac'], 'bwd', k['bwd']['ms'], k['bwd']['frac'], d['clocks'].get('sm_mhz'))"
done
done
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q 2>&1 | tail -3
