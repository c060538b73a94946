exec > gpurun_out/ovh2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
EXTRA="" bash scripts/gpu_overhead.sh; cat gpurun_out/overhead.log
EXTRA="--no-graph" bash scripts/gpu_overhead.sh; cat gpurun_out/overhead.log
