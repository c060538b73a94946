exec > gpurun_out/modes.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -15; echo pytest=$?
N=1 OPTS="--partition=1 --partition=3 --partition=4" CONFIGS="c2 c3 c4 c5" bash scripts/gpu_sweep.sh
cat gpurun_out/sweep_n1.log
