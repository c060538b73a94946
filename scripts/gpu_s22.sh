exec > gpurun_out/s22.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
