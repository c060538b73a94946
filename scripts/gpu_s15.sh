exec > gpurun_out/s15.log 2>&1
timeout 900 python -m pytest tests/test_autograd.py -m gpu -x -q 2>&1 | tail -30
