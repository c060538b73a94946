exec > gpurun_out/s17.log 2>&1
timeout 300 python -m pytest tests/test_projector.py -x -q 2>&1 | tail -25
timeout 300 python scripts/fused_probe.py
timeout 300 python scripts/proj_probe.py
