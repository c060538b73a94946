exec > gpurun_out/s25.log 2>&1
timeout 120 python -m pytest tests/test_projector.py -x -q 2>&1 | tail -5
echo "== cluster 2"; timeout 120 python scripts/proj_probe.py
echo "== cluster 1"; HB_PROJ_CLUSTER=1 timeout 120 python scripts/proj_probe.py
timeout 200 python scripts/fused_probe.py
