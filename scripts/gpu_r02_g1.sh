cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm --format=csv > gpurun_out/g1_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/g1_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/g1_pytest.log
