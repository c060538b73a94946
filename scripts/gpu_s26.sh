exec > gpurun_out/s26.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"projector|gemm|Kernel|nvjet|sm100" -c 5 -o gpurun_out/s26_proj python scripts/proj_one.py > /dev/null 2>&1; echo ncu=$?
