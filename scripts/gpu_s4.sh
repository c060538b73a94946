exec > gpurun_out/s4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:segments -s 6 -c 2 -o gpurun_out/s4_tiny python bench.py --config c2 --scale 4096 --steps 5 --warmup 3 --no-e2e --no-cpu --no-clocks --no-graph
echo rc=$?
