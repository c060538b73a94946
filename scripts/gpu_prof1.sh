exec > gpurun_out/prof1.log 2>&1
CMD="python bench.py --config c2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-clocks"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
$CMD > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:segments_kernel -s 6 -c 2 -o gpurun_out/prof_c2 $CMD > gpurun_out/ncu_full.log 2>&1; echo full=$?
ls -la gpurun_out
