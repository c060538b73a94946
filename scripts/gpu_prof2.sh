exec > gpurun_out/prof2.log 2>&1
CMD="python bench.py --config c2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-clocks"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:segments -c 30 --csv --log-file gpurun_out/launches_c2_r2.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
$CMD > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:segments -s 6 -c 2 -o gpurun_out/prof_c2_tma $CMD > gpurun_out/ncu_full.log 2>&1; echo full=$?
