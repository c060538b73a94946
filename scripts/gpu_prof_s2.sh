# session-2 evidence for profiles/: default bench line, launch list, full capture of both kernels (C2, N=1)
exec > gpurun_out/prof_s2.log 2>&1
python bench.py > gpurun_out/s2_bench_default_n1.json 2> gpurun_out/s2_bench_default_n1.err; echo bench=$?
CMD="python bench.py --config c2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-clocks"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:segments -c 30 --csv --log-file gpurun_out/s2_c2_n1_launches.csv $CMD > /dev/null 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:segments -s 6 -c 2 -o gpurun_out/s2_c2_n1_full $CMD > /dev/null 2>&1; echo full=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s2_bench_reference_n1.json 2>&1; echo ref=$?
