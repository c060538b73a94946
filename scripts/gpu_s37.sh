# session 3: push vs pull forward at N=4 (A/B), then profiles evidence at N=1 (default bench, launch list, full capture)
exec > gpurun_out/s37.log 2>&1
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for rep in 1 2; do
  for m in 1 2; do
    $T --master-port 2978$rep$m bench.py --gpus 4 --config c2x4 --matrix c4w4,c2,c4,c3 --no-e2e --no-nccl --no-overlap --steps 300 --matrix-steps 300 --fwd-mode $m > gpurun_out/s37_mode${m}_$rep.json 2> gpurun_out/s37_mode${m}_$rep.err; echo "mode $m rep $rep rc=$?"
  done
done
python bench.py > gpurun_out/s37_bench_default_n1.json 2> gpurun_out/s37_bench_default_n1.err; echo bench=$?
CMD="python bench.py --config c2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-clocks --matrix ''"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:segments -c 40 --csv --log-file gpurun_out/s37_c2_n1_launches.csv python bench.py --config c2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-clocks --matrix "" > /dev/null 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:segments -s 6 -c 2 -o gpurun_out/s37_c2_n1_full python bench.py --config c2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-clocks --matrix "" > /dev/null 2>&1; echo full=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s37_bench_reference_n1.json 2>&1; echo ref=$?
