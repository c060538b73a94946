# session 3: A/B base vs new kernels (graph per step for both), then the new default bench at N=4 and N=1
exec > gpurun_out/s35.log 2>&1
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --config c2x4 --matrix c3x4,c4w4,c4,c3 --no-e2e --no-nccl --no-overlap --steps 300 --matrix-steps 300 --graph-per-step"
for rep in 1 2; do
  HB_LIB_PATH=$PWD/ab/libhetbridge_base.so $T --master-port 2973$rep $B > gpurun_out/s35_base_$rep.json 2> gpurun_out/s35_base_$rep.err; echo "base $rep rc=$?"
  $T --master-port 2974$rep $B > gpurun_out/s35_new_$rep.json 2> gpurun_out/s35_new_$rep.err; echo "new $rep rc=$?"
done
for rep in 1 2; do
  HB_LIB_PATH=$PWD/ab/libhetbridge_base.so timeout 300 python bench.py --no-e2e --no-cpu --matrix c3,c4,c5 --graph-per-step > gpurun_out/s35_n1_base_$rep.json 2> gpurun_out/s35_n1_base_$rep.err; echo "n1 base $rep rc=$?"
  timeout 300 python bench.py --no-e2e --no-cpu --matrix c3,c4,c5 --graph-per-step > gpurun_out/s35_n1_new_$rep.json 2> gpurun_out/s35_n1_new_$rep.err; echo "n1 new $rep rc=$?"
done
s=$(date +%s); $T --master-port 29751 bench.py --gpus 4 > gpurun_out/s35_bench_n4.json 2> gpurun_out/s35_bench_n4.err; echo "bench4 rc=$? secs=$(( $(date +%s) - s ))"
s=$(date +%s); timeout 300 python bench.py > gpurun_out/s35_bench_n1.json 2> gpurun_out/s35_bench_n1.err; echo "bench1 rc=$? secs=$(( $(date +%s) - s ))"
