# the driver's exact commands at N=4 and N=2 (default config), both arms
exec > gpurun_out/s27.log 2>&1
for n in 4 2; do
  s=$(date +%s)
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n > gpurun_out/s27_bench_n$n.json 2> gpurun_out/s27_bench_n$n.err; echo "ours n=$n rc=$? secs=$(( $(date +%s) - s ))"
  s=$(date +%s)
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n bench.py --impl reference --gpus $n --steps 3 --warmup 3 > gpurun_out/s27_ref_n$n.json 2> gpurun_out/s27_ref_n$n.err; echo "ref n=$n rc=$? secs=$(( $(date +%s) - s ))"
done
