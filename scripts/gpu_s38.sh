# session 3: A/B at N=4: forward pull vs push, reduce carveout default vs 100
exec > gpurun_out/s38.log 2>&1
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --config c2x4 --matrix c4w4,c2,c4,c3x4 --no-e2e --no-nccl --no-overlap --steps 300 --matrix-steps 300"
p=29800
for rep in 1 2; do
  p=$((p+1)); $T --master-port $p $B --fwd-mode 1 > gpurun_out/s38_pull_$rep.json 2> gpurun_out/s38_pull_$rep.err; echo "pull $rep rc=$?"
  p=$((p+1)); $T --master-port $p $B --fwd-mode 2 > gpurun_out/s38_push_$rep.json 2> gpurun_out/s38_push_$rep.err; echo "push $rep rc=$?"
  p=$((p+1)); HB_RED_CARVEOUT=100 $T --master-port $p $B --fwd-mode 1 > gpurun_out/s38_co100_$rep.json 2> gpurun_out/s38_co100_$rep.err; echo "co100 $rep rc=$?"
done
for rep in 1 2; do
  timeout 300 python bench.py --no-e2e --no-cpu --matrix c3,c4,c5 > gpurun_out/s38_n1_def_$rep.json 2> gpurun_out/s38_n1_def_$rep.err; echo "n1 def $rep rc=$?"
  HB_RED_CARVEOUT=100 timeout 300 python bench.py --no-e2e --no-cpu --matrix c3,c4,c5 > gpurun_out/s38_n1_co100_$rep.json 2> gpurun_out/s38_n1_co100_$rep.err; echo "n1 co100 $rep rc=$?"
done
