# session 3: fan-out reduce (one term read, several accumulators): parity N=1..4 + A/B (HB_RED_FAN) at N=4 and N=1
exec > gpurun_out/s36.log 2>&1
s=$(date +%s); timeout 1200 python -m pytest tests/ -m gpu -x -q > gpurun_out/s36_pytest_gpu.log 2>&1; echo "pytest rc=$? secs=$(( $(date +%s) - s ))"
tail -3 gpurun_out/s36_pytest_gpu.log
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --config c2x4 --matrix c3x4,c4w4,c4,c3 --no-e2e --no-nccl --no-overlap --steps 300 --matrix-steps 300"
for rep in 1 2; do
  HB_RED_FAN=0 $T --master-port 2976$rep $B > gpurun_out/s36_nofan_$rep.json 2> gpurun_out/s36_nofan_$rep.err; echo "nofan $rep rc=$?"
  $T --master-port 2977$rep $B > gpurun_out/s36_fan_$rep.json 2> gpurun_out/s36_fan_$rep.err; echo "fan $rep rc=$?"
  HB_RED_FAN=0 timeout 300 python bench.py --no-e2e --no-cpu --matrix c3,c4,c5 > gpurun_out/s36_n1_nofan_$rep.json 2> gpurun_out/s36_n1_nofan_$rep.err; echo "n1 nofan $rep rc=$?"
  timeout 300 python bench.py --no-e2e --no-cpu --matrix c3,c4,c5 > gpurun_out/s36_n1_fan_$rep.json 2> gpurun_out/s36_n1_fan_$rep.err; echo "n1 fan $rep rc=$?"
done
