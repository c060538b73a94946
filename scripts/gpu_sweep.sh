# usage: N=4 [CONFIGS=..] [OPTS=..] bash scripts/gpu_sweep.sh  -> gpurun_out/sweep_n$N.log
exec > gpurun_out/sweep_n${N}.log 2>&1
run() { # config, opts
  if [ "$N" = "1" ]; then timeout 300 python bench.py --config $1 --steps 50 --warmup 5 --no-e2e --no-cpu --no-clocks $2;
  else timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29520 bench.py --gpus $N --config $1 --steps 50 --warmup 5 --no-e2e --no-clocks --no-nccl $2 2>/dev/null; fi | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['per_kernel']; print('$1', '$2', 'step', d['ms_per_step'], 'tstar', d['roofline']['step_tstar_ms_measured_peaks'], 'frac', d['roofline']['step_frac_of_tstar'], 'fwd', k['fwd']['ms'], k['fwd']['tstar_ms'], k['fwd']['bound'], 'bwd', k['bwd']['ms'], k['bwd']['tstar_ms'], k['bwd']['bound'])"
}
for c in ${CONFIGS:-c2 c3 c4 c5}; do
  for o in ${OPTS:-"--fwd-mode=1" "--fwd-mode=2"}; do run $c "$o"; done
done
