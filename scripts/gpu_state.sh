# state sweep at N=${N}: one bench line per config (CUDA-graph timed loop, isolated per-kernel timing)
exec > gpurun_out/state_n${N}${TAG}.log 2>&1
for c in ${CONFIGS:-c2 c3 c4 c5}; do
  if [ "$N" = "1" ]; then timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-e2e --no-cpu $EXTRA;
  else timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29580 bench.py --gpus $N --config $c --steps 300 --warmup 10 --no-e2e $EXTRA 2>/dev/null; fi | tail -1 > gpurun_out/state_${c}_n${N}${TAG}.json
  python -c "import json; d=json.load(open('gpurun_out/state_${c}_n${N}${TAG}.json')); k=d['roofline']['per_kernel']; print('$c N=$N', 'step', d['ms_per_step'], 'value', d['value'], 'tstar', d['roofline']['step_tstar_ms_measured_peaks'], 'frac', d['roofline']['step_frac_of_tstar'], 'fwd', k['fwd']['ms'], k['fwd']['tstar_ms'], k['fwd']['bound'], 'bwd', k['bwd']['ms'], k['bwd']['tstar_ms'], k['bwd']['bound'], 'nccl', (d.get('nccl_comparison') or {}).get('ms_per_step'), 'overlap', (d.get('overlap_with_pp_p2p') or {}).get('overlap_efficiency'))"
done
