exec > gpurun_out/s10.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for p in 0 1; do
HB_PARTITION=$p timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29590 tests/mgpu_worker.py c2 c3 c4 c5 c1 2>&1 | grep -cE '"parity": true' | tr '\n' ' '; echo " ok-configs partition=$p"
done
MODES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 scripts/sweep_probe.py c2x4:1,8 c3x4:1,4 c4w4:1,4 c5:1 c3:1 c4:1 2>&1 | grep "^{"
for c in c2 c3 c4 c5; do python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['per_kernel']; print('$c N=1 step', d['ms_per_step'], 'frac', d['roofline']['step_frac_of_tstar'], 'fwd', k['fwd']['ms'], k['fwd']['frac'], 'bwd', k['bwd']['ms'], k['bwd']['frac'])"; done
