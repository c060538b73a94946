exec > gpurun_out/s21.log 2>&1
run() { echo "== $*"; env "$@" MODES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 scripts/sweep_probe.py c2w4:4,1 c2x4:8,1 c4w4:4,1 c3x4:1 c2:1 c4:1 2>&1 | grep "^{"; }
run X=1
run HB_RED_CHUNK=32768
for c in c2 c3 c4; do CUDA_VISIBLE_DEVICES=0 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['per_kernel']; print('$c N=1 step', d['ms_per_step'], 'frac', d['roofline']['step_frac_of_tstar'], 'fwd', k['fwd']['ms'], k['fwd']['frac'], 'bwd', k['bwd']['ms'], k['bwd']['frac'])"; done
