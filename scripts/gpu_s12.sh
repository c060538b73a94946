exec > gpurun_out/s12.log 2>&1
for i in 1 2; do
for L in libhetbridge_r0.so libhetbridge.so; do echo "== $L"
for c in c2 c3; do HB_RED_ENGINE=ldg HB_LIB_PATH=$PWD/paper_2605_27678_b200/$L python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['per_kernel']; print('$c N=1 step', d['ms_per_step'], 'frac', d['roofline']['step_frac_of_tstar'], 'fwd', k['fwd']['ms'], k['fwd']['frac'], 'bwd', k['bwd']['ms'], k['bwd']['frac'])"; done
done; done
