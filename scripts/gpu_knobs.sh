exec > gpurun_out/knobs.log 2>&1
for kb in 32 16 8; do for rc in 32768 8192; do for c in c2w4 c4w4; do
HB_TMA_CHUNK_KB=$kb HB_RED_CHUNK=$rc timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29570 bench.py --gpus 4 --config $c --steps 300 --warmup 10 --no-e2e --no-clocks --no-nccl 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tma=$kb red=$rc $c', 'step', d['ms_per_step'], 'tstar', d['roofline']['step_tstar_ms_measured_peaks'])"
done; done; done
for kb in 32 16 8; do for rc in 32768 8192; do
HB_TMA_CHUNK_KB=$kb HB_RED_CHUNK=$rc timeout 300 python bench.py --config c2 --steps 300 --warmup 10 --no-e2e --no-clocks --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=1 tma=$kb red=$rc c2', 'step', d['ms_per_step'])"
done; done
