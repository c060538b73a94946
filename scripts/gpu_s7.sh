exec > gpurun_out/s7.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python scripts/ovh_probe.py c2
HB_LIB_PATH=$PWD/paper_2605_27678_b200/libhetbridge_old.so python scripts/ovh_probe.py c2
for p in 0 1; do
HB_PARTITION=$p timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29590 tests/mgpu_worker.py c2 c3 c4 c5 c1 2>&1 | grep -cE '"parity": true' | tr '\n' ' '; echo " ok-configs partition=$p"
done
for L in libhetbridge_old.so libhetbridge.so; do echo "== $L"
HB_LIB_PATH=$PWD/paper_2605_27678_b200/$L MODES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 scripts/sweep_probe.py c2w4:1,64 c4w4:1,4 c2:1 c3:1 c4:1 2>&1 | grep "^{"
done
