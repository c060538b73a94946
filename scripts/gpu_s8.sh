exec > gpurun_out/s8.log 2>&1
for i in 1 2; do
for L in libhetbridge_old.so libhetbridge.so libhetbridge_post1.so; do echo "== $L"
HB_LIB_PATH=$PWD/paper_2605_27678_b200/$L MODES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 scripts/sweep_probe.py c2w4:64,4 c4w4:4 2>&1 | grep "^{"
done; done
for p in 0; do
HB_PARTITION=$p timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29590 tests/mgpu_worker.py c2 c3 c4 c5 c1 2>&1 | grep -cE '"parity": true' | tr '\n' ' '; echo " ok-configs partition=$p"
HB_LIB_PATH=$PWD/paper_2605_27678_b200/libhetbridge_post1.so HB_PARTITION=$p timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29590 tests/mgpu_worker.py c2 c3 c4 c5 c1 2>&1 | grep -cE '"parity": true' | tr '\n' ' '; echo " ok-configs post1 partition=$p"
done
