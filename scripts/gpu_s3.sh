exec > gpurun_out/s3.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 scripts/sweep_probe.py c2w4:1,2,4,16,64 c4w4:1,4,16 c2:1,4 c4:1,4 2>&1 | grep -v Warning
