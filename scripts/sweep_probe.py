"""Bytes-vs-time sweep under torchrun (N GPUs, one process each).

For each (config, scale, fwd_mode): build the runtime, capture R forward (or
backward) ops into one CUDA graph (host out of the loop), time replays, max over
ranks. Prints one line per case: per-op µs and per-GPU NVLink ingress / HBM bytes
from bench.traffic_model, so slope (bandwidth) and intercept (fixed cost) can be fit.

  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 scripts/sweep_probe.py c2w4:1,4,16 c4w4:1,4
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2605_27678_b200 import bridge as hbb, configs  # noqa: E402

R = int(os.environ.get("R", "20"))
MODES = [int(m) for m in os.environ.get("MODES", "1,2").split(",")]


def main():
    rank, N = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    st = torch.cuda.Stream(priority=-1)
    for arg in sys.argv[1:]:
        name, scales = arg.split(":")
        for sc in [int(x) for x in scales.split(",")]:
            cfg = configs.get(name, scale=sc)
            plan = hbb.plan_bridge(cfg.edge())
            sp = bench.make_splice(cfg)
            r2g = configs.rank_to_gpu(plan.world, N)
            tm = bench.traffic_model(cfg, N)
            for mode in MODES:
                rt = hbb.BridgeRuntime(plan, sp, n_gpus=N, my_gpu=rank, rank_to_gpu=r2g, mb_slots=2,
                                       fwd_mode=mode, partition=int(os.environ.get("PART", "0")),
                                       blocks_per_sm=int(os.environ.get("BPS", "0")))
                rt.exchange_handles()
                mb = [0]

                def f():
                    rt.forward(mb[0], st)
                    rt.seed_forward_record(mb[0])
                    mb[0] += 1

                def b():
                    rt.seed_forward_record(mb[0])
                    rt.backward(mb[0], 1.0, st)
                    mb[0] += 1

                res = []
                for body in (f, b):
                    with torch.cuda.stream(st):
                        for _ in range(3):
                            body()
                        torch.cuda.synchronize()
                        dist.barrier()
                        g = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(g, stream=st):
                            for _ in range(R):
                                body()
                        g.replay()
                        torch.cuda.synchronize()
                        dist.barrier()
                        torch.cuda.synchronize()
                        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                        e0.record(st)
                        for _ in range(5):
                            g.replay()
                        e1.record(st)
                    torch.cuda.synchronize()
                    res.append(e0.elapsed_time(e1) / (5 * R) * 1e3)
                    del g
                t = torch.tensor(res, device=dev, dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                if rt.status():
                    raise RuntimeError("device timeout")
                if rank == 0:
                    print(json.dumps({"cfg": name, "scale": sc, "mode": mode, "fwd_us": round(t[0].item(), 2),
                                      "bwd_us": round(t[1].item(), 2),
                                      "fwd_nvl_mb": max(tm["fwd_nvl"]) / 1e6, "fwd_hbm_mb": max(tm["fwd_hbm"]) / 1e6,
                                      "bwd_nvl_mb": max(tm["bwd_nvl"]) / 1e6, "bwd_hbm_mb": max(tm["bwd_hbm"]) / 1e6}),
                          flush=True)
                rt.close()
                torch.cuda.synchronize()
                dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
