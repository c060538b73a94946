"""NVLink probe (torchrun, N=2): copy-engine peer copy vs the boundary kernels' peer pulls.

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/nvl_probe.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_27678_b200 import bridge as hbb  # noqa: E402
from paper_2605_27678_b200 import grid as hbg  # noqa: E402


def timeit(fn, iters=10):
    fn()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def main():
    rank = int(os.environ["RANK"])
    N = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    out = {}
    nbytes = 512 << 20
    # (1) copy engine: rank 0 copies from GPU1 into GPU0 (same process sees both devices)
    if rank == 0 and torch.cuda.device_count() >= 2:
        a = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
        b = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")
        for _ in range(3):
            b.copy_(a)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10):
            b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        out["copy_engine_peer_gbs"] = nbytes / (e0.elapsed_time(e1) / 10) / 1e6
        del a, b
    dist.barrier()
    W = nbytes // 2  # bf16 elements of one sample
    cases = []
    for part in (1, 4):
        for push in (False, True):
            tag = ("push" if push else "pull") + ("_tma" if part == 4 else "_ldg")
            cases += [
                (tag + "_one_way", hbg.ModuleLayout("enc", dp=1), hbg.ModuleLayout("llm", dp=1, rank_offset=1), [1, 0], push, part),
                (tag + "_bidir", hbg.ModuleLayout("enc", dp=2), hbg.ModuleLayout("llm", tp=2, dp=1), [0, 1], push, part),
            ]
    for name, src, dst, r2g, push, part in cases:
        B = src.dp
        plan = hbb.plan_bridge(hbg.BoundaryEdge(src, dst, B, W))
        rt = hbb.BridgeRuntime(plan, n_gpus=N, my_gpu=rank, rank_to_gpu=r2g, fwd_mode=2 if push else 1,
                               partition=part)
        rt.exchange_handles()
        mb = [0]

        def fwd_only():
            rt.forward(mb[0])
            mb[0] += 1

        fwd_ms = timeit(fwd_only)
        out[name] = {"fwd_ms": round(fwd_ms, 4), "gbs_per_gpu": round(W * 2 / fwd_ms / 1e6, 1)}
        rt.close()
    if rank == 0:
        print(json.dumps(out))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
