"""Fused projector forward vs cuBLAS GEMM into the source shards + pulled
forward reshard, under torchrun (N GPUs), full width, host out of the loop
(R ops captured in one CUDA graph), max over ranks."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2605_27678_b200 import bridge as hbb, configs  # noqa: E402

R = 10


def timed(body, st, dev):
    with torch.cuda.stream(st):
        for _ in range(2):
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
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(st)
        for _ in range(3):
            g.replay()
        e1.record(st)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / (3 * R) * 1e3], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return round(t.item(), 2)


def main():
    rank, N = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    st = torch.cuda.Stream()
    for name in sys.argv[1:]:
        cfg = configs.get(name)
        plan = hbb.plan_bridge(cfg.edge())
        r2g = configs.rank_to_gpu(plan.world, N)
        rt = hbb.BridgeRuntime(plan, n_gpus=N, my_gpu=rank, rank_to_gpu=r2g)
        rt.exchange_handles()
        d_h, K = cfg.hidden, 1280
        srcs = rt.local_ranks(hbb.SLOT_SRC_ACT)
        views = [rt.buffer(r, hbb.SLOT_SRC_ACT).view(-1, d_h) for r in srcs]
        rows = sum(v.shape[0] for v in views)
        x = torch.randn(rows, K, device=dev).to(torch.bfloat16)
        w = torch.randn(d_h, K, device=dev).to(torch.bfloat16)
        xs = list(torch.split(x, [v.shape[0] for v in views]))
        mb = [0]

        def fused():
            rt.forward_projected(mb[0], x, w, st)
            rt.backward(mb[0], 1.0, st)
            mb[0] += 1

        def unfused():
            for xi, v in zip(xs, views):
                torch.matmul(xi, w.t(), out=v)
            rt.forward(mb[0], st)
            rt.backward(mb[0], 1.0, st)
            mb[0] += 1

        def gemm_only():
            for xi, v in zip(xs, views):
                torch.matmul(xi, w.t(), out=v)

        res = {"cfg": name, "N": N, "K": K, "rows_per_gpu": rows,
               "fused_proj_fwd_bwd_us": timed(fused, st, dev),
               "cublas_then_fwd_bwd_us": timed(unfused, st, dev),
               "cublas_gemm_only_us": timed(gemm_only, st, dev)}
        if rank == 0:
            print(json.dumps(res), flush=True)
        rt.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
