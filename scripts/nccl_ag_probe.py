"""NCCL all-gather bandwidth at the C2 fan-in shape (per-rank shard 8 x 576 x 4096 bf16),
to see what NVLS (switch multicast) buys over point-to-point copies on this box.
  NCCL_NVLS_ENABLE=0|1 torchrun --nproc-per-node N scripts/nccl_ag_probe.py"""
import json
import os

import torch
import torch.distributed as dist

rank, N = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
n = 8 * 576 * 4096
x = torch.randn(n, device="cuda").to(torch.bfloat16)
out = torch.empty(N * n, device="cuda", dtype=torch.bfloat16)
for _ in range(5):
    dist.all_gather_into_tensor(out, x)
torch.cuda.synchronize()
dist.barrier()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
R = 20
e0.record()
for _ in range(R):
    dist.all_gather_into_tensor(out, x)
e1.record()
torch.cuda.synchronize()
t = torch.tensor([e0.elapsed_time(e1) / R], device="cuda", dtype=torch.float64)
dist.all_reduce(t, op=dist.ReduceOp.MAX)
ingress = (N - 1) * n * 2
if rank == 0:
    print(json.dumps({"N": N, "nvls": os.environ.get("NCCL_NVLS_ENABLE"), "ms": round(t.item(), 4),
                      "ingress_gbs_per_gpu": round(ingress / (t.item() * 1e-3) / 1e9, 1)}), flush=True)
dist.destroy_process_group()
