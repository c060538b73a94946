"""Host runtime worker (one process per GPU, torchrun): builds the topology's
HostRuntime (groups, NCCL world + PP communicators, boundary execs, streams),
fills every boundary shard and stage buffer with hashed values, runs steps of
the graph-aware 1F1B dispatch table and checks on every rank:
  * NC forward: each destination shard equals the index-map restatement of the
    regenerated source shards (bit-exact); NC backward: each source gradient
    equals the restatement of the regenerated destination gradients (beta=0);
  * P2P: each stage's act_in / grad_in equal the neighbour's act_out / grad_out;
and times steps with NC only, P2P only and both (overlap). Prints one JSON
line per topology from rank 0.

  torchrun --nproc-per-node N tests/runtime_worker.py [topology ...]
"""
import json
import os
import sys

import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import bench  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    all_ok = True
    for name in sys.argv[1:] or ["c5w4", "join4", "fig4a", "c5"]:
        res = bench.run_host_runtime(name, rank, world, dev)
        if res is None:
            continue
        all_ok &= res["parity"]
        if rank == 0:
            print(json.dumps(res), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if all_ok else 1)


if __name__ == "__main__":
    main()
