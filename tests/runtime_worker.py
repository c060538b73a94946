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
import statistics
import sys

import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import bench  # noqa: E402
from paper_2605_27678_b200 import bridge as hbb  # noqa: E402
from paper_2605_27678_b200 import parity as P  # noqa: E402
from paper_2605_27678_b200 import runtime as R  # noqa: E402
from paper_2605_27678_b200 import sched as S  # noqa: E402
from paper_2605_27678_b200.grid import ModuleLayout  # noqa: E402


def topology(name):
    """(modules, edges, global batch, feature width, pp bytes)"""
    if name == "c5w4":  # C5 at 4 GPUs: vit{dp1}@0 -> llm{pp3}@1-3
        return [ModuleLayout("vit", rank_offset=0), ModuleLayout("llm", pp=3, rank_offset=1)], [(0, 1)], 8, 576 * 512, 1 << 22
    if name == "join4":  # Fig. 4(a) shape at 4 GPUs: E1 pp2, E2 pp1 -> LLM pp1 (a join of two NC edges)
        return ([ModuleLayout("E1", pp=2, rank_offset=0), ModuleLayout("E2", rank_offset=2),
                 ModuleLayout("LLM", rank_offset=3)], [(0, 2), (1, 2)], 8, 576 * 256, 1 << 20)
    if name == "fig4a":  # PAPER Fig. 4(a): E1 pp2, E2 pp1, LLM pp3 (6 GPUs)
        mods, edges = S.fig4a_modules()
        return mods, edges, 8, 576 * 256, 1 << 20
    if name == "c5":  # BASELINE C5: vit{dp2}@0-1 -> llm{tp2,pp3}@2-7 (8 GPUs), bf16 h4096, 16 img x 576
        return ([ModuleLayout("vit", dp=2, rank_offset=0), ModuleLayout("llm", tp=2, pp=3, rank_offset=2)],
                [(0, 1)], 16, 576 * 4096, 16 * 576 * 4096 * 2)
    raise KeyError(name)


def hkey(*a):
    k = 0
    for x in a:
        k = k * 131 + x + 1
    return k * 7919


def run(name, rank, world, dev, steps=3):
    mods, edges, B, W, ppb = topology(name)
    if max(m.rank_end() for m in mods) > world:
        return None
    rt = R.HostRuntime(mods, edges, B, W, nmb=4, pp_bytes=ppb, skip=R.SKIP_COMPUTE)
    ok = True
    views = [rt.edge_runtime(k) for k in range(len(edges))]
    # fill boundary shards (every buffer set = microbatch slot) and stage buffers
    for k, v in enumerate(views):
        for mb in range(rt.nmb):
            for slot in (hbb.SLOT_SRC_ACT, hbb.SLOT_DST_GRAD):
                if v.buffer_numel(rank, slot) and v.rank_to_gpu[rank] == rank:
                    try:
                        b = v.buffer(rank, slot, mb)
                    except hbb.HetBridgeError:
                        b = None
                    if b is not None:
                        b.copy_(bench.fill_values(b.numel(), hkey(k, slot, mb, rank), b.dtype, dev))
    for mb in range(rt.nmb):
        for which in (R.ACT_OUT, R.GRAD_OUT):
            t = rt.stage_buffer(which, mb)
            if t is not None:
                t.view(torch.int16).copy_(bench.fill_values(t.numel() // 2, hkey(9, which, mb, rank), torch.bfloat16,
                                                            dev).view(torch.int16))
    torch.cuda.synchronize()
    dist.barrier()
    rt.step()
    ms_first = rt.last_step_ms()
    torch.cuda.synchronize()
    dist.barrier()
    # NC checks
    for k, v in enumerate(views):
        fwd_map, bwd_map = hbb.index_forward(v.plan), hbb.index_backward(v.plan, balanced=True)
        for mb in range(rt.nmb):
            def regen(r, slot, _k=k, _mb=mb, _v=v):
                n = _v.buffer_numel(r, slot)
                dt = _v.act_dtype if slot == hbb.SLOT_SRC_ACT else _v.grad_in_dtype
                return bench.fill_values(n, hkey(_k, slot, _mb, r), dt, dev)
            if v.buffer_numel(rank, hbb.SLOT_DST_ACT):
                out = v.buffer(rank, hbb.SLOT_DST_ACT, mb)
                exp, cov = P.expected_forward(fwd_map, rank, out.numel(), regen)
                ok &= cov == out.numel() and bool(torch.equal(out.view(torch.int16), exp.view(torch.int16)))
            if v.buffer_numel(rank, hbb.SLOT_SRC_GRAD):
                got = v.buffer(rank, hbb.SLOT_SRC_GRAD, mb)
                exp = P.expected_backward(bwd_map, rank, torch.zeros_like(got), 0.0, regen)
                ok &= bool(torch.equal(got, exp))
    # P2P checks: neighbours in my module's PP group
    pp = rt.group(2)
    if rt.module >= 0 and len(pp) > 1:
        i = pp.index(rank)
        for mb in range(rt.nmb):
            if i > 0:
                exp = bench.fill_values(ppb // 2, hkey(9, R.ACT_OUT, mb, pp[i - 1]), torch.bfloat16, dev)
                ok &= bool(torch.equal(rt.stage_buffer(R.ACT_IN, mb).view(torch.int16), exp.view(torch.int16)))
            if i + 1 < len(pp):
                exp = bench.fill_values(ppb // 2, hkey(9, R.GRAD_OUT, mb, pp[i + 1]), torch.bfloat16, dev)
                ok &= bool(torch.equal(rt.stage_buffer(R.GRAD_IN, mb).view(torch.int16), exp.view(torch.int16)))
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    rt.close()
    # overlap: the same table with one traffic class skipped
    times = {}
    for label, skip in (("nc_only", R.SKIP_COMPUTE | R.SKIP_P2P), ("p2p_only", R.SKIP_COMPUTE | R.SKIP_NC),
                        ("both", R.SKIP_COMPUTE)):
        r2 = R.HostRuntime(mods, edges, B, W, nmb=4, pp_bytes=ppb, skip=skip)
        r2.step()
        r2.last_step_ms()
        ts = []
        for _ in range(steps):
            dist.barrier()
            r2.step()
            ts.append(r2.last_step_ms())
        t = torch.tensor([statistics.median(ts)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        times[label] = round(t.item(), 4)
        r2.close()
    tb, tp, both = times["nc_only"], times["p2p_only"], times["both"]
    overlap = (tb + tp - both) / max(1e-9, min(tb, tp))
    return {"topology": name, "n_gpus": world, "parity": flag.item() == 0, "rows": rt.rows,
            "first_step_ms": round(ms_first, 3), "step_ms": times, "overlap": round(overlap, 3),
            "how": "HostRuntime.step over the 1F1B dispatch table (event-only compute); NC = boundary exec "
                   "fwd/bwd on the boundary stream, P2P = NCCL send/recv on the PP communicator"}


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    all_ok = True
    for name in sys.argv[1:] or ["c5w4", "join4", "fig4a", "c5"]:
        res = run(name, rank, world, dev)
        if res is None:
            continue
        all_ok &= res["parity"]
        if rank == 0:
            print(json.dumps(res), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if all_ok else 1)


if __name__ == "__main__":
    main()
