"""Multi-GPU parity worker (one process per GPU, launched by torchrun).

Every process builds the same plan, maps logical rank r to GPU floor(r*N/world),
fills the buffers of its resident ranks from one seeded global tensor, and runs
the boundary forward/backward through the C-ABI with peers' rows pulled over
NVSwitch (CUDA-IPC-mapped buffers, in-kernel epoch barrier). Each process checks
its own ranks against the oracle: forward bit-exact, backward (beta=1 into fp32)
within 1e-6. Prints one JSON line per config from rank 0.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mgpu_worker.py [configs...]
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

from paper_2605_27678_b200 import bridge as hbb  # noqa: E402
from paper_2605_27678_b200 import configs  # noqa: E402
from parity_core import ProcessDriver, bind_caller_buffers, group_parity, make_splice, o_layout  # noqa: E402

STRICT = os.environ.get("HB_STRICT", "0") == "1"


def run(name, rank, N, dev, steps=3):
    cfg = configs.get(name, scale=64)
    plan = hbb.plan_bridge(cfg.edge())
    sp = make_splice(cfg)
    r2g = configs.rank_to_gpu(plan.world, N)
    local = [r for r in range(plan.world) if r2g[r] == rank]
    rt = hbb.BridgeRuntime(plan, sp, n_gpus=N, my_gpu=rank, rank_to_gpu=r2g, act_dtype=torch.bfloat16,
                           grad_in_dtype=torch.bfloat16, grad_out_dtype=torch.float32, timeout_s=30.0,
                           fwd_mode=int(os.environ.get("HB_FWD_MODE", "0")),
                           partition=int(os.environ.get("HB_PARTITION", "0")), strict_provenance=STRICT)
    rt.exchange_handles()
    pad = int(os.environ.get("HB_BIND_PAD", "-1"))
    if pad >= 0:  # caller-owned (row-strided when pad > 0) buffers, mapped by peers through CUDA IPC
        tdt = {"bf16": torch.bfloat16, "fp32": torch.float32}
        dt = {hbb.SLOT_SRC_ACT: tdt[cfg.act], hbb.SLOT_DST_ACT: tdt[cfg.act], hbb.SLOT_TEXT: tdt[cfg.act],
              hbb.SLOT_DST_GRAD: tdt[cfg.grad_in], hbb.SLOT_SRC_GRAD: torch.float32}
        bind_caller_buffers(rt.bind, rt.buffer_numel, cfg, local, lambda r: dev, lambda sl: dt[sl], pad)
        rt.exchange_bindings()
    ok, worst = group_parity(cfg, ProcessDriver(rt, local), steps=steps, strict=STRICT)
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    w = torch.tensor([worst], dtype=torch.float64, device=dev)
    dist.all_reduce(w, op=dist.ReduceOp.MAX)
    rt.close()
    return flag.item() == 0, w.item(), r2g


def run_projected(name, rank, N, dev):
    """Fused projector forward (tcgen05 GEMM pushing rows to every destination,
    local or peer) == GEMM into the source shards + the pulled forward reshard."""
    from paper_2605_27678_b200.projector import projector_gemm

    base = configs.get(name)
    cfg = configs.get(name, scale=base.hidden // 256)
    d_h, K = cfg.hidden, 128
    plan = hbb.plan_bridge(cfg.edge())
    r2g = configs.rank_to_gpu(plan.world, N)
    rts = []
    for _ in range(2):
        rt = hbb.BridgeRuntime(plan, n_gpus=N, my_gpu=rank, rank_to_gpu=r2g, timeout_s=30.0)
        rt.exchange_handles()
        rts.append(rt)
    rt_a, rt_b = rts
    srcs = rt_a.local_ranks(hbb.SLOT_SRC_ACT)
    g = torch.Generator(device=dev).manual_seed(11)
    w = (torch.randn(d_h, K, device=dev, generator=g) / K ** 0.5).to(torch.bfloat16)
    xs = []
    for r in srcs:  # rows of source rank r: deterministic in r (tp replicas of a shard share them)
        t, c, p, d = o_layout(cfg.src).coord(r)
        n = rt_a.buffer_numel(r, hbb.SLOT_SRC_ACT) // d_h
        xs.append(torch.randn(n, K, device=dev, generator=torch.Generator(device=dev).manual_seed(1000 + d))
                  .to(torch.bfloat16))
    x = torch.cat(xs) if xs else torch.zeros(0, K, device=dev, dtype=torch.bfloat16)
    ok = True
    for step in range(2):
        torch.cuda.synchronize()
        dist.barrier()
        rt_a.forward_projected(step, x, w)  # no local source rank: protocol-only launch
        y = projector_gemm(x, w) if x.shape[0] else x
        o = 0
        for r in srcs:
            b = rt_b.buffer(r, hbb.SLOT_SRC_ACT)
            n = b.numel() // d_h
            b.copy_(y[o:o + n].reshape(-1))
            o += n
        rt_b.forward(step)
        torch.cuda.synchronize()
        for rt in rts:
            rt.seed_forward_record(step)
            rt.backward(step, 0.0)
        torch.cuda.synchronize()
        if rt_a.status() or rt_b.status():
            raise RuntimeError("flag wait timed out")
        for r in rt_a.local_ranks(hbb.SLOT_DST_ACT):
            ok &= bool(torch.equal(rt_a.buffer(r, hbb.SLOT_DST_ACT), rt_b.buffer(r, hbb.SLOT_DST_ACT)))
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    for rt in rts:
        rt.close()
    return flag.item() == 0, 0.0, r2g


def run_autograd(name, rank, N, dev):
    """boundary() autograd op across processes with zero-copy binding: the
    caller's shards are bound (exchanged through CUDA IPC), no staging copy;
    forward bit-exact and source gradients against the oracle."""
    from oracle import oracle as O
    from paper_2605_27678_b200.autograd import boundary

    cfg = configs.get(name, scale=256)
    plan = hbb.plan_bridge(cfg.edge())
    r2g = configs.rank_to_gpu(plan.world, N)
    rt = hbb.BridgeRuntime(plan, n_gpus=N, my_gpu=rank, rank_to_gpu=r2g, act_dtype=torch.float32,
                           grad_in_dtype=torch.float32, grad_out_dtype=torch.float32, timeout_s=30.0, mb_slots=2)
    rt.exchange_handles()
    src, dst = o_layout(cfg.src), o_layout(cfg.dst)
    B, W = cfg.batch, cfg.width
    SI, DI = O.intervals(B, src.dp), O.intervals(B, dst.dp)
    ok = True
    for mb in range(2):
        rng = np.random.default_rng(100 + mb)
        X = rng.standard_normal((B, W))
        G = rng.standard_normal((B, W))
        src_ranks = rt.local_ranks(hbb.SLOT_SRC_ACT)
        xs = [torch.tensor(X[SI[src.coord(r)[3]][0]:SI[src.coord(r)[3]][0] + SI[src.coord(r)[3]][1]], device=dev,
                           dtype=torch.float32, requires_grad=True) for r in src_ranks]
        outs = boundary(rt, mb, *xs)
        outs = outs if isinstance(outs, tuple) else (outs,)
        for r, x in zip(src_ranks, xs):  # no staging copy: the runtime reads the caller's tensor
            ok &= rt.buffer(r, hbb.SLOT_SRC_ACT, mb % 2).data_ptr() == x.data_ptr()
        shards = {r: X[SI[src.coord(r)[3]][0]:SI[src.coord(r)[3]][0] + SI[src.coord(r)[3]][1]]
                  for r in src.stage_ranks(src.pp - 1)}
        ref, _, _ = O.bridge_forward(src, dst, B, W, shards)
        loss = 0
        gd = {}
        for r in dst.stage_ranks(0):
            d = dst.coord(r)[3]
            gd[r] = G[DI[d][0]:DI[d][0] + DI[d][1]]
        for r, o in zip(rt.local_ranks(hbb.SLOT_DST_ACT), outs):
            ok &= bool(np.array_equal(o.detach().cpu().numpy(), ref[r].astype(np.float32)))
            loss = loss + (o * torch.tensor(gd[r], device=dev, dtype=torch.float32)).sum()
        torch.cuda.synchronize()
        dist.barrier()
        loss.backward()  # c2 / c3: every GPU hosts destination ranks, so every GPU runs the backward op
        refb, _, _ = O.bridge_backward(src, dst, B, W, gd)
        torch.cuda.synchronize()
        for r, x in zip(src_ranks, xs):
            ok &= bool(np.allclose(x.grad.cpu().numpy(), refb[r], rtol=1e-6, atol=1e-6))
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    rt.close()
    return flag.item() == 0, 0.0, r2g


def run_vocab_parallel(name, rank, N, dev):
    """Vocab-parallel text embedding across processes: logical rank r on GPU
    r % N, so the TP pairs of the CP splice straddle GPUs; every rank's table
    shard is exported with the bindings (CUDA IPC) and the splice gathers each
    text row from its owner's shard. Checked against splicing table[ids] on a
    one-GPU runtime of this process (all ranks resident)."""
    from paper_2605_27678_b200 import grid as hbg

    cfg = configs.get(name, scale=64)
    plan = hbb.plan_bridge(cfg.edge())
    sp = make_splice(cfg)
    r2g = [r % N for r in range(plan.world)]
    vocab, tp = 998, cfg.dst.tp
    rows = (vocab + tp - 1) // tp
    g = torch.Generator(device="cpu").manual_seed(11)
    table = torch.randn(vocab, cfg.hidden, generator=g).to(torch.bfloat16)
    rt = hbb.BridgeRuntime(plan, sp, n_gpus=N, my_gpu=rank, rank_to_gpu=r2g, text_embedding=True, timeout_s=30.0)
    rt.exchange_handles()
    ref = hbb.BridgeRuntime(plan, sp)  # every rank resident here, text pre-embedded
    keep = []
    for r in range(plan.world):
        if rt.buffer_numel(r, hbb.SLOT_DST_ACT) and r2g[r] == rank:
            t = hbg.coord_of_rank(cfg.dst, r).tp_idx
            piece = torch.zeros(rows, cfg.hidden, dtype=torch.bfloat16)
            lo, hi = t * rows, min(vocab, (t + 1) * rows)
            piece[: hi - lo] = table[lo:hi]
            piece = piece.to(dev)
            keep.append(piece)
            rt.set_text_embedding_shard(r, piece, t * rows, vocab)
    rt.exchange_bindings()
    for r in range(plan.world):
        n = rt.buffer_numel(r, hbb.SLOT_SRC_ACT)
        if n:
            x = torch.randn(n, generator=g).to(torch.bfloat16)
            ref.buffer(r, hbb.SLOT_SRC_ACT).copy_(x)
            if r2g[r] == rank:
                rt.buffer(r, hbb.SLOT_SRC_ACT).copy_(x)
        n = rt.buffer_numel(r, hbb.SLOT_TEXT) // cfg.hidden  # text rows = token ids
        if n:
            ids = torch.randint(0, vocab, (n,), generator=g, dtype=torch.int32)
            ref.buffer(r, hbb.SLOT_TEXT).copy_(table[ids.long()].reshape(-1))
            if r2g[r] == rank:
                rt.buffer(r, hbb.SLOT_TEXT).copy_(ids)
    torch.cuda.synchronize()
    dist.barrier()
    rt.validate()
    rt.forward(0)
    ref.forward(0)
    torch.cuda.synchronize()
    ok = rt.status() == 0
    for r in range(plan.world):
        if r2g[r] == rank and rt.buffer_numel(r, hbb.SLOT_DST_ACT):
            ok &= bool(torch.equal(rt.buffer(r, hbb.SLOT_DST_ACT), ref.buffer(r, hbb.SLOT_DST_ACT)))
    dist.barrier()
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    rt.close()
    ref.close()
    return flag.item() == 0, 0.0, r2g


def main():
    rank = int(os.environ["RANK"])
    N = int(os.environ["WORLD_SIZE"])
    local_rank = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist.init_process_group("nccl", device_id=dev)
    names = sys.argv[1:] or ["c2", "c3", "c4", "c5", "c1"]
    all_ok = True
    proj = os.environ.get("HB_PROJ", "0") == "1"
    ag = os.environ.get("HB_AUTOGRAD", "0") == "1"
    vp = os.environ.get("HB_VOCAB_PAR", "0") == "1"
    for name in names:
        fn = run_projected if proj else run_autograd if ag else run_vocab_parallel if vp else run
        ok, worst, r2g = fn(name, rank, N, dev)
        all_ok &= ok
        if rank == 0:
            print(json.dumps({"config": name, "n_gpus": N, "parity": ok, "bwd_max_rel": worst,
                              "rank_to_gpu": r2g}), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if all_ok else 1)


if __name__ == "__main__":
    main()
