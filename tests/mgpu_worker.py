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

from oracle import oracle as O  # noqa: E402
from paper_2605_27678_b200 import bridge as hbb  # noqa: E402
from paper_2605_27678_b200 import configs  # noqa: E402


def o_layout(l):
    return O.Layout(l.name, l.tp, l.cp, l.pp, l.dp, l.rank_offset)


STRICT = os.environ.get("HB_STRICT", "0") == "1"


def bf16_round(a):
    return torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16).double().numpy()


def run(name, rank, N, dev, steps=3):
    cfg = configs.get(name, scale=64)
    plan = hbb.plan_bridge(cfg.edge())
    sp = None
    if cfg.splice:
        s = cfg.splice
        sp = hbb.SpliceSpec(s["Q"], s["S"], cfg.hidden, cfg.tokens, s["codes"], s["text_mode"])
    r2g = configs.rank_to_gpu(plan.world, N)
    local = [r for r in range(plan.world) if r2g[r] == rank]
    rt = hbb.BridgeRuntime(plan, sp, n_gpus=N, my_gpu=rank, rank_to_gpu=r2g, act_dtype=torch.bfloat16,
                           grad_in_dtype=torch.bfloat16, grad_out_dtype=torch.float32, timeout_s=30.0,
                           fwd_mode=int(os.environ.get("HB_FWD_MODE", "0")),
                           partition=int(os.environ.get("HB_PARTITION", "0")), strict_provenance=STRICT)
    rt.exchange_handles()
    src, dst = o_layout(cfg.src), o_layout(cfg.dst)
    B, W = cfg.batch, cfg.width
    SI, DI = O.intervals(B, src.dp), O.intervals(B, dst.dp)
    rng = np.random.default_rng(17)
    X = bf16_round(rng.standard_normal((B, W)))
    shards = {}
    for r in src.stage_ranks(src.pp - 1):
        t, c, p, d = src.coord(r)
        shards[r] = bf16_round(X[SI[d][0]:SI[d][0] + SI[d][1]] + (8.0 * t if t else 0.0))
        if r in local:
            rt.buffer(r, hbb.SLOT_SRC_ACT).copy_(torch.from_numpy(shards[r].reshape(-1)).to(dev).to(torch.bfloat16))
    L = cfg.splice["S"] // dst.cp if sp else 0
    text = None
    if sp:
        codes = cfg.splice["codes"]
        text = bf16_round(rng.standard_normal((int((codes < 0).sum()), cfg.hidden)))
        for r in local:
            b = rt.buffer(r, hbb.SLOT_TEXT)
            if b is None:
                continue
            c = dst.coord(r)[1]
            sl = codes.reshape(-1, cfg.splice["S"])[:, c * L:(c + 1) * L].reshape(-1)
            b.copy_(torch.from_numpy(text[[-1 - int(x) for x in sl if x < 0]].reshape(-1)).to(dev).to(b.dtype))
    ref, _, _ = O.bridge_forward(src, dst, B, W, shards)
    ok = True
    worst = 0.0
    for step in range(steps):
        # fresh gradients every step; source gradients accumulate (beta=1)
        G = {}
        vg = {}
        for r in dst.stage_ranks(0):
            t, c, p, d = dst.coord(r)
            n = (cfg.splice["Q"] * L * cfg.hidden) if sp else DI[d][1] * W
            # strict: every rank its own gradient (pins the tp=0 data path);
            # default: contract gradients, tp replicas of a (cp, dp) cell equal
            seed = 100 * step + (r if STRICT else 10 * c + d)
            g = bf16_round(np.random.default_rng(seed).standard_normal(n))
            G[r] = g
            gg = g
            if sp:
                gg = O.splice_backward(cfg.splice["codes"], cfg.splice["Q"], cfg.splice["S"], cfg.hidden, c * L, L,
                                       g.reshape(-1, cfg.hidden), DI[d][1] * cfg.tokens)
            vg[r] = gg.reshape(-1, W)
            if r in local:
                rt.buffer(r, hbb.SLOT_DST_GRAD).copy_(torch.from_numpy(g).to(dev).to(torch.bfloat16))
        if step == 0:
            for r in local:
                b = rt.buffer(r, hbb.SLOT_SRC_GRAD)
                if b is not None:
                    b.zero_()
            acc = {r: np.zeros(SI[src.coord(r)[3]][1] * W) for r in src.stage_ranks(src.pp - 1)}
        torch.cuda.synchronize()
        dist.barrier()
        rt.forward(step)
        rt.backward(step, 1.0)
        torch.cuda.synchronize()
        if rt.status():
            raise RuntimeError("flag wait timed out")
        for r in local:
            if r in ref:
                exp = ref[r]
                if sp:
                    c = dst.coord(r)[1]
                    exp = O.splice_forward(cfg.splice["codes"], cfg.splice["Q"], cfg.splice["S"], cfg.hidden, c * L,
                                           L, exp.reshape(-1, cfg.hidden), text)
                got = rt.buffer(r, hbb.SLOT_DST_ACT).double().cpu().numpy()
                ok &= bool(np.array_equal(got, exp.reshape(-1)))
        refb, _, _ = O.bridge_backward(src, dst, B, W, vg)
        for r in refb:
            acc[r] = acc[r] + refb[r].reshape(-1)
            if r in local:
                got = rt.buffer(r, hbb.SLOT_SRC_GRAD).double().cpu().numpy()
                rel = float(np.max(np.abs(got - acc[r]) / np.maximum(1.0, np.abs(acc[r]))))
                worst = max(worst, rel)
                ok &= rel <= 1e-6
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
    for name in names:
        ok, worst, r2g = (run_projected if proj else run)(name, rank, N, dev)
        all_ok &= ok
        if rank == 0:
            print(json.dumps({"config": name, "n_gpus": N, "parity": ok, "bwd_max_rel": worst,
                              "rank_to_gpu": r2g}), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if all_ok else 1)


if __name__ == "__main__":
    main()
