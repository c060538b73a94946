"""N>1 host logic on CPU: world_size-2 gloo processes.

Each process compiles the plan independently (identical on
every rank), keeps only the index-map segments whose destination rank the
logical-rank->GPU map places on it (exactly the set the device runtime
uploads), reads peers' source rows from buffers exchanged over gloo (standing
in for CUDA-IPC-mapped peer memory), and the gathered result must equal the
oracle's whole-edge forward/backward.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import O, hbb
from paper_2605_27678_b200 import configs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = configs.get(name, scale=1024)
        W = 5 if not cfg.splice else cfg.width
        if cfg.splice:
            W = cfg.tokens * 8
        edge = cfg.edge().__class__(cfg.src, cfg.dst, cfg.batch, W)
        plan = hbb.plan_bridge(edge)
        sp = None
        if cfg.splice:
            s = cfg.splice
            sp = hbb.SpliceSpec(s["Q"], s["S"], 8, cfg.tokens, s["codes"], s["text_mode"])
        text = hbb.export_plan(plan)
        texts = [None] * world
        dist.all_gather_object(texts, text)
        assert all(t == text for t in texts), "plan differs across processes"
        r2g = configs.rank_to_gpu(plan.world, world)
        fwd = [s for s in hbb.index_forward(plan, sp) if r2g[s[3]] == rank]
        bwd = [s for s in hbb.index_backward(plan, sp) if r2g[s[0]] == rank]
        # every process owns a disjoint part of the work; together they cover it
        counts = [None] * world
        dist.all_gather_object(counts, (len(fwd), len(bwd)))
        assert sum(c[0] for c in counts) == len(hbb.index_forward(plan, sp))
        assert sum(c[1] for c in counts) == len(hbb.index_backward(plan, sp))

        rng = np.random.default_rng(5)
        src = O.Layout(cfg.src.name, cfg.src.tp, cfg.src.cp, cfg.src.pp, cfg.src.dp, cfg.src.rank_offset)
        dst = O.Layout(cfg.dst.name, cfg.dst.tp, cfg.dst.cp, cfg.dst.pp, cfg.dst.dp, cfg.dst.rank_offset)
        B = cfg.batch
        SI = O.intervals(B, src.dp)
        X = rng.standard_normal((B, W))
        shards = {r: X[SI[src.coord(r)[3]][0]:SI[src.coord(r)[3]][0] + SI[src.coord(r)[3]][1]]
                  for r in src.stage_ranks(src.pp - 1)}
        # local buffers only; peers' buffers arrive over gloo ("peer memory")
        mine = {(r, hbb.SLOT_SRC_ACT): shards[r].reshape(-1) for r in shards if r2g[r] == rank}
        ntext = int((np.asarray(cfg.splice["codes"]) < 0).sum()) if sp else 0
        T = rng.standard_normal((ntext, 8)) if sp else None
        if sp:
            L = cfg.splice["S"] // dst.cp
            for r in dst.stage_ranks(0):
                if r2g[r] == rank:
                    c = dst.coord(r)[1]
                    sl = cfg.splice["codes"][c * L:(c + 1) * L]
                    mine[(r, hbb.SLOT_TEXT)] = T[[-1 - int(x) for x in sl if x < 0]].reshape(-1)
        allbufs = [None] * world
        dist.all_gather_object(allbufs, mine)
        peer = {k: v for d in allbufs for k, v in d.items()}
        out = {}
        for (sr, ss, so, dr, ds, do, n) in fwd:
            buf = out.setdefault(dr, np.full(hbb.buffer_elems(plan, dr, ds, sp), np.nan))
            buf[do:do + n] = peer[(sr, ss)][so:so + n]
        outs = [None] * world
        dist.all_gather_object(outs, out)
        if rank == 0:
            got = {k: v for d in outs for k, v in d.items()}
            ref, _, _ = O.bridge_forward(src, dst, B, W, shards)
            for r, a in ref.items():
                exp = a
                if sp:
                    c = dst.coord(r)[1]
                    exp = O.splice_forward(cfg.splice["codes"], 1, cfg.splice["S"], 8, c * L, L,
                                           a.reshape(-1, 8), T)
                np.testing.assert_array_equal(got[r], exp.reshape(-1))
        # backward: destination gradients live on their owners' GPUs
        grads = {}
        for r in dst.stage_ranks(0):
            n = hbb.buffer_elems(plan, r, hbb.SLOT_DST_GRAD, sp)
            grads[r] = np.random.default_rng(1000 + r).standard_normal(n)
        mine = {(r, hbb.SLOT_DST_GRAD): g for r, g in grads.items() if r2g[r] == rank}
        allbufs = [None] * world
        dist.all_gather_object(allbufs, mine)
        peer = {k: v for d in allbufs for k, v in d.items()}
        res = {}
        for (dr, ds, do, n, terms) in bwd:
            buf = res.setdefault(dr, np.full(hbb.buffer_elems(plan, dr, ds, sp), np.nan))
            acc = np.zeros(n)
            for (tr, ts, to) in terms:
                acc = acc + peer[(tr, ts)][to:to + n]
            buf[do:do + n] = acc
        outs = [None] * world
        dist.all_gather_object(outs, res)
        if rank == 0:
            got = {k: v for d in outs for k, v in d.items()}
            DI = O.intervals(B, dst.dp)
            vg = {}
            for r, g in grads.items():
                if sp:
                    c = dst.coord(r)[1]
                    g = O.splice_backward(cfg.splice["codes"], 1, cfg.splice["S"], 8, c * L, L, g.reshape(-1, 8),
                                          DI[0][1] * cfg.tokens)
                vg[r] = g.reshape(-1, W)
            refb, _, _ = O.bridge_backward(src, dst, B, W, vg)
            for r, a in refb.items():
                np.testing.assert_allclose(got[r], a.reshape(-1), rtol=0, atol=1e-12)
        q.put((rank, "ok"))
    except Exception as exc:  # surfaced to the parent
        q.put((rank, repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_two_process_partition_matches_oracle(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: "ok", 1: "ok"}, res
    assert all(p.exitcode == 0 for p in procs)
