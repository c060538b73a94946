"""Group parity against the oracle, shared by the multi-process worker
(tests/mgpu_worker.py, one process per GPU) and the single-process group tests
(tests/test_local_group.py, hb_exec_open_peers_local).

A *driver* exposes the resident ranks it can read and write (``local``),
``buf(rank, slot)``, ``fwd(mb)``, ``bwd(mb, beta)``, ``sync()`` and
``status()``. The inputs are one seeded global tensor split by the layouts,
so every process derives the same values; each driver checks its own ranks:
forward bit-exact, backward (beta=1 into fp32, over several steps) within
|a-b|/max(1,|b|) <= 1e-6 of the oracle's doubles (SURVEY §8(a) tolerances).
"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle import oracle as O  # noqa: E402
from paper_2605_27678_b200 import bridge as hbb  # noqa: E402
from paper_2605_27678_b200 import configs  # noqa: E402


def o_layout(l):
    return O.Layout(l.name, l.tp, l.cp, l.pp, l.dp, l.rank_offset)


def bf16_round(a):
    return torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16).double().numpy()


def make_splice(cfg):
    if not cfg.splice:
        return None
    s = cfg.splice
    return hbb.SpliceSpec(s["Q"], s["S"], cfg.hidden, cfg.tokens, s["codes"], s["text_mode"])


def group_parity(cfg, drv, steps: int = 3, strict: bool = False):
    """Returns (ok, worst backward relative error) over the driver's ranks."""
    src, dst = o_layout(cfg.src), o_layout(cfg.dst)
    B, W = cfg.batch, cfg.width
    SI, DI = O.intervals(B, src.dp), O.intervals(B, dst.dp)
    sp = cfg.splice
    rng = np.random.default_rng(17)
    X = bf16_round(rng.standard_normal((B, W)))
    shards = {}
    for r in src.stage_ranks(src.pp - 1):
        t, c, p, d = src.coord(r)
        shards[r] = bf16_round(X[SI[d][0]:SI[d][0] + SI[d][1]] + (8.0 * t if t else 0.0))
        if r in drv.local:
            b = drv.buf(r, hbb.SLOT_SRC_ACT)
            b.copy_(torch.from_numpy(shards[r]).to(b.device).to(torch.bfloat16).reshape(b.shape))
    L = sp["S"] // dst.cp if sp else 0
    text = None
    if sp:
        codes = sp["codes"]
        text = bf16_round(rng.standard_normal((int((codes < 0).sum()), cfg.hidden)))
        for r in drv.local:
            b = drv.buf(r, hbb.SLOT_TEXT)
            if b is None:
                continue
            c = dst.coord(r)[1]
            sl = codes.reshape(-1, sp["S"])[:, c * L:(c + 1) * L].reshape(-1)
            b.copy_(torch.from_numpy(text[[-1 - int(x) for x in sl if x < 0]]).to(b.device).to(b.dtype).reshape(b.shape))
    ref, _, _ = O.bridge_forward(src, dst, B, W, shards)
    if sp and sp.get("text_mode") == hbb.TEXT_INPLACE:
        # the caller's embedding layer already wrote the text rows into the
        # slice; vision positions hold garbage (NaN) the boundary must replace
        for r in drv.local:
            if r not in ref:
                continue
            c = dst.coord(r)[1]
            full = O.splice_forward(sp["codes"], sp["Q"], sp["S"], cfg.hidden, c * L, L,
                                    np.zeros_like(ref[r]).reshape(-1, cfg.hidden), text)
            sl = np.asarray(sp["codes"]).reshape(-1, sp["S"])[:, c * L:(c + 1) * L].reshape(-1)
            full[sl >= 0] = np.nan
            b = drv.buf(r, hbb.SLOT_DST_ACT)
            b.copy_(torch.from_numpy(full.reshape(-1)).to(b.device).to(b.dtype).reshape(b.shape))
    ok = True
    worst = 0.0
    acc = {}
    for step in range(steps):
        # fresh gradients every step; source gradients accumulate (beta=1)
        vg = {}
        for r in dst.stage_ranks(0):
            t, c, p, d = dst.coord(r)
            n = (sp["Q"] * L * cfg.hidden) if sp else DI[d][1] * W
            # strict: every rank its own gradient (pins the tp=0 data path);
            # default: contract gradients, tp replicas of a (cp, dp) cell equal
            seed = 100 * step + (r if strict else 10 * c + d)
            g = bf16_round(np.random.default_rng(seed).standard_normal(n))
            gg = g
            if sp:
                gg = O.splice_backward(sp["codes"], sp["Q"], sp["S"], cfg.hidden, c * L, L,
                                       g.reshape(-1, cfg.hidden), DI[d][1] * cfg.tokens)
            vg[r] = gg.reshape(-1, W)
            if r in drv.local:
                b = drv.buf(r, hbb.SLOT_DST_GRAD)
                b.copy_(torch.from_numpy(g).to(b.device).to(torch.bfloat16).reshape(b.shape))
        if step == 0:
            for r in drv.local:
                b = drv.buf(r, hbb.SLOT_SRC_GRAD)
                if b is not None:
                    b.zero_()
            acc = {r: np.zeros(SI[src.coord(r)[3]][1] * W) for r in src.stage_ranks(src.pp - 1)}
        drv.sync()
        drv.fwd(step)
        drv.bwd(step, 1.0)
        drv.sync()
        if drv.status():
            raise RuntimeError("flag wait timed out")
        for r in drv.local:
            if r in ref:
                exp = ref[r]
                if sp:
                    c = dst.coord(r)[1]
                    exp = O.splice_forward(sp["codes"], sp["Q"], sp["S"], cfg.hidden, c * L, L,
                                           exp.reshape(-1, cfg.hidden), text)
                got = drv.buf(r, hbb.SLOT_DST_ACT).double().cpu().numpy().reshape(-1)
                ok &= bool(np.array_equal(got, exp.reshape(-1)))
        refb, _, _ = O.bridge_backward(src, dst, B, W, vg)
        for r in refb:
            acc[r] = acc[r] + refb[r].reshape(-1)
            if r in drv.local:
                got = drv.buf(r, hbb.SLOT_SRC_GRAD).double().cpu().numpy().reshape(-1)
                rel = float(np.max(np.abs(got - acc[r]) / np.maximum(1.0, np.abs(acc[r]))))
                worst = max(worst, rel)
                ok &= rel <= 1e-6
    return ok, worst


class LocalGroupDriver:
    """Adapter of a :class:`hbb.LocalGroup` (every rank readable)."""

    def __init__(self, group):
        self.g = group
        self.local = list(range(group.plan.world))

    def buf(self, r, slot):
        return self.g.buffer(r, slot)

    def fwd(self, mb):
        self.g.forward(mb)

    def bwd(self, mb, beta):
        self.g.backward(mb, beta)

    def sync(self):
        torch.cuda.synchronize()
        self.g.synchronize()

    def status(self):
        return self.g.status()


class ProcessDriver:
    """Adapter of one process's :class:`hbb.BridgeRuntime` in a torchrun group."""

    def __init__(self, rt, local):
        self.rt, self.local = rt, local

    def buf(self, r, slot):
        return self.rt.buffer(r, slot)

    def fwd(self, mb):
        self.rt.forward(mb)

    def bwd(self, mb, beta):
        self.rt.backward(mb, beta)

    def sync(self):
        import torch.distributed as dist

        torch.cuda.synchronize()
        dist.barrier()

    def status(self):
        return self.rt.status()


def row_width(cfg, slot):
    if cfg.splice and slot in (hbb.SLOT_DST_ACT, hbb.SLOT_DST_GRAD, hbb.SLOT_TEXT):
        return cfg.hidden
    return cfg.width


def bind_caller_buffers(bind, numel_of, cfg, ranks, device_of, dtype_of, pad=0):
    """Caller-owned buffers for every (rank, slot) in ``ranks``: [rows, W + pad]
    allocations bound through their [:, :W] view (row stride W + pad; pad=0:
    packed). Returns {(rank, slot): view}."""
    out = {}
    for r in ranks:
        for slot in (hbb.SLOT_SRC_ACT, hbb.SLOT_DST_ACT, hbb.SLOT_DST_GRAD, hbb.SLOT_SRC_GRAD, hbb.SLOT_TEXT):
            n = numel_of(r, slot)
            if not n:
                continue
            w = row_width(cfg, slot)
            full = torch.full((n // w, w + pad), float("nan"), dtype=dtype_of(slot), device=device_of(r))
            v = full[:, :w]
            bind(r, slot, v)
            out[(r, slot)] = v
    return out


def config(name, scale=64):
    return configs.get(name, scale=scale)
