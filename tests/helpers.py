"""Test-side helpers: layouts of the BASELINE configs, seeded inputs, and a
numpy executor of the product's index maps (used only to check the index
builder on CPU against the oracle; the device path is tested in -m gpu)."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2605_27678_b200 import bridge as hbb  # noqa: E402
from paper_2605_27678_b200 import grid as hbg  # noqa: E402


def to_hb(l: O.Layout) -> hbg.ModuleLayout:
    return hbg.ModuleLayout(l.name, l.tp, l.cp, l.pp, l.dp, l.rank_offset)


def hb_plan(src: O.Layout, dst: O.Layout, B: int, W: int):
    return hbb.plan_bridge(hbg.BoundaryEdge(to_hb(src), to_hb(dst), B, W))


def source_shards(src: O.Layout, B: int, W: int, rng, perturb_replicas=True, dtype=np.float64):
    """One array per source last-stage rank. Replicas of a shard get identical
    values unless perturb_replicas (then non-leader replicas differ, which
    exercises exactly which replica's copy the data path reads)."""
    X = rng.standard_normal((B, W))
    SI = O.intervals(B, src.dp)
    out = {}
    for r in src.stage_ranks(src.pp - 1):
        t, c, p, d = src.coord(r)
        st, n = SI[d]
        a = X[st:st + n].copy()
        if perturb_replicas and (t or c):
            a += 1000.0 * (t + 1) + 100.0 * (c + 1)
        out[r] = a.astype(dtype)
    return out


def dest_grads(dst: O.Layout, B: int, W: int, rng, perturb_replicas=True, contract=False):
    """contract=True: gradients that honour bridge.hpp:33-36 — tp replicas of a
    (cp, dp) cell identical, cp replicas different (they are summed)."""
    G = rng.standard_normal((B, W))
    DI = O.intervals(B, dst.dp)
    out = {}
    for r in dst.stage_ranks(0):
        t, c, p, d = dst.coord(r)
        st, n = DI[d]
        a = G[st:st + n].copy()
        if contract:
            a += 100.0 * c
        elif perturb_replicas and (t or c):
            a += 1000.0 * (t + 1) + 100.0 * (c + 1)
        out[r] = a
    return out


def apply_forward(plan, bufs: dict, splice=None):
    """Execute the forward index map on numpy buffers {(rank, slot): 1-D array}."""
    out = {}
    for (sr, ss, so, dr, ds, do, n) in hbb.index_forward(plan, splice):
        key = (dr, ds)
        if key not in out:
            out[key] = np.full(hbb.buffer_elems(plan, dr, ds, splice), np.nan)
        out[key][do:do + n] = bufs[(sr, ss)][so:so + n]
    return out


def apply_backward(plan, bufs: dict, splice=None, prev: dict | None = None, beta=0.0, balanced=False):
    out = {}
    for (dr, ds, do, n, terms) in hbb.index_backward(plan, splice, balanced):
        key = (dr, ds)
        if key not in out:
            out[key] = np.full(hbb.buffer_elems(plan, dr, ds, splice), np.nan)
        acc = np.zeros(n)
        for (r, s, o) in terms:
            acc = acc + bufs[(r, s)][o:o + n]
        if beta:
            acc = beta * prev[key][do:do + n] + acc
        out[key][do:do + n] = acc
    return out
