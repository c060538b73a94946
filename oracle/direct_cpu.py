"""ORACLE-side CPU baseline — test/bench infrastructure only, never the product.

The "direct CPU executor" of SURVEY §8(d): the boundary's forward copies and
backward sum-accumulates executed straight from an ownership index map on the
host, over all cores (numpy slices in a thread pool; numpy releases the GIL for
the copies and the ufuncs). It is an informative upper bound for a CPU
implementation of the path. The reference's own CPU path is the oracle over
simnet (one runnable rank at a time, so one core). bench.py reports it next to
that in `cpu_baseline.direct`.

Layout: bf16 tensors are uint16 arrays of bf16 bits; accumulators are float32.
"""
from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

PIECE = 1 << 20  # elements per work item


def _bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    return (u16.astype(np.uint32) << 16).view(np.float32)


def _pieces_fwd(fwd_map):
    for (sr, ss, so, dr, ds, do, n) in fwd_map:
        for a in range(0, n, PIECE):
            b = min(n, a + PIECE)
            yield (sr, ss, so + a, dr, ds, do + a, b - a)


def _pieces_bwd(bwd_map):
    for (dr, ds, do, n, terms) in bwd_map:
        for a in range(0, n, PIECE):
            b = min(n, a + PIECE)
            yield (dr, ds, do + a, b - a, [(tr, ts, to + a) for (tr, ts, to) in terms])


def run(fwd_map, bwd_map, bufs: dict, beta: float = 1.0, threads: int | None = None, repeats: int = 2):
    """Execute forward then backward `repeats` times; returns (best seconds, threads).

    bufs[(rank, slot)]: 1-D arrays (uint16 bf16 bits for copies and gradient
    terms, float32 for the accumulators). Terms are summed in order from +0.0 in
    fp32, then accumulated as beta*dst + sum, as the device kernels do."""
    threads = threads or os.cpu_count() or 1
    fw = list(_pieces_fwd(fwd_map))
    bw = list(_pieces_bwd(bwd_map))

    def copy(p):
        sr, ss, so, dr, ds, do, n = p
        bufs[(dr, ds)][do:do + n] = bufs[(sr, ss)][so:so + n]

    def reduce(p):
        dr, ds, do, n, terms = p
        acc = np.zeros(n, dtype=np.float32)
        for (tr, ts, to) in terms:
            acc += _bf16_to_f32(bufs[(tr, ts)][to:to + n])
        dst = bufs[(dr, ds)][do:do + n]
        if beta:
            dst *= np.float32(beta)
            dst += acc
        else:
            dst[:] = acc

    best = float("inf")
    with ThreadPoolExecutor(max_workers=threads) as ex:
        for _ in range(repeats):
            t0 = time.perf_counter()
            list(ex.map(copy, fw))
            list(ex.map(reduce, bw))
            best = min(best, time.perf_counter() - t0)
    return best, threads
