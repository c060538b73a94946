"""The informative all-core CPU executor (oracle/direct_cpu.py) that
bench.py reports next to the oracle baseline: same results as the oracle."""
import numpy as np
import pytest

from helpers import O, hb_plan, hbb
from oracle import direct_cpu


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bits."""
    u = x.astype(np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def bits_to_f64(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


@pytest.mark.parametrize("src,dst", [
    (O.Layout("vit", dp=8), O.Layout("llm", tp=4, dp=2)),          # C2 fan-in
    (O.Layout("enc", tp=4, dp=2), O.Layout("llm", dp=8)),          # C3 fan-out
    (O.Layout("vit", dp=2), O.Layout("llm", tp=2, pp=3, rank_offset=2)),  # C5 non-colocated
])
def test_direct_executor_matches_oracle(src, dst):
    B, W = 16, 24
    plan = hb_plan(src, dst, B, W)
    rng = np.random.default_rng(5)
    SI, DI = O.intervals(B, src.dp), O.intervals(B, dst.dp)
    X = bf16_bits(rng.standard_normal((B, W)))
    G = bf16_bits(rng.standard_normal((B, W)))
    bufs = {}
    shards, grads = {}, {}
    for r in src.stage_ranks(src.pp - 1):
        a, n = SI[src.coord(r)[3]]
        bufs[(r, hbb.SLOT_SRC_ACT)] = X[a:a + n].reshape(-1).copy()
        shards[r] = bits_to_f64(X[a:a + n])
        bufs[(r, hbb.SLOT_SRC_GRAD)] = np.zeros(n * W, dtype=np.float32)
    for r in dst.stage_ranks(0):
        a, n = DI[dst.coord(r)[3]]
        bufs[(r, hbb.SLOT_DST_ACT)] = np.zeros(n * W, dtype=np.uint16)
        bufs[(r, hbb.SLOT_DST_GRAD)] = G[a:a + n].reshape(-1).copy()
        grads[r] = bits_to_f64(G[a:a + n])
    sec, threads = direct_cpu.run(hbb.index_forward(plan), hbb.index_backward(plan, balanced=True), bufs,
                                  beta=0.0, repeats=1)
    assert sec > 0 and threads >= 1
    fwd, _, _ = O.bridge_forward(src, dst, B, W, shards)
    for r, a in fwd.items():
        np.testing.assert_array_equal(bits_to_f64(bufs[(r, hbb.SLOT_DST_ACT)]), a.reshape(-1))
    bwd, _, _ = O.bridge_backward(src, dst, B, W, grads)
    for r, a in bwd.items():
        got = bufs[(r, hbb.SLOT_SRC_GRAD)].astype(np.float64)
        np.testing.assert_allclose(got, a.reshape(-1), rtol=0, atol=1e-6 * max(1.0, np.abs(a).max()))
