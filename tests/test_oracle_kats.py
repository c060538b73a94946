"""Pins the oracle itself: the SPEC.md prose known-answer tests for the bridge
and splice made executable
against the oracle restatement running over the reference simnet/grid."""
import itertools

import numpy as np
import pytest

from helpers import O, dest_grads, source_shards


def test_fan_in_forward_kat():
    """fan-in 2, B=8, W=3: dest shard 0 = rows 0..3 of the global tensor, in order."""
    X = np.arange(24, dtype=float).reshape(8, 3)
    for dst in (O.Layout("llm", dp=2, rank_offset=4), O.Layout("llm", tp=2, dp=2, rank_offset=4)):
        src = O.Layout("enc", dp=4)
        out, led, _ = O.bridge_forward(src, dst, 8, 3, {r: X[2 * r:2 * r + 2] for r in range(4)})
        for r in dst.stage_ranks(0):
            d = dst.coord(r)[3]
            np.testing.assert_array_equal(out[r], X[4 * d:4 * d + 4])
        # fan-in fwd boundary bytes = 8 rows * 3 * 8 B = 192
        assert led[("enc->llm/fwd/send", "forward")] == (4, 192)


def test_fan_in_colocated_forward():
    src, dst = O.Layout("enc", dp=4), O.Layout("llm", dp=2, tp=2)
    X = np.arange(24, dtype=float).reshape(8, 3)
    out, led, _ = O.bridge_forward(src, dst, 8, 3, {r: X[2 * r:2 * r + 2] for r in range(4)})
    for r in range(4):
        np.testing.assert_array_equal(out[r], X[4 * (r // 2):4 * (r // 2) + 4])
    gathers = {k: v for k, v in led.items() if "all_gather" in k[0]}
    assert all(m == 2 for m, _ in gathers.values())  # 2-member groups: n(n-1) = 2 messages


def test_fan_out_nc_forward_one_message_per_dest_leader():
    """fan-out 2 NC: each dest leader receives exactly one message of (B/DP_v)*W elements."""
    src, dst = O.Layout("enc", dp=2), O.Layout("llm", dp=4, rank_offset=2)
    X = np.arange(24, dtype=float).reshape(8, 3)
    out, led, _ = O.bridge_forward(src, dst, 8, 3, {0: X[:4], 1: X[4:]})
    assert led[("enc->llm/fwd/send", "forward")] == (4, 4 * 2 * 3 * 8)
    for r in range(2, 6):
        np.testing.assert_array_equal(out[r], X[2 * (r - 2):2 * (r - 2) + 2])


def test_fan_in_backward_split_kat():
    """fan-in 2: dest grad [0,4) splits [0,2) -> src dp0, [2,4) -> src dp1."""
    src, dst = O.Layout("enc", dp=4), O.Layout("llm", dp=2, rank_offset=4)
    G = np.arange(24, dtype=float).reshape(8, 3) * 0.5
    out, _, _ = O.bridge_backward(src, dst, 8, 3, {4: G[:4], 5: G[4:]})
    for r in range(4):
        np.testing.assert_array_equal(out[r], G[2 * r:2 * r + 2])


def test_fan_out_colocated_backward_gathers_siblings():
    """fan-out 2 colocated: source rank rebuilds its [0,4) grad from two sibling intervals."""
    src, dst = O.Layout("enc", tp=2, dp=2), O.Layout("llm", dp=4)
    G = np.arange(24, dtype=float).reshape(8, 3)
    out, led, _ = O.bridge_backward(src, dst, 8, 3, {r: G[2 * r:2 * r + 2] for r in range(4)})
    for r in range(4):
        s = src.coord(r)[3]
        np.testing.assert_array_equal(out[r], G[4 * s:4 * s + 4])
    assert any("bwd/all_gather" in k[0] for k in led)


def test_equal_dp_colocated_identity_and_zero_messages():
    src, dst = O.Layout("enc", dp=4), O.Layout("llm", dp=4)
    rng = np.random.default_rng(0)
    sh = {r: rng.standard_normal((2, 5)) for r in range(4)}
    out, led, _ = O.bridge_forward(src, dst, 8, 5, sh)
    for r in range(4):
        np.testing.assert_array_equal(out[r], sh[r])
    assert sum(m for m, _ in led.values()) == 0


LAYOUT_SWEEP = [
    (O.Layout("enc", dp=4), O.Layout("llm", tp=2, dp=2, rank_offset=4)),
    (O.Layout("enc", tp=2, dp=2), O.Layout("llm", dp=8, rank_offset=4)),
    (O.Layout("enc", dp=2), O.Layout("llm", tp=2, cp=2, pp=2, rank_offset=2)),
    (O.Layout("enc", dp=8), O.Layout("llm", tp=4, dp=2)),
    (O.Layout("enc", tp=4, dp=2), O.Layout("llm", dp=8)),
    (O.Layout("enc", dp=8), O.Layout("llm", tp=2, cp=4)),
    (O.Layout("enc", pp=4, dp=2), O.Layout("llm", dp=8)),
    (O.Layout("vision", tp=4, dp=2), O.Layout("language", tp=2, pp=2, dp=2)),
]


@pytest.mark.parametrize("src,dst", LAYOUT_SWEEP)
def test_round_trip_ownership_and_conservation(src, dst):
    """after fwd then bwd with grad := output, every source owner gets exactly its
    own interval back (identity), and payload is conserved in both directions."""
    B, W = 16, 4
    rng = np.random.default_rng(1)
    sh = source_shards(src, B, W, rng, perturb_replicas=False)
    out, _, _ = O.bridge_forward(src, dst, B, W, sh)
    assert sum(a.size for a in out.values()) == B * W * len(dst.stage_ranks(0)) // dst.dp
    grads = {r: a.copy() for r, a in out.items()}
    if dst.cp > 1:  # cp replicas are summed: give the contribution to cp=0 only
        for r in grads:
            if dst.coord(r)[1]:
                grads[r][:] = 0.0
    back, _, _ = O.bridge_backward(src, dst, B, W, grads)
    assert set(back) == set(sh)
    for r in sh:
        np.testing.assert_array_equal(back[r], sh[r])


def test_nc_message_count_is_max_dp():
    """cross-boundary messages = max(DP_u, DP_v) per direction."""
    for du, dv in itertools.product((1, 2, 4), repeat=2):
        src, dst = O.Layout("enc", dp=du), O.Layout("llm", tp=2, dp=dv, rank_offset=du)
        sh = {r: np.zeros((8 // du, 2)) for r in range(du)}
        _, led, _ = O.bridge_forward(src, dst, 8, 2, sh)
        assert led[("enc->llm/fwd/send", "forward")][0] == max(du, dv)
        assert O.cross_boundary_messages(src, dst, 8) == max(du, dv)


def test_tp_replica_grads_ignored_cp_summed():
    """bridge.hpp:33-36: tp replicas hand back identical grads (only tp=0 read), cp replicas summed."""
    src, dst = O.Layout("enc", dp=2), O.Layout("llm", tp=2, cp=2, rank_offset=2)
    B, W = 4, 3
    g = {}
    for r in dst.stage_ranks(0):
        t, c, p, d = dst.coord(r)
        g[r] = np.full((4, 3), 1.0 + 10 * c + 100 * t)
    out, led, _ = O.bridge_backward(src, dst, B, W, g)
    for r in (0, 1):
        np.testing.assert_array_equal(out[r], np.full((2, 3), 1.0 + 11.0))
    assert any("all_reduce" in k[0] for k in led)


def test_determinism_of_ledgers():
    src, dst = O.Layout("enc", dp=8), O.Layout("llm", tp=2, cp=4)
    rng = np.random.default_rng(3)
    sh = source_shards(src, 16, 4, rng)
    a = O.bridge_forward(src, dst, 16, 4, sh)
    b = O.bridge_forward(src, dst, 16, 4, sh)
    assert a[1] == b[1]
    for r in a[0]:
        np.testing.assert_array_equal(a[0][r], b[0][r])


def test_missing_leader_shard():
    src, dst = O.Layout("enc", dp=2), O.Layout("llm", dp=2, rank_offset=2)
    with pytest.raises(O.OracleError) as ei:
        O.bridge_forward(src, dst, 4, 2, {0: np.zeros((2, 2))})
    assert O.error_name(ei.value.code) == "MissingSourceShard"


# ---- splice (tinymodel.hpp:94-112)
def test_cp_token_slice():
    assert [O.cp_token_slice(12, 3, c) for c in range(3)] == [(0, 4), (4, 4), (8, 4)]
    with pytest.raises(O.OracleError) as ei:
        O.cp_token_slice(10, 4, 0)
    assert O.error_name(ei.value.code) == "DivisibilityViolation"


def test_assemble_tokens_reference_layout():
    """Vision tokens at [0,S_v), text at the rest; only slice positions materialised."""
    S, S_v, d_h, n = 6, 2, 3, 2
    vis = np.arange(n * S_v * d_h, dtype=float).reshape(n, S_v * d_h) + 100
    txt = np.arange(n * (S - S_v) * d_h, dtype=float).reshape(n, (S - S_v) * d_h) + 500
    for c in range(2):
        out = O.assemble_tokens(S, S_v, d_h, vis, txt, 3 * c, 3)
        for q in range(n):
            for i, p in enumerate(range(3 * c, 3 * c + 3)):
                exp = vis[q].reshape(S_v, d_h)[p] if p < S_v else txt[q].reshape(S - S_v, d_h)[p - S_v]
                np.testing.assert_array_equal(out[q * 3 + i], exp)


def test_split_vision_grad_zeros_outside_slice_and_sum_over_cp():
    S, S_v, d_h, n, cp = 8, 3, 2, 2, 4
    L = S // cp
    rng = np.random.default_rng(0)
    tok = [rng.standard_normal((n * L, d_h)) for _ in range(cp)]
    parts = [O.split_vision_grad(S, S_v, d_h, n, tok[c], c * L, L) for c in range(cp)]
    total = sum(parts)
    for q in range(n):
        for p in range(S_v):
            c = p // L
            np.testing.assert_array_equal(total[q].reshape(S_v, d_h)[p], tok[c][q * L + p - c * L])
            for c2 in range(cp):
                if c2 != c:
                    assert not parts[c2][q].reshape(S_v, d_h)[p].any()


def test_generalised_splice_equals_reference_special_case():
    S, S_v, d_h, n = 10, 4, 3, 3
    rng = np.random.default_rng(2)
    vis = rng.standard_normal((n, S_v * d_h))
    txt = rng.standard_normal((n, (S - S_v) * d_h))
    q = np.arange(n)[:, None]
    p = np.arange(S)[None, :]
    codes = np.where(p < S_v, q * S_v + p, -1 - (q * (S - S_v) + (p - S_v)))
    for st, ln in ((0, 5), (5, 5), (0, 10)):
        a = O.assemble_tokens(S, S_v, d_h, vis, txt, st, ln)
        b = O.splice_forward(codes, n, S, d_h, st, ln, vis.reshape(-1, d_h), txt.reshape(-1, d_h))
        np.testing.assert_array_equal(a, b)
        g = rng.standard_normal((n * ln, d_h))
        np.testing.assert_array_equal(O.split_vision_grad(S, S_v, d_h, n, g, st, ln).reshape(-1, d_h),
                                      O.splice_backward(codes, n, S, d_h, st, ln, g, n * S_v))


def test_reference_gaussian_stream_is_deterministic():
    a = O.gaussian(1234, "bnd/s0", 16)
    b = O.gaussian(1234, "bnd/s0", 16)
    c = O.gaussian(1234, "bnd/s1", 16)
    np.testing.assert_array_equal(a, b)
    assert not np.array_equal(a, c)
    assert abs(O.gaussian(7, "x", 20000).std() - 1.0) < 0.05
