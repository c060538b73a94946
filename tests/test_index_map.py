"""Ownership index builder (csrc/hb/index_map.cpp) vs the oracle, on CPU.

A numpy executor applies the product's forward copy map and backward
sum map (tests/helpers.py) and must reproduce the oracle's whole-edge
bridge_forward / bridge_backward (and the splice composition) — exactly for
placement, to double rounding for sums. Replica inputs are perturbed so the
check also pins which replica's copy each route reads.
"""
import itertools

import numpy as np
import pytest

from helpers import O, apply_backward, apply_forward, dest_grads, hb_plan, hbb, source_shards
from paper_2605_27678_b200 import configs


def check_plain(src, dst, B, W, seed=0):
    rng = np.random.default_rng(seed)
    plan = hb_plan(src, dst, B, W)
    sh = source_shards(src, B, W, rng)
    ref, _, _ = O.bridge_forward(src, dst, B, W, sh)
    got = apply_forward(plan, {(r, hbb.SLOT_SRC_ACT): a.reshape(-1) for r, a in sh.items()})
    assert {k[0] for k in got} == set(ref)
    for r, a in ref.items():
        np.testing.assert_array_equal(got[(r, hbb.SLOT_DST_ACT)], a.reshape(-1))
    g = dest_grads(dst, B, W, rng)
    refb, _, _ = O.bridge_backward(src, dst, B, W, g)
    gotb = apply_backward(plan, {(r, hbb.SLOT_DST_GRAD): a.reshape(-1) for r, a in g.items()})
    assert {k[0] for k in gotb} == set(refb)
    for r, a in refb.items():
        np.testing.assert_allclose(gotb[(r, hbb.SLOT_SRC_GRAD)], a.reshape(-1), rtol=0, atol=1e-12)
    # the runtime's default map (terms from the holder's tp replicas in turn) on
    # gradients that honour the tp-replica contract
    gc = dest_grads(dst, B, W, rng, contract=True)
    refc, _, _ = O.bridge_backward(src, dst, B, W, gc)
    gotc = apply_backward(plan, {(r, hbb.SLOT_DST_GRAD): a.reshape(-1) for r, a in gc.items()}, balanced=True)
    for r, a in refc.items():
        np.testing.assert_allclose(gotc[(r, hbb.SLOT_SRC_GRAD)], a.reshape(-1), rtol=0, atol=1e-12)


def test_sweep_vs_oracle():
    n = 0
    for stp, spp, sdp in itertools.product((1, 2), (1, 2), (1, 2, 4)):
        for dtp, dcp, dpp, ddp in itertools.product((1, 2), (1, 2), (1, 2), (1, 2, 4)):
            s = O.Layout("enc", stp, 1, spp, sdp, 0)
            for colo in (True, False):
                d = O.Layout("llm", dtp, dcp, dpp, ddp, 0 if colo else s.world_size)
                if colo and s.world_size != d.world_size:
                    continue
                try:
                    hb_plan(s, d, 8, 3)
                except hbb.HetBridgeError:
                    continue
                check_plain(s, d, 8, 3, seed=n)
                n += 1
    assert n > 300


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c5"])
def test_baseline_configs_scaled(name):
    cfg = configs.get(name, scale=512)
    s = O.Layout(cfg.src.name, cfg.src.tp, cfg.src.cp, cfg.src.pp, cfg.src.dp, cfg.src.rank_offset)
    d = O.Layout(cfg.dst.name, cfg.dst.tp, cfg.dst.cp, cfg.dst.pp, cfg.dst.dp, cfg.dst.rank_offset)
    check_plain(s, d, cfg.batch, 5)


def splice_case(src, dst, B, S_v, d_h, Q, S, codes, text_mode, seed=0):
    rng = np.random.default_rng(seed)
    W = S_v * d_h
    plan = hb_plan(src, dst, B, W)
    sp = hbb.SpliceSpec(Q, S, d_h, S_v, codes, text_mode)
    sh = source_shards(src, B, W, rng)
    fwd, _, _ = O.bridge_forward(src, dst, B, W, sh)
    text = rng.standard_normal((int((np.asarray(codes) < 0).sum()), d_h))
    L = S // dst.cp
    bufs = {(r, hbb.SLOT_SRC_ACT): a.reshape(-1) for r, a in sh.items()}
    for r in dst.stage_ranks(0):
        c = dst.coord(r)[1]
        if text_mode == hbb.TEXT_SLICE:
            sl = np.asarray(codes).reshape(Q, S)[:, c * L:(c + 1) * L].reshape(-1)
            bufs[(r, hbb.SLOT_TEXT)] = text[[-1 - int(x) for x in sl if x < 0]].reshape(-1)
        else:
            bufs[(r, hbb.SLOT_TEXT)] = text.reshape(-1)
    got = apply_forward(plan, bufs, sp)
    for r in dst.stage_ranks(0):
        c = dst.coord(r)[1]
        exp = O.splice_forward(codes, Q, S, d_h, c * L, L, fwd[r].reshape(-1, d_h), text)
        np.testing.assert_array_equal(got[(r, hbb.SLOT_DST_ACT)], exp.reshape(-1))
    tg = {r: rng.standard_normal((Q * L, d_h)) for r in dst.stage_ranks(0)}
    vrows = (B // dst.dp) * S_v
    vg = {r: O.splice_backward(codes, Q, S, d_h, dst.coord(r)[1] * L, L, tg[r], vrows).reshape(-1, W)
          for r in dst.stage_ranks(0)}
    refb, _, _ = O.bridge_backward(src, dst, B, W, vg)
    gotb = apply_backward(plan, {(r, hbb.SLOT_DST_GRAD): a.reshape(-1) for r, a in tg.items()}, sp)
    for r, a in refb.items():
        np.testing.assert_array_equal(gotb[(r, hbb.SLOT_SRC_GRAD)], a.reshape(-1))
    # balanced map on contract gradients: tp replicas of a (cp, dp) cell identical
    cell = {}
    tc = {}
    for r in dst.stage_ranks(0):
        t, c, p, d = dst.coord(r)
        if (c, d) not in cell:
            cell[(c, d)] = rng.standard_normal((Q * L, d_h))
        tc[r] = cell[(c, d)]
    vc = {r: O.splice_backward(codes, Q, S, d_h, dst.coord(r)[1] * L, L, tc[r], vrows).reshape(-1, W)
          for r in dst.stage_ranks(0)}
    refc, _, _ = O.bridge_backward(src, dst, B, W, vc)
    gotc = apply_backward(plan, {(r, hbb.SLOT_DST_GRAD): a.reshape(-1) for r, a in tc.items()}, sp, balanced=True)
    for r, a in refc.items():
        np.testing.assert_array_equal(gotc[(r, hbb.SLOT_SRC_GRAD)], a.reshape(-1))


@pytest.mark.parametrize("text_mode", [0, 1])
def test_c4_fused_sequence_splice(text_mode):
    cfg = configs.get("c4", scale=256)
    s, d = O.Layout("vit", dp=8), O.Layout("llm", tp=2, cp=4)
    sp = cfg.splice
    splice_case(s, d, cfg.batch, cfg.tokens, 8, 1, sp["S"], sp["codes"], text_mode)


def test_reference_layout_splice():
    s, d = O.Layout("enc", dp=4), O.Layout("llm", cp=2, dp=2)
    n, S, S_v = 4, 10, 3
    q = np.arange(n)[:, None]
    p = np.arange(S)[None, :]
    codes = np.where(p < S_v, q * S_v + p, -1 - (q * (S - S_v) + (p - S_v)))
    splice_case(s, d, 8, S_v, 4, n, S, codes.reshape(-1), 0)


def test_nc_splice_with_cp_and_tp():
    s, d = O.Layout("enc", dp=2), O.Layout("llm", tp=2, cp=2, rank_offset=2)
    B, S, S_v = 4, 12, 2
    q = np.arange(B)[:, None]
    p = np.arange(S)[None, :]
    codes = np.where(p < S_v, q * S_v + p, -1 - (q * (S - S_v) + (p - S_v)))
    splice_case(s, d, B, S_v, 4, B, S, codes.reshape(-1), 0)


def test_segments_coalesce_to_shard_pieces():
    """C2: every destination rank materialises 4 contiguous source shards -> 4 segments each;
    backward: one select segment per source rank."""
    cfg = configs.get("c2")
    plan = hbb.plan_bridge(cfg.edge())
    fwd = hbb.index_forward(plan)
    assert len(fwd) == 32
    assert all(n == 8 * cfg.width for *_, n in fwd)
    bwd = hbb.index_backward(plan)
    assert len(bwd) == 8 and all(len(t) == 1 for *_, t in bwd)


def test_c4_index_is_row_granular_and_single_term():
    cfg = configs.get("c4")
    sp = hbb.SpliceSpec(cfg.splice["Q"], cfg.splice["S"], cfg.hidden, cfg.tokens, cfg.splice["codes"],
                        cfg.splice["text_mode"])
    plan = hbb.plan_bridge(cfg.edge())
    bwd = hbb.index_backward(plan, sp)
    assert all(len(t) == 1 for *_, t in bwd)  # each vision token lives in exactly one cp slice
    assert sum(n for _, _, _, n, _ in bwd) == cfg.batch * cfg.width
    fwd = hbb.index_forward(plan, sp)
    per_rank = {}
    for (_, _, _, dr, _, _, n) in fwd:
        per_rank[dr] = per_rank.get(dr, 0) + n
    assert all(v == cfg.splice["S"] // 4 * cfg.hidden for v in per_rank.values())


def test_fault_injection_detected():
    """corrupting one fan-in backward interval must fail parity."""
    src, dst = O.Layout("enc", dp=4), O.Layout("llm", tp=2, dp=2, rank_offset=4)
    B, W = 8, 3
    rng = np.random.default_rng(0)
    plan = hb_plan(src, dst, B, W)
    g = dest_grads(dst, B, W, rng, perturb_replicas=False)
    refb, _, _ = O.bridge_backward(src, dst, B, W, g)
    segs = hbb.index_backward(plan)
    bufs = {(r, hbb.SLOT_DST_GRAD): a.reshape(-1) for r, a in g.items()}
    dr, ds, do, n, terms = segs[1]
    bad = [(terms[0][0], terms[0][1], (terms[0][2] + n) % (4 * W))]  # wrong recorded interval
    out = np.zeros(n)
    for (r, s, o) in bad:
        out += bufs[(r, s)][o:o + n]
    assert not np.array_equal(out, refb[dr].reshape(-1)[do:do + n])


def test_splice_spec_validation():
    plan = hb_plan(O.Layout("enc", dp=2), O.Layout("llm", cp=2), 2, 6)
    with pytest.raises(hbb.HetBridgeError) as ei:  # duplicate vision row
        hbb.index_forward(plan, hbb.SpliceSpec(1, 4, 3, 2, [0, 0, -1, -2]))
    assert ei.value.code == "InvalidArgument"
    with pytest.raises(hbb.HetBridgeError) as ei:  # width != S_v * d_h
        hbb.index_forward(plan, hbb.SpliceSpec(1, 4, 2, 2, [0, 1, -1, -2]))
    assert ei.value.code == "ShapeMismatch"
    with pytest.raises(hbb.HetBridgeError) as ei:  # S % cp
        hbb.index_forward(plan, hbb.SpliceSpec(1, 3, 3, 2, [0, 1, -1]))
    assert ei.value.code == "DivisibilityViolation"


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_balanced_backward_spreads_serving_ranks(name):
    """Default runtime map: the gradient return of a tp>1 destination is served
    by every tp replica, not only tp=0 (the reference reads tp=0 only)."""
    cfg = configs.get(name, scale=256)
    plan = hbb.plan_bridge(cfg.edge())
    sp = None
    if cfg.splice:
        s = cfg.splice
        sp = hbb.SpliceSpec(s["Q"], s["S"], cfg.hidden, cfg.tokens, s["codes"], s["text_mode"])
    def served(balanced):
        load = {}
        for (_, _, _, n, terms) in hbb.index_backward(plan, sp, balanced):
            for (r, _, _) in terms:
                load[r] = load.get(r, 0) + n
        return load
    strict, bal = served(False), served(True)
    assert sum(strict.values()) == sum(bal.values())
    tp0 = {r for r in strict}
    assert all(plan_coord_tp(cfg.dst, r) == 0 for r in tp0)
    assert len(bal) == cfg.dst.tp * len(strict)
    assert max(bal.values()) <= 0.6 * max(strict.values())


def plan_coord_tp(layout, r):
    from paper_2605_27678_b200 import grid as hbg
    return hbg.coord_of_rank(layout, r).tp_idx


def random_codes(rng, n_vis_rows, Q, S):
    """A placeholder table with every vision row of the shard at a random position
    (images split across sequences and CP slices, tokens out of order) and text
    rows numbered in position order elsewhere."""
    pos = rng.choice(Q * S, size=n_vis_rows, replace=False)
    codes = np.full(Q * S, 0, dtype=np.int64)
    vis = np.zeros(Q * S, dtype=bool)
    vis[pos] = True
    codes[pos] = rng.permutation(n_vis_rows)
    text_idx = np.cumsum(~vis) - 1
    codes[~vis] = -1 - text_idx[~vis]
    return codes.astype(np.int32)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("text_mode", [0, 1])
def test_random_placeholder_tables(seed, text_mode):
    """Scattered vision tokens: runs break at every discontinuity, slices start and
    end mid-image; placement stays bit-exact and the gradient return exact."""
    rng = np.random.default_rng(100 + seed)
    s = [O.Layout("vit", dp=4), O.Layout("vit", tp=2, dp=2), O.Layout("vit", dp=8)][seed % 3]
    d = [O.Layout("llm", tp=2, cp=2), O.Layout("llm", cp=4), O.Layout("llm", tp=2, cp=2, dp=2)][seed % 3]
    B, S_v, d_h = 8, 3, 2
    Q = 2
    S = 8 * d.cp
    n_vis = (B // d.dp) * S_v
    codes = random_codes(rng, n_vis, Q, S)
    splice_case(s, d, B, S_v, d_h, Q, S, codes, text_mode, seed=seed)


@pytest.mark.parametrize("name", ["c4", "c4w4"])
def test_in_place_splice_writes_only_vision_rows(name):
    """HB_TEXT_INPLACE: the forward map is the copy splice's map without its text
    runs (the caller's embedding layer wrote those rows), the TEXT buffer is
    gone, and the backward map is unchanged."""
    base = configs.get(name, scale=64)
    ip = configs.get(name, scale=64)
    ip.splice = dict(ip.splice, text_mode=hbb.TEXT_INPLACE)
    plan = hbb.plan_bridge(base.edge())

    def spec(cfg):
        s = cfg.splice
        return hbb.SpliceSpec(s["Q"], s["S"], cfg.hidden, cfg.tokens, s["codes"], s["text_mode"])

    f_copy, f_ip = hbb.index_forward(plan, spec(base)), hbb.index_forward(plan, spec(ip))
    assert all(s[1] != hbb.SLOT_TEXT for s in f_ip)
    # same vision placements (runs may coalesce differently once text runs are gone)
    def cover(fm):
        out = set()
        for (sr, ss, so, dr, ds, do, n) in fm:
            if ss == hbb.SLOT_TEXT:
                continue
            for k in range(0, n, base.hidden):
                out.add((sr, ss, so + k, dr, ds, do + k))
        return out
    assert cover(f_ip) == cover(f_copy)
    assert any(s[1] == hbb.SLOT_TEXT for s in f_copy)
    for r in range(plan.world):
        assert hbb.buffer_elems(plan, r, hbb.SLOT_TEXT, spec(ip)) == 0
        assert hbb.buffer_elems(plan, r, hbb.SLOT_DST_ACT, spec(ip)) == hbb.buffer_elems(plan, r, hbb.SLOT_DST_ACT,
                                                                                         spec(base))
    assert hbb.index_backward(plan, spec(ip)) == hbb.index_backward(plan, spec(base))
