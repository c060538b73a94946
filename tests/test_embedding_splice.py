"""Text-embedding lookup fused into the CP splice (
tinymodel.hpp:97-101 builds the fused sequence from text embeddings and vision
rows). With ``text_embedding=True`` the TEXT slot holds int32 token ids and the
forward gathers each text row from the embedding table; the result must be
bit-identical to splicing the pre-embedded rows table[ids]."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from helpers import hbb  # noqa: E402

from paper_2605_27678_b200 import configs  # noqa: E402


def _spec(cfg):
    s = cfg.splice
    return hbb.SpliceSpec(s["Q"], s["S"], cfg.hidden, cfg.tokens, s["codes"], s["text_mode"])


@pytest.mark.parametrize("partition", [0, 1, 3])
def test_embedding_gather_equals_pre_embedded_text(partition):
    cfg = configs.get("c4", scale=64)
    plan = hbb.plan_bridge(cfg.edge())
    sp = _spec(cfg)
    vocab, d_h = 997, cfg.hidden
    table = torch.randn(vocab, d_h, device="cuda").to(torch.bfloat16)
    rt_e = hbb.BridgeRuntime(plan, sp, text_embedding=True, partition=partition)
    rt_p = hbb.BridgeRuntime(plan, sp, partition=partition)
    rt_e.set_text_embedding(table)
    g = torch.Generator(device="cuda").manual_seed(3)
    for r in rt_e.local_ranks(hbb.SLOT_SRC_ACT):
        x = torch.randn(rt_e.buffer_numel(r, hbb.SLOT_SRC_ACT), device="cuda", generator=g).to(torch.bfloat16)
        rt_e.buffer(r, hbb.SLOT_SRC_ACT).copy_(x)
        rt_p.buffer(r, hbb.SLOT_SRC_ACT).copy_(x)
    for r in rt_e.local_ranks(hbb.SLOT_TEXT):
        ids_buf = rt_e.buffer(r, hbb.SLOT_TEXT)
        assert ids_buf.dtype == torch.int32
        ids = torch.randint(0, vocab, (ids_buf.numel(),), device="cuda", generator=g, dtype=torch.int32)
        ids_buf.copy_(ids)
        rt_p.buffer(r, hbb.SLOT_TEXT).copy_(table[ids.long()].reshape(-1))
    rt_e.forward(0)
    rt_p.forward(0)
    torch.cuda.synchronize()
    assert rt_e.status() == 0
    for r in rt_e.local_ranks(hbb.SLOT_DST_ACT):
        assert torch.equal(rt_e.buffer(r, hbb.SLOT_DST_ACT), rt_p.buffer(r, hbb.SLOT_DST_ACT)), f"rank {r}"
    rt_e.close()
    rt_p.close()


def test_embedding_bad_token_id_reported():
    cfg = configs.get("c4", scale=64)
    plan = hbb.plan_bridge(cfg.edge())
    rt = hbb.BridgeRuntime(plan, _spec(cfg), text_embedding=True)
    table = torch.zeros(10, cfg.hidden, device="cuda", dtype=torch.bfloat16)
    rt.set_text_embedding(table)
    r = rt.local_ranks(hbb.SLOT_TEXT)[0]
    rt.buffer(r, hbb.SLOT_TEXT).fill_(3)
    rt.buffer(r, hbb.SLOT_TEXT)[5] = 10  # == vocab: out of range
    rt.forward(0)
    torch.cuda.synchronize()
    with pytest.raises(hbb.HetBridgeError) as ei:
        rt.status()
    assert ei.value.code == "InvalidArgument"
    rt.close()


def test_embedding_requires_table_and_splice():
    cfg = configs.get("c4", scale=64)
    plan = hbb.plan_bridge(cfg.edge())
    rt = hbb.BridgeRuntime(plan, _spec(cfg), text_embedding=True)
    with pytest.raises(hbb.HetBridgeError):
        rt.forward(0)  # no table set
    rt.close()
    with pytest.raises(hbb.HetBridgeError):
        hbb.BridgeRuntime(hbb.plan_bridge(configs.get("c2", scale=64).edge()), text_embedding=True)


@pytest.mark.parametrize("partition", [0, 1, 3])
def test_embedding_bad_row_left_unwritten(partition):
    """A bad id's row is left untouched by both copy engines (TMA: the chunk's
    good row pieces are stored one by one; LDG: the row is skipped)."""
    cfg = configs.get("c4", scale=64)
    plan = hbb.plan_bridge(cfg.edge())
    rt = hbb.BridgeRuntime(plan, _spec(cfg), text_embedding=True, partition=partition)
    table = torch.ones(10, cfg.hidden, device="cuda", dtype=torch.bfloat16)
    rt.set_text_embedding(table)
    for r in rt.local_ranks(hbb.SLOT_SRC_ACT):
        rt.buffer(r, hbb.SLOT_SRC_ACT).fill_(2.0)
    for r in rt.local_ranks(hbb.SLOT_TEXT):
        rt.buffer(r, hbb.SLOT_TEXT).fill_(3)
    r0 = rt.local_ranks(hbb.SLOT_TEXT)[0]
    rt.buffer(r0, hbb.SLOT_TEXT)[5] = -4  # out of range
    for r in rt.local_ranks(hbb.SLOT_DST_ACT):
        rt.buffer(r, hbb.SLOT_DST_ACT).fill_(7.0)
    rt.forward(0)
    torch.cuda.synchronize()
    with pytest.raises(hbb.HetBridgeError):
        rt.status()
    untouched = 0
    for r in rt.local_ranks(hbb.SLOT_DST_ACT):
        rows = rt.buffer(r, hbb.SLOT_DST_ACT).view(-1, cfg.hidden).float()
        sentinel = (rows == 7.0).all(dim=1)
        assert bool(((rows == 1.0) | (rows == 2.0)).all(dim=1)[~sentinel].all()), f"rank {r}: garbage row"
        untouched += int(sentinel.sum())
        if r != r0:
            assert int(sentinel.sum()) == 0, f"rank {r}"
    assert untouched == 1
    rt.close()


def _vp_case(n_gpus, rank_to_gpu=None, partition=0, vocab=998):
    """Vocab-parallel table (each TP rank of a destination cell holds vocab/tp
    rows, separate allocations, tp order) against splicing pre-embedded rows
    table[ids] with a plain runtime: bit-identical destination slices."""
    cfg = configs.get("c4", scale=64)  # llm{tp2, cp4}: TP groups {0,1}, {2,3}, ...
    plan = hbb.plan_bridge(cfg.edge())
    sp = _spec(cfg)
    tp = cfg.dst.tp
    table = torch.randn(vocab, cfg.hidden, device="cuda").to(torch.bfloat16)
    rows = (vocab + tp - 1) // tp
    if n_gpus == 1:
        grp = None
        rts = [hbb.BridgeRuntime(plan, sp, text_embedding=True, partition=partition)]
        r2g = [0] * plan.world
        devs = [torch.device("cuda", 0)]
    else:
        devs_i = list(range(n_gpus)) if torch.cuda.device_count() >= n_gpus else [0] * n_gpus
        grp = hbb.LocalGroup(plan, sp, devices=devs_i, rank_to_gpu=rank_to_gpu, text_embedding=True,
                             partition=partition, timeout_s=20.0)
        rts, r2g = grp.rts, grp.rank_to_gpu
        devs = [torch.device("cuda", d) for d in devs_i]
    rt_p = hbb.BridgeRuntime(plan, sp, partition=partition)
    shards = {}
    try:
        for r in range(plan.world):
            rt = rts[r2g[r]]
            if rt.buffer_numel(r, hbb.SLOT_DST_ACT) == 0:
                continue
            t = configs_tp_index(cfg, r)
            piece = torch.zeros(rows, cfg.hidden, dtype=torch.bfloat16, device=devs[r2g[r]])
            lo, hi = t * rows, min(vocab, (t + 1) * rows)
            piece[: hi - lo].copy_(table[lo:hi])
            shards[r] = piece
            rt.set_text_embedding_shard(r, piece, t * rows, vocab)
        g = torch.Generator(device="cpu").manual_seed(5)
        for r in range(plan.world):
            rt = rts[r2g[r]]
            if rt.buffer_numel(r, hbb.SLOT_SRC_ACT):
                x = torch.randn(rt.buffer_numel(r, hbb.SLOT_SRC_ACT), generator=g).to(torch.bfloat16)
                rt.buffer(r, hbb.SLOT_SRC_ACT).copy_(x)
                rt_p.buffer(r, hbb.SLOT_SRC_ACT).copy_(x)
            if rt.buffer_numel(r, hbb.SLOT_TEXT):
                ids_buf = rt.buffer(r, hbb.SLOT_TEXT)
                ids = torch.randint(0, vocab, (ids_buf.numel(),), generator=g, dtype=torch.int32)
                ids_buf.copy_(ids)
                rt_p.buffer(r, hbb.SLOT_TEXT).copy_(table[ids.long().cuda()].reshape(-1))
        for rt in rts:
            assert rt.validate() > 0
        if grp is not None:
            grp.forward(0)
            grp.synchronize()
        else:
            rts[0].forward(0)
        rt_p.forward(0)
        torch.cuda.synchronize()
        for rt in rts:
            assert rt.status() == 0
        for r in range(plan.world):
            rt = rts[r2g[r]]
            if rt.buffer_numel(r, hbb.SLOT_DST_ACT):
                got = rt.buffer(r, hbb.SLOT_DST_ACT).cpu()
                assert torch.equal(got, rt_p.buffer(r, hbb.SLOT_DST_ACT).cpu()), f"rank {r}"
    finally:
        if grp is not None:
            grp.close()
        else:
            rts[0].close()
        rt_p.close()


def configs_tp_index(cfg, r):
    from paper_2605_27678_b200 import grid as hbg

    return hbg.coord_of_rank(cfg.dst, r).tp_idx


@pytest.mark.parametrize("partition", [0, 1, 3])
def test_vocab_parallel_gather_one_gpu(partition):
    _vp_case(1, partition=partition)


@pytest.mark.parametrize("partition", [0, 3])
def test_vocab_parallel_gather_across_gpus(partition):
    """TP pairs split over two GPUs (rank r on GPU r % 2): half of every text
    row's owners sit on the peer, so the gathers cross the peer wait."""
    _vp_case(2, rank_to_gpu=[r % 2 for r in range(8)], partition=partition)


def test_vocab_parallel_shards_must_tile_the_vocab():
    cfg = configs.get("c4", scale=64)
    plan = hbb.plan_bridge(cfg.edge())
    rt = hbb.BridgeRuntime(plan, _spec(cfg), text_embedding=True)
    try:
        a = torch.zeros(10, cfg.hidden, device="cuda", dtype=torch.bfloat16)
        b = torch.zeros(12, cfg.hidden, device="cuda", dtype=torch.bfloat16)
        for r in rt.local_ranks(hbb.SLOT_DST_ACT):
            t = configs_tp_index(cfg, r)
            rt.set_text_embedding_shard(r, a if t == 0 else b, 10 * t, 22)
        with pytest.raises(hbb.HetBridgeError) as ei:
            rt.forward(0)
        assert ei.value.code == "ShapeMismatch"
    finally:
        rt.close()
