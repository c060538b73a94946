"""1F1B-paired cycle graph (hb_exec_graph_capture what=4): step k runs the
forward of buffer set k concurrently with the backward of set k-1. The two ops
touch disjoint buffers, so one paired cycle must leave every buffer bit for bit
as the same ops run one after the other: fwd(0), bwd(S-1), fwd(1), bwd(0), ...
Checked at one GPU and on a 2-GPU exec group (virtual GPUs sharing cuda:0 when
the box has one GPU; both grids capped so all four kernels are co-resident)."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from parity_core import make_splice  # noqa: E402

from paper_2605_27678_b200 import bridge as hbb  # noqa: E402
from paper_2605_27678_b200 import configs  # noqa: E402

DT = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}
SLOTS = (hbb.SLOT_SRC_ACT, hbb.SLOT_DST_ACT, hbb.SLOT_DST_GRAD, hbb.SLOT_SRC_GRAD, hbb.SLOT_TEXT)


def _bufs(rts, plan, r2g, S):
    out = {}
    for r in range(plan.world):
        rt = rts[r2g[r]]
        for slot in SLOTS:
            if rt.buffer_numel(r, slot) == 0:
                continue
            for k in range(S):
                b = rt.buffer(r, slot, k)
                if b is not None:
                    out[(r, slot, k)] = b
    return out


def _run(name, n, devices, cap, what=None):
    cfg = configs.get(name, scale=64)
    plan = hbb.plan_bridge(cfg.edge())
    S = 3
    kw = dict(act_dtype=DT[cfg.act], grad_in_dtype=DT[cfg.grad_in], grad_out_dtype=torch.float32, mb_slots=S,
              max_ctas=cap, timeout_s=20.0)
    if n == 1:
        rts = [hbb.BridgeRuntime(plan, make_splice(cfg), **kw)]
        r2g = [0] * plan.world
        streams = [torch.cuda.Stream()]
        group = None
    else:
        group = hbb.LocalGroup(plan, make_splice(cfg), devices=devices, **kw)
        rts, r2g, streams = group.rts, group.rank_to_gpu, group.streams
    try:
        bufs = _bufs(rts, plan, r2g, S)
        gen = torch.Generator(device="cpu").manual_seed(7)
        for key, b in sorted(bufs.items()):
            if key[1] == hbb.SLOT_TEXT and b.dtype == torch.int32:
                continue
            b.copy_(torch.randn(b.numel(), generator=gen).to(b.dtype))
        torch.cuda.synchronize()
        init = {k: b.clone() for k, b in bufs.items()}

        # serial reference on the same buffers: fwd(k), bwd(k-1) in cycle order (graphs, one op each)
        for rt, st in zip(rts, streams):
            for k in range(S):
                rt.capture_step(k, 1.0, stream=st, what=rt.GRAPH_FWD)
                rt.capture_step(k, 1.0, stream=st, what=rt.GRAPH_BWD)
        for k in range(S):
            for rt, st in zip(rts, streams):
                rt.replay_step(k, st, rt.GRAPH_FWD)
            for rt, st in zip(rts, streams):
                rt.replay_step((k + S - 1) % S, st, rt.GRAPH_BWD)
        torch.cuda.synchronize()
        serial = {k: b.clone() for k, b in bufs.items()}

        for k, b in bufs.items():
            b.copy_(init[k])
        torch.cuda.synchronize()
        w = rts[0].GRAPH_PAIRED if what is None else what
        for rt, st in zip(rts, streams):
            rt.capture_step(0, 1.0, stream=st, what=w)
        before = [rt.stats()["launches"] for rt in rts]
        for rt, st in zip(rts, streams):
            rt.replay_step(0, st, w)
        if w == rts[0].GRAPH_PAIRED_FUSED:  # one launch per pair: the fused kernel ran (not fused: C3's fan-out)
            expect = 2 * S if name == "c3" else S
            assert [rt.stats()["launches"] - b for rt, b in zip(rts, before)] == [expect] * len(rts)
        torch.cuda.synchronize()
        for rt in rts:
            assert rt.status() == 0
        for k, b in bufs.items():
            assert torch.equal(b.view(torch.uint8), serial[k].view(torch.uint8)), f"buffer {k} differs"
    finally:
        if group is not None:
            group.close()
        else:
            rts[0].close()


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_paired_cycle_equals_serial_one_gpu(name):
    _run(name, 1, [0], 148)


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_paired_cycle_equals_serial_group(name):
    n = 2
    devs = list(range(n)) if torch.cuda.device_count() >= n else [0] * n
    _run(name, n, devs, 48)


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_fused_paired_cycle_equals_serial_one_gpu(name):
    """what=5: each pair in one warp-specialised launch (TMA lane for the forward,
    15 warps for the gradient return)."""
    _run(name, 1, [0], 0, what=hbb.BridgeRuntime.GRAPH_PAIRED_FUSED)


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_fused_paired_cycle_equals_serial_group(name):
    n = 2
    devs = list(range(n)) if torch.cuda.device_count() >= n else [0] * n
    _run(name, n, devs, 48, what=hbb.BridgeRuntime.GRAPH_PAIRED_FUSED)


def _schedule(name, n, fuse):
    """Exec.paired in a 1F1B order (F0 F1 [F2|B0] [F3|B1] B2 B3, beta=1) against
    the same ops issued one by one; `fuse[g]` False makes GPU g issue its pairs
    as two launches while its peers fuse."""
    cfg = configs.get(name, scale=64)
    plan = hbb.plan_bridge(cfg.edge())
    S = 3
    devs = list(range(n)) if torch.cuda.device_count() >= n else [0] * n
    kw = dict(act_dtype=DT[cfg.act], grad_in_dtype=DT[cfg.grad_in], grad_out_dtype=torch.float32, mb_slots=S,
              max_ctas=48, timeout_s=20.0)
    group = hbb.LocalGroup(plan, make_splice(cfg), devices=devs, **kw)
    try:
        bufs = _bufs(group.rts, plan, group.rank_to_gpu, S)
        gen = torch.Generator(device="cpu").manual_seed(11)
        for key, b in sorted(bufs.items()):
            if key[1] == hbb.SLOT_TEXT and b.dtype == torch.int32:
                continue
            b.copy_(torch.randn(b.numel(), generator=gen).to(b.dtype))
        torch.cuda.synchronize()
        init = {k: b.clone() for k, b in bufs.items()}
        for op, mb in (("f", 0), ("f", 1), ("b", 0), ("f", 2), ("b", 1), ("f", 3), ("b", 2), ("b", 3)):
            group.forward(mb) if op == "f" else group.backward(mb, 1.0)
        group.synchronize()
        serial = {k: b.clone() for k, b in bufs.items()}
        for k, b in bufs.items():
            b.copy_(init[k])
        torch.cuda.synchronize()
        group.forward(0)
        group.forward(1)
        fused = group.paired(2, 0, 1.0, fuse) + group.paired(3, 1, 1.0, fuse)
        group.backward(2, 1.0)
        group.backward(3, 1.0)
        group.synchronize()
        assert all(rt.status() == 0 for rt in group.rts)
        for k, b in bufs.items():
            assert torch.equal(b.view(torch.uint8), serial[k].view(torch.uint8)), f"buffer {k} differs"
        return fused
    finally:
        group.close()


@pytest.mark.parametrize("name", ["c2", "c4", "c5"])
def test_exec_paired_schedule(name):
    fused = _schedule(name, 2, None)
    assert all(fused), "the fused kernel should serve these partitions"


def test_exec_paired_mixed_with_separate_launches():
    """GPU 1 issues its pairs as two launches while GPU 0 fuses: each op is
    still one op of every peer's epoch sequence."""
    assert _schedule("c2", 2, [True, False]) == [True, False, True, False]


def test_exec_paired_rejects_unknown_backward():
    cfg = configs.get("c2", scale=64)
    rt = hbb.BridgeRuntime(hbb.plan_bridge(cfg.edge()), make_splice(cfg), mb_slots=2, act_dtype=torch.bfloat16,
                           grad_in_dtype=torch.bfloat16, grad_out_dtype=torch.float32)
    try:
        with pytest.raises(hbb.HetBridgeError) as ei:
            rt.paired(1, 0)
        assert ei.value.code == "UnknownMicrobatch"
        rt.forward(0)
        rt.forward(1)
        with pytest.raises(hbb.HetBridgeError):  # 3 % 2 == 1: set 1 still holds microbatch 1
            rt.paired(3, 0)
        assert rt.paired(2, 0) in (True, False)
    finally:
        rt.close()
