"""Static race and bounds check of the device tables (hb_exec_validate).

compute-sanitizer is closed on the GPU pool (gpurun refuses it: runs under it
left GPUs needing a reset; profiles/r02/sanitizer_refused.log), so the
global-memory hazards of the boundary kernels are checked where they come
from: the descriptor tables each exec uploads. Every config, in every
partition mode and forward mode, at 1 GPU and on 2/4-GPU exec groups (virtual
GPUs sharing cuda:0, or real ones), must be free of out-of-bounds runs,
overlapping writes, reads overlapping writes, peer reads ahead of the peer
wait, and chunks handed out twice. Then a real caller error — two ranks'
destination buffers bound to overlapping memory — must be reported as a
write/write race before any kernel runs.
"""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from parity_core import make_splice  # noqa: E402

from paper_2605_27678_b200 import bridge as hbb  # noqa: E402
from paper_2605_27678_b200 import configs  # noqa: E402

ALL = ["c1", "c2", "c3", "c4", "c4ip", "c5", "c3p", "appc", "c2x4", "c3x4", "c4w4", "c5w4"]
DT = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}


def _kw(cfg):
    return dict(act_dtype=DT[cfg.act], grad_in_dtype=DT[cfg.grad_in], grad_out_dtype=torch.float32)


@pytest.mark.parametrize("partition", [0, 1, 2, 3])
@pytest.mark.parametrize("name", ALL)
def test_one_gpu_tables_clean(name, partition):
    cfg = configs.get(name, scale=64)
    rt = hbb.BridgeRuntime(hbb.plan_bridge(cfg.edge()), make_splice(cfg), mb_slots=2, partition=partition, **_kw(cfg))
    try:
        assert rt.validate() > 0
    finally:
        rt.close()


@pytest.mark.parametrize("mode", [dict(), dict(fwd_mode=2), dict(strict_provenance=True), dict(partition=1)])
@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5", "c3p", "appc", "c4w4"])
def test_group_tables_clean(name, n, mode):
    cfg = configs.get(name, scale=64)
    plan = hbb.plan_bridge(cfg.edge())
    if plan.world < n:
        pytest.skip(f"{name} has {plan.world} logical ranks")
    devs = list(range(n)) if torch.cuda.device_count() >= n else [0] * n
    g = hbb.LocalGroup(plan, make_splice(cfg), devices=devs, mb_slots=2, **_kw(cfg), **mode)
    try:
        assert sum(rt.validate() for rt in g.rts) > 0  # (a GPU of the group may have no work of its own)
    finally:
        g.close()


def test_strided_bindings_clean():
    """Caller buffers with a row stride: every run must stay inside one row."""
    cfg = configs.get("c2", scale=64)
    rt = hbb.BridgeRuntime(hbb.plan_bridge(cfg.edge()), **_kw(cfg))
    keep = []
    try:
        for slot in (hbb.SLOT_SRC_ACT, hbb.SLOT_DST_ACT):
            for r in rt.local_ranks(slot):
                n = rt.buffer_numel(r, slot)
                W = cfg.edge().feature_width
                rows = n // W
                t = torch.zeros(rows, W + 64, device="cuda", dtype=DT[cfg.act])
                keep.append(t)
                rt.bind(r, slot, t[:, :W], 0)
        assert rt.validate() > 0
    finally:
        rt.close()


def test_overlapping_destination_bindings_reported():
    cfg = configs.get("c2", scale=64)
    rt = hbb.BridgeRuntime(hbb.plan_bridge(cfg.edge()), **_kw(cfg))
    try:
        r0, r1 = rt.local_ranks(hbb.SLOT_DST_ACT)[:2]
        n = rt.buffer_numel(r0, hbb.SLOT_DST_ACT)
        big = torch.zeros(n + n // 2, device="cuda", dtype=DT[cfg.act])
        rt.bind(r0, hbb.SLOT_DST_ACT, big[:n], 0)
        rt.bind(r1, hbb.SLOT_DST_ACT, big[n // 2:n // 2 + n], 0)  # half of r0's rows again
        with pytest.raises(hbb.HetBridgeError, match="write/write race") as ei:
            rt.validate()
        assert ei.value.code == "ValidationError"
    finally:
        rt.close()


def test_source_aliasing_destination_reported():
    """A rank's destination bound over another rank's source shard: the forward
    would overwrite rows other CTAs are still reading."""
    cfg = configs.get("c2", scale=64)
    rt = hbb.BridgeRuntime(hbb.plan_bridge(cfg.edge()), **_kw(cfg))
    try:
        r = rt.local_ranks(hbb.SLOT_DST_ACT)[0]
        s = rt.local_ranks(hbb.SLOT_SRC_ACT)[-1]
        src = rt.buffer(s, hbb.SLOT_SRC_ACT, 0)
        n = rt.buffer_numel(r, hbb.SLOT_DST_ACT)
        big = torch.zeros(n + src.numel(), device="cuda", dtype=DT[cfg.act])
        rt.bind(s, hbb.SLOT_SRC_ACT, big[:src.numel()], 0)
        rt.bind(r, hbb.SLOT_DST_ACT, big[:n], 0)
        with pytest.raises(hbb.HetBridgeError, match="race"):
            rt.validate()
    finally:
        rt.close()
