"""Multi-exec parity in ONE process (hb_exec_open_peers_local): one exec per
(virtual) GPU of the group, every op launched on every GPU's stream from this
thread, the execs meeting in the same in-kernel barrier (arrival epochs,
"started" posts, lazy peer waits) and pulling rows from each other's regions
through the same remote queues, TMA rings and fan-out paths as a torchrun
group over NVSwitch.

On a one-GPU box the group's execs share cuda:0 (max_ctas keeps their grids
co-resident), so the driver's single-GPU `-m gpu` run exercises the whole
cross-GPU protocol; with >= N devices the same test runs on N real GPUs with
peer access over NVLink. Parity is against the oracle (tests/parity_core.py).
"""
import pytest

torch = pytest.importorskip("torch")

from parity_core import LocalGroupDriver, group_parity, make_splice  # noqa: E402

from paper_2605_27678_b200 import bridge as hbb  # noqa: E402
from paper_2605_27678_b200 import configs  # noqa: E402

pytestmark = pytest.mark.gpu

CONFIGS = ["c1", "c2", "c3", "c4", "c4ip", "c5", "c3p", "appc", "c2x4", "c3x4", "c4w4"]


def _group(name, n, devices, **kw):
    cfg = configs.get(name, scale=64)
    plan = hbb.plan_bridge(cfg.edge())
    if plan.world < n:
        pytest.skip(f"{name} has {plan.world} logical ranks")
    sp = make_splice(cfg)
    g = hbb.LocalGroup(plan, sp, devices=devices, act_dtype=torch.bfloat16 if cfg.act == "bf16" else torch.float32,
                       grad_in_dtype=torch.bfloat16 if cfg.grad_in == "bf16" else torch.float32,
                       grad_out_dtype=torch.float32, timeout_s=20.0, **kw)
    return cfg, g


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("name", CONFIGS)
def test_virtual_gpus_on_one_device(name, n):
    """n execs sharing cuda:0: the whole protocol on one physical GPU."""
    cfg, g = _group(name, n, [0] * n)
    try:
        ok, worst = group_parity(cfg, LocalGroupDriver(g), steps=2)
        assert g.status() == 0
        assert ok, f"{name} n={n}: parity failed (bwd worst {worst:.3g})"
    finally:
        g.close()


@pytest.mark.parametrize("mode", [dict(fwd_mode=2), dict(partition=1), dict(strict_provenance=True)])
@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_virtual_gpus_modes(name, mode):
    """push forward, contiguous partition and strict provenance across execs."""
    cfg, g = _group(name, 2, [0, 0], **mode)
    try:
        ok, worst = group_parity(cfg, LocalGroupDriver(g), steps=2, strict=bool(mode.get("strict_provenance")))
        assert g.status() == 0
        assert ok, f"{name} {mode}: parity failed (bwd worst {worst:.3g})"
    finally:
        g.close()


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5", "c3p"])
def test_real_gpus_one_process(name, n):
    """one process, n real GPUs, peer access over NVLink (skips below n GPUs)."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cfg, g = _group(name, n, list(range(n)))
    try:
        ok, worst = group_parity(cfg, LocalGroupDriver(g), steps=2)
        assert ok, f"{name} n={n}: parity failed (bwd worst {worst:.3g})"
    finally:
        g.close()


def test_open_peers_local_rejects_mismatched_group():
    cfg = configs.get("c2", scale=64)
    plan = hbb.plan_bridge(cfg.edge())
    a = hbb.BridgeRuntime(plan, n_gpus=2, my_gpu=0, rank_to_gpu=configs.rank_to_gpu(8, 2))
    b = hbb.BridgeRuntime(plan, n_gpus=2, my_gpu=1, rank_to_gpu=configs.rank_to_gpu(8, 2), mb_slots=2)
    with pytest.raises(hbb.HetBridgeError):
        a.open_peers_local([a, b])  # different buffer-set count: not the same symmetric layout
    a.close()
    b.close()


def _dtypes(cfg):
    tdt = {"bf16": torch.bfloat16, "fp32": torch.float32}
    return {hbb.SLOT_SRC_ACT: tdt[cfg.act], hbb.SLOT_DST_ACT: tdt[cfg.act], hbb.SLOT_TEXT: tdt[cfg.act],
            hbb.SLOT_DST_GRAD: tdt[cfg.grad_in], hbb.SLOT_SRC_GRAD: torch.float32}


@pytest.mark.parametrize("pad", [0, 40])
@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5", "c3p"])
def test_caller_bound_buffers_across_execs(name, pad):
    """a7 DeviceShard: every rank's slots are caller-owned tensors (row-strided
    when pad > 0), bound on their exec and read/written in place by peers."""
    from parity_core import bind_caller_buffers

    cfg, g = _group(name, 2, [0, 0])
    try:
        dt = _dtypes(cfg)
        bufs = bind_caller_buffers(g.bind, lambda r, s: hbb.buffer_elems(g.plan, r, s, g.splice), cfg,
                                   range(g.plan.world), lambda r: torch.device("cuda", 0), lambda s: dt[s], pad)
        assert bufs
        drv = LocalGroupDriver(g)
        ok, worst = group_parity(cfg, drv, steps=2)
        assert ok, f"{name} pad={pad}: parity failed (bwd worst {worst:.3g})"
        for (r, slot), v in bufs.items():  # the runtime wrote the caller's tensors, and nothing else
            base = v.as_strided((v.shape[0], v.shape[1] + pad), (v.stride(0), 1))
            if pad:
                assert bool(torch.isnan(base[:, v.shape[1]:].float()).all()), f"rank {r} slot {slot}: padding written"
            if slot in (hbb.SLOT_DST_ACT, hbb.SLOT_SRC_GRAD):
                assert not bool(torch.isnan(v.float()).any()), f"rank {r} slot {slot}: row not written"
    finally:
        g.close()


def test_out_of_turn_peer_detected():
    """Race/protocol check (the device analogue of simnet's out-of-turn check,
    R:core/src/simnet.cpp:202-207): a peer's "started" count two ops ahead of
    this launch's epoch cannot happen under the end-of-launch contract, so the
    kernel reports it (GroupMismatch) instead of reading the peer's buffers."""
    from paper_2605_27678_b200.bridge import _CAI

    cfg, g = _group("c2", 2, [0, 0])
    try:
        ok, _ = group_parity(cfg, LocalGroupDriver(g), steps=1)
        assert ok and g.status() == 0
        rt0 = g.rts[0]
        # region base of exec 0: its first buffer sits 4 KiB after the signal pad
        ptrs = [rt0.buffer(r, s).data_ptr() for r in range(g.plan.world) if g.rank_to_gpu[r] == 0
                for s in range(5) if rt0.buffer_numel(r, s)]
        words = torch.as_tensor(_CAI(min(ptrs) - 4096, 4096), device="cuda:0").view(torch.int32)
        # forward "started" word of GPU 1 in GPU 0's pad, pushed past any legal value:
        # GPU 1's own post of the next op may land before or after GPU 0 reads the
        # word, so +3 keeps it >= e+2 (two ops ahead) either way (+2 could read e+1,
        # which is legal: a peer may already have started the following op)
        words[1] += 3
        torch.cuda.synchronize()
        g.forward(1)
        g.synchronize()
        with pytest.raises(hbb.HetBridgeError) as ei:
            rt0.status()
        assert ei.value.code == "GroupMismatch"
        assert g.rts[1].status() == 0
        # recovery: every exec of the group resets its protocol state, then the
        # same execs (tables, peers) run correct steps again
        g.reset_protocol()
        assert all(rt.status() == 0 for rt in g.rts)
        ok, _ = group_parity(cfg, LocalGroupDriver(g), steps=2)
        assert ok and all(rt.status() == 0 for rt in g.rts)
    finally:
        g.close()
