"""Runtime guards: captured graphs are dropped when the
device tables are rebuilt, in-flight microbatches may not share a buffer set,
the fused projector validates its operand shape, and the autograd op never
returns an alias of the runtime's gradient buffer."""
import ctypes

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from helpers import hbb  # noqa: E402

from paper_2605_27678_b200 import _lib, configs  # noqa: E402


def _rt(name="c2", **kw):
    cfg = configs.get(name, scale=64)
    return cfg, hbb.BridgeRuntime(hbb.plan_bridge(cfg.edge()), **kw)


def test_bind_invalidates_captured_graphs():
    cfg, rt = _rt(mb_slots=2)
    st = torch.cuda.Stream()
    rt.capture_step(0, 1.0, True, st)
    rt.replay_step(0, st)
    torch.cuda.synchronize()
    r = rt.local_ranks(hbb.SLOT_SRC_ACT)[0]
    t = torch.zeros(rt.buffer_numel(r, hbb.SLOT_SRC_ACT), device="cuda", dtype=torch.bfloat16)
    rt.bind(r, hbb.SLOT_SRC_ACT, t, 0)  # rebuilds the tables: the old graph would read freed memory
    with pytest.raises(hbb.HetBridgeError, match="recapture"):
        rt.replay_step(0, st)
    rt.capture_step(0, 1.0, True, st)  # recapture works and reads the bound tensor
    rt.replay_step(0, st)
    torch.cuda.synchronize()
    assert rt.status() == 0
    rt.close()


def test_inflight_microbatches_need_distinct_buffer_sets():
    cfg, rt = _rt(mb_slots=2)
    rt.forward(0)
    rt.forward(1)  # sets 0 and 1
    with pytest.raises(hbb.HetBridgeError, match="shares buffer set"):
        rt.forward(2)  # set 0 still holds microbatch 0's activations
    rt.backward(0, 0.0)
    rt.forward(2)  # set 0 is free again
    with pytest.raises(hbb.HetBridgeError):
        rt.forward(-1)
    rt.backward(1, 0.0)
    rt.backward(2, 0.0)
    torch.cuda.synchronize()
    rt.close()


def test_forward_projected_checks_operand_rows():
    base = configs.get("c2")
    cfg = configs.get("c2", scale=base.hidden // 256)
    plan = hbb.plan_bridge(cfg.edge())
    rt = hbb.BridgeRuntime(plan)
    d_h, K = cfg.hidden, 128
    rows = sum(rt.buffer_numel(r, hbb.SLOT_SRC_ACT) for r in rt.local_ranks(hbb.SLOT_SRC_ACT)) // d_h
    w = torch.randn(d_h, K, device="cuda").to(torch.bfloat16)
    short = torch.randn(rows - 128, K, device="cuda").to(torch.bfloat16)
    with pytest.raises(hbb.HetBridgeError) as ei:
        rt.forward_projected(0, short, w)
    assert ei.value.code == "ShapeMismatch"
    # the C-ABI checks the row count too (a caller bypassing the Python face)
    L = _lib.lib()
    st = L.hb_exec_forward_projected(rt._h, 0, ctypes.c_void_p(short.data_ptr()), short.shape[0], K,
                                     ctypes.c_void_p(w.data_ptr()), K, d_h, K,
                                     ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 13  # ShapeMismatch
    x = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
    rt.forward_projected(0, x, w)
    torch.cuda.synchronize()
    rt.close()


@pytest.mark.parametrize("zero_copy", [False, True])
def test_autograd_gradient_is_not_an_alias(zero_copy):
    from paper_2605_27678_b200.autograd import boundary

    cfg, rt = _rt(mb_slots=1, grad_out_dtype=torch.bfloat16)
    srcs = rt.local_ranks(hbb.SLOT_SRC_ACT)
    xs = [torch.randn(rt.buffer_numel(r, hbb.SLOT_SRC_ACT) // cfg.width, cfg.width, device="cuda")
          .to(torch.bfloat16).requires_grad_(True) for r in srcs]
    outs = boundary(rt, 0, *xs, zero_copy=zero_copy)
    if zero_copy:  # the caller's shards are the runtime's source buffers: no staging copy
        assert all(rt.buffer(r, hbb.SLOT_SRC_ACT).data_ptr() == x.data_ptr() for r, x in zip(srcs, xs))
    sum(o.float().sum() for o in outs).backward()
    g0 = [x.grad.clone() for x in xs]
    if not zero_copy:
        ptrs = {rt.buffer(r, hbb.SLOT_SRC_GRAD).data_ptr() for r in srcs}
        assert not any(x.grad.data_ptr() in ptrs for x in xs)
    outs = boundary(rt, 1, *xs, zero_copy=zero_copy)  # reuses buffer set 0
    (2 * sum(o.float().sum() for o in outs)).backward()
    for x, g in zip(xs, g0):
        assert torch.equal(x.grad.float(), 3 * g.float())  # g0 + 2*g0, not an overwritten alias
    rt.close()
