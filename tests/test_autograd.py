"""Autograd binding and the colocated three-phase packed boundary tensor
(S:371-374).

GPU tests compare against the CPU oracle (placement, gradient return) and
against a plain PyTorch restatement of the whole step: a toy projector
"encoder", the boundary, and a "LLM" loss on its PP0 inputs; the encoder
weight gradient through the three phases must equal the one autograd computes
without any boundary (the boundary is a pure placement, so the two agree to
fp32 summation order). Contract inputs: tp replicas of the LLM receive
identical gradients (bridge.hpp:33-36).
"""
import numpy as np
import pytest

from helpers import O, hbb

from paper_2605_27678_b200 import configs


def test_autograd_module_surface():
    import paper_2605_27678_b200 as pkg

    ag = pkg.autograd
    assert callable(ag.boundary) and hasattr(ag, "PackedBoundary")


torch = pytest.importorskip("torch")
DEV = "cuda:0"


def _o(l):
    return O.Layout(l.name, l.tp, l.cp, l.pp, l.dp, l.rank_offset)


def _require_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c2", "c3", "c5"])
def test_boundary_autograd_vs_oracle(name):
    _require_gpu()
    from paper_2605_27678_b200.autograd import boundary

    cfg = configs.get(name, scale=256)
    plan = hbb.plan_bridge(cfg.edge())
    rt = hbb.BridgeRuntime(plan, act_dtype=torch.float32, grad_in_dtype=torch.float32,
                           grad_out_dtype=torch.float32)
    src, dst = _o(cfg.src), _o(cfg.dst)
    B, W = cfg.batch, cfg.width
    SI, DI = O.intervals(B, src.dp), O.intervals(B, dst.dp)
    rng = np.random.default_rng(3)
    X = rng.standard_normal((B, W))
    src_ranks = rt.local_ranks(hbb.SLOT_SRC_ACT)
    xs = []
    for r in src_ranks:
        d = src.coord(r)[3]
        xs.append(torch.tensor(X[SI[d][0]:SI[d][0] + SI[d][1]], device=DEV, dtype=torch.float32,
                               requires_grad=True))
    outs = boundary(rt, 0, *xs)
    outs = outs if isinstance(outs, tuple) else (outs,)
    ref, _, _ = O.bridge_forward(src, dst, B, W, {r: x.detach().cpu().double().numpy() for r, x in zip(src_ranks, xs)})
    dst_ranks = rt.local_ranks(hbb.SLOT_DST_ACT)
    G = rng.standard_normal((B, W))
    loss = 0
    gd = {}
    for r, o in zip(dst_ranks, outs):
        np.testing.assert_array_equal(o.detach().cpu().numpy(), ref[r].astype(np.float32))
        d = dst.coord(r)[3]
        g = G[DI[d][0]:DI[d][0] + DI[d][1]]  # tp replicas: identical gradients
        gd[r] = g
        loss = loss + (o * torch.tensor(g, device=DEV, dtype=torch.float32)).sum()
    loss.backward()
    refb, _, _ = O.bridge_backward(src, dst, B, W, gd)
    for r, x in zip(src_ranks, xs):
        np.testing.assert_allclose(x.grad.cpu().numpy(), refb[r], rtol=1e-6, atol=1e-6)
    rt.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c2", "c3"])
@pytest.mark.parametrize("n_mb", [1, 3])
def test_three_phase_packed_boundary_matches_plain_autograd(name, n_mb):
    _require_gpu()
    from paper_2605_27678_b200.autograd import PackedBoundary

    cfg = configs.get(name, scale=256)
    plan = hbb.plan_bridge(cfg.edge())
    rt = hbb.BridgeRuntime(plan, act_dtype=torch.float32, grad_in_dtype=torch.float32,
                           grad_out_dtype=torch.float32, mb_slots=n_mb)
    src, dst = _o(cfg.src), _o(cfg.dst)
    B, W = cfg.batch, cfg.width
    SI, DI = O.intervals(B, src.dp), O.intervals(B, dst.dp)
    torch.manual_seed(0)
    d_in = 16
    w = torch.randn(d_in, W, device=DEV, requires_grad=True)
    feats = [torch.randn(B, d_in, device=DEV) for _ in range(n_mb)]
    Gs = [torch.randn(B, W, device=DEV) for _ in range(n_mb)]

    # plain autograd restatement: each LLM DP shard sees its slice of the
    # projected batch, weighted by that slice of G. tp replicas of the LLM
    # compute one loss together, so a shard counts once (its tp=0 rank).
    dst_ranks = [r for r in range(plan.world) if hbb.buffer_elems(plan, r, hbb.SLOT_DST_ACT) > 0]
    loss_ref = 0
    for mb in range(n_mb):
        y = feats[mb] @ w
        for r in dst_ranks:
            t, c, p, d = dst.coord(r)
            if t == 0:
                sl = slice(DI[d][0], DI[d][0] + DI[d][1])
                loss_ref = loss_ref + (y[sl] * Gs[mb][sl]).sum()
    (gw_ref,) = torch.autograd.grad(loss_ref, w)

    # phase 1: encoder forward once over the window, projector output written
    # straight into the boundary's source buffers, colocated forward transform
    pb = PackedBoundary(rt, n_mb)
    enc = []
    for mb in range(n_mb):
        y = feats[mb] @ w
        outs = []
        for r in pb.src_ranks:
            t, c, p, d = src.coord(r)
            o = y[SI[d][0]:SI[d][0] + SI[d][1]]
            # encoder tp replicas hold the same activation; its gradient enters the
            # encoder graph once (through the tp=0 copy)
            outs.append(o if t == 0 else o.detach())
        enc.append(outs)
    leaves = pb.forward(enc)
    # phase 2: detached LLM over per-microbatch views; its gradients accumulate
    # on the packed tensor (the DST_GRAD buffers)
    for mb in range(n_mb):
        loss = 0
        for r in pb.dst_ranks:
            v = pb.view(mb, r)
            assert v.is_leaf and v.requires_grad
            d = dst.coord(r)[3]
            loss = loss + (v * Gs[mb][DI[d][0]:DI[d][0] + DI[d][1]]).sum()
        loss.backward()
        for r in pb.dst_ranks:
            buf = rt.buffer(r, hbb.SLOT_DST_GRAD, mb)
            assert pb.view(mb, r).grad.data_ptr() == buf.data_ptr()  # landed in place
    assert w.grad is None  # the encoder graph is not touched in phase 2
    # phase 3: gradient handoff, colocated backward transform, encoder backward
    pb.backward()
    torch.testing.assert_close(w.grad, gw_ref, rtol=1e-5, atol=1e-4)
    assert pb.phase == 0
    rt.close()
