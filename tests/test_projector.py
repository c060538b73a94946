"""Projector GEMM (tcgen05 / TMEM / TMA, csrc/kernels/projector_gemm.cu) vs a
plain PyTorch fp32 reference of the same op (bf16 inputs, fp32 accumulate,
bf16 output; tolerance: 1 bf16 ulp of the output magnitude plus fp32
summation-order noise)."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _ref(x, w):
    return (x.float() @ w.float().t()).to(torch.bfloat16)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 512, 128), (576, 4096, 1024), (4608, 4096, 1280),
                                   # long K (the deep 2-SM ring, half-row epilogue) and more m-tile groups
                                   # than one rasterisation group, with a ragged last group and last pair
                                   (4480, 1024, 4096), (2400, 768, 2048)])
def test_projector_gemm_vs_torch(M, N, K):
    from paper_2605_27678_b200.projector import projector_gemm

    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    y = projector_gemm(x, w)
    torch.cuda.synchronize()
    ref = _ref(x, w)
    torch.testing.assert_close(y.float(), ref.float(), rtol=1.6e-2, atol=1e-2)


def test_projector_rows_fan_out():
    """Each output row lands in every destination row of its table entry."""
    from paper_2605_27678_b200.projector import projector_gemm_rows

    M, N, K = 256, 512, 128
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    outs = [torch.zeros(M, N, device="cuda", dtype=torch.bfloat16) for _ in range(3)]
    perm = torch.randperm(M, device="cuda")
    rows = torch.zeros(M, 3, dtype=torch.int64, device="cuda")
    for f, o in enumerate(outs[:2]):  # rows scattered through a permutation
        rows[:, f] = o.data_ptr() + perm * (N * 2)
    rows[::2, 2] = outs[2].data_ptr() + torch.arange(0, M, 2, device="cuda") * (N * 2)  # sparse third target
    projector_gemm_rows(x, w, rows.reshape(-1), 3)
    torch.cuda.synchronize()
    ref = _ref(x, w).float()
    for o in outs[:2]:
        torch.testing.assert_close(o[perm].float(), ref, rtol=1.6e-2, atol=1e-2)
    torch.testing.assert_close(outs[2][::2].float(), ref[::2], rtol=1.6e-2, atol=1e-2)
    assert torch.count_nonzero(outs[2][1::2]) == 0


@pytest.mark.parametrize("name", ["c2", "c3", "c1"])
def test_fused_projector_forward_equals_gemm_then_reshard(name):
    """hb_exec_forward_projected (projector GEMM whose epilogue writes every
    destination row) is bit-identical to the same GEMM into the source shards
    followed by the forward reshard."""
    from paper_2605_27678_b200 import bridge as hbb
    from paper_2605_27678_b200 import configs
    from paper_2605_27678_b200.projector import projector_gemm

    cfg = configs.get(name, scale=4096 // 256 if name != "c3" else 5120 // 256)
    d_h, K = cfg.hidden, 128
    assert d_h == 256
    plan = hbb.plan_bridge(cfg.edge())
    rt_a = hbb.BridgeRuntime(plan)
    rt_b = hbb.BridgeRuntime(plan)
    srcs = rt_a.local_ranks(hbb.SLOT_SRC_ACT)
    rows = sum(rt_a.buffer_numel(r, hbb.SLOT_SRC_ACT) for r in srcs) // d_h
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(rows, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(d_h, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    rt_a.forward_projected(0, x, w)
    y = projector_gemm(x, w)
    o = 0
    for r in srcs:
        b = rt_b.buffer(r, hbb.SLOT_SRC_ACT)
        n = b.numel() // d_h
        b.copy_(y[o:o + n].reshape(-1))
        o += n
    rt_b.forward(0)
    torch.cuda.synchronize()
    for r in rt_a.local_ranks(hbb.SLOT_DST_ACT):
        assert torch.equal(rt_a.buffer(r, hbb.SLOT_DST_ACT), rt_b.buffer(r, hbb.SLOT_DST_ACT)), f"rank {r}"
    # the backward still works after a fused forward (records are shared)
    rt_a.backward(0, 0.0)
    torch.cuda.synchronize()
    assert rt_a.status() == 0
    rt_a.close()
    rt_b.close()
