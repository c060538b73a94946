"""Device parity: the sm_100a kernels through the C-ABI vs the CPU oracle.

Every config of BASELINE.json (C1-C5) runs with all logical ranks resident on
cuda:0 at reduced hidden width (the index maps depend on the layouts, not on
the width) against the oracle; full-width runs check size-independent
properties against plain PyTorch restatements.

Tolerances: forward placement bit-exact; backward with beta=0
value-exact (single-term returns; -0.0 == +0.0); backward with beta=1 into an
fp32 accumulator |a-b|/max(1,|b|) <= 1e-6 vs the double-precision oracle;
multi-term (cp>1 non-splice) fp32 sums <= 1e-6.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from helpers import O, hbb, hbg, to_hb  # noqa: E402

from paper_2605_27678_b200 import configs  # noqa: E402

pytestmark = pytest.mark.gpu

DEV = "cuda:0"
TDT = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}
REL_TOL = 1e-6


def _require_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def o_layout(l):
    return O.Layout(l.name, l.tp, l.cp, l.pp, l.dp, l.rank_offset)


def run_case(cfg, seed=0, beta=0.0, perturb=True, partition=0):
    """Fill every resident rank's inputs, run fwd+bwd on the device, compare with the oracle."""
    _require_gpu()
    rng = np.random.default_rng(seed)
    W = cfg.width
    plan = hbb.plan_bridge(cfg.edge())
    sp = None
    if cfg.splice:
        s = cfg.splice
        sp = hbb.SpliceSpec(s["Q"], s["S"], cfg.hidden, cfg.tokens, s["codes"], s["text_mode"])
    # perturbed replicas pin the reference data path replica for replica
    # (strict provenance); contract inputs (tp replicas of a gradient cell
    # identical, bridge.hpp:33-36) run the default replica-balanced backward
    rt = hbb.BridgeRuntime(plan, sp, act_dtype=TDT[cfg.act], grad_in_dtype=TDT[cfg.grad_in],
                           grad_out_dtype=TDT[cfg.grad_out], partition=partition, strict_provenance=perturb)
    src, dst = o_layout(cfg.src), o_layout(cfg.dst)
    B = cfg.batch
    SI, DI = O.intervals(B, src.dp), O.intervals(B, dst.dp)
    X = rng.standard_normal((B, W))
    shards = {}
    for r in src.stage_ranks(src.pp - 1):
        t, c, p, d = src.coord(r)
        a = X[SI[d][0]:SI[d][0] + SI[d][1]].copy()
        if perturb and (t or c):
            a = a + 10.0 * (t + 1)
        buf = rt.buffer(r, hbb.SLOT_SRC_ACT)
        buf.copy_(torch.from_numpy(a.reshape(-1)).to(DEV).to(buf.dtype))
        shards[r] = buf.float().cpu().numpy().astype(np.float64).reshape(-1, W)
    text_np = {}
    if sp is not None:
        codes = cfg.splice["codes"]
        ntext = int((codes < 0).sum())
        T = rng.standard_normal((ntext, cfg.hidden))
        L = cfg.splice["S"] // dst.cp
        for r in dst.stage_ranks(0):
            t, c, p, d = dst.coord(r)
            buf = rt.buffer(r, hbb.SLOT_TEXT)
            if buf is None:
                continue
            if cfg.splice["text_mode"] == hbb.TEXT_SLICE:
                sl = codes.reshape(-1, cfg.splice["S"])[:, c * L:(c + 1) * L].reshape(-1)
                rows = T[[-1 - int(x) for x in sl if x < 0]]
            else:
                rows = T[: buf.numel() // cfg.hidden]
            buf.copy_(torch.from_numpy(rows.reshape(-1)).to(DEV).to(buf.dtype))
            text_np[r] = torch.from_numpy(T).to(buf.dtype).double().numpy()
        if cfg.splice["text_mode"] == hbb.TEXT_INPLACE:
            # in place: the LLM's embedding layer wrote the text rows into the slice;
            # the vision positions hold NaN until the boundary scatters into them
            for r in dst.stage_ranks(0):
                t, c, p, d = dst.coord(r)
                out = rt.buffer(r, hbb.SLOT_DST_ACT)
                text_np[r] = torch.from_numpy(T).to(out.dtype).double().numpy()
                full = O.splice_forward(codes, cfg.splice["Q"], cfg.splice["S"], cfg.hidden, c * L, L,
                                        np.zeros((DI[d][1] * cfg.tokens, cfg.hidden)), text_np[r])
                sl = codes.reshape(-1, cfg.splice["S"])[:, c * L:(c + 1) * L].reshape(-1)
                full[sl >= 0] = np.nan
                out.copy_(torch.from_numpy(full.reshape(-1)).to(DEV).to(out.dtype))
    rt.forward(0)
    torch.cuda.synchronize()
    ref, _, _ = O.bridge_forward(src, dst, B, W, shards)
    for r, a in ref.items():
        if sp is not None:
            t, c, p, d = dst.coord(r)
            L = cfg.splice["S"] // dst.cp
            a = O.splice_forward(cfg.splice["codes"], cfg.splice["Q"], cfg.splice["S"], cfg.hidden, c * L, L,
                                 a.reshape(-1, cfg.hidden), text_np[r])
        got = rt.buffer(r, hbb.SLOT_DST_ACT).double().cpu().numpy()
        np.testing.assert_array_equal(got, a.reshape(-1), err_msg=f"{cfg.name} forward rank {r}")

    # backward
    grads = {}
    vgrads = {}
    G = rng.standard_normal((B, W))
    for r in dst.stage_ranks(0):
        t, c, p, d = dst.coord(r)
        buf = rt.buffer(r, hbb.SLOT_DST_GRAD)
        if sp is None:
            a = G[DI[d][0]:DI[d][0] + DI[d][1]].copy()
            if perturb and t:
                a = a + 3.0 * t  # tp replicas differ: checks which copy the data path reads
        elif perturb:
            a = rng.standard_normal(buf.numel())
        else:
            a = np.random.default_rng(1000 * seed + 10 * c + d).standard_normal(buf.numel())
        buf.copy_(torch.from_numpy(a.reshape(-1)).to(DEV).to(buf.dtype))
        g = buf.double().cpu().numpy()
        if sp is not None:
            L = cfg.splice["S"] // dst.cp
            g = O.splice_backward(cfg.splice["codes"], cfg.splice["Q"], cfg.splice["S"], cfg.hidden, c * L, L,
                                  g.reshape(-1, cfg.hidden), DI[d][1] * cfg.tokens)
        vgrads[r] = g.reshape(-1, W)
    prev = {}
    for r in src.stage_ranks(src.pp - 1):
        buf = rt.buffer(r, hbb.SLOT_SRC_GRAD)
        if beta:
            buf.copy_(torch.randn(buf.numel(), device=DEV).to(buf.dtype))
        else:
            buf.fill_(float("nan"))  # beta=0 must overwrite, never read
        prev[r] = buf.double().cpu().numpy()
    rt.backward(0, beta)
    torch.cuda.synchronize()
    assert rt.status() == 0
    refb, _, _ = O.bridge_backward(src, dst, B, W, vgrads)
    for r, a in refb.items():
        exp = a.reshape(-1) + (beta * prev[r] if beta else 0.0)
        got = rt.buffer(r, hbb.SLOT_SRC_GRAD).double().cpu().numpy()
        if cfg.grad_out == "fp32":
            rel = np.max(np.abs(got - exp) / np.maximum(1.0, np.abs(exp))) if exp.size else 0.0
            if beta == 0 and (dst.cp == 1 or sp is not None):
                np.testing.assert_array_equal(got, exp.astype(np.float32), err_msg=f"{cfg.name} bwd rank {r}")
            assert rel <= REL_TOL, f"{cfg.name} bwd rank {r}: rel {rel}"
        else:
            exp_c = torch.from_numpy(exp).to(TDT[cfg.grad_out]).double().numpy()
            rel = np.max(np.abs(got - exp_c) / np.maximum(1.0, np.abs(exp_c)))
            assert rel <= 8e-3, f"{cfg.name} bwd rank {r}: rel {rel}"
    rt.close()


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c4ip", "c5"])
@pytest.mark.parametrize("beta", [0.0, 1.0])
def test_configs_scaled_vs_oracle(name, beta):
    run_case(configs.get(name, scale=64), seed=sum(map(ord, name)), beta=beta)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5", "c2x4", "c3x4"])
@pytest.mark.parametrize("beta", [0.0, 1.0])
def test_configs_balanced_backward_vs_oracle(name, beta):
    """Default runtime (replica-balanced gradient return) on contract inputs."""
    run_case(configs.get(name, scale=64), seed=len(name) + 7, beta=beta, perturb=False)


@pytest.mark.parametrize("partition", [1, 2, 3, 4])
@pytest.mark.parametrize("name", ["c2", "c4", "c5"])
def test_partition_modes_vs_oracle(name, partition):
    """Every CTA work split (contiguous, interleaved, dynamic, TMA bulk) gives identical results."""
    run_case(configs.get(name, scale=64), seed=7, beta=1.0, partition=partition)


def test_odd_width_all_partition_modes():
    for partition in (1, 2, 3, 4):
        cfg = configs.get("c2", scale=64)
        cfg.tokens, cfg.hidden = 1, 3
        cfg.act = cfg.grad_in = cfg.grad_out = "fp32"
        run_case(cfg, seed=3, beta=1.0, partition=partition)


def test_reference_layout_splice_vs_oracle():
    """Reference-faithful splice: each sample one sequence, vision at [0,S_v) (tinymodel.hpp:24-26)."""
    cfg = configs.get("c4", scale=64)
    n = 8  # samples (= sequences) per destination shard
    S, S_v = 64, cfg.tokens
    cfg.src = hbg.ModuleLayout("vit", dp=8)
    cfg.dst = hbg.ModuleLayout("llm", tp=2, cp=4)
    cfg.batch = n
    q = np.arange(n)[:, None]
    p = np.arange(S)[None, :]
    codes = np.where(p < S_v, q * S_v + p, -1 - (q * (S - S_v) + (p - S_v))).astype(np.int32)
    cfg.splice = {"Q": n, "S": S, "codes": codes.reshape(-1), "text_mode": hbb.TEXT_FULL}
    run_case(cfg, seed=5, beta=1.0)


@pytest.mark.parametrize("act,gin,gout", [("fp32", "fp32", "fp32"), ("bf16", "bf16", "bf16"),
                                          ("fp16", "fp16", "fp32"), ("bf16", "fp32", "fp32")])
def test_dtype_matrix(act, gin, gout):
    cfg = configs.get("c2", scale=128)
    cfg.act, cfg.grad_in, cfg.grad_out = act, gin, gout
    run_case(cfg, seed=11, beta=1.0)


@pytest.mark.parametrize("act,gin,gout", [("fp32", "fp32", "fp32"), ("bf16", "bf16", "bf16"),
                                          ("fp16", "fp16", "fp32"), ("bf16", "fp32", "fp16")])
def test_fan_out_return_dtypes(act, gin, gout):
    """C3 on one GPU: the four encoder TP replicas of each source shard share one
    fan-out reduce segment (terms read once, four accumulators)."""
    cfg = configs.get("c3", scale=128)
    cfg.act, cfg.grad_in, cfg.grad_out = act, gin, gout
    run_case(cfg, seed=13, beta=1.0)


@pytest.mark.parametrize("partition", [1, 2, 3, 4])
@pytest.mark.parametrize("beta", [0.0, 1.0])
def test_fan_out_return_partitions(partition, beta):
    run_case(configs.get("c3", scale=64), seed=17, beta=beta, partition=partition)


def test_fan_out_return_unaligned_rows():
    """W=3 fp32 rows: the fan-out kernel's scalar tail path."""
    cfg = configs.get("c3", scale=64)
    cfg.tokens, cfg.hidden = 1, 3
    cfg.act = cfg.grad_in = cfg.grad_out = "fp32"
    run_case(cfg, seed=19, beta=1.0)


def test_nc_cp_reduction_multi_term():
    """NC edge into an LLM with cp=2: backward sums two cp contributions (fp32, fixed order)."""
    cfg = configs.get("c5", scale=64)
    cfg.dst = hbg.ModuleLayout("llm", tp=1, cp=2, pp=3, rank_offset=2)
    cfg.logical_world = 8
    run_case(cfg, seed=3, beta=0.0)


def test_odd_width_unaligned_rows():
    """W=3 fp32 rows (12 B) exercise the unaligned scalar paths of both kernels."""
    cfg = configs.get("c2", scale=64)
    cfg.tokens, cfg.hidden = 1, 3
    cfg.act = cfg.grad_in = cfg.grad_out = "fp32"
    run_case(cfg, seed=2, beta=1.0)


# ---------------------------------------------------------------- full width


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_full_size_round_trip_identity(name):
    """Full BASELINE shapes: forward placement equals a plain PyTorch
    restatement, and feeding each destination its own activations as gradient
    returns every source owner exactly its own shard (ownership round trip)."""
    _require_gpu()
    cfg = configs.get(name)
    plan = hbb.plan_bridge(cfg.edge())
    sp = None
    if cfg.splice:
        s = cfg.splice
        sp = hbb.SpliceSpec(s["Q"], s["S"], cfg.hidden, cfg.tokens, s["codes"], s["text_mode"])
    rt = hbb.BridgeRuntime(plan, sp, act_dtype=torch.bfloat16, grad_in_dtype=torch.bfloat16,
                           grad_out_dtype=torch.float32)
    src, dst = o_layout(cfg.src), o_layout(cfg.dst)
    W = cfg.width
    SI, DI = O.intervals(cfg.batch, src.dp), O.intervals(cfg.batch, dst.dp)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(7)
    X = torch.randn(cfg.batch, W, generator=gen, device=DEV).to(torch.bfloat16)
    for r in src.stage_ranks(src.pp - 1):
        d = src.coord(r)[3]
        rt.buffer(r, hbb.SLOT_SRC_ACT).copy_(X[SI[d][0]:SI[d][0] + SI[d][1]].reshape(-1))
    if sp is not None:
        for r in dst.stage_ranks(0):
            b = rt.buffer(r, hbb.SLOT_TEXT)
            if b is not None:
                b.fill_(0.5)
    rt.forward(0)
    torch.cuda.synchronize()
    codes = torch.from_numpy(cfg.splice["codes"].astype(np.int64)).to(DEV) if sp is not None else None
    for r in dst.stage_ranks(0):
        t, c, p, d = dst.coord(r)
        got = rt.buffer(r, hbb.SLOT_DST_ACT)
        if sp is None:
            exp = X[DI[d][0]:DI[d][0] + DI[d][1]].reshape(-1)
        else:
            L = cfg.splice["S"] // dst.cp
            cs = codes[c * L:(c + 1) * L]
            vis = X[DI[d][0]:DI[d][0] + DI[d][1]].reshape(-1, cfg.hidden)
            exp = torch.where((cs >= 0)[:, None], vis[cs.clamp(min=0)],
                              torch.full_like(vis[:1], 0.5)).reshape(-1)
        assert torch.equal(got, exp), f"{name} full forward rank {r}"
        rt.buffer(r, hbb.SLOT_DST_GRAD).copy_(got)
    rt.backward(0, 0.0)
    torch.cuda.synchronize()
    for r in src.stage_ranks(src.pp - 1):
        d = src.coord(r)[3]
        got = rt.buffer(r, hbb.SLOT_SRC_GRAD)
        exp = X[SI[d][0]:SI[d][0] + SI[d][1]].reshape(-1).float()
        assert torch.equal(got, exp), f"{name} full round trip rank {r}"
    rt.close()


def test_microbatch_records():
    """backward without a forward record -> UnknownMicrobatch; a record is consumed once."""
    _require_gpu()
    cfg = configs.get("c2", scale=256)
    rt = hbb.BridgeRuntime(hbb.plan_bridge(cfg.edge()))
    with pytest.raises(hbb.HetBridgeError) as ei:
        rt.backward(3)
    assert ei.value.code == "UnknownMicrobatch"
    rt.forward(3)
    with pytest.raises(hbb.HetBridgeError):
        rt.forward(3)
    rt.backward(3)
    with pytest.raises(hbb.HetBridgeError) as ei:
        rt.backward(3)
    assert ei.value.code == "UnknownMicrobatch"
    rt.seed_forward_record(9)
    rt.backward(9)
    torch.cuda.synchronize()
    rt.close()


def test_mb_slots_rotate_buffers():
    """Two microbatches in flight use distinct buffer sets (mb % slots)."""
    _require_gpu()
    cfg = configs.get("c2", scale=256)
    plan = hbb.plan_bridge(cfg.edge())
    rt = hbb.BridgeRuntime(plan, mb_slots=2)
    for s in range(2):
        for r in range(8):
            rt.buffer(r, hbb.SLOT_SRC_ACT, s).fill_(float(10 * s + r))
    rt.forward(0)
    rt.forward(1)
    torch.cuda.synchronize()
    for s in range(2):
        out0 = rt.buffer(0, hbb.SLOT_DST_ACT, s).float().view(4, -1)
        assert torch.equal(out0[:, 0].cpu(), torch.tensor([10.0 * s + i for i in range(4)]))
    rt.close()


# ---------------------------------------------------------------- golden fixtures


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5", "spec_fanin2_nc"])
def test_device_matches_golden_fixture(name):
    """Device path vs the committed oracle fixtures (no oracle library needed at run time)."""
    _require_gpu()
    import json
    import os

    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    with open(os.path.join(gold, name + ".json")) as f:
        meta = json.load(f)
    arr = dict(np.load(os.path.join(gold, name + ".npz")))
    src, dst = O.Layout(*meta["src"]), O.Layout(*meta["dst"])
    B, W = meta["B"], meta["W"]
    plan = hbb.plan_bridge(hbg.BoundaryEdge(to_hb(src), to_hb(dst), B, W))
    sp = None
    if "splice" in meta:
        s = meta["splice"]
        sp = hbb.SpliceSpec(s["Q"], s["S"], meta["hidden"], meta["tokens"], s["codes"], s["text_mode"])
    # fixture gradients differ across tp replicas: the reference data path (strict)
    rt = hbb.BridgeRuntime(plan, sp, act_dtype=torch.float32, grad_in_dtype=torch.float32,
                           grad_out_dtype=torch.float32, strict_provenance=True)
    SI = O.intervals(B, src.dp)
    X = torch.from_numpy(arr["X"]).to(DEV)
    for r in src.stage_ranks(src.pp - 1):
        d = src.coord(r)[3]
        rt.buffer(r, hbb.SLOT_SRC_ACT).copy_(X[SI[d][0]:SI[d][0] + SI[d][1]].reshape(-1))
    if sp is not None:
        codes = np.asarray(meta["splice"]["codes"])
        L = meta["splice"]["S"] // dst.cp
        for r in dst.stage_ranks(0):
            c = dst.coord(r)[1]
            sl = codes.reshape(-1, meta["splice"]["S"])[:, c * L:(c + 1) * L].reshape(-1)
            rows = [-1 - int(x) for x in sl if x < 0]
            if meta["splice"]["text_mode"] != 1:
                rows = list(range(len(arr["text"])))
            b = rt.buffer(r, hbb.SLOT_TEXT)
            b.copy_(torch.from_numpy(arr["text"][rows].reshape(-1)).to(DEV)[: b.numel()])
    for r in dst.stage_ranks(0):
        rt.buffer(r, hbb.SLOT_DST_GRAD).copy_(torch.from_numpy(arr[f"grad_r{r}"].reshape(-1)).to(DEV))
    rt.forward(0)
    rt.backward(0, 0.0)
    torch.cuda.synchronize()
    for r in dst.stage_ranks(0):
        got = rt.buffer(r, hbb.SLOT_DST_ACT).cpu().numpy()
        np.testing.assert_array_equal(got, arr[f"fwd_r{r}"].reshape(-1), err_msg=f"{name} fwd rank {r}")
    for r in src.stage_ranks(src.pp - 1):
        got = rt.buffer(r, hbb.SLOT_SRC_GRAD).cpu().numpy()
        np.testing.assert_allclose(got, arr[f"bwd_r{r}"].reshape(-1), rtol=1e-6, atol=1e-6,
                                   err_msg=f"{name} bwd rank {r}")
    rt.close()


def test_cuda_graph_replay_matches_direct_calls():
    _require_gpu()
    cfg = configs.get("c4", scale=64)
    plan = hbb.plan_bridge(cfg.edge())
    s = cfg.splice
    sp = hbb.SpliceSpec(s["Q"], s["S"], cfg.hidden, cfg.tokens, s["codes"], s["text_mode"])
    outs = []
    for use_graph in (False, True, "cycle"):
        rt = hbb.BridgeRuntime(plan, sp, mb_slots=2)
        g = torch.Generator(device=DEV)
        g.manual_seed(3)
        for k in range(2):
            for r in range(8):
                for slot in (hbb.SLOT_SRC_ACT, hbb.SLOT_TEXT, hbb.SLOT_DST_GRAD):
                    b = rt.buffer(r, slot, k)
                    if b is not None:
                        b.copy_(torch.randn(b.numel(), generator=g, device=DEV).to(b.dtype))
                rt.buffer(r, hbb.SLOT_SRC_GRAD, k).zero_()
        st = torch.cuda.Stream()
        if use_graph == "cycle":  # one graph = a step on each buffer set in turn
            rt.capture_step(0, 1.0, True, st, what=rt.GRAPH_CYCLE)
            for i in range(2):
                rt.replay_step(0, st, rt.GRAPH_CYCLE)
        elif use_graph:
            for k in range(2):
                rt.capture_step(k, 1.0, True, st)
            for i in range(4):
                rt.replay_step(i % 2, st)
        else:
            for i in range(4):
                rt.forward(i, st)
                rt.backward(i, 1.0, st)
        st.synchronize()
        outs.append([rt.buffer(r, sl, k).clone() for k in range(2) for r in range(8)
                     for sl in (hbb.SLOT_DST_ACT, hbb.SLOT_SRC_GRAD)])
        assert rt.stats()["launches"] == 8
        if use_graph is True:  # forward-only and backward-only graphs replay too
            rt.capture_step(0, 1.0, stream=st, what=rt.GRAPH_FWD)
            rt.capture_step(0, 1.0, stream=st, what=rt.GRAPH_BWD)
            rt.replay_step(0, st, rt.GRAPH_FWD)
            rt.replay_step(0, st, rt.GRAPH_BWD)
            st.synchronize()
            assert rt.stats()["launches"] == 10
        rt.close()
    for other in outs[1:]:
        for a, b in zip(outs[0], other):
            assert torch.equal(a, b)
