"""Device parity over a sweep of layout pairs (the CPU sweep of
tests/test_index_map.py::test_sweep_vs_oracle, on the GPU): every 5th valid
(encoder, LLM) pair of <= 8 ranks — tp, pp in {1, 2}, cp in {1, 2}, dp in {1, 2, 4},
colocated and disjoint — runs forward + accumulated backward on an exec group of
up to four (virtual) GPUs and is compared with the oracle: placement bit-exact,
gradients within 1e-6. Equal-DP, fan-in, fan-out, deliver and cp-reduce
routes all occur in the sample."""
import itertools

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from parity_core import LocalGroupDriver, group_parity  # noqa: E402

from paper_2605_27678_b200 import bridge as hbb  # noqa: E402
from paper_2605_27678_b200.configs import BoundaryConfig  # noqa: E402
from paper_2605_27678_b200.grid import ModuleLayout  # noqa: E402


def _sample(every=5):
    cases, k = [], 0
    for stp, spp, sdp in itertools.product((1, 2), (1, 2), (1, 2, 4)):
        for dtp, dcp, dpp, ddp in itertools.product((1, 2), (1, 2), (1, 2), (1, 2, 4)):
            s = ModuleLayout("enc", tp=stp, pp=spp, dp=sdp)
            for colo in (True, False):
                d = ModuleLayout("llm", tp=dtp, cp=dcp, pp=dpp, dp=ddp, rank_offset=0 if colo else s.world_size())
                if colo and s.world_size() != d.world_size():
                    continue
                if d.rank_end() > 8:
                    continue
                try:
                    hbb.plan_bridge(hbb.BoundaryEdge(s, d, 8, 256))
                except hbb.HetBridgeError:
                    continue
                if k % every == 0:
                    cases.append((s, d))
                k += 1
    return cases


CASES = _sample()


def _label(case):
    s, d = case
    return f"enc-tp{s.tp}pp{s.pp}dp{s.dp}__llm-tp{d.tp}cp{d.cp}pp{d.pp}dp{d.dp}@{d.rank_offset}"


@pytest.mark.parametrize("case", CASES, ids=[_label(c) for c in CASES])
def test_layout_sweep_on_exec_group(case):
    s, d = case
    cfg = BoundaryConfig("sweep", _label(case), s, d, 8, 4, 64)  # 8 samples of 4 tokens x 64
    plan = hbb.plan_bridge(cfg.edge())
    n = min(4, plan.world)
    devs = list(range(n)) if torch.cuda.device_count() >= n else [0] * n
    g = hbb.LocalGroup(plan, None, devices=devs, act_dtype=torch.bfloat16, grad_in_dtype=torch.bfloat16,
                       grad_out_dtype=torch.float32, timeout_s=20.0)
    try:
        ok, worst = group_parity(cfg, LocalGroupDriver(g), steps=2)
        assert ok, f"{_label(case)}: worst backward rel {worst}"
        assert all(rt.status() == 0 for rt in g.rts)
    finally:
        g.close()


def test_sweep_covers_every_route():
    kinds = set()
    for s, d in CASES:
        p = hbb.plan_bridge(hbb.BoundaryEdge(s, d, 8, 256))
        text = hbb.export_plan(p)
        for key in ("gather", "deliver", "reduce", "send", "bcast"):
            if key in text.lower():
                kinds.add(key)
    assert len(CASES) >= 30
    assert {"gather", "deliver", "reduce"} <= kinds, kinds
