"""Plan compilation: product plan_bridge/export_plan vs the oracle, and the
SPEC.md prose known-answer tests."""
import itertools

import pytest

from helpers import O, hb_plan, to_hb
from paper_2605_27678_b200 import HetBridgeError
from paper_2605_27678_b200 import bridge as B
from paper_2605_27678_b200 import grid as G


def edge(src, dst, Bt=8, W=3):
    return G.BoundaryEdge(to_hb(src), to_hb(dst), Bt, W)


def sweep_layouts():
    for stp, spp, sdp in itertools.product((1, 2), (1, 2), (1, 2, 4)):
        for dtp, dcp, dpp, ddp in itertools.product((1, 2), (1, 2), (1, 2), (1, 2, 4)):
            s = O.Layout("enc", stp, 1, spp, sdp, 0)
            for colo in (True, False):
                d = O.Layout("llm", dtp, dcp, dpp, ddp, 0 if colo else s.world_size)
                if colo and s.world_size != d.world_size:
                    continue
                yield s, d


def test_export_text_identical_to_oracle_sweep():
    n = 0
    for s, d in sweep_layouts():
        for Bt in (8, 16):
            try:
                ref = O.export_plan(s, d, Bt, 3)
            except O.OracleError as e:
                ref = ("err", e.code)
            try:
                got = B.export_plan(hb_plan(s, d, Bt, 3))
            except HetBridgeError as e:
                got = ("err", e.status)
            assert got == ref, (s, d, Bt)
            n += 1
    assert n > 400


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_export_identical_on_baseline_configs(name):
    from paper_2605_27678_b200 import configs

    cfg = configs.get(name)
    s = O.Layout(cfg.src.name, cfg.src.tp, cfg.src.cp, cfg.src.pp, cfg.src.dp, cfg.src.rank_offset)
    d = O.Layout(cfg.dst.name, cfg.dst.tp, cfg.dst.cp, cfg.dst.pp, cfg.dst.dp, cfg.dst.rank_offset)
    assert B.export_plan(B.plan_bridge(cfg.edge())) == O.export_plan(s, d, cfg.batch, cfg.width)


def test_export_elem_bytes_scaling():
    p = hb_plan(O.Layout("enc", dp=4), O.Layout("llm", dp=2, rank_offset=4), 8, 3)
    t8, t2 = B.export_plan(p, 8), B.export_plan(p, 2)
    assert "bytes=48" in t8 and "bytes=12" in t2  # [0,2) x 3 elems x {8,2} B


# ---- classify_dp_relation
def test_classify_kats():
    assert B.classify_dp_relation(edge(O.Layout("u", dp=4), O.Layout("v", dp=2))) == B.DpRelation(B.DpKind.FanIn, 2)
    assert B.classify_dp_relation(edge(O.Layout("u", dp=8), O.Layout("v", dp=8))) == B.DpRelation(B.DpKind.Equal, 1)
    assert B.classify_dp_relation(edge(O.Layout("u", dp=2), O.Layout("v", dp=8))) == B.DpRelation(B.DpKind.FanOut, 4)
    with pytest.raises(HetBridgeError) as ei:
        B.classify_dp_relation(edge(O.Layout("u", dp=3), O.Layout("v", dp=2)))
    assert ei.value.code == "NonIntegerFan"


# ---- plan_bridge
def test_nc_plan_kat():
    """NC enc tp1 dp4 -> llm tp2 dp2, B=8: 4 records; dest0 gets [0,2) then [2,4); 1 TP peer each."""
    src, dst = O.Layout("enc", tp=1, dp=4), O.Layout("llm", tp=2, dp=2, rank_offset=4)
    p = hb_plan(src, dst, 8, 3)
    assert p.placement == G.Placement.NonColocated
    assert p.cross_boundary_messages() == 4
    lines = B.export_plan(p).splitlines()
    sends = [ln for ln in lines if ln.startswith("fwd send")]
    assert sends[:2] == ["fwd send r0 -> r4 [0,2) bytes=48", "fwd send r1 -> r4 [2,4) bytes=48"]
    assert "fwd broadcast root=r4 group=[4,5] [0,4) bytes=96" in lines
    assert O.interval_oracle(8, 4, 2)[0] == [(0, (0, 2)), (1, (2, 2))]


def test_width_invariance_of_cross_boundary_messages():
    """S:171 / acceptance 4: NC fan-in 2 at B=8; TP widths {1,2,4} never change the count."""
    for stp, dtp in itertools.product((1, 2, 4), (1, 2, 4)):
        src = O.Layout("enc", tp=stp, dp=4)
        dst = O.Layout("llm", tp=dtp, dp=2, rank_offset=src.world_size)
        p = hb_plan(src, dst, 8, 3)
        assert p.cross_boundary_messages() == max(4, 2)


def test_colocated_locality():
    """S:172 / acceptance 5: equal-DP colocated -> no collective; fan-in ratio 2 -> groups of exactly 2."""
    eq = B.export_plan(hb_plan(O.Layout("enc", dp=8), O.Layout("llm", dp=8), 16, 3))
    assert "all_gather" not in eq and "deliver" not in eq and "send" not in eq
    fan = B.export_plan(hb_plan(O.Layout("enc", dp=8), O.Layout("llm", tp=2, dp=4), 16, 3))
    groups = [ln.split("group=")[1].split()[0] for ln in fan.splitlines() if "fwd all_gather" in ln]
    assert groups and all(len(g.strip("[]").split(",")) == 2 for g in groups)
    _, led, _ = O.bridge_forward(O.Layout("enc", dp=8), O.Layout("llm", dp=8), 16, 3,
                                 {r: __import__("numpy").zeros((2, 3)) for r in range(8)})
    assert sum(m for m, _ in led.values()) == 0


def test_plan_intervals_equal_interval_oracle():
    """Acceptance 3: plan interval records == brute-force interval oracle, B <= 64, dp in {1,2,4,8}."""
    for Bt in range(1, 65):
        for du, dv in itertools.product((1, 2, 4, 8), repeat=2):
            if Bt % du or Bt % dv:
                continue
            src, dst = O.Layout("enc", dp=du), O.Layout("llm", dp=dv, rank_offset=du)
            text = B.export_plan(hb_plan(src, dst, Bt, 1))
            got = [[] for _ in range(dv)]
            for ln in text.splitlines():
                if ln.startswith("fwd send"):
                    _, _, a, _, b, iv, _ = ln.split()
                    s_leader, d_leader = int(a[1:]), int(b[1:])
                    st, en = (int(x) for x in iv.strip("[)").split(","))
                    got[d_leader - du].append((s_leader, (st, en - st)))
            brute = [[] for _ in range(dv)]
            for j in range(Bt):
                s, d = j * du // Bt, j * dv // Bt
                if brute[d] and brute[d][-1][0] == s:
                    brute[d][-1] = (s, (brute[d][-1][1][0], brute[d][-1][1][1] + 1))
                else:
                    brute[d].append((s, (j, 1)))
            assert got == brute == O.interval_oracle(Bt, du, dv)


def test_plan_errors():
    with pytest.raises(HetBridgeError) as ei:  # PartialOverlap, not PlanInfeasible
        hb_plan(O.Layout("a", dp=6), O.Layout("b", dp=4, rank_offset=4), 24, 1)
    assert ei.value.code == "PartialOverlap"
    with pytest.raises(HetBridgeError) as ei:
        hb_plan(O.Layout("a", dp=4), O.Layout("b", dp=2, rank_offset=4), 6, 1)
    assert ei.value.code == "IndivisibleBatch"
    with pytest.raises(HetBridgeError) as ei:
        hb_plan(O.Layout("a", dp=4), O.Layout("b", dp=2, rank_offset=4), 8, 0)
    assert ei.value.code == "InvalidArgument"


def test_plan_is_deterministic():
    s, d = O.Layout("vit", dp=8), O.Layout("llm", tp=2, cp=4)
    assert len({B.export_plan(hb_plan(s, d, 16, 5)) for _ in range(5)}) == 1
