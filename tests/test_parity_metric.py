"""parity_compare / ParityReport (oracle.hpp:53-75) and the
bench's counter-hash inputs (CPU)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import bench  # noqa: E402

from paper_2605_27678_b200 import parity as P  # noqa: E402
from paper_2605_27678_b200._lib import HetBridgeError  # noqa: E402


def test_identical_states_report_zero():
    a = {"x": np.arange(6.0).reshape(2, 3), "y": np.ones(4)}
    rep = P.parity_compare(a, {k: v.copy() for k, v in a.items()}, tolerance=1e-10)
    assert rep.passed and all(i.max_rel == 0.0 for i in rep.items)
    assert "parity tensor=x max_rel=0 pass=1" in rep.render_machine()


def test_worst_first_and_metric():
    a = {"small": np.array([1.0, 2.0]), "big": np.array([10.0, 0.5])}
    b = {"small": np.array([1.0, 2.0 + 1e-9]), "big": np.array([12.0, 0.5])}
    rep = P.parity_compare(a, b, tolerance=1e-6)
    assert [i.tensor for i in rep.items] == ["big", "small"]
    assert rep.items[0].max_rel == pytest.approx(2.0 / 12.0)  # |a-b| / max(1, |b|)
    assert rep.items[1].max_rel == pytest.approx(1e-9 / 2.0)
    assert not rep.passed


def test_structure_mismatch():
    with pytest.raises(HetBridgeError) as ei:
        P.parity_compare({"a": np.zeros(2)}, {"b": np.zeros(2)})
    assert ei.value.code == "StructureMismatch"
    with pytest.raises(HetBridgeError):
        P.parity_compare({"a": np.zeros(2)}, {"a": np.zeros(3)})


def test_fill_values_deterministic_and_finite():
    a = bench.fill_values(100_000, bench.input_key(1, 0, 3), torch.bfloat16, "cpu")
    b = bench.fill_values(100_000, bench.input_key(1, 0, 3), torch.bfloat16, "cpu")
    c = bench.fill_values(100_000, bench.input_key(1, 0, 4), torch.bfloat16, "cpu")
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    assert not torch.equal(a.view(torch.int16), c.view(torch.int16))
    f = a.float()
    assert torch.isfinite(f).all() and (f.abs() >= 2.0 ** -9).all() and (f.abs() < 2.0 ** 7).all()
    assert (f < 0).any() and (f > 0).any()
    # positions are distinguishable: few equal neighbours (a misplaced run is detected)
    assert float((a[1:] == a[:-1]).float().mean()) < 0.01
    assert torch.equal(bench.fill_values(1000, 5, torch.float32, "cpu"), bench.fill_values(1000, 5, torch.bfloat16,
                                                                                              "cpu").float())


def test_restatement_matches_numpy_executor():
    """expected_forward/backward equal the numpy executor of the same maps."""
    from helpers import apply_backward, apply_forward

    from paper_2605_27678_b200 import bridge as hbb
    from paper_2605_27678_b200 import configs

    cfg = configs.get("c3", scale=256)
    plan = hbb.plan_bridge(cfg.edge())
    fwd, bwd = hbb.index_forward(plan), hbb.index_backward(plan, balanced=True)
    bufs = {}
    for r in range(plan.world):
        for slot in (hbb.SLOT_SRC_ACT, hbb.SLOT_DST_GRAD):
            n = hbb.buffer_elems(plan, r, slot)
            if n:
                bufs[(r, slot)] = bench.fill_values(n, bench.input_key(0, slot, r), torch.bfloat16, "cpu")
    npb = {k: v.float().double().numpy() for k, v in bufs.items()}
    ref_f = apply_forward(plan, npb)
    prev = {}
    for r in range(plan.world):
        n = hbb.buffer_elems(plan, r, hbb.SLOT_SRC_GRAD)
        if n:
            prev[(r, hbb.SLOT_SRC_GRAD)] = np.linspace(-3, 3, n)
    ref_b = apply_backward(plan, npb, prev=prev, beta=1.0, balanced=True)
    for (r, slot), exp in ref_f.items():
        got, cov = P.expected_forward(fwd, r, hbb.buffer_elems(plan, r, slot), lambda a, b: bufs[(a, b)])
        assert cov == exp.size and np.array_equal(got.float().double().numpy(), exp)
    for (r, slot), exp in ref_b.items():
        pv = torch.from_numpy(prev[(r, slot)]).float()
        got = P.expected_backward(bwd, r, pv, 1.0, lambda a, b: bufs[(a, b)])
        assert np.max(np.abs(got.double().numpy() - exp) / np.maximum(1, np.abs(exp))) < 1e-6
