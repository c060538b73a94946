"""The roofline's algorithmic bytes (bench.traffic_model, DESIGN §4/§6) against the
per-GPU figures SURVEY §8(d) derives by hand for the 8-GPU configs, and the
payload accounting of the BASELINE metric. CPU only."""
import pytest

import bench
from paper_2605_27678_b200 import configs

MB = 1e6
PK = {"hbm_gbs": 6539.2, "nvl_gbs": 770.0}


def tm8(name):
    return bench.traffic_model(configs.get(name), 8)


def test_c2_fan_in_8_gpus():
    t = tm8("c2")
    # fwd: out 151.0 MB + own read 37.75 + served to 3 peers -> 302.0 MB HBM, 113.2 MB NVLink in
    assert all(x == pytest.approx(302.0 * MB, rel=1e-3) for x in t["fwd_hbm"])
    assert all(x == pytest.approx(113.2 * MB, rel=1e-3) for x in t["fwd_nvl"])
    # bwd: 37.75 MB bf16 read + fp32 accumulator read-modify-write
    assert all(x == pytest.approx(188.7 * MB, rel=1e-3) for x in t["bwd_hbm"])
    assert not any(t["bwd_nvl"])


def test_c3_fan_out_8_gpus():
    t = tm8("c3")
    assert all(x == pytest.approx(94.4 * MB, rel=1e-3) for x in t["fwd_hbm"])
    assert not any(t["fwd_nvl"])
    assert all(x == pytest.approx(141.6 * MB, rel=1e-3) for x in t["bwd_nvl"])
    assert all(x == pytest.approx(943.7 * MB, rel=1e-3) for x in t["bwd_hbm"])


def test_c4_cp_splice_8_gpus():
    t = tm8("c4")
    # each GPU writes its 8192-position slice (67.1 MB) and reads what it copies locally
    assert all(x == pytest.approx(134.2 * MB, rel=1e-3) for x in t["fwd_hbm"])
    # vision rows from other GPUs: whole images (4.72 MB each), 3-4 per slice
    img = 576 * 4096 * 2
    assert all(x % img == 0 and 3 * img <= x <= 4 * img for x in t["fwd_nvl"])
    # grads come back from one of the two TP replicas (the owner's own GPU when it holds one)
    assert 0 < sum(t["bwd_nvl"]) <= sum(t["fwd_nvl"]) / 2


def test_c5_noncolocated_8_gpus():
    t = tm8("c5")
    # dest leader's TP pair (GPUs 2, 3) each ingest 16 images; the return splits over both replicas
    assert t["fwd_nvl"][2] == t["fwd_nvl"][3] == pytest.approx(75.5 * MB, rel=1e-3)
    assert sum(t["fwd_nvl"]) == t["fwd_nvl"][2] + t["fwd_nvl"][3]
    assert t["bwd_nvl"][0] == t["bwd_nvl"][1] == pytest.approx(37.75 * MB, rel=1e-3)
    assert t["bwd_hbm"][2] == t["bwd_hbm"][3]  # balanced return: both replicas serve half


def test_tstar_8_gpus_binding_resource():
    f = bench.kernel_bound(tm8("c2"), "fwd", 1.0, PK, 8)
    b = bench.kernel_bound(tm8("c2"), "bwd", 1.0, PK, 8)
    assert f["bound"] == "nvlink" and f["tstar_ms"] * 1e3 == pytest.approx(113.25e6 / 770e9 * 1e6, rel=5e-3)
    assert b["bound"] == "hbm" and b["tstar_ms"] * 1e3 == pytest.approx(188.74e6 / 6539.2e9 * 1e6, rel=5e-3)
    assert bench.kernel_bound(tm8("c3"), "bwd", 1.0, PK, 8)["bound"] == "nvlink"


def test_one_gpu_is_hbm_only():
    for name in ("c2", "c3", "c4", "c5"):
        t = bench.traffic_model(configs.get(name), 1)
        assert t["fwd_nvl"] == [0] and t["bwd_nvl"] == [0]


def test_payload_bytes():
    fwd, bwd = bench.payload_bytes(configs.get("c2"))
    assert fwd == 8 * 32 * 576 * 4096 * 2  # every LLM rank's 32-sample shard
    assert bwd == 64 * 576 * 4096 * 2      # every sample's gradient returned once


def test_reference_arm_line_contract():
    """`bench.py --impl reference` (the reference CPU path on host cores) prints one
    JSON line with the contract's keys; runs here without a GPU."""
    import json
    import os
    import subprocess
    import sys

    if not os.path.exists(os.path.join(bench.ROOT, "oracle", "_ref", "libhb_oracle.so")):
        pytest.skip("oracle not built")
    r = subprocess.run([sys.executable, os.path.join(bench.ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=300,
                       env={**os.environ, "RANK": "0"})
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    assert line["e2e"] == {"value": line["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]


def test_nvlink_egress_balances_ingress():
    """Every byte one GPU pulls over NVLink is served by another: total egress
    equals total ingress, per direction, for every config at 2, 4 and 8 GPUs."""
    for name in ("c2", "c3", "c4", "c5"):
        for n in (2, 4, 8):
            t = bench.traffic_model(configs.get(name), n)
            for kind in ("fwd", "bwd"):
                assert sum(t[kind + "_nvl"]) == sum(t[kind + "_nvl_out"])


def test_paired_bound_is_the_shared_resource_bound():
    """A 1F1B-paired step shares each GPU's HBM and links between the two ops:
    its bound is max over GPUs of max(HBM sum, NVLink sum), never more than the
    serial sum of the two kernels' bounds and never less than either of them."""
    for name in ("c2", "c3", "c4"):
        for n in (1, 4, 8):
            t = bench.traffic_model(configs.get(name), n)
            paired, crit = bench.paired_bound(t, PK, n)
            f = bench.kernel_bound(t, "fwd", 1.0, PK, n)["tstar_ms"]
            b = bench.kernel_bound(t, "bwd", 1.0, PK, n)["tstar_ms"]
            assert max(f, b) * (1 - 1e-3) <= paired <= (f + b) * (1 + 1e-3)  # (kernel_bound rounds to 0.1 us)
            assert crit is not None and crit[1] in ("hbm", "nvlink")
    # one GPU: everything is HBM, so pairing cannot beat the serial sum
    t = bench.traffic_model(configs.get("c2"), 1)
    paired, _ = bench.paired_bound(t, PK, 1)
    f = bench.kernel_bound(t, "fwd", 1.0, PK, 1)["tstar_ms"]
    b = bench.kernel_bound(t, "bwd", 1.0, PK, 1)["tstar_ms"]
    assert paired == pytest.approx(f + b, rel=1e-3)


def test_reduce_kernel_label_follows_the_kernel_that_runs(monkeypatch):
    cfg = configs.get("c4")
    assert bench.reduce_kernel_name(cfg, bench.traffic_model(cfg, 1)).startswith("reduce_segments_kernel<")
    assert bench.reduce_kernel_name(cfg, bench.traffic_model(cfg, 4)).startswith("reduce_segments_stream_kernel<")
    monkeypatch.setenv("HB_RED_STREAM", "0")
    assert bench.reduce_kernel_name(cfg, bench.traffic_model(cfg, 4)).startswith("reduce_segments_kernel<")


def test_payload_counts_what_the_boundary_writes():
    """The forward payload is the destination elements the boundary writes: the
    whole destination shards for copy splices (= DST_ACT sizes), only the vision
    rows for the in-place splice (the LLM's embedding layer wrote the text)."""
    from paper_2605_27678_b200 import bridge as hbb

    for name in ("c1", "c2", "c3", "c4", "c5"):
        cfg = configs.get(name)
        plan = hbb.plan_bridge(cfg.edge())
        sp = bench.make_splice(cfg)
        dst = sum(hbb.buffer_elems(plan, r, hbb.SLOT_DST_ACT, sp) for r in range(plan.world))
        assert bench.payload_bytes(cfg)[0] == dst * bench.DT_SIZE[cfg.act]
    c4, ip = configs.get("c4"), configs.get("c4ip")
    vision = 16 * 576 * 4096 * 2 * 2  # 16 images x 576 tokens x d_h, bf16, written into both tp replicas
    assert bench.payload_bytes(ip)[0] == vision
    assert bench.payload_bytes(ip)[1] == bench.payload_bytes(c4)[1]
    t, ti = bench.traffic_model(c4, 8), bench.traffic_model(ip, 8)
    assert all(a < b for a, b in zip(ti["fwd_hbm"], t["fwd_hbm"]))
    assert ti["fwd_nvl"] == t["fwd_nvl"]
