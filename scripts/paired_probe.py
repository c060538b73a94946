"""Fused paired step kernel vs the serial cycle at N=1 (one GPU, full-size
configs): per-step time of graph what=5 (one paired_step_kernel launch per
step) and what=3 (forward then backward), CUDA events. Under ncu the launch
list shows the kernels each graph runs. Measurement tool only.

  python scripts/paired_probe.py [c2 c4 ...]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_27678_b200 import bridge as hbb  # noqa: E402
from paper_2605_27678_b200 import configs  # noqa: E402

TDT = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}


def one(name, slots=4, cycles=int(os.environ.get("PROBE_CYCLES", "25"))):
    cfg = configs.get(name)
    plan = hbb.plan_bridge(cfg.edge())
    rt = hbb.BridgeRuntime(plan, bench.make_splice(cfg), act_dtype=TDT[cfg.act], grad_in_dtype=TDT[cfg.grad_in],
                           grad_out_dtype=TDT[cfg.grad_out], mb_slots=slots)
    st = torch.cuda.Stream()
    dev = torch.device("cuda", 0)
    try:
        bench.fill_inputs(rt, list(range(plan.world)), slots, dev)
        out = {"config": name}
        for label, what in (("serial", rt.GRAPH_CYCLE), ("fused", rt.GRAPH_PAIRED_FUSED)):
            rt.capture_step(0, cfg.beta, True, st, what=what)
            rt.replay_step(0, st, what)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(cycles):
                rt.replay_step(0, st, what)
            b.record(st)
            st.synchronize()
            out[label + "_ms_per_step"] = round(a.elapsed_time(b) / (cycles * slots), 5)
        assert rt.status() == 0
        return out
    finally:
        rt.close()


if __name__ == "__main__":
    for n in sys.argv[1:] or ["c2", "c3", "c4", "c4ip", "c5"]:
        print(json.dumps(one(n)), flush=True)
