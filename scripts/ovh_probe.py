"""Fixed-cost probe on one GPU: tiny C2 step, graph replay, variants."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_27678_b200 import bridge as hbb, configs
cfg = configs.get("c2", scale=4096)
plan = hbb.plan_bridge(cfg.edge())
res = {}
for part in (1, 3, 4):
    rt = hbb.BridgeRuntime(plan, partition=part, mb_slots=1)
    st = torch.cuda.Stream()
    for name, fn in (("fwd", lambda: rt.capture_step(0, 1.0, False, st)), ("fwdbwd", lambda: rt.capture_step(0, 1.0, True, st))):
        fn()
        for _ in range(20): rt.replay_step(0, st)
        st.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(st)
        for _ in range(200): rt.replay_step(0, st)
        e1.record(st); st.synchronize()
        res[f"part{part}_{name}_us"] = round(e0.elapsed_time(e1) / 200 * 1e3, 2)
    rt.close()
# empty-kernel floor: torch tiny op
x = torch.zeros(1, device="cuda")
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        x.add_(1)
    for _ in range(20): g.replay()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(st)
    for _ in range(200): g.replay()
    e1.record(st); st.synchronize()
res["torch_tiny_graph_us"] = round(e0.elapsed_time(e1) / 200 * 1e3, 2)
print(json.dumps(res))
