"""Fixed-cost probe on one GPU: tiny steps (hidden /4096) with the host out of the loop.

R fwd / bwd / fwd+bwd ops are captured into ONE CUDA graph (torch capture around
the C-ABI launches), so the mean per op is the GPU-side cost, not the Python +
cudaGraphLaunch dispatch rate. Also: the same for a one-CTA torch op."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_27678_b200 import bridge as hbb, configs  # noqa: E402

R = 50


def per_op_us(body, st):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        body()  # warm (and prepare tables) outside the capture
        st.synchronize()
        with torch.cuda.graph(g, stream=st):
            for _ in range(R):
                body()
    with torch.cuda.stream(st):  # replay() launches on the current stream
        for _ in range(3):
            g.replay()
        st.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(st)
        for _ in range(10):
            g.replay()
        e1.record(st)
    st.synchronize()
    return round(e0.elapsed_time(e1) / (10 * R) * 1e3, 2)


name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = configs.get(name, scale=int(os.environ.get("SCALE", "4096")))
plan = hbb.plan_bridge(cfg.edge())
sp = None
if cfg.splice:
    s = cfg.splice
    sp = hbb.SpliceSpec(s["Q"], s["S"], cfg.hidden, cfg.tokens, s["codes"], s["text_mode"])
res = {"config": cfg.name, "scale": os.environ.get("SCALE", "4096")}
st = torch.cuda.Stream()
for part in (1, 3, 4):
    for bps in (0, 1):
        rt = hbb.BridgeRuntime(plan, sp, partition=part, mb_slots=1, blocks_per_sm=bps)
        mb = [0]

        def f():
            rt.forward(mb[0], st)
            mb[0] += 1
        res[f"part{part}_bps{bps}_fwd_us"] = per_op_us(f, st)

        def b():
            rt.seed_forward_record(mb[0])
            rt.backward(mb[0], 1.0, st)
            mb[0] += 1
        res[f"part{part}_bps{bps}_bwd_us"] = per_op_us(b, st)

        def fb():
            rt.forward(mb[0], st)
            rt.backward(mb[0], 1.0, st)
            mb[0] += 1
        res[f"part{part}_bps{bps}_fwdbwd_us"] = per_op_us(fb, st)
        rt.close()
x = torch.zeros(1, device="cuda")
res["torch_tiny_op_us"] = per_op_us(lambda: x.add_(1), st)
y = torch.zeros(148 * 2 * 512, device="cuda")
res["torch_296x512_op_us"] = per_op_us(lambda: y.add_(1), st)
print(json.dumps(res))
