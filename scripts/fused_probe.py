"""Fused projector + forward reshard vs (GEMM into the source shards, then the
forward reshard), C2 layouts on one GPU at full size (d_h 4096, K = encoder width)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_27678_b200 import bridge as hbb, configs  # noqa: E402
from paper_2605_27678_b200.projector import projector_gemm  # noqa: E402


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for name in ("c2", "c3"):
    cfg = configs.get(name)
    plan = hbb.plan_bridge(cfg.edge())
    rt = hbb.BridgeRuntime(plan)
    d_h = cfg.hidden
    srcs = rt.local_ranks(hbb.SLOT_SRC_ACT)
    views = [rt.buffer(r, hbb.SLOT_SRC_ACT).view(-1, d_h) for r in srcs]
    rows = sum(v.shape[0] for v in views)
    for K in (1024, 1280):
        x = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
        w = torch.randn(d_h, K, device="cuda").to(torch.bfloat16)
        xs = list(torch.split(x, [v.shape[0] for v in views]))
        mb = [0]

        def fused():
            rt.forward_projected(mb[0], x, w)
            rt.seed_forward_record(-1)
            rt.backward  # noqa: B018
            mb[0] += 1

        def fused_step():
            rt.forward_projected(0, x, w)
            rt.seed_forward_record(0)
            rt.backward(0, 1.0)

        def cublas_step():
            for xi, v in zip(xs, views):
                torch.matmul(xi, w.t(), out=v)
            rt.forward(0)
            rt.backward(0, 1.0)

        def ours_step():
            for xi, v in zip(xs, views):
                projector_gemm(xi, w, out=v)
            rt.forward(0)
            rt.backward(0, 1.0)

        def gemm_only():
            for xi, v in zip(xs, views):
                torch.matmul(xi, w.t(), out=v)

        res = {"cfg": name, "K": K, "rows": rows, "d_h": d_h,
               "fused_proj_fwd_bwd_ms": round(t(fused_step), 4),
               "cublas_gemm_then_fwd_bwd_ms": round(t(cublas_step), 4),
               "our_gemm_then_fwd_bwd_ms": round(t(ours_step), 4),
               "cublas_gemms_only_ms": round(t(gemm_only), 4)}
        print(json.dumps(res), flush=True)
    rt.close()
