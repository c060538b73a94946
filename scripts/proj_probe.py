"""Projector GEMM throughput vs cuBLAS (torch.matmul) on the projector shapes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_27678_b200.projector import projector_gemm_rows  # noqa: E402


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


for M, N, K in [(4608, 4096, 1024), (4608, 4096, 1280), (4608, 5120, 1280), (16384, 4096, 4096), (8192, 8192, 8192)]:
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    rows = out.data_ptr() + torch.arange(M, device="cuda", dtype=torch.int64) * (N * 2)  # row table built once
    ms = t(lambda: projector_gemm_rows(x, w, rows, 1))
    ms_cb = t(lambda: torch.matmul(x, w.t(), out=out))
    fl = 2 * M * N * K
    print(json.dumps({"M": M, "N": N, "K": K, "ours_ms": round(ms, 4), "ours_tflops": round(fl / ms / 1e9, 1),
                      "cublas_ms": round(ms_cb, 4), "cublas_tflops": round(fl / ms_cb / 1e9, 1),
                      "out_gbs_ours": round(M * N * 2 / ms / 1e6, 1)}))
