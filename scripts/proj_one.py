import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_27678_b200.projector import projector_gemm
M, N, K = 4608, 4096, 1280
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    projector_gemm(x, w, out)
torch.matmul(x, w.t(), out=out)
torch.cuda.synchronize()
