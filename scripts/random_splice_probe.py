"""GPU parity on random placeholder tables (to promote into tests/test_gpu_parity.py
once it has run on a B200): scattered vision tokens, images split across
sequences and CP slices, both text numberings, several partitions. Uses the
GPU test suite's run_case (device result vs the oracle).

  python scripts/random_splice_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from paper_2605_27678_b200 import bridge as hbb, configs  # noqa: E402
from paper_2605_27678_b200 import grid as hbg  # noqa: E402
from test_gpu_parity import run_case  # noqa: E402
from test_index_map import random_codes  # noqa: E402

cases = [(hbg.ModuleLayout("vit", dp=4), hbg.ModuleLayout("llm", tp=2, cp=2)),
         (hbg.ModuleLayout("vit", tp=2, dp=2), hbg.ModuleLayout("llm", cp=4)),
         (hbg.ModuleLayout("vit", dp=8), hbg.ModuleLayout("llm", tp=2, cp=2, dp=2))]
n = 0
for seed in range(6):
    for text_mode in (hbb.TEXT_FULL, hbb.TEXT_SLICE):
        for partition in (0, 1, 3):
            rng = np.random.default_rng(100 + seed)
            src, dst = cases[seed % 3]
            cfg = configs.get("c4", scale=64)
            cfg.src, cfg.dst = src, dst
            cfg.batch, cfg.tokens, cfg.hidden = 8, 3, 8 * (1 + seed % 2)  # 16 B or 32 B rows (bf16)
            Q, S = 2, 16 * dst.cp
            n_vis = (cfg.batch // dst.dp) * cfg.tokens
            cfg.splice = {"Q": Q, "S": S, "codes": random_codes(rng, n_vis, Q, S), "text_mode": text_mode}
            for beta in (0.0, 1.0):
                run_case(cfg, seed=seed, beta=beta, perturb=False, partition=partition)
                n += 1
print(f"random placeholder tables: {n} device cases match the oracle")
