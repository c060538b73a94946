"""Generate the committed golden fixtures (run here, where /root/reference exists).

Inputs come from the reference's own GaussianStream (matrix.cpp:136-180),
seed 1234, tag "bnd/s<j>" per global sample j and "grad/r<r>" per destination
rank, as SURVEY.md §8(d) prescribes; outputs from the oracle (restated bridge
over the reference simnet/grid). Fixtures are small so they live in git and
travel to the GPU box, where the oracle library is not needed to check them.

  python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402
from paper_2605_27678_b200 import configs  # noqa: E402

CASES = {
    # name: (config, scale, width override)
    "c1": ("c1", 512, None),
    "c2": ("c2", 512, None),
    "c3": ("c3", 512, None),
    "c4": ("c4", 512, None),
    "c5": ("c5", 512, None),
    "spec_fanin2_nc": (None, None, None),
}


def layouts(cfg):
    l = lambda m: O.Layout(m.name, m.tp, m.cp, m.pp, m.dp, m.rank_offset)  # noqa: E731
    return l(cfg.src), l(cfg.dst)


def make(name):
    if name == "spec_fanin2_nc":  # S:155-157 known answer: fan-in 2, B=8, W=3
        src, dst, B, W, splice = O.Layout("enc", dp=4), O.Layout("llm", tp=2, dp=2, rank_offset=4), 8, 3, None
        hidden, tokens = 3, 1
    else:
        cfg = configs.get(CASES[name][0], scale=CASES[name][1])
        if not cfg.splice:
            cfg.tokens = 4  # keep fixtures small: W = 4 tokens x 8 hidden
        src, dst = layouts(cfg)
        B, W, splice, hidden, tokens = cfg.batch, cfg.width, cfg.splice, cfg.hidden, cfg.tokens
    SI, DI = O.intervals(B, src.dp), O.intervals(B, dst.dp)
    X = np.stack([O.gaussian(1234, f"bnd/s{j}", W) for j in range(B)])
    X = X.astype(np.float32).astype(np.float64)  # exactly representable in fp32 (and the fixture dtype)
    shards = {r: X[SI[src.coord(r)[3]][0]:SI[src.coord(r)[3]][0] + SI[src.coord(r)[3]][1]]
              for r in src.stage_ranks(src.pp - 1)}
    fwd, led_f, _ = O.bridge_forward(src, dst, B, W, shards)
    arrays = {"X": X}
    text = None
    if splice:
        codes = splice["codes"]
        text = np.stack([O.gaussian(1234, f"txt/q{i}", hidden) for i in range(int((codes < 0).sum()))])
        text = text.astype(np.float32).astype(np.float64)
        arrays["text"] = text
        L = splice["S"] // dst.cp
    grads, vg = {}, {}
    for r in dst.stage_ranks(0):
        t, c, p, d = dst.coord(r)
        if splice:
            arrays[f"fwd_r{r}"] = O.splice_forward(splice["codes"], splice["Q"], splice["S"], hidden, c * L, L,
                                                   fwd[r].reshape(-1, hidden), text)
            g = O.gaussian(1234, f"grad/r{r}", splice["Q"] * L * hidden).astype(np.float32).astype(np.float64)
            vg[r] = O.splice_backward(splice["codes"], splice["Q"], splice["S"], hidden, c * L, L,
                                      g.reshape(-1, hidden), DI[d][1] * tokens).reshape(-1, W)
        else:
            arrays[f"fwd_r{r}"] = fwd[r]
            g = O.gaussian(1234, f"grad/r{r}", DI[d][1] * W).astype(np.float32).astype(np.float64)
            vg[r] = g.reshape(-1, W)
        grads[r] = g
        arrays[f"grad_r{r}"] = g
    bwd, led_b, _ = O.bridge_backward(src, dst, B, W, vg)
    for r, a in bwd.items():
        arrays[f"bwd_r{r}"] = a
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **{k: v.astype(np.float32) for k, v in arrays.items()})
    meta = {"name": name, "src": [src.name, src.tp, src.cp, src.pp, src.dp, src.rank_offset],
            "dst": [dst.name, dst.tp, dst.cp, dst.pp, dst.dp, dst.rank_offset], "B": B, "W": W,
            "hidden": hidden, "tokens": tokens, "seed": 1234,
            "ledger_fwd": {f"{k[0]}|{k[1]}": v for k, v in led_f.items()},
            "ledger_bwd": {f"{k[0]}|{k[1]}": v for k, v in led_b.items()},
            "export_plan": O.export_plan(src, dst, B, W),
            "generator": "tests/golden/make_golden.py (oracle over reference simnet/grid)"}
    if splice:
        meta["splice"] = {"Q": splice["Q"], "S": splice["S"], "text_mode": splice["text_mode"],
                          "codes": [int(x) for x in splice["codes"]]}
    with open(os.path.join(HERE, f"{name}.json"), "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    for n in CASES:
        make(n)
        print("wrote", n)
