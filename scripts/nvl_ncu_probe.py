#!/usr/bin/env python
"""NVLink bytes of one GPU's boundary kernels, for ncu.

One process drives an N-GPU exec group (hb_exec_open_peers_local: peer access
over NVSwitch, no CUDA IPC, no NCCL), fills every GPU's buffers with the
bench's hashed inputs, then launches GPU 0's forward and backward alone with
the cross-GPU barrier off (HB_DEBUG_NO_SYNC=1, set below before the library
loads; safe here because every peer's inputs were written and synchronised
beforehand and nothing else runs). GPU 0's kernels pull their remote rows from
the peers exactly as in a group step, so ncu's nvlrx/nvltx counters on device
0 measure that kernel's NVLink traffic, while a single process and kernel
replay of device-0 memory keep ncu away from the multi-process deadlock of the
round-1 attempt.

  ncu --devices 0 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\\
      nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum \\
      -k regex:segments --csv --log-file out.csv python scripts/nvl_ncu_probe.py --config c2x4 --gpus 4

Without ncu it prints the kernels' one-way times (GPU 0 alone, CUDA events)
and the index map's expected ingress bytes on GPU 0.
"""
import argparse
import json
import os
import sys

os.environ["HB_DEBUG_NO_SYNC"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_27678_b200 import bridge as hbb  # noqa: E402
from paper_2605_27678_b200 import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2x4")
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    cfg = configs.get(a.config)
    plan = hbb.plan_bridge(cfg.edge())
    sp = bench.make_splice(cfg)
    N = a.gpus
    tdt = {"bf16": torch.bfloat16, "fp32": torch.float32}
    g = hbb.LocalGroup(plan, sp, devices=list(range(N)), act_dtype=tdt[cfg.act], grad_in_dtype=tdt[cfg.grad_in],
                       grad_out_dtype=tdt[cfg.grad_out], max_ctas=0)
    for gi, rt in enumerate(g.rts):
        with torch.cuda.device(gi):
            local = [r for r in range(plan.world) if g.rank_to_gpu[r] == gi]
            bench.fill_inputs(rt, local, 1, torch.device("cuda", gi))
    for gi in range(N):
        torch.cuda.synchronize(gi)
    rt0, st0 = g.rts[0], g.streams[0]
    times = {"fwd": [], "bwd": []}
    mb = 0
    for rep in range(a.reps + 1):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        with torch.cuda.device(0):
            ev[0].record(st0)
            rt0.forward(mb, st0)
            ev[1].record(st0)
            rt0.backward(mb, cfg.beta, st0)
            ev[2].record(st0)
            st0.synchronize()
        mb += 1
        if rep:  # the first is a warm-up
            times["fwd"].append(ev[0].elapsed_time(ev[1]))
            times["bwd"].append(ev[1].elapsed_time(ev[2]))
    tm = bench.traffic_model(cfg, N)
    print(json.dumps({"config": cfg.name, "n_gpus": N, "gpu": 0,
                      "fwd_ms_alone": min(times["fwd"]), "bwd_ms_alone": min(times["bwd"]),
                      "fwd_nvl_in_bytes": tm["fwd_nvl"][0], "bwd_nvl_in_bytes": tm["bwd_nvl"][0],
                      "fwd_hbm_bytes": tm["fwd_hbm"][0], "bwd_hbm_bytes": tm["bwd_hbm"][0],
                      "status": rt0.status()}), flush=True)
    g.close()


if __name__ == "__main__":
    main()
