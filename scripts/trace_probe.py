"""Per-CTA timeline of one boundary launch (HB_TRACE=1 diagnostics).

Runs each config's forward-only and backward-only graphs back to back (steady
state), then reads the last launch's per-CTA %globaltimer stamps and reports,
per GPU: per-op time (CUDA events), kernel span (first entry -> last exit),
entry spread, arrival / peer-wait / first-chunk latencies, the tail after the
last CTA finished its work, and the GPUs' entry skew (globaltimer is one clock
per GPU; cross-GPU numbers are indicative).

  HB_TRACE=1 torchrun --nproc-per-node N scripts/trace_probe.py c4w4 c2x4 ...
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("HB_TRACE", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2605_27678_b200 import bridge as hbb, configs  # noqa: E402


def pct(x, q):
    return float(np.percentile(x, q)) if len(x) else float("nan")


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    N = world
    stream = torch.cuda.Stream(priority=-1)
    tdt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}
    pk = bench.peaks()
    for spec in sys.argv[1:]:
        name, _, sc = spec.partition(":")
        scale = int(sc or 1)
        cfg = configs.get(name, scale=scale)
        plan = hbb.plan_bridge(cfg.edge())
        sp = bench.make_splice(cfg)
        r2g = configs.rank_to_gpu(plan.world, N)
        local = [r for r in range(plan.world) if r2g[r] == rank]
        slots = 2
        rt = hbb.BridgeRuntime(plan, sp, n_gpus=N, my_gpu=rank, rank_to_gpu=r2g, act_dtype=tdt[cfg.act],
                               grad_in_dtype=tdt[cfg.grad_in], grad_out_dtype=tdt[cfg.grad_out], mb_slots=slots)
        if N > 1:
            rt.exchange_handles()
        for s in range(slots):
            for r in local:
                for slot in (hbb.SLOT_SRC_ACT, hbb.SLOT_DST_GRAD, hbb.SLOT_TEXT, hbb.SLOT_SRC_GRAD):
                    b = rt.buffer(r, slot, s)
                    if b is not None:
                        b.normal_()
        for mb in range(3):
            rt.forward(mb, stream)
            rt.backward(mb, cfg.beta, stream)
        torch.cuda.synchronize()
        if N > 1:
            dist.barrier()
        tm = bench.traffic_model(cfg, N)
        res = {}
        for kind, what in (("fwd", 0), ("bwd", 2)):
            for k in range(slots):
                rt.capture_step(k, cfg.beta, True, stream, what=what)
            for k in range(slots):
                rt.replay_step(k, stream, what)
            torch.cuda.synchronize()
            if N > 1:
                dist.barrier()
            K = 100
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record(stream)
            for i in range(K):
                rt.replay_step(i % slots, stream, what)
            b.record(stream)
            stream.synchronize()
            ms = a.elapsed_time(b) / K
            tr = rt.trace(0 if kind == "fwd" else 1).astype(np.int64)
            ent, arr, peers, first, done, ext, nch, nrem = (tr[:, i] for i in range(8))
            t0 = ent.min()
            w = peers > 0
            st = {
                "op_us": round(ms * 1e3, 2),
                "tstar_us": round(bench.kernel_bound(tm, kind, ms, pk, N)["tstar_ms"] * 1e3, 2),
                "grid": int(len(ent)),
                "span_us": round((ext.max() - t0) / 1e3, 2),
                "entry_spread_us": round((ent.max() - t0) / 1e3, 2),
                "arrive_p50_us": round(pct(arr - ent, 50) / 1e3, 2),
                "peers_wait_p50_us": round(pct((peers - ent)[w], 50) / 1e3, 2) if w.any() else None,
                "peers_max_from_t0_us": round(((peers[w]).max() - t0) / 1e3, 2) if w.any() else None,
                "first_p50_us": round(pct((first - ent)[first > 0], 50) / 1e3, 2),
                "first_max_from_t0_us": round(((first[first > 0]).max() - t0) / 1e3, 2) if (first > 0).any() else None,
                "done_p50_from_t0_us": round(pct(done - t0, 50) / 1e3, 2),
                "done_max_from_t0_us": round((done.max() - t0) / 1e3, 2),
                "tail_us": round((ext.max() - done.max()) / 1e3, 2),
                "chunks": int(nch.sum()), "remote_chunks": int(nrem.sum()),
                "chunks_max": int(nch.max()), "idle_ctas": int((nch == 0).sum()),
                "t0_ns": int(t0),
            }
            res[kind] = st
        # the same ops with the host out of the loop: R steps (fwd+bwd) captured in ONE graph
        R = 16
        mbc = [100]

        def step():
            rt.forward(mbc[0] % slots + slots * (mbc[0] // slots), stream)
            rt.backward(mbc[0] % slots + slots * (mbc[0] // slots), cfg.beta, stream)
            mbc[0] += 1

        with torch.cuda.stream(stream):
            step()
            torch.cuda.synchronize()
            if N > 1:
                dist.barrier()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for _ in range(R):
                    step()
            g.replay()
            torch.cuda.synchronize()
            if N > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(stream)
            for _ in range(5):
                g.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        res["fwd"]["step_in_graph_us"] = round(e0.elapsed_time(e1) / (5 * R) * 1e3, 2)
        for k in range(slots):
            rt.capture_step(k, cfg.beta, True, stream, what=1)
        torch.cuda.synchronize()
        if N > 1:
            dist.barrier()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(stream)
        for i in range(100):
            rt.replay_step(i % slots, stream, 1)
        b.record(stream)
        stream.synchronize()
        res["fwd"]["step_graph_per_step_us"] = round(a.elapsed_time(b) / 100 * 1e3, 2)
        del g
        allr = [None] * N
        if N > 1:
            dist.all_gather_object(allr, res)
        else:
            allr = [res]
        if rank == 0:
            for kind in ("fwd", "bwd"):
                t0s = [r[kind]["t0_ns"] for r in allr]
                skew = [round((t - min(t0s)) / 1e3, 2) for t in t0s]
                for g, r in enumerate(allr):
                    d = dict(r[kind])
                    d.pop("t0_ns")
                    print(json.dumps({"cfg": spec, "N": N, "gpu": g, "kind": kind, "entry_skew_us": skew[g], **d}),
                          flush=True)
        rt.close()
        torch.cuda.synchronize()
        if N > 1:
            dist.barrier()
    if N > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
