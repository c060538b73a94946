"""Copy-engine peer copy one-way vs bidirectional (2 GPUs, one process): the
baseline SM-issued TMA pulls are compared against."""
# copy-engine peer copy: one-way vs bidirectional, and concurrent with an SM TMA pull
import torch, json, time
n = 512 << 20
d0, d1 = torch.device("cuda", 0), torch.device("cuda", 1)
a0 = torch.empty(n, dtype=torch.uint8, device=d0); b0 = torch.empty(n, dtype=torch.uint8, device=d0)
a1 = torch.empty(n, dtype=torch.uint8, device=d1); b1 = torch.empty(n, dtype=torch.uint8, device=d1)
s0 = torch.cuda.Stream(d0); s1 = torch.cuda.Stream(d1)
def run(bidir, reps=10):
    for _ in range(2):
        with torch.cuda.stream(s0): b0.copy_(a1, non_blocking=True)   # pull 1 -> 0 (issued on GPU 0)
        if bidir:
            with torch.cuda.stream(s1): b1.copy_(a0, non_blocking=True)
    torch.cuda.synchronize(d0); torch.cuda.synchronize(d1)
    t = time.perf_counter()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(s0)
    if bidir: e[2].record(s1)
    for _ in range(reps):
        with torch.cuda.stream(s0): b0.copy_(a1, non_blocking=True)
        if bidir:
            with torch.cuda.stream(s1): b1.copy_(a0, non_blocking=True)
    e[1].record(s0)
    if bidir: e[3].record(s1)
    torch.cuda.synchronize(d0); torch.cuda.synchronize(d1)
    ms = e[0].elapsed_time(e[1]) / reps
    out = {"gbs_gpu0": n / (ms * 1e-3) / 1e9}
    if bidir:
        ms1 = e[2].elapsed_time(e[3]) / reps
        out["gbs_gpu1"] = n / (ms1 * 1e-3) / 1e9
    return out
print(json.dumps({"ce_one_way": run(False), "ce_bidir": run(True), "can_access": torch.cuda.can_device_access_peer(0, 1)}))
