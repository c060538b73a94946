"""Summarise an ncu report (and optional launch-list CSV) into profiles/.

usage: python scripts/ncu_summary.py <report.ncu-rep> <out-prefix> [launches.csv]
Writes <out-prefix>.json (per-kernel metrics) and, for bench.py, the
per-direction DRAM traffic file profiles/traffic_<cfg>_n<N>.json when asked
with --traffic <cfg> <N>.
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "nvlrx__bytes.sum", "nvltx__bytes.sum",
]


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        k = {"kernel": r[hdr.index("Kernel Name")].strip()}
        for m in METRICS:
            if m in hdr:
                k[m] = {"value": r[hdr.index(m)], "unit": units[hdr.index(m)]}
        res.append(k)
    return res


def to_bytes(v):
    x = float(v["value"].replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(v["unit"], 1)


if __name__ == "__main__":
    args = sys.argv[1:]
    traffic = None
    if "--traffic" in args:
        i = args.index("--traffic")
        traffic = (args[i + 1], args[i + 2])
        del args[i:i + 3]
    rep, prefix = args[0], args[1]
    ks = summarise(rep)
    doc = {"report": rep, "kernels": ks}
    if len(args) > 2:
        doc["launch_list_csv"] = args[2]
    with open(prefix + ".json", "w") as f:
        json.dump(doc, f, indent=1)
    for k in ks:
        print(k["kernel"][:70], {m: k[m]["value"] + " " + k[m]["unit"] for m in METRICS[:5] if m in k})
    if traffic:
        t = {}
        for k in ks:
            d = "fwd" if "copy_segments" in k["kernel"] else "bwd"
            t.setdefault(d, int(to_bytes(k["dram__bytes_read.sum"]) + to_bytes(k["dram__bytes_write.sum"])))
        with open(f"profiles/traffic_{traffic[0]}_n{traffic[1]}.json", "w") as f:
            json.dump(t, f)
        print(t)
