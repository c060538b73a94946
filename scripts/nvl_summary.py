#!/usr/bin/env python
"""Summarise an ncu NVLink capture of scripts/nvl_ncu_probe.py into one JSON
file per (config, N): per kernel the ncu duration, DRAM bytes, NVLink rx/tx
bytes (all and user data), achieved NVLink GB/s against the measured peer-copy
peak (770 GB/s, B200_PROFILING.md) and the 900 GB/s nominal, and the wasted
traffic ratio nvlrx user bytes / the index map's ingress bytes for GPU 0.

  python scripts/nvl_summary.py CSV PLAIN_JSON OUT_JSON [--label TEXT]

CSV: `ncu --devices 0 --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,
nvltx__bytes_data_user.sum --clock-control none -k regex:segments --csv`;
PLAIN_JSON: the probe's line run without ncu (one-way times, expected bytes).
ncu times are cold-cache, serialised and of GPU 0 alone (peers idle, barrier
off): they bound the kernel's NVLink rate, they are not bench values.
"""
import argparse
import collections
import csv
import json
import statistics

PEAK_MEASURED = 770.0
PEAK_NOMINAL = 900.0


def load_csv(path):
    rows = [r for r in csv.DictReader(line for line in open(path) if line.startswith('"'))]
    launches = collections.OrderedDict()
    for r in rows:
        k = (int(r["ID"]), r["Kernel Name"], r["Grid Size"], r["Block Size"])
        launches.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return launches


def kind_of(name):
    return "fwd" if "copy_segments" in name else "bwd"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("plain")
    ap.add_argument("out")
    ap.add_argument("--label", default="")
    a = ap.parse_args()
    plain = None
    for line in open(a.plain):
        line = line.strip()
        if line.startswith("{"):
            plain = json.loads(line)
            break
    launches = load_csv(a.csv)
    per = collections.defaultdict(list)
    names = {}
    for (lid, name, grid, block), m in launches.items():
        k = kind_of(name)
        per[k].append(m)
        names[k] = (name.split("(")[0].replace("void ", "").replace("unnamed>::", ""), grid, block)
    out = {"label": a.label, "config": plain["config"], "n_gpus": plain["n_gpus"], "gpu": 0,
           "source": {"csv": a.csv, "plain": a.plain},
           "method": "one process drives the N-GPU exec group (open_peers_local); GPU 0's forward and backward run "
                     "alone with every peer's inputs resident, ncu --devices 0 single-pass counters (no replay "
                     "across ranks), --clock-control none; times cold-cache and serialised",
           "kernels": {}}
    for k, ms in per.items():
        med = lambda key: statistics.median(x[key] for x in ms)  # noqa: E731
        t_ns = med("gpu__time_duration.sum")
        rx_user = med("nvlrx__bytes_data_user.sum")
        rx_all = med("nvlrx__bytes.sum")
        tx_all = med("nvltx__bytes.sum")
        expect = plain[f"{k}_nvl_in_bytes"]
        gbs = rx_user / t_ns if t_ns else 0.0
        out["kernels"][k] = {
            "kernel": names[k][0], "grid": names[k][1], "block": names[k][2], "launches": len(ms),
            "ncu_us": round(t_ns / 1e3, 2),
            "plain_us_alone": round(plain[f"{k}_ms_alone"] * 1e3, 2),
            "dram_read_bytes": med("dram__bytes_read.sum"), "dram_write_bytes": med("dram__bytes_write.sum"),
            "hbm_bytes_index_map": plain[f"{k}_hbm_bytes"],
            "nvlrx_bytes": rx_all, "nvlrx_user_bytes": rx_user, "nvltx_bytes": tx_all,
            "nvltx_user_bytes": med("nvltx__bytes_data_user.sum"),
            "nvl_in_bytes_index_map": expect,
            "nvl_wasted_ratio": round(rx_user / expect, 4) if expect else None,
            "nvl_protocol_overhead": round(rx_all / rx_user, 4) if rx_user else None,
            "achieved_nvl_gbs": round(gbs, 1),
            "frac_of_770_measured": round(gbs / PEAK_MEASURED, 4),
            "frac_of_900_nominal": round(gbs / PEAK_NOMINAL, 4),
        }
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")
    for k, v in out["kernels"].items():
        print(out["config"], out["n_gpus"], k, v["kernel"], v["ncu_us"], "us",
              v["achieved_nvl_gbs"], "GB/s", "wasted", v["nvl_wasted_ratio"])


if __name__ == "__main__":
    main()
