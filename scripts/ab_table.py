#!/usr/bin/env python
"""Side-by-side step / fwd / bwd ms of bench.py JSON lines (headline + config
matrix), one row per file: python scripts/ab_table.py a.json b.json ..."""
import json
import sys


def rows(path):
    for line in open(path):
        if line.startswith("{"):
            d = json.loads(line)
            rf = d["roofline"]["per_kernel"]
            out = {d["config"]["name"]: (d["ms_per_step"], d["roofline"]["step_frac_of_tstar"], rf["fwd"]["ms"],
                                         rf["bwd"]["ms"], (d.get("parity") or {}).get("pass", True))}
            for k, v in (d.get("config_matrix") or {}).items():
                if k not in out and "ms_per_step" in v:
                    out[k] = (v["ms_per_step"], v["frac_of_tstar"], v["fwd_ms"], v["bwd_ms"], (v.get("parity") or {}).get("pass", True))
            return out
    return {}


if __name__ == "__main__":
    for p in sys.argv[1:]:
        r = rows(p)
        print(p.split("/")[-1].ljust(28), "  ".join(f"{k}:{v[0]*1e3:.1f}us({v[1]:.2f}) f{v[2]*1e3:.1f} b{v[3]*1e3:.1f}"
                                                    f"{'' if v[4] else ' PARITY-FAIL'}" for k, v in r.items()))
