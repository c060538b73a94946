"""Summaries of gpurun_out artefacts: trace-probe jsonl and bench JSON lines."""
import json
import sys


def lines(f):
    return [json.loads(l) for l in open(f) if l.startswith("{")]


for f in sys.argv[1:]:
    if f.endswith(".jsonl"):
        for d in lines(f):
            print(d["cfg"], d["N"], d["gpu"], d["kind"], "op", d["op_us"], "T*", d["tstar_us"], "span", d["span_us"],
                  "pw50", d["peers_wait_p50_us"], "pmax", d["peers_max_from_t0_us"], "f50", d["first_p50_us"],
                  "d50", d["done_p50_from_t0_us"], "dmax", d["done_max_from_t0_us"], "tail", d["tail_us"],
                  "ch", d["chunks"], d["remote_chunks"], "ingraph", d.get("step_in_graph_us"),
                  "stepgraph", d.get("step_graph_per_step_us"))
    else:
        for d in lines(f):
            r = d.get("roofline", {})
            print(f, d.get("config", {}).get("name"), "value", d["value"], "ms", d["ms_per_step"], "frac_step",
                  r.get("step_frac_of_tstar"), "fwd", r.get("per_kernel", {}).get("fwd", {}).get("ms"),
                  r.get("per_kernel", {}).get("fwd", {}).get("tstar_ms"), "bwd",
                  r.get("per_kernel", {}).get("bwd", {}).get("ms"), r.get("per_kernel", {}).get("bwd", {}).get("tstar_ms"),
                  "clk", (d.get("clocks") or {}).get("sm_mhz"))
            for k, v in (d.get("config_matrix") or {}).items():
                print("   ", k, {x: v.get(x) for x in ["ms_per_step", "tstar_ms", "frac_of_tstar", "fwd_ms", "fwd_tstar_ms",
                                                    "bwd_ms", "bwd_tstar_ms", "error"]},
                      (v.get("overlap_with_pp_p2p") or {}).get("overlap"))
