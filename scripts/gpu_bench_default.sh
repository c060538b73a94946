exec > gpurun_out/bench_default.log 2>&1
python bench.py > gpurun_out/bench_default.json; echo rc=$?
cat gpurun_out/bench_default.json
for c in c3 c4 c5; do python bench.py --config $c --no-cpu > gpurun_out/bench_$c.json; echo $c rc=$?; done
python - <<'PY'
import json
for c in ["default","c3","c4","c5"]:
    d=json.load(open(f"gpurun_out/bench_{c}.json"))
    print(c, d["value"], d["ms_per_step"], "frac_step", d["roofline"]["step_frac_of_tstar"], "dom", d["roofline"]["kernel"], d["roofline"]["frac"], "e2e", d["e2e"]["value"], d["e2e"]["ms_per_step"], "clk", d["clocks"])
PY
