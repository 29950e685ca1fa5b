#!/bin/bash
# phase probe at C2 / C1 / C3 and one short bench line
mkdir -p gpurun_out
for d in 25600000 1000000 110000000; do
  timeout 300 python tools/phase_probe.py $d ${SEL:-mstopk} >> gpurun_out/phase_probe.log 2>&1
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?"
python - <<'PY'
import json
l = json.loads(open("gpurun_out/bench_quick.json").read().strip().splitlines()[-1])
print("ms/step", round(l["ms_per_step"]*1e3,1), "us; roofline", {k: l["roofline"][k] for k in ("achieved","frac","ms_per_launch")}, "stages", {k: round(v["ms_per_launch"]*1e3,1) for k,v in l["stages"].items()})
PY
