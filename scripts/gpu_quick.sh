#!/bin/bash
# Quick GPU iteration: parity tests, then a short bench at cfg3 without the CPU baseline and the dense leg.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t.txt 2>&1; tail -4 gpurun_out/t.txt
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/bq.json 2> gpurun_out/bq.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bq.json").read().strip().splitlines()[-1])
print("us/step", round(d["us_per_step"], 1), "phases", {k: round(v, 1) for k, v in d["phases_us"].items() if k != "note"},
      "frac", round(d["step_roofline"]["frac"], 3), "fallback", d.get("fallback_rows"), "err", d.get("device_error"))
PY
tail -3 gpurun_out/bq.err
