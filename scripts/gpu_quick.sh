#!/bin/bash
# Quick GPU iteration: parity tests, then a short bench at cfg3 without the CPU baseline and the dense leg.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/t.txt 2>&1; tail -4 gpurun_out/t.txt
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-dense ${BENCH_ARGS} > gpurun_out/bq.json 2> gpurun_out/bq.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bq.json").read().strip().splitlines()[-1])
print("us/step", round(d["us_per_step"], 1), "median", round(d["step_us"]["median"], 1), "p10/p90",
      round(d["step_us"]["p10"], 1), round(d["step_us"]["p90"], 1), "eager median", round(d["eager_step_us"]["median"], 1),
      "launch", d["config"]["launch"][:40])
print("phases", {k: round(v, 1) for k, v in d["phases_us"].items() if k != "note"},
      "frac", round(d["step_roofline"]["frac"], 3), "attend frac", round(d["roofline"]["frac"], 3),
      "fallback", d.get("fallback_rows"), "err", d.get("device_error"), "e2e", round(d["e2e"]["value"]))
PY
tail -3 gpurun_out/bq.err
