#!/bin/bash
# Small / latency-bound configs: step time and per-kernel phases (serialised) for each config.
mkdir -p gpurun_out/small
for c in ${CONFIGS:-cfg2_s50 cfg2_s10 cfg4_t0 cfg1}; do
  timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --no-dense > gpurun_out/small/$c.json 2> gpurun_out/small/$c.err
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/small/*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "failed", e); continue
    print(f.split("/")[-1][:-5], "median", round(d["step_us"]["median"], 1), "frac", round(d["step_roofline"]["frac"], 3),
          {k: round(v, 1) for k, v in d.get("phases_us", {}).items() if k != "note"}, d["config"].get("launch", "")[:30])
PY
