#!/bin/bash
# A/B/C of one build under different values of an environment variable:
#   scripts/ab_env.sh VAR "v1 v2 v3" [rounds]
VAR=$1; VALS=$2; R=${3:-2}
mkdir -p gpurun_out/abe
for r in $(seq 1 $R); do
  for v in $VALS; do
    env $VAR=$v timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-dense ${BENCH_ARGS} > gpurun_out/abe/$v.$r.json 2>gpurun_out/abe/$v.$r.err
  done
done
python - "$VALS" <<'PY'
import json, glob, sys
for v in sys.argv[1].split():
    for f in sorted(glob.glob(f"gpurun_out/abe/{v}.[0-9]*.json")):
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
        except Exception as e:
            print(v, f, "failed", open(f.replace(".json", ".err")).read()[-300:]); continue
        print(v, "median", round(d["step_us"]["median"], 1), "p10", round(d["step_us"]["p10"], 1), "mean", round(d["us_per_step"], 1),
              {k: round(x, 1) for k, x in d["phases_us"].items() if k != "note"}, "fb", d["fallback_rows"], "err", d["device_error"])
PY
