#!/bin/bash
# A/B/... on one box: round-robin `bench.py` runs of several repo copies (each a full tree with
# its own built libsdattn.so), $ROUNDS rounds (default 3); BENCH_ARGS: extra bench flags.
mkdir -p gpurun_out/abn
R=${ROUNDS:-3}
for r in $(seq 1 $R); do
  i=0
  for d in "$@"; do
    timeout 300 python $d/bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-dense ${BENCH_ARGS} > gpurun_out/abn/v${i}_$r.json 2>/dev/null
    i=$((i+1))
  done
done
python - "$@" <<'PY'
import json, glob, sys
for i, d in enumerate(sys.argv[1:]):
    for f in sorted(glob.glob(f"gpurun_out/abn/v{i}_*.json")):
        try:
            x = json.loads(open(f).read().strip().splitlines()[-1])
        except Exception as e:
            print(d, f, "failed", e); continue
        print(f"{d:8s}", "median", round(x["step_us"]["median"], 1), "mean", round(x["us_per_step"], 1),
              {k: round(v, 1) for k, v in x["phases_us"].items() if k != "note"}, "fb", x["fallback_rows"])
PY
