# per-phase times of the smaller BASELINE configs
for c in cfg2_s50 cfg2_s10 cfg4_t0; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/ph_$c.json 2>/dev/null
  python - "$c" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ph_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(sys.argv[1], "median", round(d["step_us"]["median"], 1), {k: round(v, 1) for k, v in d["phases_us"].items() if k != "note"}, "frac", round(d["step_roofline"]["frac"], 3))
PY
done
