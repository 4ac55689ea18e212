timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t30.txt 2>&1; tail -3 gpurun_out/t30.txt
for d in ab/a .; do
  timeout 300 python $d/bench.py --config cfg3_fp8 --steps 50 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/fp8_$(basename $d).json 2>/dev/null
  python - $d <<'PY'
import json, sys, os
d = json.loads(open(f"gpurun_out/fp8_{os.path.basename(sys.argv[1])}.json").read().strip().splitlines()[-1])
print(sys.argv[1], "cfg3_fp8 median", round(d["step_us"]["median"], 1), {k: round(v, 1) for k, v in d["phases_us"].items() if k != "note"}, "frac", round(d["step_roofline"]["frac"], 3), "fb", d["fallback_rows"])
PY
done
