#!/bin/bash
# A/B on one box: alternate `bench.py` runs of two repo copies (A = $1, B = $2;
# each a full tree with its own built libsdattn.so), 3 rounds, then ncu of the
# kernel regex $3 (optional) in both.
A=$1; B=$2; K=${3:-}
mkdir -p gpurun_out/ab
for r in 1 2 3; do
  for v in A B; do
    d=$([ $v = A ] && echo $A || echo $B)
    timeout 300 python $d/bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-dense ${BENCH_ARGS} > gpurun_out/ab/$v$r.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob
for v in "AB":
    for f in sorted(glob.glob(f"gpurun_out/ab/{v}[0-9].json")):
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
        except Exception as e:
            print(v, f, "failed", e); continue
        print(v, f[-7:-5], "median", round(d["step_us"]["median"], 1), "mean", round(d["us_per_step"], 1),
              {k: round(x, 1) for k, x in d["phases_us"].items() if k != "note"}, "fb", d["fallback_rows"])
PY
if [ -n "$K" ]; then
  for v in A B; do
    d=$([ $v = A ] && echo $A || echo $B)
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:$K -s 3 -c 1 -o gpurun_out/ab/ncu_$v \
      python $d/bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-dense --no-graph > gpurun_out/ab/ncu_$v.log 2>&1
  done
fi
