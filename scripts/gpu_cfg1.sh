timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t32.txt 2>&1; tail -2 gpurun_out/t32.txt
for d in ab/a .; do
  timeout 300 python $d/bench.py --sweep configs --sweep-configs cfg1,cfg2_s50 --steps 20 > gpurun_out/c1_$(basename $d).jsonl 2>/dev/null
  python - $d <<'PY'
import json, sys, os
for l in open(f"gpurun_out/c1_{os.path.basename(sys.argv[1])}.jsonl"):
    d = json.loads(l); print(sys.argv[1], d["config"], "median", round(d["fused_us"]["median"], 1), "dense", round(d["dense_us"], 1))
PY
done
