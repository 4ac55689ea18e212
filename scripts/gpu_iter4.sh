timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t4.txt 2>&1; tail -3 gpurun_out/t4.txt
bash scripts/ab.sh ab/a .
timeout 900 python bench.py --sweep configs --sweep-configs cfg1,cfg2_s50,cfg4_t33,cfg5 --steps 20 > gpurun_out/sw4.jsonl 2> gpurun_out/sw4.err
python - <<'PY'
import json
for l in open("gpurun_out/sw4.jsonl"):
    d = json.loads(l); print(d["config"], "median", round(d["fused_us"]["median"], 1), "p90", round(d["fused_us"]["p90"], 1), "frac", round(d["frac"], 3), "dense", round(d["dense_us"], 1), "fb", d["fallback_rows"])
PY
tail -2 gpurun_out/sw4.err
