timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t9.txt 2>&1; tail -3 gpurun_out/t9.txt
timeout 300 python scripts/diag_mha.py 4 2 | head -2
timeout 900 python bench.py --sweep table1 --steps 20 > gpurun_out/t1b.jsonl 2>gpurun_out/t1b.err
python - <<'PY'
import json
for l in open("gpurun_out/t1b.jsonl"):
    d = json.loads(l)
    print("B", d["B"], "S", d["S"], "backend_us", round(d["backend_us"]["median"], 1), "x dense", round(d["speedup_vs_dense"], 2), "paper", d["paper_speedup_vs_flashinfer_h100"], "frac_u", round(d["frac_union_bytes"], 2))
PY
tail -2 gpurun_out/t1b.err
