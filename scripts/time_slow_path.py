"""Cost of the fused select's exact slow path (every row forced onto it) vs the fast path, cfg3."""
import os, sys, json
sys.path.insert(0, os.environ.get("SD_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, workloads, paper_2605_24168_b200 as sd
case = workloads.config_case("cfg3", device="cuda")
kv, sk = sd.KVCache.from_case(case), sd.SketchCache.from_case(case)
def t(fn, n=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
print(json.dumps({"fast_us": t(lambda: sd.sparse_decode_fused(case.q, kv, sk, S=50.0)),
                  "all_rows_slow_us": t(lambda: sd.sparse_decode_fused(case.q, kv, sk, S=50.0, force_slow_path=True))}))
