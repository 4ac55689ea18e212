"""Unfused top-k (sd_topk_select over materialised cfg3 scores) and the fused slow path, timed."""
import os, sys, json
sys.path.insert(0, os.environ.get("SD_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, workloads, paper_2605_24168_b200 as sd
case = workloads.config_case("cfg3", device="cuda")
kv, sk = sd.KVCache.from_case(case), sd.SketchCache.from_case(case)
sc = sd.sparse_index_score(case.q, kv, sk)
def t(fn, n=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
print(json.dumps({"topk_select_us": t(lambda: sd.topk_select(sc, case.seq_lens, 131072, S=50.0, num_kv_heads=8)),
                  "fused_all_rows_slow_us": t(lambda: sd.sparse_decode_fused(case.q, kv, sk, S=50.0, force_slow_path=True))}))
