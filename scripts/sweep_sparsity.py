"""Fused step time vs sparsity at one config (Table-1-style sweep on B200).

    python scripts/sweep_sparsity.py [--config cfg3] [--S 2,5,10,20,50,100,200,500]

Prints one JSON line per S: us/step (CUDA events over 20 steps after 5 warm-up,
4 rotating query sets), union rows, algorithmic bytes, GB/s, and the dense
decode time for the speedup column.
"""
import argparse, json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_2605_24168_b200 as sd
from paper_2605_24168_b200 import roofline as RL

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--S", default="2,5,10,20,50,100,200,500")
ap.add_argument("--B", type=int, default=0)
a = ap.parse_args()
cfg = dict(workloads.CONFIGS[a.config])
if a.B:
    cfg["B"] = a.B
case = workloads.make_case(cfg["B"], cfg["Hq"], cfg["Hkv"], cfg["N"], dtype=cfg["dtype"], sketch=True, seed=5, device="cuda")
kv, sk = sd.KVCache.from_case(case), sd.SketchCache.from_case(case)
scale = 1 / math.sqrt(128)
gen = torch.Generator(device="cuda").manual_seed(3)
qs = [case.q] + [torch.randn(case.q.shape, generator=gen, device="cuda").to(case.q.dtype) for _ in range(3)]
out = torch.empty_like(case.q)
lse = torch.empty(case.q.shape[:2], dtype=torch.float32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

def timeit(fn, n=20):
    for i in range(5):
        fn(qs[i % 4])
    torch.cuda.synchronize()
    e0.record()
    for i in range(n):
        fn(qs[i % 4])
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3

dense_us = timeit(lambda q: sd.dense_decode(q, kv, scale=scale, out=out, lse=lse), n=5)
for S in [float(x) for x in a.S.split(",")]:
    _, _, idx, cnt = sd.sparse_decode_fused(case.q, kv, sk, S=S, scale=scale, return_idx=True)
    B, Hq, k = idx.shape
    x = idx.view(B, cfg["Hkv"], -1).long().sort(-1).values
    new = torch.ones_like(x, dtype=torch.bool)
    new[..., 1:] = x[..., 1:] != x[..., :-1]
    E = int((new & (x >= 0)).sum())
    us = timeit(lambda q: sd.sparse_decode_fused(q, kv, sk, S=S, scale=scale, out=out, lse=lse))
    m = RL.sparse_step_bytes(B, Hq, cfg["Hkv"], cfg["N"], k, union_rows_total=E)
    sd.clear_device_error()
    sd.sparse_decode_fused(case.q, kv, sk, S=S, scale=scale, out=out, lse=lse)
    fb = sd.read_stats()["fallback_rows"]
    print(json.dumps({"config": a.config, "B": B, "S": S, "k": k, "us": round(us, 1), "union_rows": E,
                      "bytes": m["total_union"], "gbs": round(m["total_union"] / us / 1e3, 1),
                      "frac": round(m["total_union"] / us / 1e3 / 6540.2, 3), "dense_us": round(dense_us, 1),
                      "speedup": round(dense_us / us, 2), "fallback_rows": fb}))
