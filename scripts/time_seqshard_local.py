"""Per-rank step of the sequence-sharded cfg5 (N_loc = 2^17 of 2^20 tokens, B=1, Hq=32, Hkv=8,
k_b = 10486 from the global length) on one GPU: local top-k (materialised scores + radix) and
cut + attend, vs the fused single-GPU path at the same local geometry."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, workloads, paper_2605_24168_b200 as sd
dev = "cuda"
NG, P = 1 << 20, 8
nl = NG // P
case = workloads.make_case(1, 32, 8, nl, seed=9000, device=dev)
kv, sk = sd.KVCache.from_case(case), sd.SketchCache.from_case(case)
glens = torch.tensor([NG], dtype=torch.int32, device=dev)
k = sd.budget_k(100.0, NG)
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
cs, ci = sd.seqshard_local_topk(case.q, kv, sk, glens, NG, 100.0, k_max=k)
allc = torch.stack([cs] * P)
res = {"local_topk_us": t(lambda: sd.seqshard_local_topk(case.q, kv, sk, glens, NG, 100.0, k_max=k)),
       "cut_attend_us": t(lambda: sd.seqshard_cut_attend(case.q, kv, glens, allc, ci, 0, 100.0)),
       "index_score_us": t(lambda: sd.sparse_index_score(case.q, kv, sk)),
       "fused_same_k_us": t(lambda: sd.sparse_decode_fused(case.q, kv, sk, k_fixed=k))}
print(json.dumps(res))
