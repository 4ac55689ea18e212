"""One small fused step per shape for compute-sanitizer (memcheck / racecheck)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_2605_24168_b200 as sd

for (B, Hq, Hkv, lens, S) in [(2, 32, 8, [20000, 9000], 50.0), (1, 32, 8, [70001], 2.0), (2, 16, 2, [5000, 64], 10.0)]:
    case = workloads.make_case(B, Hq, Hkv, lens, seed=5, dist="needle", n_needles=10).to("cuda")
    kv, sk = sd.KVCache.from_case(case), sd.SketchCache.from_case(case)
    out, lse, idx, cnt = sd.sparse_decode_fused(case.q, kv, sk, S=S, scale=1 / math.sqrt(128), return_idx=True)
    sd.dense_decode(case.q, kv, scale=1 / math.sqrt(128))
torch.cuda.synchronize()
print("sanitize run done; device error", sd.read_device_error())
