"""One small fused step (G = 4) for compute-sanitizer racecheck."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_2605_24168_b200 as sd

case = workloads.make_case(1, 8, 2, [9000], seed=5, dist="needle", n_needles=10).to("cuda")
kv, sk = sd.KVCache.from_case(case), sd.SketchCache.from_case(case)
sd.sparse_decode_fused(case.q, kv, sk, S=50.0, scale=1 / math.sqrt(128), return_idx=True)
torch.cuda.synchronize()
print("done", sd.read_device_error())
