"""Timeline of the gather-attend's CTAs at cfg3 (debug build with -DSD_ATTEND_TRACE):
per CTA start (after its PDL wait), first unit ready, end, units processed; printed
relative to the earliest start.  Run from a tree built by scripts/mkvariant.sh.
"""
import ctypes, math, os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
import paper_2605_24168_b200 as sd
import workloads

cfg = workloads.CONFIGS["cfg3"]
case = workloads.make_case(cfg["B"], cfg["Hq"], cfg["Hkv"], cfg["N"], dtype=cfg["dtype"], sketch=cfg["sketch"], seed=3, device="cuda:0")
dc = case
kv, sk = sd.KVCache.from_case(dc), sd.SketchCache.from_case(dc)
lib = sd.load_library() if hasattr(sd, "load_library") else None
from paper_2605_24168_b200 import _capi
L = _capi.load()
L.sd_debug_attend_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
n = 2 * torch.cuda.get_device_properties(0).multi_processor_count
for rep in range(5):
    out = sd.sparse_decode_fused(dc.q, kv, sk, S=cfg["S"], scale=1 / math.sqrt(128))
    torch.cuda.synchronize()
buf = np.zeros((n, 4), dtype=np.uint64)
assert L.sd_debug_attend_trace(buf.ctypes.data, n) == 0
t0 = buf[:, 0].min()
st = (buf[:, 0] - t0) / 1e3
fu = (buf[:, 1] - t0) / 1e3
en = (buf[:, 2] - t0) / 1e3
it = buf[:, 3]
q = lambda a: " ".join(f"{np.percentile(a, p):7.2f}" for p in (0, 10, 50, 90, 100))
print("percentiles 0/10/50/90/100 (us from the first CTA start)")
print("start     ", q(st))
print("first unit", q(fu))
print("end       ", q(en))
print("units     ", q(it.astype(float)))
print("mean busy fraction", float(np.mean(en - st) / en.max()))
