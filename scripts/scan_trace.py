"""Timeline of the scan's CTAs at cfg3 (debug build with -DSD_SCAN_TRACE): per CTA the
time its PDL wait returned and its end, relative to the earliest; run from a tree built
by scripts/mkvariant.sh."""
import ctypes, math, os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
import paper_2605_24168_b200 as sd
import workloads
from paper_2605_24168_b200 import _capi

cfg = workloads.CONFIGS["cfg3"]
case = workloads.make_case(cfg["B"], cfg["Hq"], cfg["Hkv"], cfg["N"], dtype=cfg["dtype"], sketch=cfg["sketch"], seed=3,
                           device="cuda:0")
kv, sk = sd.KVCache.from_case(case), sd.SketchCache.from_case(case)
L = _capi.load()
L.sd_debug_scan_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
n = (cfg["N"] // 8192) * cfg["B"] * cfg["Hkv"]
for rep in range(5):
    sd.sparse_decode_fused(case.q, kv, sk, S=cfg["S"], scale=1 / math.sqrt(128))
    torch.cuda.synchronize()
buf = np.zeros((n, 2), dtype=np.uint64)
assert L.sd_debug_scan_trace(buf.ctypes.data, n) == 0
t0 = buf[:, 0].min()
st, en = (buf[:, 0] - t0) / 1e3, (buf[:, 1] - t0) / 1e3
q = lambda a: " ".join(f"{np.percentile(a, p):7.2f}" for p in (0, 10, 50, 90, 99, 100))
print("percentiles 0/10/50/90/99/100 (us from the first CTA's PDL release)")
print("start   ", q(st))
print("end     ", q(en))
print("duration", q(en - st))
busy = (en - st).sum() / (en.max() * 592)
print("SM-slot busy fraction (592 slots)", round(float(busy), 3))
