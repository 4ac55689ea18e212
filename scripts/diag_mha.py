"""MHA (Hq = Hkv = 32, G = 1) rows that leave the fused fast path (Table-2 layout, N = 128K):
host recomputation of each row's sample bracket, band and region counts from the unfused scores."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, workloads, paper_2605_24168_b200 as sd
B, N = int(sys.argv[1]) if len(sys.argv) > 1 else 4, 131072
S = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
case = workloads.make_case(B, 32, 32, N, seed=5000 + B, device="cuda")
kv = sd.KVCache(case.k_pages, case.v_pages, case.page_table, case.seq_lens, N)
sk = sd.SketchCache.from_case(case)
k = sd.budget_k(S, N)
sd.clear_device_error()
out, lse, idx, cnt = sd.sparse_decode_fused(case.q, kv, sk, S=S, return_idx=True)
torch.cuda.synchronize()
print("fallback_rows", sd.read_stats()["fallback_rows"], "err", sd.read_device_error(), "k", k)
sc = sd.sparse_index_score(case.q, kv, sk)[:, :, :N].cpu().numpy()
def keys(x):
    u = x.view(np.uint32).astype(np.uint64)
    return np.where(u & 0x80000000, (~u) & 0xFFFFFFFF, u | 0x80000000).astype(np.uint64)
npg = N // 16; cap_pages = 256; spg = -(-npg // cap_pages); ns = -(-npg // spg)
pos = np.concatenate([np.arange(16) + p * spg * 16 for p in range(ns)]); f = len(pos) / N
mu = k * f; sdv = math.sqrt(k * f * (1 - f)); r_lo = math.ceil(mu + 4 * sdv + 1); r_hi = math.floor(mu - 4 * sdv)
print("r_lo", r_lo, "r_hi", r_hi)
worst = []
for b in range(B):
    for h in range(32):
        kk = keys(sc[b, h]); srt = np.sort(kk)[::-1]; tau = srt[k - 1]
        samp = np.sort(kk[pos])[::-1]
        lo = (samp[r_lo - 1] >> 13) << 13; hi = ((samp[r_hi - 1] >> 13) << 13) | 0x1FFF
        sure = int((kk > hi).sum()); inb = (kk >= lo) & (kk <= hi); band = int(inb.sum())
        reg = np.bincount(np.arange(N)[inb] // 1024, minlength=N // 1024).max()
        ties = int((kk == tau).sum())
        ok = sure <= k <= sure + band
        worst.append((not ok, band, reg, ties, b, h))
worst.sort(reverse=True)
print("worst rows (miss, band, max per 1024-token region, ties at tau, b, h):", worst[:8])
