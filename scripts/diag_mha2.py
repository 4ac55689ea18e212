"""Find the (query, row) of the Table-2 MHA sweep (B=16, N=128K) that leaves the fused fast path."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, workloads, paper_2605_24168_b200 as sd
B, N, S = 16, 131072, float(sys.argv[1]) if len(sys.argv) > 1 else 20.0
case = workloads.make_case(B, 32, 32, N, seed=5000 + B, device="cuda")
kv = sd.KVCache(case.k_pages, case.v_pages, case.page_table, case.seq_lens, N)
sk = sd.SketchCache.from_case(case)
g = torch.Generator(device="cuda"); g.manual_seed(17)
qs = [case.q] + [torch.randn(case.q.shape, generator=g, device="cuda").to(case.q.dtype) for _ in range(3)]
k = sd.budget_k(S, N)
def keys(x):
    u = x.view(np.uint32).astype(np.uint64)
    return np.where(u & 0x80000000, (~u) & 0xFFFFFFFF, u | 0x80000000).astype(np.uint64)
npg = N // 16; spg = -(-npg // 256); ns = -(-npg // spg)
pos = np.concatenate([np.arange(16) + p * spg * 16 for p in range(ns)]); f = len(pos) / N
mu = k * f; sdv = math.sqrt(k * f * (1 - f)); r_lo = math.ceil(mu + 4 * sdv + 1); r_hi = math.floor(mu - 4 * sdv)
for qi, q in enumerate(qs):
    sd.clear_device_error()
    out, lse, idx, cnt = sd.sparse_decode_fused(q, kv, sk, S=S, return_idx=True)
    torch.cuda.synchronize()
    fb = sd.read_stats()["fallback_rows"]
    if not fb:
        print(f"q{qi}: no fallback"); continue
    sc = sd.sparse_index_score(q, kv, sk)[:, :, :N].cpu().numpy()
    res = []
    for b in range(B):
        for h in range(32):
            kk = keys(sc[b, h]); tau = np.sort(kk)[::-1][k - 1]
            samp = np.sort(kk[pos])[::-1]
            lo = (samp[r_lo - 1] >> 13) << 13; hi = ((samp[r_hi - 1] >> 13) << 13) | 0x1FFF
            sure = int((kk > hi).sum()); inb = (kk >= lo) & (kk <= hi); band = int(inb.sum())
            reg = np.bincount(np.arange(N)[inb] // 1024, minlength=N // 1024).max()
            ties = int((kk == tau).sum())
            res.append((not (sure <= k <= sure + band), band, int(reg), ties, b, h))
    res.sort(reverse=True)
    print(f"q{qi}: fallback_rows={fb}; worst (miss, band, max/region, ties, b, h):", res[:4])
