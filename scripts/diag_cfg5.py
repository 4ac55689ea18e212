"""Which cfg5 (N = 2^20, B = 1, Hq = 32, Hkv = 8, S = 100) rows leave the fused fast path, and why:
recompute each row's sample bracket on the host from the unfused fp32 indexer scores."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, workloads, paper_2605_24168_b200 as sd

case = workloads.config_case("cfg5", device="cuda", seed=6000)
N, S = 1 << 20, 100.0
kv = sd.KVCache(case.k_pages, case.v_pages, case.page_table, case.seq_lens, N)
sk = sd.SketchCache.from_case(case)
g = torch.Generator(device="cuda"); g.manual_seed(17)
qs = [case.q] + [torch.randn(case.q.shape, generator=g, device="cuda").to(case.q.dtype) for _ in range(5)]
k = sd.budget_k(S, N)
def keys(x):  # order-preserving map of fp32
    u = x.view(np.uint32).astype(np.uint64)
    return np.where(u & 0x80000000, (~u) & 0xFFFFFFFF, u | 0x80000000).astype(np.uint64)
npg = N // 16; cap_pages = 256; spg = -(-npg // cap_pages); ns_pages = -(-npg // spg)
pos = np.concatenate([np.arange(16) + p * spg * 16 for p in range(ns_pages)])
pos = pos[pos < N]; f = len(pos) / N
mu = k * f; sdv = math.sqrt(k * f * (1 - f))
r_lo = math.ceil(mu + 4 * sdv + 1); r_hi = math.floor(mu - 4 * sdv)
print("k", k, "n_s", len(pos), "r_lo", r_lo, "r_hi", r_hi)
for qi, q in enumerate(qs):
    sd.clear_device_error()
    out, lse, idx, cnt = sd.sparse_decode_fused(q, kv, sk, S=S, return_idx=True)
    torch.cuda.synchronize()
    fb = sd.read_stats()["fallback_rows"]
    sc = sd.sparse_index_score(q, kv, sk)[0, :, :N].cpu().numpy()
    bad = []
    for h in range(32):
        kk = keys(sc[h])
        srt = np.sort(kk)[::-1]
        tau = srt[k - 1]
        samp = np.sort(kk[pos])[::-1]
        lo_key, hi_key = samp[r_lo - 1], samp[r_hi - 1]
        lo_bin = (lo_key >> 13) << 13; hi_bin = ((hi_key >> 13) << 13) | 0x1FFF
        sure = int((kk > hi_bin).sum()); band = int(((kk >= lo_bin) & (kk <= hi_bin)).sum())
        ok = sure <= k <= sure + band
        ties = int((kk == tau).sum())
        if not ok or ties > 1:
            bad.append((h, sure, band, ties))
    print(f"q{qi}: fallback_rows={fb} host-bracket-misses/ties={bad[:6]}")
