"""Parity rules between the CUDA path and the fp64 oracle (SURVEY.md 8(c),
BASELINE.json north_star).

* Index sets: |I_gpu| = k_b, strictly increasing, in range; every token whose
  oracle score exceeds tau + 1e-5*M_row is selected and every selected token
  scores >= tau - 1e-5*M_row (tau = oracle k-th score, M_row = max |score|).
  Exact ties (bit-identical fp32 scores) are checked bit-exactly elsewhere.
* Outputs are compared with oracle.attend_given(I_gpu) so that selection
  ambiguity cannot leak into output error: max_d |o - o_ref| / max_d |o_ref|.
"""
import numpy as np
import torch

import oracle

SEL_REL_GAP = 1e-5          # BASELINE.json: "gap exceeds 1e-5 relative"
OUT_TOL_BF16 = 1e-2         # BASELINE.json: "within 1e-2 max relative error for bf16 KV"
OUT_TOL_F32 = 1e-5          # fp32 KV (cfg1)
LSE_TOL = 1e-3              # SURVEY.md 8(c) proposal: |dlse| <= 1e-3 max(1, |lse|)


def check_selection(idx_row, count, scores, k):
    """idx_row: np int array (the GPU row), scores: oracle fp64 scores [N]."""
    N = scores.shape[0]
    assert count == k, f"count {count} != k {k}"
    sel = np.asarray(idx_row[:count], dtype=np.int64)
    assert sel.size == k
    assert np.all((sel >= 0) & (sel < N)), "index out of range"
    assert np.all(np.diff(sel) > 0), "indices not strictly increasing"
    ref = oracle.topk_select(scores, k)
    tau = scores[ref].min()
    M = max(np.abs(scores).max(), 1e-300)
    band = SEL_REL_GAP * M
    chosen = np.zeros(N, dtype=bool)
    chosen[sel] = True
    must = scores > tau + band
    assert np.all(chosen[must]), f"missed {np.flatnonzero(must & ~chosen)[:8]} (tau={tau}, band={band})"
    assert np.all(scores[sel] >= tau - band), "selected a clearly-losing token"
    return sel


def check_region_selection(idx_row, count, scores, n_sink, n_local, heavy_fraction=0.0, k_abs=0):
    """NEXT-1: all sinks [0, lo) and locals [hi, N) kept, plus the
    middle's top-kh under the same tolerance rule as check_selection."""
    N = scores.shape[0]
    lo = min(n_sink, N)
    hi = max(lo, N - min(n_local, N))
    kh = oracle.heavy_budget(N, n_sink, n_local, heavy_fraction, k_abs)
    total = lo + (N - hi) + kh
    assert count == total, f"count {count} != {total}"
    sel = np.asarray(idx_row[:count], dtype=np.int64)
    assert np.all(np.diff(sel) > 0), "indices not strictly increasing"
    edge = np.concatenate([np.arange(0, lo), np.arange(hi, N)])
    assert np.isin(edge, sel).all(), "a sink / local token is missing"
    mid = sel[(sel >= lo) & (sel < hi)]
    if kh > 0:
        check_selection(mid - lo, kh, scores[lo:hi], kh)
    else:
        assert mid.size == 0
    return sel


def rel_err(o, ref):
    o = np.asarray(o, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return np.abs(o - ref).max() / max(np.abs(ref).max(), 1e-30)


def check_lse(lse, ref):
    assert abs(lse - ref) <= LSE_TOL * max(1.0, abs(ref)), (lse, ref)


def host_subcase(case, b):
    """A single-sequence host copy of sequence b of a (device) DecodeCase, with
    its pages renumbered 0..n-1 (inputs only; used to feed the oracle)."""
    from workloads.gen import DecodeCase
    N = int(case.seq_lens[b].item())
    npg = (N + case.page_size - 1) // case.page_size
    pages = case.page_table[b, :npg].long()
    kp = case.k_pages[pages].cpu()
    vp = case.v_pages[pages].cpu()
    sp = case.sketch_pages[pages].cpu() if case.sketch_pages is not None else None
    ch = case.channel_ids[b:b + 1].cpu() if case.channel_ids is not None else None
    return DecodeCase(B=1, Hq=case.Hq, Hkv=case.Hkv, D=case.D, page_size=case.page_size, C=case.C,
                      seq_lens=torch.tensor([N], dtype=torch.int32),
                      page_table=torch.arange(npg, dtype=torch.int32)[None],
                      q=case.q[b:b + 1].cpu(), k_pages=kp, v_pages=vp, channel_ids=ch, sketch_pages=sp,
                      seed=case.seed, dist=case.dist)


def sketch_view(case, b):
    """Sequence b of a (device) DecodeCase as oracle inputs for the SELECTION
    only: q, the sequence's sketch pages (renumbered 0..n-1) and channel ids.
    K/V are a one-page placeholder that sketch-mode scores never read, so a
    2^20-token sequence costs its 16 B/token sketch on the host, not 512 B."""
    from workloads.gen import DecodeCase
    N = int(case.seq_lens[b].item())
    npg = (N + case.page_size - 1) // case.page_size
    pages = case.page_table[b, :npg].long()
    sp = case.sketch_pages[pages].cpu()
    ph = torch.zeros((1,) + tuple(case.k_pages.shape[1:]), dtype=case.k_pages.dtype)
    return DecodeCase(B=1, Hq=case.Hq, Hkv=case.Hkv, D=case.D, page_size=case.page_size, C=case.C,
                      seq_lens=torch.tensor([N], dtype=torch.int32),
                      page_table=torch.arange(npg, dtype=torch.int32)[None],
                      q=case.q[b:b + 1].cpu(), k_pages=ph, v_pages=ph,
                      channel_ids=case.channel_ids[b:b + 1].cpu(), sketch_pages=sp, seed=case.seed, dist=case.dist)


def rows_view(case, b, g, tokens):
    """KV head g of sequence b restricted to `tokens` (ascending, unique), as a
    one-sequence, one-KV-head case whose token i is the original token
    tokens[i]: the K/V rows are gathered through the page table (pure data
    movement), q holds the group's G query heads.  oracle.attend_given on
    np.searchsorted(tokens, I) then attends over exactly the original rows I."""
    from workloads.gen import DecodeCase
    ps = case.page_size
    t = torch.as_tensor(np.asarray(tokens, dtype=np.int64), device=case.page_table.device)
    pg = case.page_table[b, t // ps].long()
    sl = t % ps
    n = int(t.numel())
    npg = (n + ps - 1) // ps
    G = case.Hq // case.Hkv

    def gather(pool):
        rows = pool[pg, sl, g]                                   # [n, D]
        out = torch.zeros((npg * ps, 1, case.D), dtype=pool.dtype, device=pool.device)
        out[:n, 0] = rows
        return out.view(npg, ps, 1, case.D).cpu()

    return DecodeCase(B=1, Hq=G, Hkv=1, D=case.D, page_size=ps, C=case.C,
                      seq_lens=torch.tensor([n], dtype=torch.int32),
                      page_table=torch.arange(npg, dtype=torch.int32)[None],
                      q=case.q[b:b + 1, g * G:(g + 1) * G].cpu(), k_pages=gather(case.k_pages),
                      v_pages=gather(case.v_pages), channel_ids=None, sketch_pages=None, seed=case.seed,
                      dist=case.dist)


def check_rows_full_size(case, b, heads, S, idx, cnt, out, lse, gpu_scores=None, scale=None, out_tol=1e-4):
    """Full-size parity of rows (b, h) for h in `heads`: the selection against
    the fp64 oracle scores (tolerance rule) and, when the GPU's own fp32 scores
    are given, bit-exact against oracle.topk_select on them; the output against
    oracle.attend_given on the GPU's selection.  idx/cnt/out/lse: host arrays."""
    scale = scale if scale is not None else 1.0 / np.sqrt(case.D)
    sv = oracle.from_case(sketch_view(case, b))
    N = int(case.seq_lens[b].item())
    k = oracle.budget_k(S, N)
    G = case.Hq // case.Hkv
    sels = {}
    for h in heads:
        scores = oracle.index_scores(sv, 0, int(h), "sketch")
        sels[h] = check_selection(idx[b, h], int(cnt[b, h]), scores, k)
        if gpu_scores is not None:
            ref = oracle.topk_select(np.asarray(gpu_scores[h][:N], dtype=np.float64), k)
            assert np.array_equal(sels[h], ref), (b, h, "not the exact top-k of the GPU's own fp32 scores")
    for g in sorted({int(h) // G for h in heads}):
        hs = [h for h in heads if int(h) // G == g]
        toks = np.unique(np.concatenate([sels[h] for h in hs]))
        rv = oracle.from_case(rows_view(case, b, g, toks))
        for h in hs:
            ro, rl = oracle.attend_given(rv, 0, int(h) - g * G, np.searchsorted(toks, sels[h]), scale)
            assert rel_err(out[b, h], ro) <= out_tol, (b, h, rel_err(out[b, h], ro))
            check_lse(float(lse[b, h]), rl)
