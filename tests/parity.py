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
