"""Algorithmic byte model of one decode step (
PAPER.md:59 Fig. 1a "Dense reads the full KV cache every step (O(N d) bytes);
Sparse ... selects k rows (O(k d) bytes)").

These are the bytes the METHOD must move, not what an implementation moves:
score round-trips, index writes and split-k partials count against the
implementation and are excluded.

  sketch scan   B*Hkv*N*C*2                (once per KV head, shared by its G q-heads)
  exact scan    B*Hkv*N*D*w                (indexer reading full keys, P:145 oracle mode)
  rows (union)  2*B*Hkv*E*D*w              E = |U_{h in group} I_h| per (b, g)
  rows (paper)  2*B*Hq*k*D*w               per-head gathers, no dedup
  q/out/lse     B*Hq*D*w_q + B*Hq*D*w_o + 4*B*Hq
  page table    4*B*ceil(N/16)
  dense         2*B*N*Hkv*D*w (+ q/out/lse + page table)
"""
from __future__ import annotations

import math
from typing import Optional, Sequence, Union

IntOrList = Union[int, Sequence[int]]


def _lens(B: int, N: IntOrList):
    return [int(N)] * B if isinstance(N, (int,)) else [int(n) for n in N]


def dense_bytes(B, N: IntOrList, Hkv, D=128, w=2, Hq=None, w_q=None, w_o=None, page_size=16,
                include_io=False) -> int:
    lens = _lens(B, N)
    kv = sum(2 * n * Hkv * D * w for n in lens)
    if not include_io:
        return kv
    Hq = Hq or Hkv
    return kv + _io(B, Hq, D, w_q or w, w_o or w) + sum(4 * math.ceil(n / page_size) for n in lens)


def gather_bytes_per_head(B, Hq, k: IntOrList, D=128, w=2) -> int:
    """Paper accounting (no GQA dedup): 2*B*Hq*k*D*w."""
    ks = _lens(B, k)
    return sum(2 * Hq * kk * D * w for kk in ks)


def gather_bytes_union(union_rows_total: int, D=128, w=2) -> int:
    """Must-move rows: sum over (b, g) of the union size E_bg, times K+V rows."""
    return 2 * union_rows_total * D * w


def expected_union(N: int, k: int, G: int) -> float:
    """E = N (1 - (1 - k/N)^G) for G independent k-subsets."""
    return N * (1.0 - (1.0 - k / N) ** G)


def indexer_bytes(B, N: IntOrList, Hkv, C=8, sketch_w=2, D=128, w=2, exact=False) -> int:
    lens = _lens(B, N)
    per = D * w if exact else C * sketch_w
    return sum(Hkv * n * per for n in lens)


def _io(B, Hq, D, w_q, w_o):
    return B * Hq * D * w_q + B * Hq * D * w_o + 4 * B * Hq


def sparse_step_bytes(B, Hq, Hkv, N: IntOrList, k: IntOrList, D=128, w=2, C=8, exact=False,
                      union_rows_total: Optional[int] = None, w_o=None, page_size=16, sketch_w=2) -> dict:
    """Per-step algorithmic bytes of the fused path; `union_rows_total` (measured
    from the selected indices) gives the must-move union model, otherwise the
    independence estimate E is used."""
    lens = _lens(B, N)
    ks = _lens(B, k)
    G = Hq // Hkv
    if union_rows_total is None:
        union_rows_total = int(round(sum(Hkv * expected_union(n, kk, G) for n, kk in zip(lens, ks))))
    idx_b = indexer_bytes(B, lens, Hkv, C, sketch_w, D, w, exact)
    io = _io(B, Hq, D, w, w_o or w)
    pt = sum(4 * math.ceil(n / page_size) for n in lens)
    uni = gather_bytes_union(union_rows_total, D, w)
    per = gather_bytes_per_head(B, Hq, ks, D, w)
    return {"indexer": idx_b, "rows_union": uni, "rows_per_head": per, "io": io, "page_table": pt,
            "total_union": idx_b + uni + io + pt, "total_per_head": idx_b + per + io + pt,
            "union_rows": union_rows_total}
