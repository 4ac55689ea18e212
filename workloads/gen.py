"""Seeded synthetic paged-KV decode workloads.

Recipe (SURVEY.md 8(d) "Value distributions"):

* Geometry follows the paper's kernel tables: GQA Hq=32, Hkv=8, D=128, page
  size 16, NHD layout inside a page (Table 1 caption), bf16
  storage (BASELINE.json north_star) or fp32 (BASELINE.json configs[0]).
* Pages of every sequence are drawn from one pool through a random
  permutation, so consecutive logical pages are never physically adjacent
  (SPEC.md:34-39 page table; gathers must go through the table).
* Distributions:
    iid     q, K, V ~ N(0, 1), rounded to the storage dtype (default).
    spec    q, K, V ~ N(0, 1)/sqrt(D), kept as one parity case.
    needle  iid plus, per (sequence, KV head), `n_needles` planted keys
            K[t] += nu*sqrt(D)*qbar/|qbar|^2 (qbar = mean query of the group),
            which lifts those logits by ~nu for every head of the group
            (SPEC.md:459 planted needle, RULER/LOFT-shaped retrieval).
    dup     iid, then 1/8 of each sequence's key rows are overwritten by copies
            of other rows: exact score ties (tie-break stress).
    equal   every key row of a (sequence, KV head) is the same vector: all
            scores tie, so the lowest indices must win.
* The Double-Sparsity channel sketch ("8 x 16-bit channels") is
  setup, not the timed path: channel_ids per (sequence, KV head) are the C
  channels with the largest mean |K|, stored ascending,
  and the sketch holds exact bf16 copies of those key channels, laid out
  head-major inside a page: sketch_pages[page][Hkv][page_size][C].

Nothing here computes a score, a selection or an attention output.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import Optional, Sequence, Union

import torch


@dataclass
class DecodeCase:
    B: int
    Hq: int
    Hkv: int
    D: int
    page_size: int
    C: int
    seq_lens: torch.Tensor            # int32 [B]
    page_table: torch.Tensor          # int32 [B][max_pages]  (-1 = unused)
    q: torch.Tensor                   # [B][Hq][D]           storage dtype
    k_pages: torch.Tensor             # [num_pages][page_size][Hkv][D]
    v_pages: torch.Tensor             # [num_pages][page_size][Hkv][D]
    channel_ids: Optional[torch.Tensor]   # int32 [B][Hkv][C]
    sketch_pages: Optional[torch.Tensor]  # bf16 [num_pages][Hkv][page_size][C]
    seed: int = 0
    dist: str = "iid"

    @property
    def G(self) -> int:
        return self.Hq // self.Hkv

    @property
    def num_pages(self) -> int:
        return int(self.k_pages.shape[0])

    @property
    def max_pages(self) -> int:
        return int(self.page_table.shape[1])

    @property
    def dtype(self) -> torch.dtype:
        return self.k_pages.dtype

    def to(self, device) -> "DecodeCase":
        mv = lambda t: None if t is None else t.to(device)
        return replace(self, seq_lens=mv(self.seq_lens), page_table=mv(self.page_table),
                       q=mv(self.q), k_pages=mv(self.k_pages), v_pages=mv(self.v_pages),
                       channel_ids=mv(self.channel_ids), sketch_pages=mv(self.sketch_pages))


def _randn(shape, gen, device, dtype, std=1.0):
    x = torch.randn(shape, generator=gen, device=device, dtype=torch.float32)
    if std != 1.0:
        x.mul_(std)
    return x.to(dtype)


def _fill_randn_(t: torch.Tensor, gen, std=1.0, chunk=4096):
    """Fill a [P, ...] tensor page-chunk by page-chunk (bounded fp32 temp)."""
    for p0 in range(0, t.shape[0], chunk):
        p1 = min(t.shape[0], p0 + chunk)
        t[p0:p1] = _randn(tuple(t[p0:p1].shape), gen, t.device, t.dtype, std)


def _token_rows(page_table_row: torch.Tensor, toks: torch.Tensor, ps: int):
    """Physical (page, slot) of logical tokens."""
    return page_table_row[toks // ps].long(), (toks % ps).long()


def make_case(B: int, Hq: int, Hkv: int, seq_lens: Union[int, Sequence[int]], *, D: int = 128,
              page_size: int = 16, C: int = 8, dtype: torch.dtype = torch.bfloat16,
              seed: int = 0, dist: str = "iid", n_needles: int = 0, nu: float = 3.0,
              sketch: bool = True, spare_pages: int = 0, device="cpu",
              sketch_dtype: torch.dtype = torch.bfloat16) -> DecodeCase:
    if Hq % Hkv:
        raise ValueError("Hq must be a multiple of Hkv")
    if isinstance(seq_lens, int):
        seq_lens = [seq_lens] * B
    seq_lens = [int(n) for n in seq_lens]
    assert len(seq_lens) == B and all(n >= 1 for n in seq_lens)
    device = torch.device(device)
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed))
    ps = page_size
    npages = [(n + ps - 1) // ps for n in seq_lens]
    max_pages = max(npages)
    total = sum(npages) + spare_pages
    perm = torch.randperm(total, generator=gen, device=device).to(torch.int32)
    page_table = torch.full((B, max_pages), -1, dtype=torch.int32, device=device)
    off = 0
    owner = torch.zeros(total, dtype=torch.long, device=device)
    for b in range(B):
        page_table[b, :npages[b]] = perm[off:off + npages[b]]
        owner[perm[off:off + npages[b]].long()] = b
        off += npages[b]

    std = 1.0 / math.sqrt(D) if dist == "spec" else 1.0
    q = _randn((B, Hq, D), gen, device, dtype, std)
    k_pages = torch.empty((total, ps, Hkv, D), dtype=dtype, device=device)
    v_pages = torch.empty((total, ps, Hkv, D), dtype=dtype, device=device)
    _fill_randn_(k_pages, gen, std)
    _fill_randn_(v_pages, gen, std)

    G = Hq // Hkv
    if dist in ("needle", "dup", "equal"):
        for b in range(B):
            N = seq_lens[b]
            for g in range(Hkv):
                if dist == "needle" and n_needles > 0:
                    n = min(n_needles, N)
                    toks = torch.randperm(N, generator=gen, device=device)[:n]
                    pg, sl = _token_rows(page_table[b], toks, ps)
                    qbar = q[b, g * G:(g + 1) * G].float().mean(0)
                    delta = nu * math.sqrt(D) * qbar / qbar.dot(qbar)
                    rows = k_pages[pg, sl, g].float() + delta
                    k_pages[pg, sl, g] = rows.to(dtype)
                elif dist == "dup" and N >= 2:
                    n = max(1, N // 8)
                    dst = torch.randperm(N, generator=gen, device=device)[:n]
                    src = torch.randint(0, N, (n,), generator=gen, device=device)
                    pd, sd = _token_rows(page_table[b], dst, ps)
                    pss, ss = _token_rows(page_table[b], src, ps)
                    k_pages[pd, sd, g] = k_pages[pss, ss, g].clone()
                elif dist == "equal":
                    toks = torch.arange(N, device=device)
                    pg, sl = _token_rows(page_table[b], toks, ps)
                    row = _randn((D,), gen, device, dtype, std)
                    k_pages[pg, sl, g] = row.expand(N, D)

    channel_ids = sketch_pages = None
    if sketch:
        assert C <= D
        channel_ids = torch.empty((B, Hkv, C), dtype=torch.int32, device=device)
        for b in range(B):
            N = seq_lens[b]
            toks = torch.arange(N, device=device)
            pg, sl = _token_rows(page_table[b], toks, ps)
            mabs = torch.zeros((Hkv, D), dtype=torch.float64, device=device)
            for t0 in range(0, N, 65536):
                rows = k_pages[pg[t0:t0 + 65536], sl[t0:t0 + 65536]]  # [n, Hkv, D]
                mabs += rows.abs().double().sum(0)
            # largest mean |K| first; stable so equal means keep the lower channel
            order = torch.sort(-mabs, dim=1, stable=True).indices[:, :C]
            channel_ids[b] = torch.sort(order, dim=1).values.to(torch.int32)
        sketch_pages = torch.empty((total, Hkv, ps, C), dtype=torch.bfloat16, device=device)
        chunk = 2048
        for p0 in range(0, total, chunk):
            p1 = min(total, p0 + chunk)
            ch = channel_ids[owner[p0:p1]].long()                       # [n, Hkv, C]
            kp = k_pages[p0:p1].permute(0, 2, 1, 3)                      # [n, Hkv, ps, D]
            idx = ch[:, :, None, :].expand(p1 - p0, Hkv, ps, C)
            sketch_pages[p0:p1] = torch.gather(kp, 3, idx).to(torch.bfloat16)
        if sketch_dtype != torch.bfloat16:
            # NEXT-4 low-precision sketch: the same channels
            # rounded to the storage type (fp8 e4m3: round to nearest, |x| <= 448)
            sketch_pages = sketch_pages.to(sketch_dtype)

    return DecodeCase(B=B, Hq=Hq, Hkv=Hkv, D=D, page_size=ps, C=C,
                      seq_lens=torch.tensor(seq_lens, dtype=torch.int32, device=device),
                      page_table=page_table, q=q, k_pages=k_pages, v_pages=v_pages,
                      channel_ids=channel_ids, sketch_pages=sketch_pages, seed=seed, dist=dist)


def _cfg4_len(t: int) -> int:
    """SWE-agentic growing context, 67 turns, 8K -> 128K (SURVEY.md 8(d) cfg 4)."""
    return 8192 + (t * 122880) // 66


# BASELINE.json configs -> concrete synthetic inputs.
CONFIGS = {
    "cfg1": dict(B=1, Hq=8, Hkv=1, N=4096, S=50.0, dtype=torch.float32, sketch=False),
    "cfg2_s10": dict(B=8, Hq=32, Hkv=8, N=32768, S=10.0, dtype=torch.bfloat16, sketch=True),
    "cfg2_s50": dict(B=8, Hq=32, Hkv=8, N=32768, S=50.0, dtype=torch.bfloat16, sketch=True),
    "cfg2_s100": dict(B=8, Hq=32, Hkv=8, N=32768, S=100.0, dtype=torch.bfloat16, sketch=True),
    "cfg3": dict(B=16, Hq=32, Hkv=8, N=131072, S=50.0, dtype=torch.bfloat16, sketch=True),
    # NEXT-4: cfg3 with the 8-channel sketch stored as fp8 e4m3 (half the indexer bytes)
    "cfg3_fp8": dict(B=16, Hq=32, Hkv=8, N=131072, S=50.0, dtype=torch.bfloat16, sketch=True,
                     sketch_dtype=torch.float8_e4m3fn),
    "cfg4_t66": dict(B=32, Hq=32, Hkv=8, N=_cfg4_len(66), S=50.0, dtype=torch.bfloat16, sketch=True),
    "cfg4_t33": dict(B=32, Hq=32, Hkv=8, N=_cfg4_len(33), S=50.0, dtype=torch.bfloat16, sketch=True),
    "cfg4_t0": dict(B=32, Hq=32, Hkv=8, N=_cfg4_len(0), S=50.0, dtype=torch.bfloat16, sketch=True),
    "cfg5": dict(B=1, Hq=32, Hkv=8, N=1 << 20, S=100.0, dtype=torch.bfloat16, sketch=True),
}


def config_case(name: str, *, seed: Optional[int] = None, device="cpu", **over) -> DecodeCase:
    c = dict(CONFIGS[name])
    c.update(over)
    if seed is None:
        seed = 1000 * (list(CONFIGS).index(name) + 1)
    return make_case(c["B"], c["Hq"], c["Hkv"], c["N"], dtype=c["dtype"], sketch=c["sketch"],
                     seed=seed, device=device,
                     **{k: v for k, v in c.items() if k in ("dist", "n_needles", "nu", "C", "sketch_dtype")})
