"""Plain, slow, fp64 CPU oracle of the sparse decode-attention hot path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): no product code may call it.

What the method computes (the oracle is its plain definition):
for every decode query (sequence b, query head h) an indexer scores all N_b
cached tokens, the k_b = max(1, ceil(N_b / S)) best-scoring tokens are kept
(ties toward the smaller token index), and exact softmax attention runs over
only those rows.  Citations: PAPER.md line numbers ("P:n"), SPEC.md line
numbers ("S:n"); DESIGN.md "Readings" lists every place the paper is silent.

Numerics: every stored value (bf16 or fp32) is decoded exactly to float64;
products of two bf16/fp32 values are exact in float64 and sums carry only
float64 rounding.  Library primitives used as single steps: numpy dot/matmul,
numpy stable argsort, numpy exp/log.  Nothing is blocked, fused or reordered.

Pins (tests/test_oracle_pins.py) tie every function below to something other
than itself: SPEC worked examples, closed forms, torch SDPA in float64,
brute force on tiny inputs, algebraic identities.  Parity status per function
is listed in DESIGN.md ("Oracle pins"); no function here is unpinned.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

__all__ = [
    "budget_k", "OracleInputs", "from_case", "index_scores",
    "topk_select", "attend", "dense_decode", "sparse_decode", "attend_given",
    "lse_merge", "seqshard_decode", "sink_local_heavy_select", "heavy_budget",
    "stochastic_select", "SparseResult",
]


def _np64(x) -> np.ndarray:
    """Decode a stored tensor (torch CPU tensor or numpy array) exactly to float64."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x.detach().to("cpu").double().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x, dtype=np.float64)


def _npint(x) -> np.ndarray:
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x.detach().to("cpu").long().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x, dtype=np.int64)


# ---------------------------------------------------------------------------
# A1  budget  ("each query-head attends to 1/S fraction of total tokens";
#              rounding S:188-196: k = max(1, ceil(N / S)), S >= 1)
# ---------------------------------------------------------------------------
def budget_k(S: float, N: int, k_fixed: int = 0) -> int:
    """k_b for one sequence.  k_fixed > 0 is the absolute-form budget (S:177-180,
    Fig 2c "K retrieved tokens"); k_fixed > N is rejected."""
    if N < 1:
        raise ValueError("N must be >= 1 (S:123 non-empty sequence)")
    if k_fixed and k_fixed > 0:
        if k_fixed > N:
            raise ValueError("k > N rejected (S:201)")
        return int(k_fixed)
    if not (S >= 1.0):
        raise ValueError("S < 1 rejected (S:192)")
    # exact ceil(N / S) for a real S: N / S is evaluated in float64 and the
    # ceiling taken; when S is integral this is the integer ceiling.
    if float(S).is_integer():
        k = -(-N // int(S))
    else:
        k = math.ceil(N / S)
    return max(1, int(k))


@dataclass
class OracleInputs:
    """float64 view of one decode step's inputs (same bits the GPU reads)."""
    q: np.ndarray             # [B][Hq][D]
    k_pages: object           # [P][ps][Hkv][D] (decoded lazily per (b, g))
    v_pages: object
    page_table: np.ndarray    # [B][max_pages] int
    seq_lens: np.ndarray      # [B]
    page_size: int
    Hkv: int
    channel_ids: Optional[np.ndarray] = None   # [B][Hkv][C]
    sketch_pages: object = None                # [P][Hkv][ps][C]
    _cache: dict = field(default_factory=dict, repr=False)

    @property
    def B(self):
        return self.q.shape[0]

    @property
    def Hq(self):
        return self.q.shape[1]

    @property
    def D(self):
        return self.q.shape[2]

    @property
    def G(self):
        return self.Hq // self.Hkv

    def _rows(self, b: int):
        """Physical (page, slot) of logical tokens 0..N_b-1, via the page table."""
        N = int(self.seq_lens[b])
        t = np.arange(N)
        return self.page_table[b][t // self.page_size], t % self.page_size

    def keys(self, b: int, g: int) -> np.ndarray:
        """K rows of sequence b, KV head g, in logical order: [N_b][D] fp64."""
        key = ("K", b, g)
        if key not in self._cache:
            pg, sl = self._rows(b)
            self._cache[key] = _np64(self.k_pages[pg, sl, g])
        return self._cache[key]

    def values(self, b: int, g: int) -> np.ndarray:
        key = ("V", b, g)
        if key not in self._cache:
            pg, sl = self._rows(b)
            self._cache[key] = _np64(self.v_pages[pg, sl, g])
        return self._cache[key]

    def sketch(self, b: int, g: int) -> np.ndarray:
        """Sketch rows (the C chosen key channels) of (b, g): [N_b][C]."""
        key = ("SK", b, g)
        if key not in self._cache:
            pg, sl = self._rows(b)
            self._cache[key] = _np64(self.sketch_pages[pg, g, sl])
        return self._cache[key]


def from_case(case) -> OracleInputs:
    """Build oracle inputs from any object with the DecodeCase attributes.

    Tensors are converted with exact widening (bf16/fp32 -> fp64).  torch
    tensors for the page pools are kept as-is and indexed lazily so that only
    the rows an oracle call touches are decoded."""
    import torch
    kp = case.k_pages.cpu() if isinstance(case.k_pages, torch.Tensor) else case.k_pages
    vp = case.v_pages.cpu() if isinstance(case.v_pages, torch.Tensor) else case.v_pages
    sp = case.sketch_pages
    if isinstance(sp, torch.Tensor):
        sp = sp.cpu()
    ch = None if case.channel_ids is None else _npint(case.channel_ids)
    # torch advanced indexing needs torch index tensors; wrap pools in a small adaptor
    return OracleInputs(q=_np64(case.q), k_pages=_TorchPool(kp), v_pages=_TorchPool(vp),
                        page_table=_npint(case.page_table), seq_lens=_npint(case.seq_lens),
                        page_size=int(case.page_size), Hkv=int(case.Hkv), channel_ids=ch,
                        sketch_pages=None if sp is None else _TorchPool(sp))


class _TorchPool:
    """Lazy fp64 decoding of a torch page pool indexed with numpy index arrays."""

    def __init__(self, t):
        self.t = t

    def __getitem__(self, idx):
        import torch
        if not isinstance(self.t, torch.Tensor):
            return np.asarray(self.t[idx], dtype=np.float64)
        idx = tuple(torch.as_tensor(i) if isinstance(i, np.ndarray) else i for i in idx)
        return self.t[idx].double().numpy()


# ---------------------------------------------------------------------------
# A2  indexer scores (unscaled; selection is invariant to the positive scale)
#   sketch mode, Double Sparsity:
#       s_hat[t] = sum_{c<C} q[h][ch[b][g][c]] * sk[b][g][t][c]
#   exact mode, oracle top-k ("exact oracle top-k selection"):
#       s_hat[t] = sum_{d<D} q[h][d] * K[b][t][g][d]
# ---------------------------------------------------------------------------
def index_scores(inp: OracleInputs, b: int, h: int, mode: str = "sketch") -> np.ndarray:
    g = h // inp.G                              # contiguous GQA groups
    q = inp.q[b, h]
    if mode == "exact":
        return inp.keys(b, g) @ q
    if mode == "sketch":
        ch = inp.channel_ids[b, g]
        return inp.sketch(b, g) @ q[ch]
    raise ValueError(mode)


# ---------------------------------------------------------------------------
# A3  exact top-k (tie rule S:200 "ties broken toward smaller token
#     index"; output "returned in increasing index order" S:112)
# ---------------------------------------------------------------------------
def topk_select(scores: np.ndarray, k: int) -> np.ndarray:
    """The k first tokens of the total order (score descending, index ascending),
    returned ascending.  A stable sort of -score keeps equal scores in index order."""
    scores = np.asarray(scores, dtype=np.float64)
    if not (1 <= k <= scores.shape[0]):
        raise ValueError("need 1 <= k <= N (S:199)")
    if not np.all(np.isfinite(scores)):
        raise ValueError("non-finite score rejected (S:160)")
    order = np.argsort(-scores, kind="stable")
    return np.sort(order[:k])


# ---------------------------------------------------------------------------
# A5  weighted softmax attention over a row set ("weighted attention given
#     sparse index and associated weights"; LSE S:124)
#     s_i = scale <q, K_i>;  m = max s_i;  e_i = w_i exp(s_i - m);  l = sum e_i
#     o = sum e_i V_i / l;   lse = m + log l          (two passes, fp64)
# ---------------------------------------------------------------------------
def attend(q: np.ndarray, K: np.ndarray, V: np.ndarray, scale: float,
           weights: Optional[np.ndarray] = None):
    if K.shape[0] == 0:
        raise ValueError("empty index list rejected (S:134)")
    s = scale * (K @ q)
    if weights is None:
        w = np.ones_like(s)
    else:
        w = np.asarray(weights, dtype=np.float64)
        if not (np.all(w > 0) and np.all(np.isfinite(w))):
            raise ValueError("weights must be finite and > 0 (S:113)")
    m = s.max()
    e = w * np.exp(s - m)
    l = e.sum()
    o = (e @ V) / l
    return o, m + math.log(l)


def attend_given(inp: OracleInputs, b: int, h: int, idx: Sequence[int], scale: float,
                 weights=None):
    """Attention of (b, h) over a GIVEN index set (used to check a GPU output on
    the GPU's own selection, SURVEY.md 8(c) parity rules)."""
    g = h // inp.G
    idx = np.asarray(idx, dtype=np.int64)
    N = int(inp.seq_lens[b])
    if idx.size and (idx.min() < 0 or idx.max() >= N):
        raise ValueError("index out of range (S:61)")
    return attend(inp.q[b, h], inp.keys(b, g)[idx], inp.values(b, g)[idx], scale, weights)


def dense_decode(inp: OracleInputs, scale: float):
    """Full softmax over all N_b rows (P:59 dense regime)."""
    o = np.zeros((inp.B, inp.Hq, inp.D))
    lse = np.zeros((inp.B, inp.Hq))
    for b in range(inp.B):
        for h in range(inp.Hq):
            g = h // inp.G
            o[b, h], lse[b, h] = attend(inp.q[b, h], inp.keys(b, g), inp.values(b, g), scale)
    return o, lse


@dataclass
class SparseResult:
    idx: List[List[np.ndarray]]   # [B][Hq] ascending int64
    o: np.ndarray                 # [B][Hq][D]
    lse: np.ndarray               # [B][Hq]
    k: np.ndarray                 # [B] budgets
    tau: np.ndarray               # [B][Hq] k-th best score
    tau_plus: np.ndarray          # [B][Hq] best excluded score (-inf if none)
    mrow: np.ndarray              # [B][Hq] max_t |score_t|


def sparse_decode(inp: OracleInputs, S: float, scale: float, mode: str = "sketch",
                  k_fixed: int = 0, rows=None) -> SparseResult:
    """The whole hot path (A1-A5) per (b, h): scores -> top-k -> attention over the
    chosen rows with EXACT full-key logits (the sketch only selects).
    `rows` optionally restricts to a list of (b, h) pairs (bounded samples)."""
    B, Hq = inp.B, inp.Hq
    res = SparseResult(idx=[[None] * Hq for _ in range(B)], o=np.full((B, Hq, inp.D), np.nan),
                       lse=np.full((B, Hq), np.nan), k=np.zeros(B, dtype=np.int64),
                       tau=np.full((B, Hq), np.nan), tau_plus=np.full((B, Hq), np.nan),
                       mrow=np.full((B, Hq), np.nan))
    todo = rows if rows is not None else [(b, h) for b in range(B) for h in range(Hq)]
    for b, h in todo:
        N = int(inp.seq_lens[b])
        k = budget_k(S, N, k_fixed)
        res.k[b] = k
        s = index_scores(inp, b, h, mode)
        I = topk_select(s, k)
        chosen = np.zeros(N, dtype=bool)
        chosen[I] = True
        res.idx[b][h] = I
        res.tau[b, h] = s[I].min()
        res.tau_plus[b, h] = s[~chosen].max() if k < N else -np.inf
        res.mrow[b, h] = np.abs(s).max()
        res.o[b, h], res.lse[b, h] = attend_given(inp, b, h, I, scale)
    return res


# ---------------------------------------------------------------------------
# Split-k / cross-shard LSE merge (flash-decoding identity; S:124 LSE):
#   lse = log sum_p exp(lse_p);   o = sum_p exp(lse_p - lse) * o_p
# An empty part has lse_p = -inf and contributes nothing.
# ---------------------------------------------------------------------------
def lse_merge(part_o: np.ndarray, part_lse: np.ndarray):
    part_o = np.asarray(part_o, dtype=np.float64)
    part_lse = np.asarray(part_lse, dtype=np.float64)
    m = np.max(part_lse, axis=0)
    safe_m = np.where(np.isfinite(m), m, 0.0)
    wts = np.exp(part_lse - safe_m)                  # exp(-inf) = 0 for empty parts
    l = wts.sum(axis=0)
    lse = safe_m + np.log(l)
    o = (wts[..., None] * part_o).sum(axis=0) / l[..., None]
    return o, lse


def seqshard_decode(inp: OracleInputs, S: float, scale: float, P: int, mode: str = "sketch"):
    """Sequence-sharded exact top-k + LSE merge, simulated in-process:
    shard r holds tokens [r*N/P, (r+1)*N/P) (contiguous); each shard keeps its local
    top-k_b (k_b of the GLOBAL N_b) in the order (score desc, index asc); the global
    cut is taken over the union of candidates in the same order; every shard attends
    over its surviving candidates; partials are LSE-merged in rank order.
    Must equal sparse_decode exactly for I and within fp64 rounding for o."""
    B, Hq = inp.B, inp.Hq
    o = np.zeros((B, Hq, inp.D))
    lse = np.zeros((B, Hq))
    idx = [[None] * Hq for _ in range(B)]
    for b in range(B):
        N = int(inp.seq_lens[b])
        k = budget_k(S, N)
        bounds = [(r * N) // P for r in range(P + 1)]
        for h in range(Hq):
            s = index_scores(inp, b, h, mode)
            cands = []
            for r in range(P):
                lo, hi = bounds[r], bounds[r + 1]
                if hi > lo:
                    loc = topk_select(s[lo:hi], min(k, hi - lo)) + lo
                    cands.append(loc)
            cand = np.concatenate(cands)
            glob = cand[topk_select(s[cand], k)]          # global cut over candidates
            idx[b][h] = np.sort(glob)
            parts_o, parts_l = [], []
            for r in range(P):
                lo, hi = bounds[r], bounds[r + 1]
                mine = glob[(glob >= lo) & (glob < hi)]
                if mine.size:
                    po, pl = attend_given(inp, b, h, mine, scale)
                else:
                    po, pl = np.zeros(inp.D), -np.inf
                parts_o.append(po)
                parts_l.append(pl)
            o[b, h], lse[b, h] = lse_merge(np.stack(parts_o), np.array(parts_l))
    return idx, o, lse


# ---------------------------------------------------------------------------
# NEXT-1  Sink + Local + heavy-fraction scaffold ("Sink(128) + Local(128)
#   + OracleTopK with heavy fraction 0.20"; Fig 2c "64 sinks always retained",
#   P:126): union of sinks [0, min(sink,N)), locals [N-min(local,N), N)
#   and the top-(heavy budget) tokens of the middle region; heavy budget
#   round-half-up(h * |middle|) or an absolute K.
# ---------------------------------------------------------------------------
def heavy_budget(N: int, n_sink: int, n_local: int, heavy_fraction: float = 0.0,
                 k_abs: int = 0) -> int:
    lo = min(n_sink, N)
    hi = max(lo, N - min(n_local, N))
    middle = hi - lo
    if k_abs > 0:
        return min(k_abs, middle)
    return min(middle, int(math.floor(heavy_fraction * middle + 0.5)))


def sink_local_heavy_select(scores: np.ndarray, n_sink: int, n_local: int,
                            heavy_fraction: float = 0.0, k_abs: int = 0) -> np.ndarray:
    N = scores.shape[0]
    lo = min(n_sink, N)
    hi = max(lo, N - min(n_local, N))
    kh = heavy_budget(N, n_sink, n_local, heavy_fraction, k_abs)
    parts = [np.arange(0, lo), np.arange(hi, N)]
    if kh > 0:
        parts.append(topk_select(scores[lo:hi], kh) + lo)
    return np.unique(np.concatenate(parts).astype(np.int64))


# ---------------------------------------------------------------------------
# NEXT-2  weighted stochastic selection (vAttention stand-in; P:145, P:158 name
#   the method but not its internals; S:233-241 design): deterministic top-k_d
#   with weight 1, plus `n_samples` tokens drawn uniformly without replacement
#   from the remainder R, each with weight |R| / n_samples.  The random draw is
#   an INPUT here (`u`: one uniform key per token; the n_samples remainder tokens
#   with the smallest keys are the sample - a uniform sample without replacement).
# ---------------------------------------------------------------------------
def stochastic_select(scores: np.ndarray, k_det: int, n_samples: int, u: np.ndarray):
    N = scores.shape[0]
    det = topk_select(scores, k_det)
    rest = np.setdiff1d(np.arange(N), det)
    ns = min(n_samples, rest.size)
    if ns == 0:
        samp, w = rest[:0], 1.0
    elif ns == rest.size:
        samp, w = rest, 1.0
    else:
        order = np.argsort(np.asarray(u)[rest], kind="stable")[:ns]
        samp, w = np.sort(rest[order]), rest.size / ns
    idx = np.concatenate([det, samp])
    wts = np.concatenate([np.ones(det.size), np.full(samp.size, w)])
    o = np.argsort(idx, kind="stable")
    return idx[o], wts[o]
