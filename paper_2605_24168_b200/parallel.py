"""Multi-GPU orchestration of the sparse decode step.

One process per GPU, `torch.distributed` for the plumbing (NCCL over NVLink on
GPUs; gloo in the CPU tests).  Two partitionings of the same step:

* KV-head sharding (BASELINE configs[3]): rank r owns KV heads
  [r*Hkv/P, (r+1)*Hkv/P) and their q-heads for every sequence and runs the
  single-GPU fused call on its shard.  The data path has NO collective (the
  o_proj all-reduce that follows in a model is outside this path).
* Sequence sharding (BASELINE configs[4]): rank r owns a contiguous token
  range of every sequence.  Exactness needs every rank's local top-k_b with
  k_b from the GLOBAL length (the global top-k is a subset of the union of the
  local top-k's), one all-gather of the candidate scores, a global cut that
  every rank computes identically (ties: lower rank, then lower local index ==
  lower global index because shards are contiguous and rank-ordered), a local
  attend over the surviving candidates, one all-gather of the normalised
  partials (o, lse) and an LSE merge in rank order (deterministic).

The local compute is injected (`SeqShardBackend`): `CudaSeqShardBackend` calls
the sm_100a library through the C ABI; the CPU tests inject an oracle-based
backend to check the protocol itself with gloo.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Protocol, Tuple

import torch
import torch.distributed as dist


# --------------------------------------------------------------------------- helpers
def head_range(Hkv: int, world: int, rank: int) -> Tuple[int, int]:
    """KV heads owned by `rank` (contiguous, equal shares)."""
    if Hkv % world:
        raise ValueError(f"Hkv={Hkv} is not divisible by world={world}")
    per = Hkv // world
    return rank * per, (rank + 1) * per


def token_bounds(N: int, world: int, page_size: int = 16) -> List[int]:
    """Contiguous token shard bounds [b_0=0, ..., b_P=N], page-aligned so that
    every shard keeps whole pages (shard r = [b_r, b_{r+1}))."""
    bounds = [((r * N) // world) // page_size * page_size for r in range(world)] + [N]
    for r in range(world):
        bounds[r] = min(bounds[r], N)
    return bounds


def all_gather_stack(t: torch.Tensor, group=None) -> torch.Tensor:
    """[P, *t.shape] in rank order."""
    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
    if t.is_cuda and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
    elif t.is_cuda:  # a CPU backend (gloo) with device tensors: stage through the host
        return all_gather_stack(t.cpu(), group).to(t.device)
    else:
        parts = list(out.unbind(0))
        dist.all_gather(parts, t.contiguous(), group=group)
        out = torch.stack(parts)
    return out


# --------------------------------------------------------------------------- KV-head sharding
@dataclass
class HeadShard:
    """The KV-head shard of a paged cache owned by one rank."""
    q: torch.Tensor            # [B][Hq/P][D]
    k_pages: torch.Tensor      # [P][ps][Hkv/P][D]
    v_pages: torch.Tensor
    sketch_pages: Optional[torch.Tensor]   # [P][Hkv/P][ps][C]
    channel_ids: Optional[torch.Tensor]    # [B][Hkv/P][C]
    page_table: torch.Tensor
    seq_lens: torch.Tensor
    h0: int                    # first KV head owned
    G: int


def shard_heads(q, k_pages, v_pages, page_table, seq_lens, sketch_pages=None, channel_ids=None,
                world: int = 1, rank: int = 0) -> HeadShard:
    """Slice a full cache into `rank`'s KV-head shard (contiguous copies)."""
    Hkv = k_pages.shape[2]
    G = q.shape[1] // Hkv
    g0, g1 = head_range(Hkv, world, rank)
    return HeadShard(q=q[:, g0 * G:g1 * G].contiguous(), k_pages=k_pages[:, :, g0:g1].contiguous(),
                     v_pages=v_pages[:, :, g0:g1].contiguous(),
                     sketch_pages=None if sketch_pages is None else sketch_pages[:, g0:g1].contiguous(),
                     channel_ids=None if channel_ids is None else channel_ids[:, g0:g1].contiguous(),
                     page_table=page_table, seq_lens=seq_lens, h0=g0, G=G)


class HeadShardedDecoder:
    """KV-head-sharded fused decode: the rank's shard only, no collective."""

    def __init__(self, shard: HeadShard, max_seq_len: int):
        from . import api
        self.api = api
        self.shard = shard
        self.kv = api.KVCache(shard.k_pages, shard.v_pages, shard.page_table, shard.seq_lens, max_seq_len)
        self.sk = None if shard.sketch_pages is None else api.SketchCache(shard.sketch_pages, shard.channel_ids)

    def decode(self, q: Optional[torch.Tensor] = None, S: float = 50.0, scale: Optional[float] = None, **kw):
        return self.api.sparse_decode_fused(self.shard.q if q is None else q, self.kv, self.sk, S=S, scale=scale, **kw)

    @staticmethod
    def gather_outputs(out: torch.Tensor, group=None) -> torch.Tensor:
        """Validation helper: [B][Hq/P][D] per rank -> [B][Hq][D] (head order)."""
        parts = all_gather_stack(out, group)            # [P][B][Hq/P][D]
        return parts.permute(1, 0, 2, 3).reshape(out.shape[0], -1, out.shape[2])


# --------------------------------------------------------------------------- sequence sharding
class SeqShardBackend(Protocol):
    def local_topk(self, global_lens: torch.Tensor, max_global: int, S: float, k_max: int
                   ) -> Tuple[torch.Tensor, torch.Tensor]:
        """Local candidates: scores fp32 [B][Hq][k_max] (-inf pad) and LOCAL indices,
        ascending local index order."""

    def cut_attend(self, global_lens: torch.Tensor, all_cand: torch.Tensor, cand_idx: torch.Tensor, rank: int,
                   S: float, scale: float) -> Tuple[torch.Tensor, torch.Tensor]:
        """This rank's normalised partial (o fp32 [B][Hq][D], lse fp32 [B][Hq])."""

    def merge(self, part_o: torch.Tensor, part_lse: torch.Tensor) -> Tuple[torch.Tensor, torch.Tensor]:
        """LSE merge of [P][B][Hq][D], [P][B][Hq] in rank order."""


class CudaSeqShardBackend:
    """The local compute of one rank through the sm_100a C ABI."""

    def __init__(self, q, kv_local, sketch_local, out_dtype=torch.float32):
        from . import api
        self.api = api
        self.q, self.kv, self.sk = q, kv_local, sketch_local
        self.out_dtype = out_dtype

    def local_topk(self, global_lens, max_global, S, k_max):
        return self.api.seqshard_local_topk(self.q, self.kv, self.sk, global_lens, max_global, S, k_max=k_max)

    def cut_attend(self, global_lens, all_cand, cand_idx, rank, S, scale):
        return self.api.seqshard_cut_attend(self.q, self.kv, global_lens, all_cand, cand_idx, rank, S, scale=scale)

    def merge(self, part_o, part_lse):
        return self.api.lse_merge(part_o, part_lse, out_dtype=self.out_dtype)


def seqshard_decode(backend: SeqShardBackend, global_lens: torch.Tensor, max_global: int, S: float,
                    scale: float, k_max: int, group=None):
    """The sequence-sharded protocol of one decode step (every rank calls it).
    Returns the merged (out, lse), identical on every rank."""
    rank = dist.get_rank(group)
    cand_scores, cand_idx = backend.local_topk(global_lens, max_global, S, k_max)
    all_cand = all_gather_stack(cand_scores, group)                     # exchange 1: candidates
    part_o, part_lse = backend.cut_attend(global_lens, all_cand, cand_idx, rank, S, scale)
    all_o = all_gather_stack(part_o, group)                             # exchange 2: partials
    all_lse = all_gather_stack(part_lse, group)
    return backend.merge(all_o, all_lse)
