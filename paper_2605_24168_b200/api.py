"""Thin Python binding over the C ABI (same names as include/sdattn.h, minus `sd_`).

Argument marshalling only: every step of the hot path runs in the sm_100a
kernels of libsdattn.so.  PyTorch supplies device memory and the current CUDA
stream.  Tensors must be CUDA and contiguous; nothing is copied or converted.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

import torch

from . import _capi as C


class SdError(RuntimeError):
    pass


def load_library():
    return C.load()


def _check(status: int, what: str):
    if status != C.SD_OK:
        lib = C.load()
        raise SdError(f"{what}: {lib.sd_status_str(status).decode()}")


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("sdattn tensors must live on the GPU (no CPU path)")
    if not t.is_contiguous():
        raise ValueError("sdattn tensors must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _dt(dtype: torch.dtype) -> int:
    if dtype == torch.bfloat16:
        return C.SD_BF16
    if dtype == torch.float32:
        return C.SD_F32
    raise ValueError(f"unsupported dtype {dtype} (bf16 or fp32)")


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


@dataclass
class KVCache:
    """Paged KV cache: k/v pages [P][page_size][Hkv][D] (NHD), page_table int32
    [B][max_pages], seq_lens int32 [B]; max_seq_len is the host-side bound."""
    k_pages: torch.Tensor
    v_pages: torch.Tensor
    page_table: torch.Tensor
    seq_lens: torch.Tensor
    max_seq_len: int

    @classmethod
    def from_case(cls, case):
        return cls(case.k_pages, case.v_pages, case.page_table, case.seq_lens,
                   int(case.seq_lens.max().item()))

    def c_struct(self) -> C.PagedKV:
        return C.PagedKV(_ptr(self.k_pages), _ptr(self.v_pages), _ptr(self.page_table), _ptr(self.seq_lens),
                         int(self.k_pages.shape[0]), int(self.max_seq_len))


@dataclass
class SketchCache:
    """Double-Sparsity sketch: pages bf16 or fp8 e4m3 (NEXT-4) [P][Hkv][page_size][C],
    channel_ids int32 [B][Hkv][C]."""
    pages: torch.Tensor
    channel_ids: torch.Tensor

    @classmethod
    def from_case(cls, case):
        if case.sketch_pages is None:
            return None
        return cls(case.sketch_pages, case.channel_ids)

    def c_struct(self) -> C.Sketch:
        dt = C.SD_E4M3 if self.pages.dtype == torch.float8_e4m3fn else C.SD_BF16
        return C.Sketch(_ptr(self.pages), _ptr(self.channel_ids), int(self.pages.shape[-1]), dt)


def geometry(q: torch.Tensor, kv: KVCache, out_dtype: Optional[torch.dtype] = None) -> C.Geometry:
    B, Hq, D = q.shape
    _, ps, Hkv, Dk = kv.k_pages.shape
    return C.Geometry(B, Hq, Hkv, D if D == Dk else -1, ps, int(kv.page_table.shape[1]),
                      _dt(kv.k_pages.dtype), _dt(q.dtype), _dt(out_dtype or q.dtype))


def make_budget(S: float = 1.0, k_fixed: int = 0, n_sink: int = 0, n_local: int = 0,
                heavy_fraction: float = 0.0) -> C.Budget:
    return C.Budget(float(S), int(k_fixed), int(n_sink), int(n_local), float(heavy_fraction))


def budget_k(S: float, N: int, k_fixed: int = 0, n_sink: int = 0, n_local: int = 0,
             heavy_fraction: float = 0.0) -> int:
    """Rows kept for one sequence of N tokens: max(1, ceil(N/S)) or k_fixed; with
    sinks / locals / a heavy fraction (NEXT-1) sinks + locals + the middle's heavy budget."""
    k = C.c_i32()
    b = make_budget(S, k_fixed, n_sink, n_local, heavy_fraction)
    _check(C.load().sd_budget_k(ctypes.byref(b), int(N), ctypes.byref(k)), "sd_budget_k")
    return k.value


_WS = {}


def workspace_size(geom: C.Geometry, budget: Optional[C.Budget], max_seq_len: int) -> int:
    n = C.c_size()
    _check(C.load().sd_workspace_size(ctypes.byref(geom), ctypes.byref(budget) if budget else None,
                                      int(max_seq_len), ctypes.byref(n)), "sd_workspace_size")
    return n.value


def workspace(nbytes: int, device=None, stream=None) -> torch.Tensor:
    """A zeroed (error word cleared) device workspace, cached per (device, stream)
    and grown on demand.  The buffer is allocated on (and recorded with) the
    stream the library enqueues on, so the caching allocator never hands a
    replaced buffer out while that stream may still use it."""
    device = torch.device(device or "cuda")
    s = stream if stream is not None else torch.cuda.current_stream(device)
    key = (device.index if device.index is not None else torch.cuda.current_device(), s.cuda_stream)
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        if ws is not None:
            ws.record_stream(s)  # the old buffer stays reserved until s passes this point
        with torch.cuda.stream(s):
            ws = torch.zeros(max(nbytes, 256) + 256, dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws


def _ws_ptr(ws: torch.Tensor):
    p = ws.data_ptr()
    return ctypes.c_void_p((p + 255) & ~255), ws.numel() - ((-p) & 255)


def read_device_error(ws: Optional[torch.Tensor] = None, stream=None) -> int:
    if ws is None:
        s = stream if stream is not None else torch.cuda.current_stream()
        ws = _WS[(torch.cuda.current_device(), s.cuda_stream)]
    code = C.c_i32()
    p, _ = _ws_ptr(ws)
    C.load().sd_read_device_error(p, ctypes.byref(code), _stream(stream))
    return code.value


def read_stats(ws: Optional[torch.Tensor] = None, stream=None) -> dict:
    """Workspace statistics (cumulative since clear_device_error): number of rows
    the fused path computed on its exact slow path."""
    if ws is None:
        s = stream if stream is not None else torch.cuda.current_stream()
        ws = _WS[(torch.cuda.current_device(), s.cuda_stream)]
    arr = (C.c_i32 * 1)()
    p, _ = _ws_ptr(ws)
    _check(C.load().sd_read_stats(p, arr, 1, _stream(stream)), "sd_read_stats")
    return {"fallback_rows": int(arr[0])}


def clear_device_error(ws: Optional[torch.Tensor] = None, stream=None):
    if ws is None:
        s = stream if stream is not None else torch.cuda.current_stream()
        ws = _WS.get((torch.cuda.current_device(), s.cuda_stream))
        if ws is None:
            return
    p, _ = _ws_ptr(ws)
    _check(C.load().sd_clear_device_error(p, _stream(stream)), "sd_clear_device_error")


# --------------------------------------------------------------------------- entry points
def sparse_index_score(q, kv: KVCache, sketch: Optional[SketchCache] = None, scores=None, stream=None):
    """A2: fp32 unscaled indexer scores [B][Hq][ld] (entries t >= N_b unwritten)."""
    g = geometry(q, kv)
    ld = (kv.max_seq_len + 63) // 64 * 64
    if scores is None:
        scores = torch.empty((g.batch, g.num_q_heads, ld), dtype=torch.float32, device=q.device)
    kvs = kv.c_struct()
    sk = sketch.c_struct() if sketch is not None else None
    _check(C.load().sd_sparse_index_score(ctypes.byref(g), ctypes.byref(kvs), ctypes.byref(sk) if sk else None,
                                          _ptr(q), _ptr(scores), int(scores.shape[-1]), _stream(stream)),
           "sd_sparse_index_score")
    return scores


def topk_select(scores, seq_lens, max_seq_len: int, S: float = 1.0, k_fixed: int = 0, num_kv_heads=None,
                k_max: Optional[int] = None, stream=None, n_sink: int = 0, n_local: int = 0,
                heavy_fraction: float = 0.0):
    """A3: (idx int32 [B][Hq][k_max] ascending, counts int32 [B][Hq])."""
    B, Hq, ld = scores.shape
    bud = make_budget(S, k_fixed, n_sink, n_local, heavy_fraction)
    if k_max is None:
        k_max = max(1, budget_k(S, max_seq_len, k_fixed, n_sink, n_local, heavy_fraction))
    Hkv = num_kv_heads or Hq
    g = C.Geometry(B, Hq, Hkv, 128, 16, (max_seq_len + 15) // 16, C.SD_BF16, C.SD_BF16, C.SD_BF16)
    idx = torch.full((B, Hq, k_max), -1, dtype=torch.int32, device=scores.device)
    counts = torch.zeros((B, Hq), dtype=torch.int32, device=scores.device)
    ws = workspace(256, scores.device, stream)
    p, n = _ws_ptr(ws)
    _check(C.load().sd_topk_select(ctypes.byref(g), _ptr(scores), ld, _ptr(seq_lens), int(max_seq_len),
                                   ctypes.byref(bud), _ptr(idx), _ptr(counts), int(k_max), p, n, _stream(stream)),
           "sd_topk_select")
    return idx, counts


def stochastic_select(scores, u, seq_lens, max_seq_len: int, k_det: int, n_samples: int, num_kv_heads=None,
                      k_max: Optional[int] = None, stream=None):
    """NEXT-2: (idx int32 [B][Hq][k_max] ascending, weights fp32 [B][Hq][k_max],
    counts int32 [B][Hq]) = deterministic top-k_det + n_samples smallest-u
    remainder tokens weighted |R| / n_samples (u: the uniform draw, an input)."""
    B, Hq, ld = scores.shape
    if k_max is None:
        k_max = max(1, min(k_det + n_samples, max_seq_len))
    Hkv = num_kv_heads or Hq
    g = C.Geometry(B, Hq, Hkv, 128, 16, (max_seq_len + 15) // 16, C.SD_BF16, C.SD_BF16, C.SD_BF16)
    idx = torch.full((B, Hq, k_max), -1, dtype=torch.int32, device=scores.device)
    wts = torch.zeros((B, Hq, k_max), dtype=torch.float32, device=scores.device)
    counts = torch.zeros((B, Hq), dtype=torch.int32, device=scores.device)
    ws = workspace(_ws_bytes_budget(g, None, max_seq_len, k_max), scores.device, stream)
    p, n = _ws_ptr(ws)
    _check(C.load().sd_stochastic_select(ctypes.byref(g), _ptr(scores), ld, _ptr(u), _ptr(seq_lens),
                                         int(max_seq_len), int(k_det), int(n_samples), _ptr(idx), _ptr(wts),
                                         _ptr(counts), int(k_max), p, n, _stream(stream)), "sd_stochastic_select")
    return idx, wts, counts


def sparse_gather_attend(q, kv: KVCache, idx, counts, weights=None, scale: Optional[float] = None,
                         out_dtype=None, out=None, lse=None, stream=None):
    """A4+A5: weighted attention over per-head index lists -> (out [B][Hq][D], lse [B][Hq])."""
    g = geometry(q, kv, out_dtype)
    scale = scale if scale is not None else 1.0 / math.sqrt(q.shape[-1])
    out = out if out is not None else torch.empty(q.shape, dtype=out_dtype or q.dtype, device=q.device)
    lse = lse if lse is not None else torch.empty(q.shape[:2], dtype=torch.float32, device=q.device)
    kvs = kv.c_struct()
    ws = workspace(workspace_size(g, None, kv.max_seq_len), q.device, stream)
    p, n = _ws_ptr(ws)
    _check(C.load().sd_sparse_gather_attend(ctypes.byref(g), ctypes.byref(kvs), _ptr(q), _ptr(idx), _ptr(counts),
                                            int(idx.shape[-1]), _ptr(weights), float(scale), _ptr(out), _ptr(lse),
                                            p, n, _stream(stream)), "sd_sparse_gather_attend")
    return out, lse


def sparse_decode_fused(q, kv: KVCache, sketch: Optional[SketchCache], S: float = 50.0, k_fixed: int = 0,
                        scale: Optional[float] = None, out_dtype=None, return_idx: bool = False, out=None,
                        lse=None, idx=None, counts=None, stream=None, n_sink: int = 0, n_local: int = 0,
                        heavy_fraction: float = 0.0, force_slow_path: bool = False):
    """A6: the fused decode step -> (out, lse) or (out, lse, idx, counts).  With
    n_sink / n_local / heavy_fraction: the Sink + Local + heavy budget (NEXT-1).
    force_slow_path: every row on the exact slow selection path (sd_sparse_decode_fused_ex
    SD_FUSED_FORCE_SLOW_PATH; same result, for tests)."""
    g = geometry(q, kv, out_dtype)
    bud = make_budget(S, k_fixed, n_sink, n_local, heavy_fraction)
    scale = scale if scale is not None else 1.0 / math.sqrt(q.shape[-1])
    out = out if out is not None else torch.empty(q.shape, dtype=out_dtype or q.dtype, device=q.device)
    lse = lse if lse is not None else torch.empty(q.shape[:2], dtype=torch.float32, device=q.device)
    if return_idx and idx is None:
        k_max = max(1, budget_k(S, kv.max_seq_len, k_fixed, n_sink, n_local, heavy_fraction))
        idx = torch.full((g.batch, g.num_q_heads, k_max), -1, dtype=torch.int32, device=q.device)
        counts = torch.zeros((g.batch, g.num_q_heads), dtype=torch.int32, device=q.device)
    kvs = kv.c_struct()
    sk = sketch.c_struct() if sketch is not None else None
    ws = workspace(workspace_size(g, bud, kv.max_seq_len), q.device, stream)
    p, n = _ws_ptr(ws)
    args = (ctypes.byref(g), ctypes.byref(kvs), ctypes.byref(sk) if sk else None, _ptr(q), ctypes.byref(bud),
            float(scale), _ptr(out), _ptr(lse), _ptr(idx), _ptr(counts), int(idx.shape[-1]) if idx is not None else 0,
            p, n)
    if force_slow_path:
        _check(C.load().sd_sparse_decode_fused_ex(*args, C.SD_FUSED_FORCE_SLOW_PATH, _stream(stream)),
               "sd_sparse_decode_fused_ex")
    else:
        _check(C.load().sd_sparse_decode_fused(*args, _stream(stream)), "sd_sparse_decode_fused")
    if return_idx:
        return out, lse, idx, counts
    return out, lse


FUSED_PHASES = ("sample", "scan", "select", "attend", "merge")


def sparse_decode_fused_timed(q, kv: KVCache, sketch: SketchCache, S: float = 50.0, k_fixed: int = 0,
                              scale: Optional[float] = None, out=None, lse=None, stream=None):
    """Measurement helper: the fused step with CUDA events between its kernels
    (serialised; synchronizes) -> (out, lse, {phase: ms})."""
    g = geometry(q, kv, None)
    bud = make_budget(S, k_fixed)
    scale = scale if scale is not None else 1.0 / math.sqrt(q.shape[-1])
    out = out if out is not None else torch.empty(q.shape, dtype=q.dtype, device=q.device)
    lse = lse if lse is not None else torch.empty(q.shape[:2], dtype=torch.float32, device=q.device)
    kvs, sk = kv.c_struct(), sketch.c_struct()
    ws = workspace(workspace_size(g, bud, kv.max_seq_len), q.device, stream)
    p, n = _ws_ptr(ws)
    ms = (ctypes.c_float * len(FUSED_PHASES))()
    _check(C.load().sd_sparse_decode_fused_timed(ctypes.byref(g), ctypes.byref(kvs), ctypes.byref(sk), _ptr(q),
                                                 ctypes.byref(bud), float(scale), _ptr(out), _ptr(lse), p, n,
                                                 _stream(stream), ms, len(FUSED_PHASES)),
           "sd_sparse_decode_fused_timed")
    return out, lse, {k: float(v) for k, v in zip(FUSED_PHASES, ms)}


def dense_decode(q, kv: KVCache, scale: Optional[float] = None, out_dtype=None, out=None, lse=None, stream=None):
    """A7: full softmax over all N_b rows -> (out, lse)."""
    g = geometry(q, kv, out_dtype)
    scale = scale if scale is not None else 1.0 / math.sqrt(q.shape[-1])
    out = out if out is not None else torch.empty(q.shape, dtype=out_dtype or q.dtype, device=q.device)
    lse = lse if lse is not None else torch.empty(q.shape[:2], dtype=torch.float32, device=q.device)
    kvs = kv.c_struct()
    ws = workspace(workspace_size(g, None, kv.max_seq_len), q.device, stream)
    p, n = _ws_ptr(ws)
    _check(C.load().sd_dense_decode(ctypes.byref(g), ctypes.byref(kvs), _ptr(q), float(scale), _ptr(out),
                                    _ptr(lse), p, n, _stream(stream)), "sd_dense_decode")
    return out, lse


def lse_merge(part_o, part_lse, out_dtype=torch.float32, out=None, lse=None, stream=None):
    """Merge normalised partials part_o [P][rows..][D], part_lse [P][rows..] -> (out, lse)."""
    P = part_o.shape[0]
    D = part_o.shape[-1]
    rows = part_lse[0].numel()
    out = out if out is not None else torch.empty(part_o.shape[1:], dtype=out_dtype, device=part_o.device)
    lse = lse if lse is not None else torch.empty(part_lse.shape[1:], dtype=torch.float32, device=part_o.device)
    _check(C.load().sd_lse_merge(int(P), int(rows), int(D), _ptr(part_o), _ptr(part_lse), _dt(out_dtype),
                                 _ptr(out), _ptr(lse), _stream(stream)), "sd_lse_merge")
    return out, lse


def seqshard_local_topk(q, kv: KVCache, sketch: Optional[SketchCache], global_seq_lens, max_global_seq_len: int,
                        S: float, k_fixed: int = 0, k_max: Optional[int] = None, stream=None):
    """Sequence shard step (1): local candidates (scores fp32, LOCAL idx int32), ascending local index."""
    g = geometry(q, kv)
    bud = make_budget(S, k_fixed)
    if k_max is None:
        k_max = budget_k(S, max_global_seq_len, k_fixed)
    cand_scores = torch.empty((g.batch, g.num_q_heads, k_max), dtype=torch.float32, device=q.device)
    cand_idx = torch.empty((g.batch, g.num_q_heads, k_max), dtype=torch.int32, device=q.device)
    kvs = kv.c_struct()
    sk = sketch.c_struct() if sketch is not None else None
    ws = workspace(_ws_bytes_budget(g, bud, kv.max_seq_len, k_max), q.device, stream)
    p, n = _ws_ptr(ws)
    _check(C.load().sd_seqshard_local_topk(ctypes.byref(g), ctypes.byref(kvs), ctypes.byref(sk) if sk else None,
                                           _ptr(q), ctypes.byref(bud), _ptr(global_seq_lens),
                                           int(max_global_seq_len), _ptr(cand_scores), _ptr(cand_idx), int(k_max),
                                           p, n, _stream(stream)), "sd_seqshard_local_topk")
    return cand_scores, cand_idx


def seqshard_cut_attend(q, kv: KVCache, global_seq_lens, all_cand, cand_idx, rank: int, S: float,
                        k_fixed: int = 0, scale: Optional[float] = None, stream=None, return_survivors: bool = False):
    """Sequence shard step (3): this rank's normalised partial (part_o fp32 [B][Hq][D], part_lse fp32 [B][Hq]),
    plus (surv_idx int32 [B][Hq][k_max] LOCAL ascending, surv_counts int32 [B][Hq]) with return_survivors."""
    g = geometry(q, kv)
    bud = make_budget(S, k_fixed)
    P = all_cand.shape[0]
    k_max = all_cand.shape[-1]
    scale = scale if scale is not None else 1.0 / math.sqrt(q.shape[-1])
    part_o = torch.empty(q.shape, dtype=torch.float32, device=q.device)
    part_lse = torch.empty(q.shape[:2], dtype=torch.float32, device=q.device)
    surv = cnt = None
    if return_survivors:
        surv = torch.full((g.batch, g.num_q_heads, k_max), -1, dtype=torch.int32, device=q.device)
        cnt = torch.zeros((g.batch, g.num_q_heads), dtype=torch.int32, device=q.device)
    kvs = kv.c_struct()
    ws = workspace(_ws_bytes_budget(g, bud, kv.max_seq_len, k_max), q.device, stream)
    p, n = _ws_ptr(ws)
    _check(C.load().sd_seqshard_cut_attend(ctypes.byref(g), ctypes.byref(kvs), _ptr(q), ctypes.byref(bud),
                                           _ptr(global_seq_lens), _ptr(all_cand), _ptr(cand_idx), int(k_max),
                                           int(P), int(rank), float(scale), _ptr(part_o), _ptr(part_lse),
                                           _ptr(surv), _ptr(cnt), p, n, _stream(stream)), "sd_seqshard_cut_attend")
    if return_survivors:
        return part_o, part_lse, surv, cnt
    return part_o, part_lse


def _ws_bytes_budget(g, bud, max_seq_len, k_max):
    n = C.c_size()
    _check(C.load().sd_workspace_size_k(ctypes.byref(g), int(max_seq_len), int(k_max), ctypes.byref(n)),
           "sd_workspace_size_k")
    return n.value


# Kernel launches enqueued by one sd_sparse_decode_fused call in sketch mode
# with bf16 KV (sample, scan, select, persistent union attend, split merge) -
# keep in sync with csrc/sd_api.cu.
LAUNCHES_PER_FUSED = 5
