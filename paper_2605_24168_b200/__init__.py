"""paper_2605_24168_b200 - B200 (sm_100a) sparse decode attention.

The hot path of arxiv 2605.24168 (indexer scan -> exact top-k -> gather-attend
-> split-k LSE merge) as a C-ABI library of hand-written CUDA kernels
(libsdattn.so, include/sdattn.h) plus this thin binding.  There is no CPU
fallback: every call runs in the CUDA library or raises.
"""
from .api import (  # noqa: F401
    KVCache, SketchCache, SdError, budget_k, clear_device_error, dense_decode, geometry, load_library,
    lse_merge, make_budget, read_device_error, read_stats, seqshard_cut_attend, seqshard_local_topk, sparse_decode_fused,
    sparse_gather_attend, sparse_index_score, topk_select, workspace, workspace_size,
)

__version__ = "0.1.0"
