"""ctypes declaration of the C ABI in include/sdattn.h (argument marshalling only).

The shared library is built in-tree (paper_2605_24168_b200/libsdattn.so, see
build.py).  There is no fallback: if the library cannot be loaded every entry
point raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsdattn.so")

SD_OK = 0
SD_ERR_INVALID_ARG = 1
SD_ERR_UNSUPPORTED = 2
SD_ERR_WORKSPACE = 3
SD_ERR_CUDA = 4
SD_ERR_DEVICE_CHECK = 5

SD_BF16 = 0
SD_F32 = 1
SD_E4M3 = 2  # fp8 e4m3 (sketch pages only, NEXT-4)
SD_FUSED_FORCE_SLOW_PATH = 1  # sd_sparse_decode_fused_ex flag

DEVERR = {0: "none", 1: "index out of range", 2: "indices not strictly increasing", 3: "empty index list",
          4: "weight <= 0 or non-finite", 5: "bad sequence length / budget", 6: "candidate overflow"}

c_i32 = ctypes.c_int32
c_f32 = ctypes.c_float
c_vp = ctypes.c_void_p
c_size = ctypes.c_size_t


class Geometry(ctypes.Structure):
    _fields_ = [("batch", c_i32), ("num_q_heads", c_i32), ("num_kv_heads", c_i32), ("head_dim", c_i32),
                ("page_size", c_i32), ("max_pages_per_seq", c_i32), ("kv_dtype", c_i32),
                ("q_dtype", c_i32), ("out_dtype", c_i32)]


class PagedKV(ctypes.Structure):
    _fields_ = [("k_pages", c_vp), ("v_pages", c_vp), ("page_table", c_vp), ("seq_lens", c_vp),
                ("num_pages", c_i32), ("max_seq_len", c_i32)]


class Sketch(ctypes.Structure):
    _fields_ = [("pages", c_vp), ("channel_ids", c_vp), ("channels", c_i32), ("dtype", c_i32)]


class Budget(ctypes.Structure):
    _fields_ = [("sparsity", ctypes.c_double), ("k_fixed", c_i32), ("n_sink", c_i32), ("n_local", c_i32),
                ("heavy_fraction", ctypes.c_double)]


P = ctypes.POINTER
_PROTOS = {
    "sd_status_str": (ctypes.c_char_p, [c_i32]),
    "sd_version": (ctypes.c_char_p, []),
    "sd_budget_k": (c_i32, [P(Budget), c_i32, P(c_i32)]),
    "sd_workspace_size": (c_i32, [P(Geometry), P(Budget), c_i32, P(c_size)]),
    "sd_workspace_size_k": (c_i32, [P(Geometry), c_i32, c_i32, P(c_size)]),
    "sd_clear_device_error": (c_i32, [c_vp, c_vp]),
    "sd_read_device_error": (c_i32, [c_vp, P(c_i32), c_vp]),
    "sd_read_stats": (c_i32, [c_vp, P(c_i32), c_i32, c_vp]),
    "sd_sparse_index_score": (c_i32, [P(Geometry), P(PagedKV), P(Sketch), c_vp, c_vp, c_i32, c_vp]),
    "sd_topk_select": (c_i32, [P(Geometry), c_vp, c_i32, c_vp, c_i32, P(Budget), c_vp, c_vp, c_i32, c_vp,
                               c_size, c_vp]),
    "sd_stochastic_select": (c_i32, [P(Geometry), c_vp, c_i32, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp,
                                     c_i32, c_vp, c_size, c_vp]),
    "sd_sparse_gather_attend": (c_i32, [P(Geometry), P(PagedKV), c_vp, c_vp, c_vp, c_i32, c_vp, c_f32, c_vp,
                                        c_vp, c_vp, c_size, c_vp]),
    "sd_sparse_decode_fused": (c_i32, [P(Geometry), P(PagedKV), P(Sketch), c_vp, P(Budget), c_f32, c_vp, c_vp,
                                       c_vp, c_vp, c_i32, c_vp, c_size, c_vp]),
    "sd_sparse_decode_fused_ex": (c_i32, [P(Geometry), P(PagedKV), P(Sketch), c_vp, P(Budget), c_f32, c_vp, c_vp,
                                          c_vp, c_vp, c_i32, c_vp, c_size, ctypes.c_uint32, c_vp]),
    "sd_sparse_decode_fused_timed": (c_i32, [P(Geometry), P(PagedKV), P(Sketch), c_vp, P(Budget), c_f32, c_vp,
                                             c_vp, c_vp, c_size, c_vp, P(c_f32), c_i32]),
    "sd_dense_decode": (c_i32, [P(Geometry), P(PagedKV), c_vp, c_f32, c_vp, c_vp, c_vp, c_size, c_vp]),
    "sd_lse_merge": (c_i32, [c_i32, c_i32, c_i32, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "sd_seqshard_local_topk": (c_i32, [P(Geometry), P(PagedKV), P(Sketch), c_vp, P(Budget), c_vp, c_i32, c_vp,
                                       c_vp, c_i32, c_vp, c_size, c_vp]),
    "sd_seqshard_cut_attend": (c_i32, [P(Geometry), P(PagedKV), c_vp, P(Budget), c_vp, c_vp, c_vp, c_i32,
                                       c_i32, c_i32, c_f32, c_vp, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
}

EXPORTS = tuple(_PROTOS)

_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libsdattn.so and declare every exported prototype.  Raises if the
    library is missing: the product has no CPU path to fall back to."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `python -m paper_2605_24168_b200.build` "
                           "(the sparse decode path only runs on the sm_100a library)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
