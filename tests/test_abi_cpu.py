"""CPU-side checks of the C ABI: the library builds/loads, exports every symbol
include/sdattn.h declares, and the host-only logic (budget arithmetic, argument
validation, workspace sizing) behaves as documented.  No kernel is launched."""
import ctypes
import os
import re

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_24168_b200 import _capi, build
    if not os.path.exists(_capi.LIB_PATH):
        build.build_library()
    return _capi.load()


def _declared():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            txt = open(os.path.join(ROOT, "include", fn)).read()
            txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
            names |= set(re.findall(r"\b(sd_[a-z0-9_]+)\s*\(", txt))
    return names


def test_exports_every_declared_symbol(lib):
    from paper_2605_24168_b200 import _capi
    decl = _declared()
    assert len(decl) >= 14
    for name in decl:
        assert hasattr(lib, name), name
    assert decl == set(_capi.EXPORTS), decl ^ set(_capi.EXPORTS)


def test_no_cpu_fallback_symbols():
    """The product package never imports the oracle (it is test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2605_24168_b200")
    for dp, _, fns in os.walk(pkg):
        for fn in fns:
            if fn.endswith(".py"):
                src = open(os.path.join(dp, fn)).read()
                assert "import oracle" not in src and "from oracle" not in src, fn


@pytest.mark.parametrize("S,N", [(50.0, 131072), (500.0, 131072), (50.0, 4096), (1.0, 9), (10.0, 32768),
                                 (100.0, 1 << 20), (3.0, 2), (2.5, 5), (7.0, 7), (1.5, 1000)])
def test_budget_matches_oracle(lib, S, N):
    from paper_2605_24168_b200 import _capi as C
    b = C.Budget(S, 0, 0, 0, 0.0)
    k = C.c_i32()
    assert lib.sd_budget_k(ctypes.byref(b), N, ctypes.byref(k)) == 0
    assert k.value == oracle.budget_k(S, N)


@pytest.mark.parametrize("S,N,want", [(1.3, 13, 10), (3.3, 33, 10), (2.3, 23, 10), (4.1, 41, 10)])
def test_budget_non_representable_sparsity(lib, S, N, want):
    """S is a double across the ABI: ceil(13 / 1.3) = 10 as in the SPEC's double
    arithmetic.  Through a float32 field, 1.3f < 1.3 and 13 / 1.3f
    = 10.0000004 would round up to 11 (likewise 33 / 3.3f, 23 / 2.3f, 41 / 4.1f)."""
    from paper_2605_24168_b200 import _capi as C
    k = C.c_i32()
    assert lib.sd_budget_k(ctypes.byref(C.Budget(S, 0, 0, 0, 0.0)), N, ctypes.byref(k)) == 0
    assert k.value == oracle.budget_k(S, N) == want


@pytest.mark.parametrize("N,n_sink,n_local,hf,kh", [(5 + 8, 4, 4, 0.7, 4), (10 + 8, 4, 4, 0.45, 5),
                                                    (10 + 8, 4, 4, 0.65, 7)])
def test_heavy_fraction_non_representable(lib, N, n_sink, n_local, hf, kh):
    """heavy_fraction is a double: round-half-up(0.7 * 5) = 4; through a
    float32 field 0.7f * 5 = 3.49999994 would round to 3 (0.45f * 10 -> 4, 0.65f * 10 -> 6)."""
    from paper_2605_24168_b200 import _capi as C
    k = C.c_i32()
    assert lib.sd_budget_k(ctypes.byref(C.Budget(1.0, 0, n_sink, n_local, hf)), N, ctypes.byref(k)) == 0
    assert oracle.heavy_budget(N, n_sink, n_local, hf) == kh
    assert k.value == n_sink + n_local + kh


def test_budget_rejections(lib):
    from paper_2605_24168_b200 import _capi as C
    k = C.c_i32()
    assert lib.sd_budget_k(ctypes.byref(C.Budget(0.5, 0, 0, 0, 0.0)), 10, ctypes.byref(k)) == C.SD_ERR_INVALID_ARG
    assert lib.sd_budget_k(ctypes.byref(C.Budget(2.0, 11, 0, 0, 0.0)), 10, ctypes.byref(k)) == C.SD_ERR_INVALID_ARG
    assert lib.sd_budget_k(ctypes.byref(C.Budget(2.0, 0, 0, 0, 0.0)), 0, ctypes.byref(k)) == C.SD_ERR_INVALID_ARG
    assert lib.sd_budget_k(ctypes.byref(C.Budget(2.0, 10, 0, 0, 0.0)), 10, ctypes.byref(k)) == 0 and k.value == 10


@pytest.mark.parametrize("N,n_sink,n_local,hf,k_abs", [(20000, 128, 128, 0.20, 0), (20000, 128, 128, 0.02, 0),
                                                       (131072, 128, 128, 0.02, 0), (200, 128, 128, 0.5, 0),
                                                       (5000, 64, 0, 0.0, 16), (77, 0, 32, 0.0, 0),
                                                       (1000, 0, 0, 0.125, 0)])
def test_budget_sink_local_heavy_matches_oracle(lib, N, n_sink, n_local, hf, k_abs):
    """NEXT-1 budget: sinks + locals + the middle's heavy
    budget, against the oracle's heavy_budget (AC8: 4205 rows at N=20000)."""
    from paper_2605_24168_b200 import _capi as C
    k = C.c_i32()
    assert lib.sd_budget_k(ctypes.byref(C.Budget(1.0, k_abs, n_sink, n_local, hf)), N, ctypes.byref(k)) == 0
    lo = min(n_sink, N)
    hi = max(lo, N - min(n_local, N))
    assert k.value == lo + (N - hi) + oracle.heavy_budget(N, n_sink, n_local, hf, k_abs)
    if (N, n_sink, n_local, hf) == (20000, 128, 128, 0.20):
        assert k.value == 4205


def test_budget_sink_local_rejections(lib):
    from paper_2605_24168_b200 import _capi as C
    k = C.c_i32()
    for bad in (C.Budget(1.0, 0, -1, 0, 0.0), C.Budget(1.0, 0, 0, -4, 0.0), C.Budget(1.0, 0, 4, 4, 1.5),
                C.Budget(1.0, 0, 4, 4, float("nan"))):
        assert lib.sd_budget_k(ctypes.byref(bad), 100, ctypes.byref(k)) == C.SD_ERR_INVALID_ARG


def _geom(C, **kw):
    g = dict(batch=2, num_q_heads=32, num_kv_heads=8, head_dim=128, page_size=16, max_pages_per_seq=64,
             kv_dtype=C.SD_BF16, q_dtype=C.SD_BF16, out_dtype=C.SD_BF16)
    g.update(kw)
    return C.Geometry(**g)


def test_validation_before_any_launch(lib):
    """Host-checked errors return before touching (fake) device pointers."""
    from paper_2605_24168_b200 import _capi as C
    fake = ctypes.c_void_p(0x1000)
    kv = C.PagedKV(fake, fake, fake, fake, 128, 1000)
    sk = C.Sketch(fake, fake, 8)
    bud = C.Budget(50.0, 0, 0, 0, 0.0)
    ws = ctypes.c_void_p(0x10000)

    def fused(g, kvv=kv, s=sk, b=bud, scale=0.1, wsb=1 << 40, wsp=ws):
        return lib.sd_sparse_decode_fused(ctypes.byref(g), ctypes.byref(kvv), ctypes.byref(s) if s else None, fake,
                                          ctypes.byref(b) if b else None, scale, fake, None, None, None, 0, wsp,
                                          wsb, None)

    assert fused(_geom(C, num_q_heads=30)) == C.SD_ERR_INVALID_ARG          # Hq % Hkv
    assert fused(_geom(C, head_dim=64)) == C.SD_ERR_UNSUPPORTED
    assert fused(_geom(C, page_size=32)) == C.SD_ERR_UNSUPPORTED
    assert fused(_geom(C, num_q_heads=48, num_kv_heads=3)) == C.SD_ERR_UNSUPPORTED  # G = 16
    assert fused(_geom(C, kv_dtype=7)) == C.SD_ERR_INVALID_ARG
    assert fused(_geom(C, q_dtype=C.SD_F32)) == C.SD_ERR_UNSUPPORTED
    assert fused(_geom(C), b=C.Budget(0.5, 0, 0, 0, 0.0)) == C.SD_ERR_INVALID_ARG   # S < 1
    assert fused(_geom(C), b=C.Budget(1.0, 5000, 0, 0, 0.0)) == C.SD_ERR_INVALID_ARG  # k > N
    assert fused(_geom(C), b=None) == C.SD_ERR_INVALID_ARG
    assert fused(_geom(C), s=C.Sketch(fake, fake, 129)) == C.SD_ERR_INVALID_ARG      # C > D
    assert fused(_geom(C), s=C.Sketch(fake, fake, 12)) == C.SD_ERR_UNSUPPORTED
    assert fused(_geom(C), scale=-1.0) == C.SD_ERR_INVALID_ARG
    assert fused(_geom(C), kvv=C.PagedKV(fake, fake, fake, fake, 128, 5000)) == C.SD_ERR_INVALID_ARG  # > pages*16
    assert fused(_geom(C), kvv=C.PagedKV(None, fake, fake, fake, 128, 100)) == C.SD_ERR_INVALID_ARG
    assert fused(_geom(C), wsb=100) == C.SD_ERR_WORKSPACE
    assert fused(_geom(C), wsp=ctypes.c_void_p(0x10010)) == C.SD_ERR_WORKSPACE     # misaligned
    # the option-flag entry: unknown flag bits are rejected before any launch
    assert lib.sd_sparse_decode_fused_ex(ctypes.byref(_geom(C)), ctypes.byref(kv), ctypes.byref(sk), fake,
                                         ctypes.byref(bud), 0.1, fake, None, None, None, 0, ws, 1 << 40, 2,
                                         None) == C.SD_ERR_INVALID_ARG
    assert lib.sd_sparse_decode_fused_ex(ctypes.byref(_geom(C, num_q_heads=30)), ctypes.byref(kv), ctypes.byref(sk),
                                         fake, ctypes.byref(bud), 0.1, fake, None, None, None, 0, ws, 1 << 40,
                                         C.SD_FUSED_FORCE_SLOW_PATH, None) == C.SD_ERR_INVALID_ARG
    assert lib.sd_lse_merge(0, 4, 128, fake, fake, 0, fake, None, None) == C.SD_ERR_INVALID_ARG
    assert lib.sd_lse_merge(2, 4, 64, fake, fake, 0, fake, None, None) == C.SD_ERR_UNSUPPORTED


def test_workspace_size_monotone(lib):
    from paper_2605_24168_b200 import _capi as C
    n1, n2, n3 = C.c_size(), C.c_size(), C.c_size()
    g = _geom(C, max_pages_per_seq=8192)
    assert lib.sd_workspace_size(ctypes.byref(g), None, 131072, ctypes.byref(n1)) == 0
    assert lib.sd_workspace_size(ctypes.byref(g), ctypes.byref(C.Budget(50.0, 0, 0, 0, 0.0)), 131072,
                                 ctypes.byref(n2)) == 0
    assert lib.sd_workspace_size(ctypes.byref(g), ctypes.byref(C.Budget(10.0, 0, 0, 0, 0.0)), 131072,
                                 ctypes.byref(n3)) == 0
    assert 0 < n1.value < n2.value < n3.value
    assert n1.value % 256 == 0 and n2.value % 256 == 0


def test_status_strings(lib):
    assert lib.sd_status_str(0) == b"SD_OK"
    assert lib.sd_status_str(3) == b"SD_ERR_WORKSPACE"
    assert b"sm_100a" in lib.sd_version()
