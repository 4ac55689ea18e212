"""CUDA path vs the fp64 oracle, element by element, through the C ABI.

Sizes span several CTA tiles (scan tile 2048 tokens, top-k tile 4096 keys,
attention tile 16 rows) and ragged tails; edge cases cover N_b = 1, k = N,
all-equal and duplicated keys, fp32 KV, ragged batches and weights.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import workloads
from parity import (SEL_REL_GAP, OUT_TOL_BF16, OUT_TOL_F32, check_lse, check_region_selection, check_rows_full_size,
                    check_selection, host_subcase, rel_err)

pytestmark = pytest.mark.gpu

SCALE = 1.0 / math.sqrt(128)


def _dev(case):
    return case.to("cuda")


def _kv(sd, case):
    return sd.KVCache.from_case(case), sd.SketchCache.from_case(case)


# --------------------------------------------------------------------------- A2
@pytest.mark.parametrize("dtype,mode", [(torch.bfloat16, "sketch"), (torch.bfloat16, "exact"),
                                        (torch.float32, "exact"), (torch.float32, "sketch")])
def test_index_score_matches_oracle(cuda_lib, dtype, mode):
    sd = cuda_lib
    lens = [1, 17, 2048, 4099, 5000]
    case = workloads.make_case(len(lens), 16, 4, lens, dtype=dtype, seed=11)
    inp = oracle.from_case(case)
    dc = _dev(case)
    kv, sk = _kv(sd, dc)
    sc = sd.sparse_index_score(dc.q, kv, sk if mode == "sketch" else None).cpu().double().numpy()
    u = 2.0 ** -24
    for b, N in enumerate(lens):
        for h in range(16):
            ref = oracle.index_scores(inp, b, h, mode)
            # fp32 forward error bound of an n-term fma/butterfly sum: n*u*sum|q_d k_d|
            g = h // 4
            if mode == "exact":
                mag, n = np.abs(inp.keys(b, g)) @ np.abs(inp.q[b, h]), 128
            else:
                mag, n = np.abs(inp.sketch(b, g)) @ np.abs(inp.q[b, h][inp.channel_ids[b, g]]), 8
            assert np.all(np.abs(sc[b, h, :N] - ref) <= n * u * mag + 1e-30), (b, h)
            # and inside the selection rule's band (1e-5 M_row), so that the rule
            # tests the selection, not indexer rounding
            assert np.abs(sc[b, h, :N] - ref).max() <= SEL_REL_GAP * max(np.abs(ref).max(), 1e-30), (b, h)


def test_index_score_fp8_sketch_matches_oracle(cuda_lib):
    """NEXT-4: the e4m3 sketch is converted exactly, so the scores meet the same
    fp32 error bound against the oracle's fp64 sum of the same e4m3 values."""
    sd = cuda_lib
    lens = [33, 4099, 9000]
    case = workloads.make_case(len(lens), 16, 4, lens, seed=13, sketch_dtype=torch.float8_e4m3fn)
    inp = oracle.from_case(case)
    dc = _dev(case)
    kv, sk = _kv(sd, dc)
    sc = sd.sparse_index_score(dc.q, kv, sk).cpu().double().numpy()
    u = 2.0 ** -24
    for b, N in enumerate(lens):
        for h in range(16):
            ref = oracle.index_scores(inp, b, h, "sketch")
            g = h // 4
            mag = np.abs(inp.sketch(b, g)) @ np.abs(inp.q[b, h][inp.channel_ids[b, g]])
            assert np.all(np.abs(sc[b, h, :N] - ref) <= 8 * u * mag + 1e-30), (b, h)
            assert np.abs(sc[b, h, :N] - ref).max() <= SEL_REL_GAP * max(np.abs(ref).max(), 1e-30), (b, h)


@pytest.mark.parametrize("dist", ["iid", "needle", "dup"])
def test_fused_fp8_sketch_matches_oracle(cuda_lib, dist):
    """NEXT-4 through the fused entry: selection against the oracle's scores of
    the same e4m3 sketch, outputs against attend_given on the selection."""
    lens = [20000, 4099, 300]
    case = workloads.make_case(len(lens), 32, 8, lens, seed=19, dist=dist, n_needles=32,
                               sketch_dtype=torch.float8_e4m3fn)
    _check_fused(cuda_lib, case, 50.0, "sketch")


def test_fused_fp8_equals_unfused_chain(cuda_lib):
    """The fp8-sketch fused step selects exactly what sd_sparse_index_score ->
    sd_topk_select select on the same e4m3 sketch."""
    sd = cuda_lib
    case = _dev(workloads.make_case(2, 32, 8, [30000, 777], seed=43, dist="needle", n_needles=40,
                                    sketch_dtype=torch.float8_e4m3fn))
    kv, sk = _kv(sd, case)
    _, _, idx_f, cnt_f = sd.sparse_decode_fused(case.q, kv, sk, S=50.0, scale=SCALE, return_idx=True)
    scores = sd.sparse_index_score(case.q, kv, sk)
    idx_u, cnt_u = sd.topk_select(scores, case.seq_lens, int(case.seq_lens.max()), S=50.0, num_kv_heads=8)
    assert torch.equal(cnt_f, cnt_u)
    k = idx_u.shape[-1]
    assert torch.equal(idx_f[..., :k], idx_u)


# --------------------------------------------------------------------------- A3
def _seeded_scores(B, H, lens, seed, kind):
    g = torch.Generator().manual_seed(seed)
    ld = (max(lens) + 63) // 64 * 64
    s = torch.zeros((B, H, ld), dtype=torch.float32)
    for b, N in enumerate(lens):
        if kind == "normal":
            s[b, :, :N] = torch.randn((H, N), generator=g)
        elif kind == "ties":
            s[b, :, :N] = torch.randint(-4, 5, (H, N), generator=g).float() * 0.25
        elif kind == "equal":
            s[b, :, :N] = 1.5
        elif kind == "signed_zero":
            v = torch.randint(0, 3, (H, N), generator=g).float() - 1.0
            v[v == 0] = -0.0
            v[:, ::3] = 0.0
            s[b, :, :N] = v
    return s


@pytest.mark.parametrize("kind", ["normal", "ties", "equal", "signed_zero"])
@pytest.mark.parametrize("S,k_fixed", [(50.0, 0), (10.0, 0), (1.0, 0), (2.5, 0), (1.0, 7)])
def test_topk_select_bit_exact(cuda_lib, kind, S, k_fixed):
    """Scores are a seeded INPUT to both sides, so the selection (an integer
    decision) is taken on identical fp32 values and must match bit for bit."""
    sd = cuda_lib
    lens = [7, 17, 4096, 5003, 131]
    B, H = len(lens), 4
    s = _seeded_scores(B, H, lens, 5, kind)
    seq = torch.tensor(lens, dtype=torch.int32)
    idx, cnt = sd.topk_select(s.cuda(), seq.cuda(), max(lens), S=S, k_fixed=k_fixed)
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    for b, N in enumerate(lens):
        k = oracle.budget_k(S, N, k_fixed) if k_fixed <= N else None
        for h in range(H):
            if k is None:
                continue
            ref = oracle.topk_select(s[b, h, :N].double().numpy(), k)
            assert cnt[b, h] == k
            assert idx[b, h, :k].tolist() == ref.tolist(), (b, h)


def test_topk_full_length_row(cuda_lib):
    """One 131,072-key row (BASELINE cfg3 row length) with heavy ties."""
    sd = cuda_lib
    N = 131072
    s = _seeded_scores(2, 2, [N, N - 5], 9, "ties")
    idx, cnt = sd.topk_select(s.cuda(), torch.tensor([N, N - 5], dtype=torch.int32).cuda(), N, S=50.0)
    for b, n in enumerate([N, N - 5]):
        for h in range(2):
            k = oracle.budget_k(50.0, n)
            ref = oracle.topk_select(s[b, h, :n].double().numpy(), k)
            assert idx[b, h, :k].cpu().tolist() == ref.tolist()


# --------------------------------------------------------------------------- A4/A5
@pytest.mark.parametrize("dtype,out_dtype", [(torch.bfloat16, torch.float32), (torch.bfloat16, torch.bfloat16),
                                             (torch.float32, torch.float32)])
@pytest.mark.parametrize("weighted", [False, True])
def test_gather_attend_matches_oracle(cuda_lib, dtype, out_dtype, weighted):
    sd = cuda_lib
    lens = [1, 40, 3000, 777]
    B, Hq, Hkv = len(lens), 8, 2
    case = workloads.make_case(B, Hq, Hkv, lens, dtype=dtype, seed=3)
    inp = oracle.from_case(case)
    dc = _dev(case)
    kv, _ = _kv(sd, dc)
    rng = np.random.default_rng(0)
    k_max = 1500
    idx = np.full((B, Hq, k_max), -1, dtype=np.int32)
    cnt = np.zeros((B, Hq), dtype=np.int32)
    w = np.ones((B, Hq, k_max), dtype=np.float32)
    for b, N in enumerate(lens):
        for h in range(Hq):
            c = int(rng.integers(1, min(N, k_max) + 1))
            sel = np.sort(rng.choice(N, c, replace=False))
            idx[b, h, :c] = sel
            cnt[b, h] = c
            if weighted:
                w[b, h, :c] = rng.uniform(0.1, 5.0, c).astype(np.float32)
    out, lse = sd.sparse_gather_attend(dc.q, kv, torch.from_numpy(idx).cuda(), torch.from_numpy(cnt).cuda(),
                                       weights=torch.from_numpy(w).cuda() if weighted else None,
                                       scale=SCALE, out_dtype=out_dtype)
    sd.clear_device_error()
    assert sd.read_device_error() == 0
    out = out.float().cpu().numpy()
    lse = lse.cpu().numpy()
    tol = OUT_TOL_BF16 if out_dtype == torch.bfloat16 else (OUT_TOL_F32 if dtype == torch.float32 else 1e-4)
    for b in range(B):
        for h in range(Hq):
            c = cnt[b, h]
            ro, rl = oracle.attend_given(inp, b, h, idx[b, h, :c], SCALE,
                                         w[b, h, :c].astype(np.float64) if weighted else None)
            assert rel_err(out[b, h], ro) <= tol, (b, h, rel_err(out[b, h], ro))
            check_lse(lse[b, h], rl)


def test_gather_attend_long_rows(cuda_lib):
    """Index lists over rows longer than 2^18 tokens (the bitmap is built in
    place in global memory, not in shared memory), GQA-union path."""
    sd = cuda_lib
    lens = [300_017, 5000]
    case = workloads.make_case(2, 8, 2, lens, seed=13)
    dc = _dev(case)
    kv, _ = _kv(sd, dc)
    rng = np.random.default_rng(2)
    k_max = 4000
    idx = np.full((2, 8, k_max), -1, dtype=np.int32)
    cnt = np.zeros((2, 8), dtype=np.int32)
    for b, N in enumerate(lens):
        for h in range(8):
            c = int(rng.integers(1, k_max + 1))
            idx[b, h, :c] = np.sort(rng.choice(N, c, replace=False))
            cnt[b, h] = c
    sd.clear_device_error()
    out, lse = sd.sparse_gather_attend(dc.q, kv, torch.from_numpy(idx).cuda(), torch.from_numpy(cnt).cuda(),
                                       scale=SCALE, out_dtype=torch.float32)
    assert sd.read_device_error() == 0
    out, lse = out.cpu().numpy(), lse.cpu().numpy()
    inp = oracle.from_case(case)
    for b in range(2):
        for h in (0, 3, 6):
            ro, rl = oracle.attend_given(inp, b, h, idx[b, h, :cnt[b, h]], SCALE)
            assert rel_err(out[b, h], ro) <= 1e-4
            check_lse(lse[b, h], rl)


def test_gather_attend_device_errors(cuda_lib):
    sd = cuda_lib
    case = _dev(workloads.make_case(1, 4, 1, 100, seed=1))
    kv, _ = _kv(sd, case)

    def run(idx_rows, counts, weights=None):
        sd.clear_device_error()
        idx = torch.tensor(idx_rows, dtype=torch.int32).cuda()[None]
        cnt = torch.tensor(counts, dtype=torch.int32).cuda()[None]
        wt = None if weights is None else torch.tensor(weights, dtype=torch.float32).cuda()[None]
        sd.sparse_gather_attend(case.q, kv, idx, cnt, weights=wt)
        return sd.read_device_error()

    ok = [[0, 5, 9], [1, 2, 3], [7, 8, 99], [0, 1, 2]]
    assert run(ok, [3, 3, 3, 3]) == 0
    assert run([[0, 5, 100], *ok[1:]], [3, 3, 3, 3]) == 1      # index >= N
    assert run([[5, 5, 9], *ok[1:]], [3, 3, 3, 3]) == 2        # not strictly increasing
    assert run(ok, [3, 0, 3, 3]) == 3                          # empty list
    assert run(ok, [3, 3, 3, 3], [[1, 1, 0.0]] + [[1, 1, 1]] * 3) == 4   # weight <= 0
    sd.clear_device_error()


# --------------------------------------------------------------------------- A7
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_dense_matches_oracle(cuda_lib, G):
    sd = cuda_lib
    lens = [1, 33, 4097, 9000]
    Hkv = 2
    case = workloads.make_case(len(lens), Hkv * G, Hkv, lens, seed=G)
    inp = oracle.from_case(case)
    dc = _dev(case)
    kv, _ = _kv(sd, dc)
    out, lse = sd.dense_decode(dc.q, kv, scale=SCALE, out_dtype=torch.float32)
    ro, rl = oracle.dense_decode(inp, SCALE)
    out, lse = out.cpu().numpy(), lse.cpu().numpy()
    for b in range(len(lens)):
        for h in range(Hkv * G):
            assert rel_err(out[b, h], ro[b, h]) <= 1e-4
            check_lse(lse[b, h], rl[b, h])


def test_dense_fp32_cfg1(cuda_lib):
    sd = cuda_lib
    case = workloads.config_case("cfg1", seed=1)
    inp = oracle.from_case(case)
    dc = _dev(case)
    kv, _ = _kv(sd, dc)
    out, lse = sd.dense_decode(dc.q, kv, scale=SCALE)
    ro, rl = oracle.dense_decode(inp, SCALE)
    for h in range(8):
        assert rel_err(out[0, h].cpu().numpy(), ro[0, h]) <= OUT_TOL_F32


# --------------------------------------------------------------------------- A6 fused
def _check_fused(sd, case, S, mode, out_dtype=torch.float32, k_fixed=0, rows=None):
    inp = oracle.from_case(case)
    dc = _dev(case)
    kv, sk = _kv(sd, dc)
    out, lse, idx, cnt = sd.sparse_decode_fused(dc.q, kv, sk if mode == "sketch" else None, S=S, k_fixed=k_fixed,
                                                scale=SCALE, out_dtype=out_dtype, return_idx=True)
    sd.clear_device_error()
    out = out.float().cpu().numpy()
    lse = lse.cpu().numpy()
    idx = idx.cpu().numpy()
    cnt = cnt.cpu().numpy()
    tol = OUT_TOL_BF16 if out_dtype == torch.bfloat16 else (OUT_TOL_F32 if case.dtype == torch.float32 else 1e-4)
    todo = rows if rows is not None else [(b, h) for b in range(case.B) for h in range(case.Hq)]
    for b, h in todo:
        N = int(case.seq_lens[b])
        k = oracle.budget_k(S, N, k_fixed)
        scores = oracle.index_scores(inp, b, h, mode)
        sel = check_selection(idx[b, h], cnt[b, h], scores, k)
        ro, rl = oracle.attend_given(inp, b, h, sel, SCALE)
        assert rel_err(out[b, h], ro) <= tol, (b, h, rel_err(out[b, h], ro))
        check_lse(lse[b, h], rl)
    return out, lse, idx, cnt


@pytest.mark.parametrize("dist", ["iid", "needle", "dup", "equal", "spec"])
def test_fused_sketch_matches_oracle(cuda_lib, dist):
    lens = [1, 100, 4099, 20000]
    case = workloads.make_case(len(lens), 32, 8, lens, seed=17, dist=dist, n_needles=64)
    _check_fused(cuda_lib, case, 50.0, "sketch")


@pytest.mark.parametrize("mode", ["sketch", "exact"])
def test_fused_all_equal_keys_take_lowest_indices(cuda_lib, mode):
    """S:204 (all scores equal, k = 3 -> {0, 1, 2}) at decode sizes: with every
    key of a (sequence, KV head) identical, every row's selection must be
    exactly the k_b lowest token indices - the only correct answer."""
    sd = cuda_lib
    lens = [1, 3, 100, 4099, 20000, 131072]
    case = _dev(workloads.make_case(len(lens), 32, 8, lens, seed=29, dist="equal", sketch=mode == "sketch"))
    kv, sk = _kv(sd, case)
    sd.clear_device_error()
    _, _, idx, cnt = sd.sparse_decode_fused(case.q, kv, sk if mode == "sketch" else None, S=50.0, scale=SCALE,
                                            return_idx=True)
    assert sd.read_device_error() == 0
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    for b, N in enumerate(lens):
        k = oracle.budget_k(50.0, N)
        for h in range(case.Hq):
            assert cnt[b, h] == k
            assert np.array_equal(idx[b, h, :k], np.arange(k)), (b, h, idx[b, h, :8])


@pytest.mark.parametrize("Hq,Hkv", [(32, 8), (8, 8), (16, 8), (16, 2)])
@pytest.mark.parametrize("dist", ["iid", "needle", "dup", "spec"])
@pytest.mark.parametrize("sketch_dtype", [torch.bfloat16, torch.float8_e4m3fn])
def test_fused_selection_is_exact_topk_of_gpu_scores(cuda_lib, Hq, Hkv, dist, sketch_dtype):
    """Where only one answer is correct it must be the one given: the fused
    selection equals, bit for bit, oracle.topk_select (ties to the lower index,
    S:200) applied to the GPU's own fp32 indexer scores (sd_sparse_index_score,
    the same fp32 arithmetic).  dup plants exact ties that straddle tau."""
    sd = cuda_lib
    lens = [1, 100, 4099, 20000, 70001]
    case = _dev(workloads.make_case(len(lens), Hq, Hkv, lens, seed=37 + Hq + Hkv, dist=dist, n_needles=64,
                                    sketch_dtype=sketch_dtype))
    kv, sk = _kv(sd, case)
    sd.clear_device_error()
    _, _, idx, cnt = sd.sparse_decode_fused(case.q, kv, sk, S=50.0, scale=SCALE, return_idx=True)
    assert sd.read_device_error() == 0
    sc = sd.sparse_index_score(case.q, kv, sk).cpu().numpy()
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    for b, N in enumerate(lens):
        k = oracle.budget_k(50.0, N)
        for h in range(Hq):
            ref = oracle.topk_select(sc[b, h, :N].astype(np.float64), k)
            assert cnt[b, h] == k
            assert np.array_equal(idx[b, h, :k], ref), (b, h)


@pytest.mark.parametrize("dist", ["iid", "dup"])
def test_fused_exact_topk_large_grid_ragged(cuda_lib, dist):
    """The scan's 4-CTA/SM shape (grids above one 3-CTA/SM wave) and its half-chunk
    CTAs in the last wave (two band sub-regions per chunk region, k_fused.cu):
    B = 16 ragged rows (a row ending inside the second half of a split chunk, one
    ending on a half boundary, short rows), every row's selection equal bit for bit
    to oracle.topk_select of the GPU's own fp32 scores (S:200 ties)."""
    sd = cuda_lib
    lens = [70001, 5000, 65536, 61440, 69000, 4097, 33333, 70001,
            50000, 8192, 12289, 69632, 45056 + 4095, 70000, 61441, 57345]
    case = _dev(workloads.make_case(len(lens), 32, 8, lens, seed=91, dist=dist, n_needles=64))
    kv, sk = _kv(sd, case)
    sd.clear_device_error()
    _, _, idx, cnt = sd.sparse_decode_fused(case.q, kv, sk, S=50.0, scale=SCALE, return_idx=True)
    assert sd.read_device_error() == 0
    assert sd.read_stats()["fallback_rows"] <= 2  # (deterministic inputs; the fast path is what this covers)
    sc = sd.sparse_index_score(case.q, kv, sk).cpu().numpy()
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    for b, N in enumerate(lens):
        k = oracle.budget_k(50.0, N)
        for h in range(32):
            ref = oracle.topk_select(sc[b, h, :N].astype(np.float64), k)
            assert cnt[b, h] == k
            assert np.array_equal(idx[b, h, :k], ref), (b, h)


def test_seq_len_above_max_seq_len_is_reported(cuda_lib):
    """sdattn.h: N_b > max_seq_len (or < 1) is a device error (SD_DEVERR_SEQLEN);
    the row reads as empty (out = 0, lse = -inf) and nothing else is touched:
    the valid rows keep their exact results, for every entry point."""
    sd = cuda_lib
    host = workloads.make_case(3, 8, 2, [5000, 3000, 4000], seed=91)
    case = _dev(host)
    inp = oracle.from_case(host)
    bad = torch.tensor([5000, 5001, 0], dtype=torch.int32, device="cuda")  # table rows hold 5008 tokens
    kvb = sd.KVCache(case.k_pages, case.v_pages, case.page_table, bad, 5000)
    sk = sd.SketchCache.from_case(case)

    def ok_row0(out, lse, sel=None):
        for h in range(8):
            if sel is None:  # dense: attention over every row of sequence 0
                ro, rl = oracle.attend_given(inp, 0, h, np.arange(5000), SCALE)
            else:
                ro, rl = oracle.attend_given(inp, 0, h, sel[h], SCALE)
            assert rel_err(out[0, h], ro) <= 1e-4
            check_lse(lse[0, h], rl)
        assert np.all(out[1:] == 0) and np.all(np.isneginf(lse[1:]))

    for mode in ("sketch", "exact"):
        sd.clear_device_error()
        out, lse, idx, cnt = sd.sparse_decode_fused(case.q, kvb, sk if mode == "sketch" else None, S=50.0,
                                                    scale=SCALE, out_dtype=torch.float32, return_idx=True)
        assert sd.read_device_error() == 5, mode
        idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
        assert np.all(cnt[1:] == 0)
        sels = {h: check_selection(idx[0, h], cnt[0, h], oracle.index_scores(inp, 0, h, mode), 100)
                for h in range(8)}
        ok_row0(out.cpu().numpy(), lse.cpu().numpy(), sels)
    sd.clear_device_error()
    out, lse = sd.dense_decode(case.q, kvb, scale=SCALE, out_dtype=torch.float32)
    assert sd.read_device_error() == 5
    ok_row0(out.cpu().numpy(), lse.cpu().numpy())
    sd.clear_device_error()
    sc = sd.sparse_index_score(case.q, kvb, sk)
    _, cnt = sd.topk_select(sc, bad, 5000, S=50.0, num_kv_heads=2)
    assert sd.read_device_error() == 5
    assert np.all(cnt.cpu().numpy()[1:] == 0) and np.all(cnt.cpu().numpy()[0] == 100)


@pytest.mark.parametrize("G,Hkv", [(1, 4), (2, 3), (8, 2)])
@pytest.mark.parametrize("S", [2.0, 10.0, 50.0])
def test_fused_sketch_group_sizes_and_sparsity(cuda_lib, G, Hkv, S):
    """Every GQA group size of the persistent union attend, including low
    sparsity (items with several 1024-row work units) and ragged lengths that
    end inside a page, a bitmap word and an 8192-token item."""
    lens = [20000, 8193, 37]
    case = workloads.make_case(len(lens), G * Hkv, Hkv, lens, seed=101 + G, dist="spec")
    _check_fused(cuda_lib, case, S, "sketch")


def test_fused_sketch_fp32_kv(cuda_lib):
    """fp32 KV with a sketch: the CUDA-core union attend + split merge path."""
    lens = [9000, 300]
    case = workloads.make_case(len(lens), 8, 2, lens, seed=61, dtype=torch.float32)
    _check_fused(cuda_lib, case, 20.0, "sketch")


def test_fused_timed_matches_untimed(cuda_lib):
    """sd_sparse_decode_fused_timed: same output as the untimed call, five
    non-negative kernel durations."""
    sd = cuda_lib
    case = _dev(workloads.make_case(2, 32, 8, [20000, 5000], seed=67, dist="needle", n_needles=16))
    kv, sk = _kv(sd, case)
    o1, l1 = sd.sparse_decode_fused(case.q, kv, sk, S=50.0, scale=SCALE)
    o2, l2, ph = sd.api.sparse_decode_fused_timed(case.q, kv, sk, S=50.0, scale=SCALE)
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    assert set(ph) == set(sd.api.FUSED_PHASES) and all(v >= 0 for v in ph.values()), ph


NEXT1_CASES = [(128, 128, 0.20, 0), (128, 128, 0.02, 0), (64, 0, 0.0, 16), (0, 32, 0.05, 0), (300, 300, 0.1, 0)]


@pytest.mark.parametrize("n_sink,n_local,hf,k_abs", NEXT1_CASES)
@pytest.mark.parametrize("mode", ["sketch", "exact"])
def test_fused_sink_local_heavy(cuda_lib, n_sink, n_local, hf, k_abs, mode):
    """NEXT-1 Sink + Local + heavy fraction through the
    fused entry (sample/scan/select in sketch mode, radix top-k in exact mode)."""
    sd = cuda_lib
    lens = [20000, 5000, 200]
    case = workloads.make_case(len(lens), 8, 2, lens, seed=71, dist="needle", n_needles=24, sketch=mode == "sketch")
    inp = oracle.from_case(case)
    dc = _dev(case)
    kv, sk = _kv(sd, dc)
    out, lse, idx, cnt = sd.sparse_decode_fused(dc.q, kv, sk if mode == "sketch" else None, S=1.0, k_fixed=k_abs,
                                                scale=SCALE, out_dtype=torch.float32, return_idx=True,
                                                n_sink=n_sink, n_local=n_local, heavy_fraction=hf)
    assert sd.read_device_error() == 0
    out, lse, idx, cnt = out.cpu().numpy(), lse.cpu().numpy(), idx.cpu().numpy(), cnt.cpu().numpy()
    for b in range(case.B):
        for h in range(case.Hq):
            scores = oracle.index_scores(inp, b, h, mode)
            sel = check_region_selection(idx[b, h], cnt[b, h], scores, n_sink, n_local, hf, k_abs)
            ro, rl = oracle.attend_given(inp, b, h, sel, SCALE)
            assert rel_err(out[b, h], ro) <= 1e-4, (b, h)
            check_lse(lse[b, h], rl)


@pytest.mark.parametrize("n_sink,n_local,hf,k_abs", NEXT1_CASES)
def test_topk_sink_local_heavy_bit_exact(cuda_lib, n_sink, n_local, hf, k_abs):
    """sd_topk_select with a NEXT-1 budget equals oracle.sink_local_heavy_select
    exactly on fp32 scores with heavy ties."""
    sd = cuda_lib
    g = torch.Generator().manual_seed(5)
    B, Hq, N = 2, 4, 7000
    sc = torch.randint(-40, 40, (B, Hq, N), generator=g).float() / 8.0  # many exact ties
    lens = torch.tensor([N, 1500], dtype=torch.int32)
    idx, cnt = sd.topk_select(sc.cuda(), lens.cuda(), N, S=1.0, k_fixed=k_abs, n_sink=n_sink, n_local=n_local,
                              heavy_fraction=hf)
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    for b in range(B):
        n = int(lens[b])
        for h in range(Hq):
            ref = oracle.sink_local_heavy_select(sc[b, h, :n].double().numpy(), n_sink, n_local, hf, k_abs)
            assert cnt[b, h] == ref.size
            np.testing.assert_array_equal(idx[b, h, :cnt[b, h]], ref)


@pytest.mark.parametrize("k_det,n_samples", [(16, 64), (10, 0), (1, 40), (10, 100000), (300, 700)])
def test_stochastic_select_matches_oracle(cuda_lib, k_det, n_samples):
    """NEXT-2: the GPU selection and weights equal
    oracle.stochastic_select on the same scores and the same uniform draw
    (ties in scores and in u to the lower index)."""
    sd = cuda_lib
    g = torch.Generator().manual_seed(9)
    B, Hq, N = 2, 4, 5000
    sc = torch.randint(-30, 30, (B, Hq, N), generator=g).float() / 4.0
    u = torch.randint(0, 4000, (B, Hq, N), generator=g).float() / 4096.0  # uniform keys with ties
    lens = torch.tensor([N, 777], dtype=torch.int32)
    idx, wts, cnt = sd.api.stochastic_select(sc.cuda(), u.cuda(), lens.cuda(), N, k_det, n_samples)
    idx, wts, cnt = idx.cpu().numpy(), wts.cpu().numpy(), cnt.cpu().numpy()
    for b in range(B):
        n = int(lens[b])
        for h in range(Hq):
            ri, rw = oracle.stochastic_select(sc[b, h, :n].double().numpy(), min(k_det, n), n_samples,
                                              u[b, h, :n].double().numpy())
            assert cnt[b, h] == ri.size, (b, h, cnt[b, h], ri.size)
            np.testing.assert_array_equal(idx[b, h, :ri.size], ri)
            np.testing.assert_allclose(wts[b, h, :ri.size], rw, rtol=1e-6)


def test_stochastic_weighted_attend_end_to_end(cuda_lib):
    """NEXT-2 selection on the GPU's own index scores -> weighted gather-attend
    == oracle.attend_given(selection, weights)."""
    sd = cuda_lib
    case = workloads.make_case(2, 8, 2, [6000, 900], seed=77)
    inp = oracle.from_case(case)
    dc = _dev(case)
    kv, sk = _kv(sd, dc)
    N = int(case.seq_lens.max())
    scores = sd.sparse_index_score(dc.q, kv, sk)
    gen = torch.Generator(device="cuda").manual_seed(4)
    u = torch.rand(scores.shape, generator=gen, device="cuda")
    idx, wts, cnt = sd.api.stochastic_select(scores, u, dc.seq_lens, N, 32, 96, num_kv_heads=2)
    out, lse = sd.sparse_gather_attend(dc.q, kv, idx, cnt, weights=wts, scale=SCALE, out_dtype=torch.float32)
    out, lse = out.cpu().numpy(), lse.cpu().numpy()
    idx, wts, cnt = idx.cpu().numpy(), wts.cpu().numpy(), cnt.cpu().numpy()
    for b in range(case.B):
        for h in range(case.Hq):
            c = int(cnt[b, h])
            ro, rl = oracle.attend_given(inp, b, h, idx[b, h, :c], SCALE, weights=wts[b, h, :c].astype(np.float64))
            assert rel_err(out[b, h], ro) <= 1e-4
            check_lse(lse[b, h], rl)


@pytest.mark.parametrize("S", [1.0, 2.0, 10.0, 100.0, 500.0])
def test_fused_exact_mode_sparsity_sweep(cuda_lib, S):
    lens = [3, 257, 6000]
    case = workloads.make_case(len(lens), 8, 2, lens, seed=23, sketch=False)
    _check_fused(cuda_lib, case, S, "exact")


def test_fused_cfg1_fp32_exact(cuda_lib):
    """BASELINE.json configs[0]: B=1, 1 KV head, 8 q-heads, N=4096, S=50 (k=82), fp32 KV."""
    case = workloads.config_case("cfg1")
    out, lse, idx, cnt = _check_fused(cuda_lib, case, 50.0, "exact")
    assert (cnt == 82).all()


def test_fused_bf16_output_and_kfixed(cuda_lib):
    case = workloads.make_case(2, 16, 2, [5000, 64], seed=31)
    _check_fused(cuda_lib, case, 1.0, "sketch", out_dtype=torch.bfloat16, k_fixed=64)


def test_fused_equals_unfused_chain(cuda_lib):
    """The fused entry and sd_sparse_index_score -> sd_topk_select select the same
    sets bit for bit (same fp32 score code) and give the same outputs."""
    sd = cuda_lib
    case = _dev(workloads.make_case(3, 32, 8, [7000, 30000, 123], seed=41, dist="needle", n_needles=40))
    kv, sk = _kv(sd, case)
    out_f, lse_f, idx_f, cnt_f = sd.sparse_decode_fused(case.q, kv, sk, S=20.0, scale=SCALE,
                                                        out_dtype=torch.float32, return_idx=True)
    sc = sd.sparse_index_score(case.q, kv, sk)
    idx_u, cnt_u = sd.topk_select(sc, case.seq_lens, kv.max_seq_len, S=20.0, num_kv_heads=8)
    assert torch.equal(cnt_f, cnt_u)
    for b in range(3):
        for h in range(32):
            c = int(cnt_u[b, h])
            assert torch.equal(idx_f[b, h, :c], idx_u[b, h, :c])
    out_u, lse_u = sd.sparse_gather_attend(case.q, kv, idx_u, cnt_u, scale=SCALE, out_dtype=torch.float32)
    assert (out_u - out_f).abs().max().item() <= 1e-5 * out_u.abs().max().item()


@pytest.mark.slow
@pytest.mark.parametrize("name,heads", [("cfg3", "all"), ("cfg2_s10", 6), ("cfg2_s50", "all"), ("cfg2_s100", 6),
                                        ("cfg4_t0", "all"), ("cfg4_t33", 6), ("cfg4_t66", 6)])
def test_fused_baseline_sizes(cuda_lib, name, heads):
    """BASELINE.json full sizes in the bench's launch configuration: for 2
    sequences, every q-head ("all") or 6 sampled heads: the selection is the
    exact top-k of the GPU's own fp32 scores (bit for bit) and within the
    tolerance rule of the fp64 oracle scores; the output matches
    oracle.attend_given on the GPU's selection."""
    sd = cuda_lib
    cfg = workloads.CONFIGS[name]
    case = workloads.config_case(name, device="cuda")
    kv, sk = _kv(sd, case)
    sd.clear_device_error()
    out, lse, idx, cnt = sd.sparse_decode_fused(case.q, kv, sk, S=cfg["S"], scale=SCALE,
                                                out_dtype=torch.float32, return_idx=True)
    assert sd.read_device_error() == 0
    assert sd.read_stats()["fallback_rows"] == 0
    sc = sd.sparse_index_score(case.q, kv, sk)
    out, lse, idx, cnt = out.cpu().numpy(), lse.cpu().numpy(), idx.cpu().numpy(), cnt.cpu().numpy()
    rng = np.random.default_rng(0)
    for b in rng.choice(case.B, 2, replace=False):
        hs = list(range(case.Hq)) if heads == "all" else sorted(rng.choice(case.Hq, heads, replace=False).tolist())
        check_rows_full_size(case, int(b), hs, cfg["S"], idx, cnt, out, lse, gpu_scores=sc[int(b)].cpu().numpy(),
                             scale=SCALE)


@pytest.mark.slow
def test_fused_cfg5_geometry_one_gpu(cuda_lib):
    """BASELINE cfg5's geometry unsharded on one GPU: B=1, Hq=32, Hkv=8,
    N=2^20, S=100 (k=10486): fast path for every row, heads of four groups
    checked bit-exactly on the GPU's scores and against the oracle."""
    sd = cuda_lib
    case = workloads.config_case("cfg5", device="cuda")
    kv, sk = _kv(sd, case)
    sd.clear_device_error()
    out, lse, idx, cnt = sd.sparse_decode_fused(case.q, kv, sk, S=100.0, scale=SCALE, out_dtype=torch.float32,
                                                return_idx=True)
    assert sd.read_device_error() == 0
    assert sd.read_stats()["fallback_rows"] == 0
    assert int(cnt.min()) == int(cnt.max()) == 10486
    # the band capacity holds the band's spread (~1/sqrt(sample ranks)) over many queries
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    for _ in range(8):
        qx = torch.randn(case.q.shape, generator=g, device="cuda").to(case.q.dtype)
        sd.sparse_decode_fused(qx, kv, sk, S=100.0, scale=SCALE)
    torch.cuda.synchronize()
    assert sd.read_stats()["fallback_rows"] == 0
    sc = sd.sparse_index_score(case.q, kv, sk)
    check_rows_full_size(case, 0, [0, 13, 22, 31], 100.0, idx.cpu().numpy(), cnt.cpu().numpy(), out.cpu().numpy(),
                         lse.cpu().numpy(), gpu_scores=sc[0].cpu().numpy(), scale=SCALE)


@pytest.mark.parametrize("N", [1 << 20, (1 << 21) - 8192, (1 << 21) + 4096])
def test_fused_maximum_lengths(cuda_lib, N):
    """The fused path at the longest sequences: 2^20 (BASELINE cfg5 on one GPU)
    and around 2^21, where the sample grows with N (rounds of 4096 tokens,
    ~N^2) so the bracket's band stays within the select's capacity: every row
    on the fast path.  Sampled rows checked one by one against the oracle."""
    sd = cuda_lib
    case = workloads.make_case(1, 8, 2, [N], seed=81, dist="needle", n_needles=16, device="cuda")
    kv, sk = _kv(sd, case)
    sd.clear_device_error()
    out, lse, idx, cnt = sd.sparse_decode_fused(case.q, kv, sk, S=100.0, scale=SCALE, out_dtype=torch.float32,
                                                return_idx=True)
    torch.cuda.synchronize()
    assert sd.read_device_error() == 0
    assert sd.read_stats()["fallback_rows"] == 0
    sub = host_subcase(case, 0)
    inp = oracle.from_case(sub)
    k = oracle.budget_k(100.0, N)
    for h in (0, 5):
        scores = oracle.index_scores(inp, 0, h, "sketch")
        sel = check_selection(idx[0, h].cpu().numpy(), int(cnt[0, h]), scores, k)
        ro, rl = oracle.attend_given(inp, 0, h, sel, SCALE)
        assert rel_err(out[0, h].cpu().numpy(), ro) <= 1e-4
        check_lse(float(lse[0, h]), rl)


@pytest.mark.slow
def test_fused_4m_tokens_fast_equals_slow(cuda_lib):
    """2^22 tokens (16 sample rounds, the longest fast-path row at S = 100):
    no row on the slow path, and the selection and outputs equal the forced
    exact slow path (full-row radix select over the same fp32 scores) bit for bit."""
    sd = cuda_lib
    N = 1 << 22
    case = workloads.make_case(1, 8, 2, [N], seed=83, device="cuda")
    kv, sk = _kv(sd, case)
    sd.clear_device_error()
    o1, l1, i1, c1 = sd.sparse_decode_fused(case.q, kv, sk, S=100.0, scale=SCALE, out_dtype=torch.float32,
                                            return_idx=True)
    torch.cuda.synchronize()
    assert sd.read_device_error() == 0
    assert sd.read_stats()["fallback_rows"] == 0
    o2, l2, i2, c2 = sd.sparse_decode_fused(case.q, kv, sk, S=100.0, scale=SCALE, out_dtype=torch.float32,
                                            return_idx=True, force_slow_path=True)
    assert torch.equal(c1, c2) and torch.equal(i1, i2)
    assert torch.equal(o1, o2) and torch.equal(l1, l2)


# --------------------------------------------------------------------------- sequence sharding (1 GPU)
def _shard_kv(sd, case, lo, hi):
    """KV cache view of tokens [lo, hi) of every sequence (lo page-aligned)."""
    assert lo % 16 == 0
    pt = case.page_table[:, lo // 16:].contiguous()
    lens = torch.clamp(case.seq_lens - lo, min=0).clamp(max=hi - lo).to(torch.int32)
    return sd.KVCache(case.k_pages, case.v_pages, pt, lens, max(1, int(lens.max()))), lens


@pytest.mark.parametrize("P,G", [(2, 4), (3, 4), (4, 4), (3, 2)])
@pytest.mark.parametrize("dist", ["dup", "needle"])
def test_seqshard_protocol_matches_oracle(cuda_lib, P, G, dist):
    """Sequence sharding on one GPU: local top-k_b per shard ->
    all candidate scores -> global cut + local attend -> LSE merge.  The union
    of the ranks' survivors is bit for bit the exact top-k_b of the GPU's own
    fp32 scores (duplicated keys: exact ties across shards go to the lower
    global index) and equals oracle.seqshard_decode's index set; the merged
    output matches oracle.seqshard_decode and oracle.attend_given on the set."""
    sd = cuda_lib
    N = 8192
    # G = 4: the fused local selection + the GQA-union attend; G = 2: materialised
    # scores + radix top-k (the general path)
    host = workloads.make_case(2, 4 * G, 4, [N, N - 77], seed=50 + P, dist=dist, n_needles=40)
    case = _dev(host)
    kv, sk = _kv(sd, case)
    S = 20.0
    glens = case.seq_lens
    k_max = sd.budget_k(S, N)
    bounds = [((r * N) // P) // 16 * 16 for r in range(P)] + [N]
    cands, cidx, kvs = [], [], []
    for r in range(P):
        kvr, _ = _shard_kv(sd, case, bounds[r], bounds[r + 1])
        cs, ci = sd.seqshard_local_topk(case.q, kvr, sk, glens, N, S, k_max=k_max)
        cands.append(cs)
        cidx.append(ci)
        kvs.append(kvr)
    all_cand = torch.stack(cands).contiguous()
    parts_o, parts_l, survs = [], [], []
    for r in range(P):
        po, pl, sv, sc_ = sd.seqshard_cut_attend(case.q, kvs[r], glens, all_cand, cidx[r], r, S, scale=SCALE,
                                                 return_survivors=True)
        parts_o.append(po)
        parts_l.append(pl)
        survs.append((sv.cpu().numpy(), sc_.cpu().numpy()))
    out, lse = sd.lse_merge(torch.stack(parts_o).contiguous(), torch.stack(parts_l).contiguous())
    assert sd.read_device_error() == 0
    out, lse = out.cpu().numpy(), lse.cpu().numpy()
    gpu_sc = sd.sparse_index_score(case.q, kv, sk).cpu().numpy()
    inp = oracle.from_case(host)
    ref_idx, ref_o, ref_lse = oracle.seqshard_decode(inp, S, SCALE, P)
    for b in range(case.B):
        Nb = int(host.seq_lens[b])
        k = oracle.budget_k(S, Nb)
        for h in range(case.Hq):
            got = np.sort(np.concatenate([sv[b, h, :c[b, h]] + bounds[r] for r, (sv, c) in enumerate(survs)]))
            assert got.size == k
            assert np.array_equal(got, oracle.topk_select(gpu_sc[b, h, :Nb].astype(np.float64), k)), (b, h)
            check_selection(got, k, oracle.index_scores(inp, b, h, "sketch"), k)
            assert np.array_equal(got, ref_idx[b][h]), (b, h)
            assert rel_err(out[b, h], ref_o[b, h]) <= 1e-4, (b, h)
            check_lse(lse[b, h], ref_lse[b, h])
            ro, rl = oracle.attend_given(inp, b, h, got, SCALE)
            assert rel_err(out[b, h], ro) <= 1e-4
            check_lse(lse[b, h], rl)


@pytest.mark.parametrize("dist", ["needle", "dup"])
def test_seqshard_local_candidates_exact(cuda_lib, dist):
    """Sequence-shard step 1 on the fused selection (k_b from the GLOBAL length,
    scores never materialised): every shard's candidates are exactly the
    top-min(k_b, N_loc) of the GPU's own fp32 indexer scores of the shard
    (ties to the lower index), ascending, with those scores bit for bit, padded
    with -1 / -inf; shards past a short sequence's end are empty."""
    sd = cuda_lib
    lens = [8192 + 5, 3000]
    case = _dev(workloads.make_case(2, 32, 8, lens, seed=71, dist=dist, n_needles=60))
    _, sk = _kv(sd, case)
    S, P, NG = 20.0, 3, max(lens)
    glens = case.seq_lens
    k_max = sd.budget_k(S, NG)
    bounds = [((r * NG) // P) // 16 * 16 for r in range(P)] + [NG]
    for r in range(P):
        kvr, loc = _shard_kv(sd, case, bounds[r], bounds[r + 1])
        sd.clear_device_error()
        cs, ci = sd.seqshard_local_topk(case.q, kvr, sk, glens, NG, S, k_max=k_max)
        sc = sd.sparse_index_score(case.q, kvr, sk)
        assert sd.read_device_error() == 0
        cs, ci, sc = cs.cpu().numpy(), ci.cpu().numpy(), sc.cpu().numpy()
        for b in range(2):
            nl = int(loc[b])
            k = min(sd.budget_k(S, lens[b]), nl)
            for h in range(32):
                exp = oracle.topk_select(sc[b, h, :nl].astype(np.float64), k) if k else np.zeros(0, np.int64)
                assert np.array_equal(ci[b, h, :k], exp), (r, b, h)
                assert np.array_equal(cs[b, h, :k].view(np.uint32), sc[b, h, exp].view(np.uint32))
                assert np.all(ci[b, h, k:] == -1) and np.all(np.isneginf(cs[b, h, k:]))


@pytest.mark.parametrize("dist", ["iid", "needle", "dup"])
def test_fused_forced_fallback_identical(cuda_lib, dist):
    """The exact per-(b, g) fallback of the fused select (sd_sparse_decode_fused_ex
    with SD_FUSED_FORCE_SLOW_PATH) gives the same index sets and the same
    outputs as the sample-bracket fast path."""
    sd = cuda_lib
    case = _dev(workloads.make_case(2, 32, 8, [20000, 3000], seed=61, dist=dist, n_needles=100))
    kv, sk = _kv(sd, case)
    a = sd.sparse_decode_fused(case.q, kv, sk, S=50.0, scale=SCALE, out_dtype=torch.float32, return_idx=True)
    sd.clear_device_error()
    b = sd.sparse_decode_fused(case.q, kv, sk, S=50.0, scale=SCALE, out_dtype=torch.float32, return_idx=True,
                               force_slow_path=True)
    assert sd.read_stats()["fallback_rows"] == case.B * case.Hq
    assert torch.equal(a[3], b[3])
    for bb in range(2):
        for h in range(32):
            c = int(a[3][bb, h])
            assert torch.equal(a[2][bb, h, :c], b[2][bb, h, :c])
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_fused_deterministic_and_large_window(cuda_lib):
    """Two calls are bitwise identical; N > one bitmap window (G=8 -> 65,536)."""
    sd = cuda_lib
    case = _dev(workloads.make_case(1, 16, 2, [70001], seed=71))
    kv, sk = _kv(sd, case)
    a = sd.sparse_decode_fused(case.q, kv, sk, S=100.0, scale=SCALE, out_dtype=torch.float32, return_idx=True)
    b = sd.sparse_decode_fused(case.q, kv, sk, S=100.0, scale=SCALE, out_dtype=torch.float32, return_idx=True)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    _check_fused(sd, workloads.make_case(1, 16, 2, [70001], seed=71), 100.0, "sketch", rows=[(0, h) for h in range(16)])


@pytest.mark.parametrize("dist,lens", [("iid", [131072, 20000]), ("needle", [70000, 9000]), ("spec", [50000])])
def test_fused_fast_path_taken(cuda_lib, dist, lens):
    """On the paper-shaped workloads the sample bracket holds: no row needs the
    exact slow path (the fast path is what the bench times)."""
    sd = cuda_lib
    case = _dev(workloads.make_case(len(lens), 32, 8, lens, seed=81, dist=dist, n_needles=80))
    kv, sk = _kv(sd, case)
    sd.sparse_decode_fused(case.q, kv, sk, S=50.0, scale=SCALE)
    sd.clear_device_error()
    sd.sparse_decode_fused(case.q, kv, sk, S=50.0, scale=SCALE)
    assert sd.read_stats()["fallback_rows"] == 0
    assert sd.read_device_error() == 0


@pytest.mark.parametrize("S,N", [(50.0, 40000), (2.0, 131072)])
def test_fused_g4_pair_select_and_ws_attend(cuda_lib, S, N):
    """G = 4 (the tensor-core scan's head-pair regions): at S = 50 the select runs
    one CTA per head pair (two 256-thread halves); at S = 2, N = 128K its band
    capacity exceeds two heads per CTA and one CTA per head reads the pair
    regions.  Both feed the warp-specialised attend (dynamic item claiming):
    parity on rows of both heads of every pair, no slow path, and two calls
    bitwise identical."""
    sd = cuda_lib
    case = workloads.make_case(1, 32, 8, [N], seed=97, dist="needle", n_needles=30)
    rows = [(0, h) for h in (0, 1, 2, 3, 14, 15, 30, 31)]
    _check_fused(sd, case, S, "sketch", rows=rows)
    dc = _dev(case)
    kv, sk = _kv(sd, dc)
    sd.clear_device_error()
    a = sd.sparse_decode_fused(dc.q, kv, sk, S=S, scale=SCALE, out_dtype=torch.float32, return_idx=True)
    assert sd.read_stats()["fallback_rows"] == 0
    b = sd.sparse_decode_fused(dc.q, kv, sk, S=S, scale=SCALE, out_dtype=torch.float32, return_idx=True)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
