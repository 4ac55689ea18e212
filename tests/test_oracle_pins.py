"""Pins of the fp64 oracle against things other than itself (CPU only).

Each test names the passage / closed form / library routine it pins to, and is
chosen so that a plausible mistake in oracle/sdoracle.py (a dropped term, a
wrong sign or index, a transposed operand, a wrong tie order) fails one of them.
"""
import itertools
import math

import numpy as np
import pytest
import torch

import oracle
from oracle import OracleInputs
import workloads


def _inputs_from_logical(K, V, q, seq_lens, page_size=4, seed=0, sketch=None, channel_ids=None):
    """Lay logical K/V [B][N][Hkv][D] into randomly permuted pages (numpy pools)."""
    rng = np.random.default_rng(seed)
    B, N, Hkv, D = K.shape
    npg = (N + page_size - 1) // page_size
    total = B * npg
    perm = rng.permutation(total)
    pt = perm.reshape(B, npg)
    kp = np.zeros((total, page_size, Hkv, D))
    vp = np.zeros((total, page_size, Hkv, D))
    sp = None
    if sketch is not None:
        C = sketch.shape[-1]
        sp = np.zeros((total, Hkv, page_size, C))
    for b in range(B):
        for t in range(N):
            p, s = pt[b, t // page_size], t % page_size
            kp[p, s] = K[b, t]
            vp[p, s] = V[b, t]
            if sp is not None:
                sp[p, :, s] = sketch[b, t]
    return OracleInputs(q=np.asarray(q, float), k_pages=kp, v_pages=vp, page_table=pt,
                        seq_lens=np.asarray(seq_lens), page_size=page_size, Hkv=Hkv,
                        channel_ids=channel_ids, sketch_pages=sp)


# --------------------------------------------------------------------------- A1
@pytest.mark.parametrize("S,N,k", [
    (1.0, 7, 7), (1.0, 131072, 131072),          # S:194 dense limit
    (50.0, 131072, 2622), (500.0, 131072, 263),
    (50.0, 4096, 82),                            # BASELINE.json configs[0] "k=82"
    (10.0, 32768, 3277), (50.0, 32768, 656), (100.0, 32768, 328),
    (100.0, 1 << 20, 10486),                     # SURVEY 8(c) reading 12
    (50.0, 1, 1), (3.0, 2, 1), (2.5, 5, 2), (2.5, 6, 3),
])
def test_budget_worked_values(S, N, k):
    assert oracle.budget_k(S, N) == k


def test_budget_rejections():
    with pytest.raises(ValueError):
        oracle.budget_k(0.5, 10)      # S < 1
    with pytest.raises(ValueError):
        oracle.budget_k(2.0, 0)       # empty sequence
    with pytest.raises(ValueError):
        oracle.budget_k(2.0, 5, k_fixed=6)   # k > N
    assert oracle.budget_k(2.0, 5, k_fixed=5) == 5


# --------------------------------------------------------------------------- A3
def test_topk_spec_examples():
    # S:203 scores [3, 1, 2], k=2 -> {0, 2};  S:204 all equal, k=3, N=10 -> {0, 1, 2}
    assert oracle.topk_select(np.array([3.0, 1.0, 2.0]), 2).tolist() == [0, 2]
    assert oracle.topk_select(np.zeros(10), 3).tolist() == [0, 1, 2]


def test_topk_bruteforce_rank_definition():
    """AC2: 1,000 random instances, ties forced by small integer scores.
    Brute force: t is selected iff fewer than k tokens precede it in the total
    order, i.e. #{u: s_u > s_t} + #{u < t: s_u == s_t} < k."""
    rng = np.random.default_rng(7)
    for _ in range(1000):
        N = int(rng.integers(1, 40))
        s = rng.integers(-3, 4, size=N).astype(float)
        k = int(rng.integers(1, N + 1))
        got = oracle.topk_select(s, k)
        want = [t for t in range(N)
                if (np.sum(s > s[t]) + np.sum(s[:t] == s[t])) < k]
        assert got.tolist() == want
        assert np.all(np.diff(got) > 0)


def test_topk_exhaustive_tiny():
    """Every score pattern over {0,1,2} for N <= 6 and every k: brute-force subset
    search for the lexicographically best set (sorted desc scores, then indices)."""
    for N in range(1, 7):
        for pat in itertools.product([0.0, 1.0, 2.0], repeat=N):
            s = np.array(pat)
            for k in range(1, N + 1):
                best = None
                for sub in itertools.combinations(range(N), k):
                    key = (sorted((-s[list(sub)]).tolist()), list(sub))
                    if best is None or key < best[0]:
                        best = (key, sub)
                assert oracle.topk_select(s, k).tolist() == list(best[1])


def test_topk_rejects():
    with pytest.raises(ValueError):
        oracle.topk_select(np.zeros(3), 4)
    with pytest.raises(ValueError):
        oracle.topk_select(np.array([0.0, np.nan]), 1)


# --------------------------------------------------------------------------- A2
def test_onehot_keys_closed_form_selection():
    """K[t] = c_t e_{t mod D} with c_t = t+1 and q = e_j: score_t = c_t if
    t = j (mod D) else 0, so the top-k are the k LAST tokens congruent to j."""
    D, N, Hkv, G = 8, 64, 2, 2
    K = np.zeros((1, N, Hkv, D))
    for t in range(N):
        for g in range(Hkv):
            K[0, t, g, t % D] = t + 1.0
    V = np.random.default_rng(0).standard_normal((1, N, Hkv, D))
    q = np.zeros((1, Hkv * G, D))
    js = [1, 6, 3, 0]
    for h, j in enumerate(js):
        q[0, h, j] = 1.0
    inp = _inputs_from_logical(K, V, q, [N])
    for h, j in enumerate(js):
        s = oracle.index_scores(inp, 0, h, "exact")
        congruent = [t for t in range(N) if t % D == j]
        for k in (1, 3, len(congruent)):
            assert oracle.topk_select(s, k).tolist() == congruent[-k:]


def test_sketch_full_channels_equals_exact():
    """with C = D and channel_ids = 0..D-1 the sketch score equals the
    exact score bit for bit (same products, same order)."""
    case = workloads.make_case(2, 8, 2, [50, 33], D=16, C=16, seed=3, dtype=torch.float32)
    inp = oracle.from_case(case)
    inp.channel_ids = np.tile(np.arange(16), (2, 2, 1))
    # rebuild the sketch for the identity channel map
    kp = case.k_pages.double().numpy()
    inp.sketch_pages = kp.transpose(0, 2, 1, 3).copy()     # [P][Hkv][ps][C=D]
    for b in range(2):
        for h in range(8):
            a = oracle.index_scores(inp, b, h, "sketch")
            e = oracle.index_scores(inp, b, h, "exact")
            assert np.array_equal(a, e)


def test_sketch_onehot_query_reads_the_named_channel():
    """q = e_{ch[c]} makes the sketch score the stored value of sketch channel c,
    which is K[t][ch[c]] (S:183 'sketch row = chosen channels of the key row')."""
    case = workloads.make_case(1, 4, 2, 45, D=32, C=8, seed=5)
    inp = oracle.from_case(case)
    for g in range(2):
        ch = inp.channel_ids[0, g]
        assert np.all(np.diff(ch) > 0) and ch.max() < 32
        for c in (0, 5, 7):
            inp.q = np.zeros_like(inp.q)
            inp.q[0, 2 * g, ch[c]] = 1.0
            s = oracle.index_scores(inp, 0, 2 * g, "sketch")
            assert np.array_equal(s, inp.keys(0, g)[:, ch[c]])


def test_needle_selected_for_every_head():
    """a key row set to c*qbar (c large) is the top-1 of every head of its group."""
    rng = np.random.default_rng(11)
    B, N, Hkv, G, D = 1, 300, 2, 4, 64
    q = rng.standard_normal((B, Hkv * G, D))
    K = rng.standard_normal((B, N, Hkv, D))
    V = rng.standard_normal((B, N, Hkv, D))
    tstar = [123, 7]
    for g in range(Hkv):
        K[0, tstar[g], g] = 50.0 * q[0, g * G:(g + 1) * G].mean(0)
    inp = _inputs_from_logical(K, V, q, [N])
    for h in range(Hkv * G):
        s = oracle.index_scores(inp, 0, h, "exact")
        assert oracle.topk_select(s, 1).tolist() == [tstar[h // G]]


# --------------------------------------------------------------------------- A5
def _sdpa(q, K, V, scale, mask=None):
    qt = torch.from_numpy(q)[None, None, None, :]
    Kt = torch.from_numpy(K)[None, None]
    Vt = torch.from_numpy(V)[None, None]
    m = None if mask is None else torch.from_numpy(mask)[None, None, None, :]
    return torch.nn.functional.scaled_dot_product_attention(qt, Kt, Vt, attn_mask=m, scale=scale)[0, 0, 0].numpy()


@pytest.mark.parametrize("N", [1, 2, 3, 17, 256, 512])
@pytest.mark.parametrize("D", [8, 128])
@pytest.mark.parametrize("G", [1, 4])
def test_dense_equals_torch_sdpa_and_full_index_sparse(N, D, G):
    """AC1 + S:136: sparse over I = [0..N) with unit weights equals dense;
    dense equals torch SDPA in float64; lse equals torch.logsumexp of the logits."""
    rng = np.random.default_rng(N * 1000 + D + G)
    Hkv = 2
    q = rng.standard_normal((1, Hkv * G, D))
    K = rng.standard_normal((1, N, Hkv, D))
    V = rng.standard_normal((1, N, Hkv, D))
    inp = _inputs_from_logical(K, V, q, [N], page_size=16)
    scale = 1.0 / math.sqrt(D)
    o, lse = oracle.dense_decode(inp, scale)
    sp = oracle.sparse_decode(inp, 1.0, scale, mode="exact")   # S=1 -> k = N
    for h in range(Hkv * G):
        g = h // G
        ref = _sdpa(q[0, h], K[0, :, g], V[0, :, g], scale)
        np.testing.assert_allclose(o[0, h], ref, rtol=1e-12, atol=1e-12)
        ref_lse = torch.logsumexp(torch.from_numpy(scale * K[0, :, g] @ q[0, h]), 0).item()
        assert abs(lse[0, h] - ref_lse) < 1e-12
        assert sp.idx[0][h].tolist() == list(range(N))
        np.testing.assert_allclose(sp.o[0, h], o[0, h], rtol=1e-12, atol=1e-13)


def test_sparse_equals_masked_sdpa():
    """sparse attention over I equals SDPA with a boolean mask built from I."""
    rng = np.random.default_rng(2)
    N, D = 256, 128
    q = rng.standard_normal((1, 4, D))
    K = rng.standard_normal((1, N, 1, D))
    V = rng.standard_normal((1, N, 1, D))
    inp = _inputs_from_logical(K, V, q, [N], page_size=16)
    res = oracle.sparse_decode(inp, 2.0, 0.09, mode="exact")
    for h in range(4):
        mask = np.zeros(N, dtype=bool)
        mask[res.idx[0][h]] = True
        ref = _sdpa(q[0, h], K[0, :, 0], V[0, :, 0], 0.09, mask)
        np.testing.assert_allclose(res.o[0, h], ref, rtol=1e-12, atol=1e-12)
        assert len(res.idx[0][h]) == 128


def test_attend_closed_forms():
    rng = np.random.default_rng(4)
    D = 16
    q = rng.standard_normal(D)
    K = rng.standard_normal((9, D))
    V = rng.standard_normal((9, D))
    # S:127 N=1 -> the value row, lse = its logit
    o, lse = oracle.attend(q, K[:1], V[:1], 0.3)
    assert np.array_equal(o, V[0]) and abs(lse - 0.3 * K[0] @ q) < 1e-15
    # S:128 identical keys -> mean of V, lse = s + log N
    Kc = np.repeat(K[:1], 9, axis=0)
    o, lse = oracle.attend(q, Kc, V, 0.3)
    np.testing.assert_allclose(o, V.mean(0), rtol=1e-13, atol=1e-14)
    assert abs(lse - (0.3 * K[0] @ q + math.log(9))) < 1e-12
    # dominant key concentrates the softmax
    Kd = K.copy()
    Kd[4] = 40.0 * q / np.linalg.norm(q)
    o, _ = oracle.attend(q, Kd, V, 1.0)
    np.testing.assert_allclose(o, V[4], atol=1e-3)
    # V = ones -> o = 1: attention weights sum to one
    o, _ = oracle.attend(q, K, np.ones_like(V), 0.7)
    np.testing.assert_allclose(o, 1.0, rtol=1e-14)


def test_weights_are_multiplicities():
    """Integer weights w_i = n_i equal unweighted attention over the multiset with
    row i repeated n_i times (w multiplies exp(s) in numerator and denominator,
    S:133).  Scaling all weights by c leaves o unchanged and shifts lse by log c."""
    rng = np.random.default_rng(9)
    D = 12
    q = rng.standard_normal(D)
    K = rng.standard_normal((6, D))
    V = rng.standard_normal((6, D))
    n = np.array([1, 3, 2, 5, 1, 4])
    o_w, lse_w = oracle.attend(q, K, V, 0.5, n.astype(float))
    o_m, lse_m = oracle.attend(q, np.repeat(K, n, axis=0), np.repeat(V, n, axis=0), 0.5)
    np.testing.assert_allclose(o_w, o_m, rtol=1e-13, atol=1e-14)
    assert abs(lse_w - lse_m) < 1e-13
    o_c, lse_c = oracle.attend(q, K, V, 0.5, 7.0 * n)
    np.testing.assert_allclose(o_c, o_w, rtol=1e-13, atol=1e-14)
    assert abs(lse_c - lse_w - math.log(7.0)) < 1e-13
    with pytest.raises(ValueError):
        oracle.attend(q, K, V, 0.5, np.array([1, 0, 1, 1, 1, 1.0]))


def test_attend_permutation_and_shift_invariance():
    """permuting I leaves (o, lse) unchanged; adding u to every key with
    u orthogonal to q leaves the logits and the output unchanged."""
    rng = np.random.default_rng(12)
    D = 32
    q = rng.standard_normal(D)
    K = rng.standard_normal((20, D))
    V = rng.standard_normal((20, D))
    o, lse = oracle.attend(q, K, V, 0.2)
    p = rng.permutation(20)
    o2, lse2 = oracle.attend(q, K[p], V[p], 0.2)
    np.testing.assert_allclose(o2, o, rtol=1e-13, atol=1e-14)
    u = rng.standard_normal(D)
    u -= (u @ q) / (q @ q) * q
    o3, lse3 = oracle.attend(q, K + u, V, 0.2)
    np.testing.assert_allclose(o3, o, rtol=1e-12, atol=1e-13)
    assert abs(lse3 - lse) < 1e-12


# --------------------------------------------------------------------------- merge
def test_lse_merge_any_chunking_equals_whole():
    rng = np.random.default_rng(13)
    D = 24
    q = rng.standard_normal(D)
    K = 2.0 * rng.standard_normal((100, D))
    V = rng.standard_normal((100, D))
    o, lse = oracle.attend(q, K, V, 0.4)
    for parts in (1, 2, 5, 13):
        cuts = np.sort(rng.choice(np.arange(1, 100), parts - 1, replace=False))
        chunks = np.split(np.arange(100), cuts)
        po, pl = zip(*[oracle.attend(q, K[c], V[c], 0.4) for c in chunks])
        # include an empty part (lse = -inf) to pin the empty-shard guard
        po = list(po) + [np.zeros(D)]
        pl = list(pl) + [-np.inf]
        mo, ml = oracle.lse_merge(np.stack(po), np.array(pl))
        np.testing.assert_allclose(mo, o, rtol=1e-12, atol=1e-13)
        assert abs(ml - lse) < 1e-12


@pytest.mark.parametrize("dist", ["iid", "dup", "equal"])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 7])
def test_seqshard_equals_unsharded(dist, P):
    case = workloads.make_case(2, 8, 2, [97, 64], D=32, seed=21 + P, dist=dist, C=8)
    inp = oracle.from_case(case)
    ref = oracle.sparse_decode(inp, 5.0, 0.17, mode="sketch")
    idx, o, lse = oracle.seqshard_decode(inp, 5.0, 0.17, P, mode="sketch")
    for b in range(2):
        for h in range(8):
            assert idx[b][h].tolist() == ref.idx[b][h].tolist()
    np.testing.assert_allclose(o, ref.o, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(lse, ref.lse, rtol=1e-12, atol=1e-12)


def test_equal_keys_select_lowest_indices_end_to_end():
    case = workloads.make_case(2, 4, 1, [40, 23], D=16, seed=2, dist="equal", dtype=torch.float32)
    inp = oracle.from_case(case)
    for mode in ("exact", "sketch"):
        res = oracle.sparse_decode(inp, 4.0, 0.25, mode=mode)
        for b, N in enumerate([40, 23]):
            k = oracle.budget_k(4.0, N)
            for h in range(4):
                assert res.idx[b][h].tolist() == list(range(k))
                # equal keys -> uniform weights over the chosen rows
                V = inp.values(b, 0)[:k]
                np.testing.assert_allclose(res.o[b, h], V.mean(0), rtol=1e-12, atol=1e-12)


# --------------------------------------------------------------------------- NEXT-1 / NEXT-2
def test_sink_local_heavy_density_ac8():
    """AC8: sink=local=128, h=0.20, N=20000 -> 4205 rows (0.2102);
    h=0.02 -> 0.0325; N <= sink+local -> every token."""
    s = np.random.default_rng(0).standard_normal(20000)
    I = oracle.sink_local_heavy_select(s, 128, 128, 0.20)
    assert I.size == 4205 and abs(I.size / 20000 - 0.2102) < 1e-4
    assert set(range(128)) <= set(I.tolist()) and set(range(20000 - 128, 20000)) <= set(I.tolist())
    I2 = oracle.sink_local_heavy_select(s, 128, 128, 0.02)
    assert abs(I2.size / 20000 - 0.0325) < 1e-4
    assert oracle.sink_local_heavy_select(s[:200], 128, 128, 0.5).tolist() == list(range(200))
    # Fig 2c absolute form: 64 sinks + K best of the rest
    I3 = oracle.sink_local_heavy_select(s, 64, 0, k_abs=16)
    assert I3.size == 80 and set(range(64)) <= set(I3.tolist())


def test_stochastic_limits_and_unbiasedness():
    """S:238-241 / AC9."""
    rng = np.random.default_rng(5)
    N = 1024
    s = rng.standard_normal(N)
    # sample_count = |R| -> everything with weight 1
    idx, w = oracle.stochastic_select(s, 10, N, rng.random(N))
    assert idx.tolist() == list(range(N)) and np.all(w == 1.0)
    # sample_count = 0 -> plain top-k
    idx, w = oracle.stochastic_select(s, 10, 0, rng.random(N))
    assert idx.tolist() == oracle.topk_select(s, 10).tolist()
    # unbiased denominator over 10,000 resamples within 1%
    m = s.max()
    exact = np.exp(s - m).sum()
    acc = 0.0
    for _ in range(10000):
        idx, w = oracle.stochastic_select(s, 16, 64, rng.random(N))
        acc += (w * np.exp(s[idx] - m)).sum()
    assert abs(acc / 10000 - exact) / exact < 0.01
