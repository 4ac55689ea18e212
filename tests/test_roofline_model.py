"""Byte model (SPEC.md:286-312 traffic_model) pinned to SPEC worked values."""
from paper_2605_24168_b200 import roofline as R


def test_spec_worked_values():
    assert R.gather_bytes_per_head(1, 1, 2622) == 1_342_464
    assert R.dense_bytes(1, 131072, 8) == 536_870_912
    assert R.dense_bytes(8, 32768, 8) == 1 << 30                          # S:458 (1 GiB cache)


def test_limits_and_ratios():
    # k = N without dedup costs G x dense (S:299 GQA amplification)
    assert R.gather_bytes_per_head(2, 32, 4096) == 4 * R.dense_bytes(2, 4096, 8)
    # G = 1: sparse/dense byte ratio is k/N exactly
    assert R.gather_bytes_per_head(1, 8, 1024) * 4 == R.dense_bytes(1, 4096, 8)
    # C=8 bf16 sketch is 1/16 of the dense key bytes
    assert R.indexer_bytes(1, 4096, 8) * 16 == R.dense_bytes(1, 4096, 8) // 2
    # union of G identical full sets is N
    assert abs(R.expected_union(1000, 1000, 4) - 1000) < 1e-9
    assert abs(R.expected_union(1000, 1, 1) - 1) < 1e-9


def test_cfg3_model_matches_survey():
    m = R.sparse_step_bytes(16, 32, 8, 131072, 2622)
    # 936.3 MB union / 956.7 MB per-head at cfg3
    assert abs(m["total_union"] / 1e6 - 936.3) < 0.5
    assert abs(m["total_per_head"] / 1e6 - 956.7) < 0.5
    assert m["indexer"] == 268_435_456
