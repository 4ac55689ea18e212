"""Seeded synthetic decode workloads (inputs only).

This module is shared by the oracle-side tests and the CUDA-side tests/bench.
It holds NO arithmetic of the method (no scores, no selection, no softmax):
it only draws random numbers, rounds them to the storage dtype and lays them
out as a paged KV cache.  See DESIGN.md "Input recipe".
"""
from .gen import DecodeCase, make_case, CONFIGS, config_case  # noqa: F401
