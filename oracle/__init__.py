"""CPU fp64 oracle for sparse decode attention (arxiv 2605.24168).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this
package.  The product (`paper_2605_24168_b200`) never imports it and has no
CPU fallback.  The oracle shares no code with the CUDA path.
"""
from .sdoracle import *  # noqa: F401,F403
from .sdoracle import __all__  # noqa: F401
