"""AdaHOP CPU oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct numpy (fp64 unless stated) implementation of what
the AdaHOP hot path computes, written from the paper (arXiv 2604.02525,
/root/reference/PAPER.md, cited as P:<line>). It shares no code with the CUDA path
(``paper_2604_02525_b200``) and imports nothing from it.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product path never does.

Parity status per function: every public function
is pinned by at least one ``-m "not gpu"`` test in tests/test_oracle_*.py against
a closed form, an invariant, a golden fixture from the paper, or brute force.
No function is "parity unpinned".
"""
from .adahop_oracle import *  # noqa: F401,F403
