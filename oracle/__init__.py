"""ORACLE — TEST INFRASTRUCTURE ONLY.

A CPU restatement of the reference solver's per-iteration hot path
(arXiv 2412.19027 / ``conic_ipm`` in /root/reference), used exclusively as

* the parity checker in ``tests/`` and ``__graft_entry__.smoke()``, and
* the CPU baseline leg of ``bench.py`` (``cpu_baseline`` / ``--impl reference``).

The product package (``paper_2412_19027_b200``) never imports, links or
executes anything here; its CUDA path fails loudly when the native library
is missing.  Parity of this oracle is pinned against golden fixtures produced
by the unmodified reference (``tests/golden/make_golden.py``).
"""
from .ipm import OracleSolver, oracle_solve  # noqa: F401
