"""CPU oracles for the sFFT4.0 hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package, and
only as the checker or the CPU baseline.  The product package
``paper_2011_05698_b200`` never imports it.
"""
from .oracle import Oracle, OracleError, available, load  # noqa: F401
