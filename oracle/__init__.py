"""CPU oracle for the Fermat path solver — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU baseline. The product path (``paper_2510_16172_b200``) never
imports it and has no CPU fallback.

Pinning: ``tests/test_oracle_pin.py`` checks every function here against the
golden vectors in ``tests/golden/`` that ``tests/golden/make_golden.py``
produced by importing the reference package (/root/reference/pkg/src) in the
build container.
"""
