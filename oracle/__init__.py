"""CPU oracle for the all-to-all spectral connectivity path (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import this package, and only as the checker / CPU baseline.  The product
path (``paper_2303_03279_b200``) never imports it.

Parity is pinned: ``tests/test_oracle.py`` checks this restatement against
golden vectors produced by running the unmodified reference
(``tests/golden/make_golden.py``) and against the reference's own on-disk
fixtures (``pkg/frontend/tests/fixtures/threshold_*.json``).
"""
from .connstream_oracle import *  # noqa: F401,F403
