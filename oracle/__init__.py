"""CPU oracle for the wavelet-tree hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package, and only as
the checker or the timed CPU baseline.  The product package
(``paper_2505_03372_b200``) never imports it.

Parity pinned: ``tests/golden/`` holds vectors produced by running the real
reference (``wtindex`` 0.1.0 under /root/reference/pkg/src) through
``tests/golden/make_golden.py``; ``tests/test_oracle_golden.py`` checks this
restatement against every one of them.
"""

from .wt_oracle import *  # noqa: F401,F403
