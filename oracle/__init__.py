"""TEST INFRASTRUCTURE ONLY — the plain CPU oracle for arXiv 1511.07983.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package.
The product path (``paper_1511_07983_b200``) never imports it; the two share
no code.  See ``oracle/rk_oracle.cpp`` for the citations of every step.
"""
from .oracle import *  # noqa: F401,F403
