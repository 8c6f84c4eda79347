"""CPU oracle for the SAECache hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package.
The product path (``paper_2605_18825_b200``) never imports it and shares no
code with it.  See ``oracle/sae_oracle.cpp`` for the implementation and its
citations into /root/reference/PAPER.md.
"""
from .oracle import *  # noqa: F401,F403
