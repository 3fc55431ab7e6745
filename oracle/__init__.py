"""The fp64 CPU oracle (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_2403_08551_b200`` never imports it and shares no code
with it.  See ``oracle/gio.cpp`` for what it computes and the paper passages
each function follows.
"""
from .gio import *  # noqa: F401,F403
