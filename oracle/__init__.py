"""fp64 CPU oracle for the DiffVC-RT decode hot path.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  It shares no code with ``paper_2601_20564_b200`` (the product) and
never imports it.
"""
from .oracle import *  # noqa: F401,F403
