"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct NumPy (fp64) implementation of what the
Nacrith hot path computes (arXiv 2602.19626, /root/reference/PAPER.md), written
from the paper and SURVEY.md §8(c).  Each function cites the passage it follows
as ``P:<line>`` or ``S:<line>`` or a SURVEY.md D-reading.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_2602_19626_b200`` + ``libnc.so``) never imports, links or executes
anything here, and this package imports nothing from the product path.  The
two share only the seeded input generators in ``synth/`` (no method
arithmetic there).

Parity status per function is listed in DESIGN.md §"Oracle pins".
Functions whose result the paper cannot pin (bpb on real data) say
"parity unpinned" in their docstring.
"""
