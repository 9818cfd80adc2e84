"""CPU oracle for the rlpyt (arXiv 1909.01500) replay + return-estimation hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1909_01500_b200``) never imports it and
shares no code with it: no kernels, helpers, constants or table generators.

Every function is a plain, slow, obviously-correct definition in float64,
Python ``int`` (exact) or mpmath, following the passage it cites:

  P:n  -> /root/reference/PAPER.md line n (the paper, LaTeX source)
  S:n  -> /root/reference/SPEC.md line n (a CPU-program spec written from the paper)
  §8c #k -> the k-th reading in SURVEY.md §8(c) / DESIGN.md "Readings"

Parity pins (tests/test_oracle_*.py) tie each function to something other than
itself: worked examples printed in SPEC.md, closed forms, exact rational
arithmetic, brute force on tiny inputs and known-answer vectors.  No function in
this package is "parity unpinned".
"""
