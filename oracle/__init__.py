"""SDRT CPU oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of the Spectral Difference
Raviart-Thomas (SDRT) semi-discrete residual and classical RK4 integration, written
from /root/reference/PAPER.md (arXiv 2105.08632):

  * reference elements and point sets      PAPER.md App. A  (lines 2325-2816)
  * RT / solution bases and Vandermondes   PAPER.md §2.1    (lines 192-248)
  * Appendix-B operator matrices           PAPER.md App. B  (lines 2828-2935)
  * residual pipeline                      PAPER.md §2.1    (lines 268-350)
  * physics (lin. adv/diff, Euler, NS)     PAPER.md §3, §5  (lines 464-496, 1658-1678,
                                                             1909-1935, 2012-2047)

Operators are built in mpmath (>= 30 significant digits) and rounded once to fp64;
the residual is the dense Appendix-B matrix form evaluated with numpy fp64.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything in this package. The product path
(``paper_2105_08632_b200``) shares no code with it.

Functions without an independent pin say "parity unpinned" in their docstring
(see DESIGN.md §Oracle pins).
"""
