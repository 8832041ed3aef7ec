"""CPU oracle for arxiv/paper_2604_00028 (sequence-aware split policy for
low-head-count decode attention).

TEST INFRASTRUCTURE ONLY.  This package is the slow, obviously-correct CPU
statement of what the B200 path computes.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_2604_00028_b200``) never imports, links or executes anything here,
and this package never imports the product path: the two share no code.
Inputs come from ``synth/`` (seeded generators, no method arithmetic).

Modules
-------
``oracle.attention``  C-att / C-part / C-comb: fp64
                      decode attention over the bf16-exact inputs, per-split
                      partials, and the log-sum-exp combine.
``oracle.policy``     C-pol: tile geometry, the guarded FA3-style default
                      (P:L23), the efficiency loop, the paper's
                      sequence-aware cascade (Fig. 3) and the
                      split partition - pure Python integers.

Citations: P:Lnn = /root/reference/PAPER.md line nn (section / figure /
table given beside it); S:Lnn = /root/reference/SPEC.md line nn.  Readings of
silent or ambiguous passages are the C-amb-* items listed in DESIGN.md §3.

Parity status: every function here is pinned by ``tests/test_oracle_*.py``
(``-m "not gpu"``) against values the paper prints, closed forms, library
routines or brute force, EXCEPT the efficiency loop beyond its single-wave
closed form, which the paper references but never defines (P:L85, P:L106,
P:L157): "parity unpinned" by the paper for those cases.
"""

from . import attention, policy  # noqa: F401
