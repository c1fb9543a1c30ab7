"""pytest plugin for tools/ref_suite.sh (test infrastructure, not product).

The reference's test_acceptance.py imports its bench/report emitters
(BenchReport, BenchRow, emit_markdown) at module level; they are out of scope
for the drop-in.  This plugin binds placeholders that raise if
called, so the criteria on the hot path (C1 oracle equivalence, C3 exact
reduction, C4 mode/run determinism, C5 feasibility, C6 monotone descent)
can run against the drop-in; C2/C7/C8 (report tallies, informational
speedup, report bolding) are deselected by ref_suite.sh.
"""
import remlot


def _out_of_scope(*_a, **_k):
    raise NotImplementedError("bench/report emitters are out of scope for the B200 drop-in")


for _name in ("BenchReport", "BenchRow", "emit_markdown"):
    if not hasattr(remlot, _name):
        setattr(remlot, _name, _out_of_scope)
