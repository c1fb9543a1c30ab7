"""The ``remlot`` import alias (paper_1704_05132_b200/compat/remlot): code
written against the reference package resolves to the drop-in's modules.

SURVEY.md 8(b) API-compat checklist: the names of reference
pkg/src/remlot/__init__.py:3-20 on the path, ``remlot.vnd`` / ``remlot.gvns``
module paths (test_vnd.py:12, test_gvns.py:9), the ``_MIN_CHUNK`` attribute
monkeypatched by test_vnd.py:172.  tools/ref_suite.sh runs the reference's
own test files through this alias on a B200 (profiles/r01_reference_suite_b200.log).
"""
import importlib
import os
import sys

COMPAT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "paper_1704_05132_b200", "compat")

# reference pkg/src/remlot/__init__.py:3-20 minus the CLI bench/report
# emitters (BenchReport, BenchRow, BenchSuite, SchemeAggregate, default_suite,
# emit_csv, emit_markdown, format_cents, load_suite, run_bench: out of scope)
NAMES = """INFEASIBLE SCHEME_HYBRID SCHEME_MULTIWORKER SCHEME_PRODUCT_PARALLEL
SCHEME_SERIAL_VND SCHEMES GvnsResult SearchState SolverConfig gvns next_strength shake
solve_scheme worker_round GeneratorConfig Instance InstanceFormatError generate_instance
parse_instance serialize_instance validate_instance enumerate_optimal DecodedPlan SetupPlan
decode evaluate evaluate_product initial_solution DEFAULT_PARALLELISM MODE_PRODUCT_PARALLEL
MODE_SERIAL NEIGHBORHOOD_COUNT VND_MODES ImprovementDelta Move apply_delta best_neighbor
enumerate_neighbors vnd vnd_pass""".split()


def _remlot():
    if COMPAT not in sys.path:
        sys.path.insert(0, COMPAT)
    return importlib.import_module("remlot")


def test_alias_exports_reference_names():
    remlot = _remlot()
    missing = [n for n in NAMES if not hasattr(remlot, n)]
    assert not missing
    assert remlot.__version__ == "0.1.0"


def test_alias_submodules_are_the_drop_in_modules(monkeypatch):
    _remlot()
    impl_vnd = importlib.import_module("paper_1704_05132_b200.vnd")
    vnd_module = importlib.import_module("remlot.vnd")
    assert vnd_module is impl_vnd
    monkeypatch.setattr(vnd_module, "_MIN_CHUNK", 1)
    assert impl_vnd._MIN_CHUNK == 1
    from remlot.gvns import _worker_rng  # noqa: F401
    assert importlib.import_module("remlot.oracle").enumerate_optimal is not None
    assert vnd_module.VND_MODES == ("serial", "product-parallel")
