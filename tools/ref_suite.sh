#!/bin/bash
# Run the reference's own test suite, unchanged, against the B200 drop-in.
#
#   tools/ref_suite.sh stage   # here (needs /root/reference): copy the
#                              # reference's tests into baseline/_ref/tests
#                              # (git-ignored, travels to the GPU box)
#   tools/ref_suite.sh run     # on a B200 box: pytest those files with
#                              # `import remlot` resolved to the drop-in
#                              # (paper_1704_05132_b200/compat/remlot)
#
# Staged: the model / plan / vnd / gvns / oracle tests, the acceptance
# criteria, and their helpers (conftest.py, reference.py).  Not staged:
# test_cli.py and test_bench.py (the reference's CLI and bench/report
# emitters, out of scope).  test_acceptance.py imports the
# emitters at module level: tools/ref_acceptance_stub.py binds placeholders
# and the criteria off the hot path (C2 report tallies, C7 informational
# speedup, C8 report bolding) are deselected; C1 and C3-C6 run.
set -e
root=$(cd "$(dirname "$0")/.." && pwd)
dst=$root/baseline/_ref/tests
case "$1" in
stage)
  src=/root/reference/pkg/tests
  mkdir -p "$dst"
  rm -rf "$dst"
  mkdir -p "$dst"
  for f in conftest.py reference.py test_model.py test_plan.py test_vnd.py test_gvns.py \
           test_oracle.py test_acceptance.py; do
    cp "$src/$f" "$dst/$f"
  done
  echo "staged $(ls "$dst" | wc -l) files into $dst"
  ;;
run)
  shift
  cd "$root/baseline/_ref"
  PYTHONPATH=$root/paper_1704_05132_b200/compat:$root:$root/tools${PYTHONPATH:+:$PYTHONPATH} \
    python -m pytest tests -q -p no:cacheprovider -p ref_acceptance_stub -s \
      --deselect tests/test_acceptance.py::test_criterion_2_scheme_quality_ordering \
      --deselect tests/test_acceptance.py::test_criterion_7_product_parallel_speedup \
      --deselect tests/test_acceptance.py::test_criterion_8_report_bold_fidelity "$@"
  ;;
*)
  echo "usage: $0 stage|run [pytest args]" >&2
  exit 2
  ;;
esac
