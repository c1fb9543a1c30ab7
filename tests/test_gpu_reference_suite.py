"""The reference's own test files for the path, unchanged, against the
drop-in (`import remlot` -> paper_1704_05132_b200/compat/remlot): model,
plan, vnd, gvns, oracle and the acceptance criteria on the path (C1 oracle
equivalence, C3-C6).  tools/ref_suite.sh stages them from /root/reference
into the git-ignored baseline/_ref/tests in the build container (the
reference does not exist on the GPU box); this test runs whatever was
staged and skips when nothing was."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

STAGED = os.path.join(ROOT, "baseline", "_ref", "tests")


@pytest.mark.skipif(not os.path.exists(os.path.join(STAGED, "test_vnd.py")),
                    reason="reference tests not staged (tools/ref_suite.sh stage)")
def test_reference_suite_passes_on_drop_in():
    out = subprocess.run(["bash", os.path.join(ROOT, "tools", "ref_suite.sh"), "run"],
                         capture_output=True, text=True, timeout=1800, cwd=ROOT)
    tail = out.stdout[-3000:] + out.stderr[-2000:]
    assert out.returncode == 0, tail
    m = re.search(r"(\d+) passed", out.stdout)
    assert m and int(m.group(1)) >= 99, tail
    assert "failed" not in out.stdout.splitlines()[-1], tail
    for crit in (1, 3, 4, 5, 6):
        if os.path.exists(os.path.join(STAGED, "test_acceptance.py")):
            assert f"ACCEPTANCE {crit} PASS" in out.stdout, tail
