"""``remlot`` import alias of the B200 drop-in (reference pkg/src/remlot/__init__.py).

Put ``paper_1704_05132_b200/compat`` on ``sys.path`` and code written against
the reference package -- ``import remlot``, ``importlib.import_module(
"remlot.vnd")``, ``from remlot.gvns import _worker_rng`` -- runs on the GPU
path unchanged.  The submodules are the drop-in's own module objects (not
copies), so ``monkeypatch.setattr(remlot.vnd, "_MIN_CHUNK", 1)`` patches what
the drop-in reads.  The reference's CLI and bench/report emitters
(``remlot.cli``, ``remlot.bench``) are out of scope and are not
aliased.
"""
import importlib
import sys

import paper_1704_05132_b200 as _impl
from paper_1704_05132_b200 import *  # noqa: F401,F403  (the reference's public names)

__version__ = _impl.__version__

# submodule name in the reference -> the drop-in's module (as in the
# reference, the package attribute ``remlot.vnd`` stays the function)
for _name, _mod in (("vnd", "vnd"), ("gvns", "gvns"), ("plan", "plan"), ("model", "model"),
                    ("oracle", "exhaustive")):
    sys.modules[__name__ + "." + _name] = importlib.import_module(_impl.__name__ + "." + _mod)
del _name, _mod
