"""Test-only alias: `import kgdist` resolves to paper_2201_02791_b200.

Used by tools/ref_suite.sh to run the reference's own test suite
(/root/reference/pkg/tests, copied to the git-ignored baseline/_ref/) against
the drop-in package. Every `kgdist.<module>` name is the package's module
object, so `from kgdist.model import X` binds our implementation. The
reference CLI (out of scope for the hot path) is loaded from its own source
copy next to the tests when present, on top of the aliased modules.
"""

import importlib
import importlib.util
import os
import sys

import paper_2201_02791_b200 as _pkg
from paper_2201_02791_b200 import *  # noqa: F401,F403

for _name in ("errors", "graph", "partition", "sampler", "model", "trainer", "evaluate", "io"):
    sys.modules[f"kgdist.{_name}"] = importlib.import_module(f"paper_2201_02791_b200.{_name}")
    globals()[_name] = sys.modules[f"kgdist.{_name}"]

_cli = os.environ.get("KGDIST_REF_CLI")
if _cli and os.path.isfile(_cli):
    _spec = importlib.util.spec_from_file_location("kgdist.cli", _cli)
    _mod = importlib.util.module_from_spec(_spec)
    sys.modules["kgdist.cli"] = _mod
    _spec.loader.exec_module(_mod)
    cli = _mod

__version__ = _pkg.__version__
