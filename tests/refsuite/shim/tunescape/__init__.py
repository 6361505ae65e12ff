"""Test-only alias: ``import tunescape`` resolves to this B200 build.

With ``tests/refsuite/shim`` on ``PYTHONPATH``, the reference's own test
suite (``/root/reference/pkg/tests``, run unmodified by
``tests/test_reference_suite.py``) imports ``tunescape.<module>`` and gets
``paper_2407_11488_b200.<module>``; ``python -m tunescape`` runs our CLI.
No reference code is imported.
"""

import importlib
import sys

_pkg = importlib.import_module("paper_2407_11488_b200")
for _name in ("errors", "expressions", "paramspace", "measure", "store", "strategies", "landscape", "cli"):
    _mod = importlib.import_module(f"paper_2407_11488_b200.{_name}")
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod

from paper_2407_11488_b200 import *  # noqa: E402,F401,F403
