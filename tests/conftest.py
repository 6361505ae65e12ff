import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "reference_golden.json"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    return json.loads(GOLDEN.read_text())


@pytest.fixture(scope="session")
def reference_pkg():
    """The unmodified reference package, when this host has it (build container)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference tree not present on this host")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.append(str(REFERENCE_SRC))
    import tunescape

    return tunescape
