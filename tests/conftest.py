import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "reference: needs the read-only reference tree (build container only)")


try:
    import hypothesis

    hypothesis.settings.register_profile("default", max_examples=50, deadline=None,
                                         suppress_health_check=[hypothesis.HealthCheck.too_slow])
    hypothesis.settings.load_profile(os.environ.get("HYPOTHESIS_PROFILE", "default"))
except ImportError:  # pragma: no cover
    pass


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference package, imported read-only (skips where absent)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference tree not present (GPU box)")
    sys.path.insert(0, str(REFERENCE_SRC))
    import batchlp
    return batchlp
