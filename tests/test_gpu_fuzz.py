"""A fixed, seeded slice of scripts/fuzz_gpu.py: random shapes (1..300 rows/columns), LP
recipes, solver limits, support mode and forced kernel families, every case against the
oracle (status, x, iterations exact; objective to 1e-9 relative)."""
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("seed", [11, 12])
def test_fuzz_slice(seed):
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "scripts"))
    import fuzz_gpu
    msgs = []
    cases, lps, bad = fuzz_gpu.run(seed, cases=40, log=msgs.append)
    assert cases == 40 and bad == 0, "\n".join(msgs[:5])
