"""INTEGRATION.md's ctypes stub (the binding a maintainer would add to batchlp) runs as
written against libblp.so and returns the same outcomes as the drop-in package."""
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _stub_source() -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    block = re.search(r"```python\n# batchlp/_blp.py.*?```", text, re.S).group(0)
    src = block.split("\n", 1)[1].rsplit("```", 1)[0]
    # the stub lives inside batchlp; here its relative imports resolve to the drop-in's model
    src = src.replace("from .model import", "from paper_1802_08557_b200.model import")
    return src.replace('"/path/to/paper_1802_08557_b200/libblp.so"', repr(str(ROOT / "paper_1802_08557_b200" / "libblp.so")))


def test_stub_parses():
    compile(_stub_source(), "INTEGRATION.md:_blp.py", "exec")


@pytest.mark.gpu
def test_stub_matches_drop_in():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1802_08557_b200 import SolverLimits, batch_solve, standard_form, workloads
    ns: dict = {}
    exec(_stub_source(), ns)
    A, b, c = workloads.afiro_arrays(300, seed=12)
    lps = [standard_form(c[k], A[k], b[k]) for k in range(len(c))]
    got = ns["solve_many"](lps, SolverLimits())
    want = batch_solve(lps).outcomes
    for g, w in zip(got, want):
        assert g.status == w.status and g.iterations_phase1 == w.iterations_phase1
        assert g.iterations_phase2 == w.iterations_phase2
        if w.primal_point is not None:
            assert np.array_equal(g.primal_point, w.primal_point) and g.objective_value == w.objective_value
