"""Loading of the golden fixtures (tests/golden/, produced by make_golden.py from the reference)
and the parity comparison shared by the oracle tests and the GPU tests."""
from __future__ import annotations

import ast
import hashlib
import json
from pathlib import Path

import numpy as np

from paper_1802_08557_b200 import workloads

GOLDEN = Path(__file__).resolve().parent / "golden"
OBJ_RTOL = 1e-9   # north star: objective within 1e-9 relative (reference sums c.x with BLAS ddot)


def obj_rel_err(got, want) -> np.ndarray:
    """True relative error |got - want| / |want| (no absolute floor).  A zero reference
    objective must be matched exactly (rel = inf otherwise, 0 when equal)."""
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    diff = np.abs(got - want)
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(diff == 0, 0.0, diff / np.abs(want))
    return rel


def obj_close(got, want) -> bool:
    return bool((obj_rel_err(got, want) <= OBJ_RTOL).all())


def _limits(d: dict) -> dict:
    return dict(max_iterations=d["max_iterations"], anti_cycling=d["anti_cycling"],
                degenerate_pivot_limit=d["degenerate_pivot_limit"])


def json_records(name: str) -> list[dict]:
    recs = json.loads((GOLDEN / name).read_text())
    for r in recs:
        r["A"] = np.asarray(r["A"], np.float64).reshape(r["m"], r["n"])
        r["b"] = np.asarray(r["b"], np.float64)
        r["c"] = np.asarray(r["c"], np.float64)
        r["limits"] = _limits(r["limits"])
    return recs


def packed_names() -> list[str]:
    return sorted(p.stem for p in GOLDEN.glob("*.npz"))


def _sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def _call(expr: str):
    """Evaluate one ``workloads.<fn>(<literal args>)`` recipe call (no general eval)."""
    node = ast.parse(expr.strip(), mode="eval").body
    assert isinstance(node, ast.Call) and isinstance(node.func, ast.Attribute) \
        and getattr(node.func.value, "id", None) == "workloads", expr
    args = [ast.literal_eval(a) for a in node.args]
    kwargs = {k.arg: ast.literal_eval(k.value) for k in node.keywords}
    return getattr(workloads, node.func.attr)(*args, **kwargs)


def packed_fixture(stem: str) -> dict:
    """Inputs regenerated from the stored recipe (sha256-pinned) + reference outcomes."""
    z = np.load(GOLDEN / f"{stem}.npz", allow_pickle=False)
    recipe = str(z["recipe"])
    if ";" in recipe:  # support mode: polytope; directions
        first, second = recipe.split(";")
        A, b = _call(first)
        c = _call(second)
    else:
        A, b, c = (np.asarray(v, np.float64) for v in _call(recipe))
        if A.ndim == 2:
            A, b, c = A[None], b[None], c[None]
    assert _sha(A, b, c) == str(z["sha256"]), f"{stem}: regenerated inputs differ from the fixture's"
    return dict(A=A, b=b, c=c, shared=bool(z["shared"]), status=z["status"], objective=z["objective"],
                x=z["x"], it1=z["it1"], it2=z["it2"], recipe=recipe)


def compare(got: dict, want: dict, label: str = "") -> None:
    """Status, x and iteration counts exactly equal; objective within OBJ_RTOL (true relative)."""
    gs, ws = np.asarray(got["status"]), np.asarray(want["status"])
    bad = np.flatnonzero(gs != ws)
    assert bad.size == 0, f"{label}: status differs at {bad[:10]} (got {gs[bad[:10]]}, want {ws[bad[:10]]})"
    for key in ("it1", "it2"):
        g, w = np.asarray(got[key]), np.asarray(want[key])
        bad = np.flatnonzero(g != w)
        assert bad.size == 0, f"{label}: {key} differs at {bad[:10]} (got {g[bad[:10]]}, want {w[bad[:10]]})"
    opt = ws == 0
    gx, wx = np.asarray(got["x"])[opt], np.asarray(want["x"])[opt]
    bad = np.flatnonzero(~(gx == wx).all(axis=1)) if gx.size else np.array([], int)
    assert bad.size == 0, f"{label}: x differs on {bad.size} optimal LPs, first {np.flatnonzero(opt)[bad[:5]]}"
    go, wo = np.asarray(got["objective"])[opt], np.asarray(want["objective"])[opt]
    rel = obj_rel_err(go, wo)
    assert (rel <= OBJ_RTOL).all(), f"{label}: objective rel err {rel.max() if rel.size else 0}"


def box_records() -> list[dict]:
    return json.loads((GOLDEN / "box.json").read_text())


def box_arrays(rec: dict):
    lo = np.asarray(rec["lower"], np.float64)[None]
    hi = np.asarray(rec["upper"], np.float64)[None]
    d = np.asarray(rec["direction"], np.float64)[None]
    return lo, hi, d


def box_message(status: int, lo, hi) -> str | None:
    if status == 0:
        return None
    if status < 0:
        return "box bounds must be finite"
    j = status - 1
    return f"lower[{j}] = {lo[j]} > upper[{j}] = {hi[j]}"


def compare_box(value, point, status, rec: dict) -> None:
    """Points exact, values within OBJ_RTOL, errors with the reference's message."""
    lo, hi, _ = box_arrays(rec)
    want = rec["outcome"]
    if "error" in want:
        assert status != 0, rec["name"]
        assert box_message(int(status), lo[0], hi[0]) == want["error"], rec["name"]
        return
    assert status == 0, f"{rec['name']}: status {status}"
    assert np.array_equal(np.asarray(point), np.asarray(want["point"])), rec["name"]
    assert obj_close(value, want["value"]), rec["name"]
