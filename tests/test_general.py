"""General-form ingest vs the reference: MPS reader, lowering to
GeneralLP, standardize + VariableMap, and the batched recovery of solver outputs.

Golden records (tests/golden/make_general_golden.py) hold the reference's own results;
lowered arrays must match bit for bit (every lowered coefficient is a copy, a
negation or the same numpy dot), warnings and error messages verbatim.
"""
import json
import warnings

import numpy as np
import pytest

from golden_io import GOLDEN
from paper_1802_08557_b200 import (BatchArrays, GeneralLP, InfeasibleBounds, ParseError, UnsupportedFeature,
                                   VariableMap, lower_to_general, parse_mps, recover_batch, standardize,
                                   standardize_batch)
from paper_1802_08557_b200.general import Sense


def _records(name):
    return json.loads((GOLDEN / name).read_text())["records"]


def _bits_equal(got, want) -> bool:
    g = np.asarray(got, dtype=np.float64).ravel()
    w = np.asarray(want, dtype=np.float64).ravel()
    return g.shape == w.shape and np.array_equal(g.view(np.int64), w.view(np.int64))


def _model_dict(m) -> dict:
    return dict(name=m.name, sense=m.objective_sense.value, objective_row=m.objective_row,
                row_types=m.row_types, row_order=m.row_order, column_order=m.column_order,
                entries=[[k[0], k[1], float(v)] for k, v in m.entries.items()],
                rhs=[[k, float(v)] for k, v in m.rhs.items()],
                ranges=[[k, float(v)] for k, v in m.ranges.items()],
                bounds=[[t, v, None if x is None else float(x)] for t, v, x in m.bounds],
                integral=sorted(m.integral_columns))


def _check_general(g, want, tag):
    assert g.sense.value == want["sense"], tag
    assert [r.value for r in g.relations] == want["relations"], tag
    assert list(g.row_names) == want["row_names"] and list(g.col_names) == want["col_names"], tag
    for key in ("c", "rows", "rhs", "lower", "upper"):
        assert _bits_equal(getattr(g, key), want[key]), (tag, key)


def _general_from(rec) -> GeneralLP:
    k, n = rec["k"], rec["n"]
    return GeneralLP.build(rec["sense"], rec["c"], np.asarray(rec["rows"]).reshape(k, n), rec["relations"],
                           rec["rhs"], rec["lower"], rec["upper"], rec["row_names"], rec["col_names"])


def _check_lowered(g, want, tag):
    if "error" in want:
        with pytest.raises(InfeasibleBounds) as err:
            standardize(g)
        assert str(err.value) == want["message"], tag
        return
    lp, vm = standardize(g)
    assert (lp.m, lp.n) == (want["m"], want["n"]), tag
    for key in ("A", "b", "c"):
        assert _bits_equal(getattr(lp, key), want[key]), (tag, key)
    v = want["vmap"]
    assert vm.sense.value == v["sense"] and vm.num_standard_vars == v["num_standard_vars"], tag
    assert _bits_equal([vm.offset], [v["offset"]]) and _bits_equal(vm.shift, v["shift"]), tag
    assert vm.plus_col.tolist() == v["plus_col"] and vm.minus_col.tolist() == v["minus_col"], tag


def test_mps_records_match_reference():
    recs = _records("mps.json")
    assert sum(r["name"].startswith("fixture:") for r in recs) == 8
    for rec in recs:
        tag = rec["name"]
        with warnings.catch_warnings(record=True) as caught:
            warnings.simplefilter("always")
            try:
                model = parse_mps(rec["text"])
                err = None
            except ParseError as e:
                model, err = None, e
        assert [str(w.message) for w in caught] == rec["parse_warnings"], tag
        if "parse_error" in rec:
            assert err is not None and str(err) == rec["parse_error"] and err.line_no == rec["line_no"], tag
            continue
        assert err is None, (tag, err)
        assert _model_dict(model) == rec["model"], tag
        with warnings.catch_warnings(record=True) as caught:
            warnings.simplefilter("always")
            try:
                g = lower_to_general(model)
                lerr = None
            except UnsupportedFeature as e:
                g, lerr = None, e
        assert [str(w.message) for w in caught] == rec["lower_warnings"], tag
        if "lower_error" in rec:
            assert lerr is not None and str(lerr) == rec["lower_error"], tag
            continue
        _check_general(g, rec["general"], tag)
        _check_lowered(g, rec["lowered"], tag)


def test_general_records_lower_like_reference():
    for rec in _records("general.json"):
        g = _general_from(rec["general"])
        _check_general(g, rec["general"], rec["name"])
        _check_lowered(g, rec["lowered"], rec["name"])


def _std_arrays(recs):
    """The reference's standard-form solver outputs as one packed BatchArrays."""
    n = max(r["lowered"]["n"] for r in recs)
    B = len(recs)
    status = np.array([r["lowered"]["std"]["status"] for r in recs], np.int8)
    obj = np.array([np.nan if r["lowered"]["std"]["objective"] is None else r["lowered"]["std"]["objective"]
                    for r in recs])
    x = np.zeros((B, n))
    for k, r in enumerate(recs):
        if r["lowered"]["std"]["x"] is not None:
            x[k, :r["lowered"]["n"]] = r["lowered"]["std"]["x"]
    it = np.zeros(B, np.int32)
    return BatchArrays(status=status, objective=obj, x=x, iterations_phase1=it, iterations_phase2=it)


def test_recover_batch_equals_reference_recovery():
    """recover_batch on the reference's own standard-form outputs == its recover_outcome, bitwise."""
    recs = [r for r in _records("general.json") if "error" not in r["lowered"]]
    fam = [r for r in recs if r["name"].startswith("family:")]
    for group in (fam, recs):
        maps = [standardize(_general_from(r["general"]))[1] for r in group]
        got = recover_batch(maps, _std_arrays(group))
        for k, r in enumerate(group):
            want = r["lowered"]["outcome"]
            assert got.status[k] == want["status"], r["name"]
            if want["status"] == 0:
                assert _bits_equal([got.objective[k]], [want["objective"]]), r["name"]
                assert _bits_equal(got.x[k], want["x"]), r["name"]
                o = got.outcome(k)
                assert o.objective_value == got.objective[k] and o.primal_point is got.x[k]
            else:
                assert np.isnan(got.objective[k]) and got.outcome(k).primal_point is None


def test_standardize_batch_packs_same_shape_family():
    recs = [r for r in _records("general.json") if r["name"].startswith("family:")]
    glps = [_general_from(r["general"]) for r in recs]
    A, b, c, maps = standardize_batch(glps)
    assert A.shape == (len(recs), recs[0]["lowered"]["m"], recs[0]["lowered"]["n"])
    for k, r in enumerate(recs):
        assert _bits_equal(A[k], r["lowered"]["A"]) and _bits_equal(b[k], r["lowered"]["b"])
        assert _bits_equal(c[k], r["lowered"]["c"])
    assert len({vm.layout_key() for vm in maps}) == 1
    mixed = [glps[0], GeneralLP.build("max", [1.0], [[1.0]], ["<="], [1.0])]
    with pytest.raises(ValueError, match="lowers to"):
        standardize_batch(mixed)


def test_general_lp_validation_messages():
    with pytest.raises(ValueError, match=r"rows has shape \(1, 2\), expected \(1, 1\)"):
        GeneralLP(Sense.MAX, np.ones(1), np.ones((1, 2)), ("<=",), np.ones(1), np.zeros(1), np.ones(1))
    with pytest.raises(ValueError, match="2 relations for 1 rows"):
        GeneralLP.build("max", [1.0], [[1.0]], ["<=", "<="], [1.0])
    with pytest.raises(ValueError, match="bounds must both have length n"):
        GeneralLP.build("max", [1.0], [[1.0]], ["<="], [1.0], lower=[0.0, 0.0])
    with pytest.raises(ValueError, match="unique"):
        GeneralLP.build("max", [1.0, 1.0], [[1.0, 1.0]], ["<="], [1.0], col_names=("a", "a"))
    with pytest.raises(InfeasibleBounds, match="variable 'x0': lower 2.0 > upper 1.0"):
        standardize(GeneralLP.build("max", [1.0], np.zeros((0, 1)), [], [], lower=[2.0], upper=[1.0]))


def test_variable_map_recovery_rules():
    vm = VariableMap(sense=Sense.MIN, offset=1.5, shift=np.array([0.0, 2.0]), plus_col=np.array([0, 2]),
                     minus_col=np.array([1, -1]), num_standard_vars=3)
    assert vm.recover_point(np.array([0.0, 2.5, 1.0])).tolist() == [-2.5, 3.0]
    assert vm.recover_objective(4.0) == -2.5


# ---- live comparisons with the reference (build container only) ----

@pytest.mark.reference
def test_parser_agrees_with_reference_on_random_text(reference):
    from hypothesis import given, settings
    from hypothesis import strategies as st

    vocab = st.sampled_from(["NAME", "ROWS", "COLUMNS", "RHS", "RANGES", "BOUNDS", "ENDATA", "OBJSENSE", "N", "L",
                             "G", "E", "UP", "FR", "x", "c1", "obj", "1", "-2.5", "'MARKER'", "'INTORG'", "*"])
    line = st.tuples(st.booleans(), st.lists(vocab, min_size=1, max_size=5)).map(
        lambda t: (" " if t[0] else "") + " ".join(t[1]))

    @settings(max_examples=300, deadline=None)
    @given(st.one_of(st.text(max_size=200), st.lists(line, max_size=12).map("\n".join)))
    def check(text):
        outs = []
        for parse, perr in ((reference.parse_mps, reference.ParseError), (parse_mps, ParseError)):
            with warnings.catch_warnings(record=True) as caught:
                warnings.simplefilter("always")
                try:
                    outs.append(("ok", _model_dict(parse(text)), [str(w.message) for w in caught]))
                except perr as e:
                    outs.append(("err", str(e), e.line_no))
        assert outs[0] == outs[1]

    check()


@pytest.mark.reference
def test_standardize_agrees_with_reference_on_random_general_lps(reference):
    from hypothesis import given, settings
    from hypothesis import strategies as st

    @st.composite
    def glps(draw):
        n, k = draw(st.integers(1, 4)), draw(st.integers(0, 4))
        val = st.floats(-1e3, 1e3, allow_nan=False).map(lambda v: float(np.round(v, 3)))
        rows = [[draw(val) for _ in range(n)] for _ in range(k)]
        lo = [draw(st.sampled_from([0.0, -np.inf, -2.5, 1.0])) for _ in range(n)]
        hi = [draw(st.sampled_from([np.inf, 4.0, 10.5])) for _ in range(n)]
        return dict(sense=draw(st.sampled_from(["min", "max"])), c=[draw(val) for _ in range(n)],
                    rows=np.asarray(rows, float).reshape(k, n),
                    rels=[draw(st.sampled_from(["<=", ">=", "="])) for _ in range(k)],
                    rhs=[draw(val) for _ in range(k)], lower=lo, upper=hi)

    @settings(max_examples=300, deadline=None)
    @given(glps())
    def check(d):
        args = (d["sense"], d["c"], d["rows"], d["rels"], d["rhs"], d["lower"], d["upper"])
        ours, theirs = GeneralLP.build(*args), reference.GeneralLP.build(*args)
        try:
            want = reference.standardize(theirs)
        except reference.InfeasibleBounds as e:
            with pytest.raises(InfeasibleBounds) as err:
                standardize(ours)
            assert str(err.value) == str(e)
            return
        lp, vm = standardize(ours)
        rlp, rvm = want
        for a, b in ((lp.A, rlp.A), (lp.b, rlp.b), (lp.c, rlp.c), (vm.shift, rvm.shift), ([vm.offset], [rvm.offset])):
            assert _bits_equal(a, b)
        assert vm.plus_col.tolist() == rvm.plus_col.tolist() and vm.minus_col.tolist() == rvm.minus_col.tolist()
        x = np.linspace(-3.0, 7.0, vm.num_standard_vars)
        assert _bits_equal(vm.recover_point(x), rvm.recover_point(x))
        assert _bits_equal([vm.recover_objective(2.75)], [rvm.recover_objective(2.75)])

    check()
