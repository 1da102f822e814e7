"""The bench CSV surface: the reference's schema (cli.py:42-46,304-333)."""
import pytest

from paper_1802_08557_b200.cli import BENCH_CSV_HEADER, EXTENDED_HEADER, main

torch = pytest.importorskip("torch")


def run(capsys, *argv):
    code = main([str(a) for a in argv])
    out, err = capsys.readouterr()
    return code, out, err


def test_header_matches_reference_schema():
    assert BENCH_CSV_HEADER == ("dim", "batch_size", "repeats", "setup_ms", "wall_ms", "lps_per_sec",
                                "n_optimal", "n_unbounded", "n_infeasible", "n_iteration_limit")


def test_bench_count_zero_emits_header_only(capsys):
    code, out, _ = run(capsys, "bench", "--count", "0")
    assert code == 0 and out == ",".join(BENCH_CSV_HEADER) + "\n"


def test_env_defaults(capsys, monkeypatch):
    monkeypatch.setenv("BATCHLP_COUNT", "0")
    code, out, _ = run(capsys, "bench", "--extended")
    assert code == 0 and out == ",".join(BENCH_CSV_HEADER + EXTENDED_HEADER) + "\n"


def test_reference_bench_matches_schema(reference, capsys):
    """The reference's own bench emits the same header (live, build container only)."""
    from batchlp.cli import BENCH_CSV_HEADER as REF_HEADER
    assert tuple(REF_HEADER) == BENCH_CSV_HEADER


@pytest.mark.gpu
def test_bench_small_cell_schema_and_counts(capsys):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1802_08557_b200 import BatchConfig, batch_solve, gen_random_lps
    code, out, _ = run(capsys, "bench", "--dims", "4", "--batch-sizes", "8", "--repeats", "2", "--seed", "5",
                       "--extended")
    assert code == 0
    header, row = out.strip().splitlines()
    assert header == ",".join(BENCH_CSV_HEADER + EXTENDED_HEADER)
    f = dict(zip(BENCH_CSV_HEADER + EXTENDED_HEADER, row.split(",")))
    assert (f["dim"], f["batch_size"], f["repeats"]) == ("4", "8", "2")
    assert float(f["wall_ms"]) > 0 and float(f["setup_ms"]) >= 0
    counts = batch_solve(gen_random_lps(4, 8, seed=5), BatchConfig()).status_counts()
    assert int(f["n_optimal"]) == counts.get("optimal", 0)
    assert int(f["n_infeasible"]) == counts.get("infeasible", 0)
    assert f["kernel"].startswith(("ctab", "warplp"))
