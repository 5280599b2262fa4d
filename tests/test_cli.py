"""CLI / harness: argument validation and CSV round trip run on CPU;
the end-to-end examples of SPEC.md:424-426 / 490-493 run on the GPU (-m gpu)."""
import io

import pytest

from paper_1204_5072_b200.cli import parse_and_run
from paper_1204_5072_b200.harness import CSV_COLUMNS, ExperimentConfig, Row, read_csv, write_csv


@pytest.mark.parametrize("argv", [
    ["kpz", "--size", "100"],                       # size must be a power of two
    ["kpz", "--scheduler", "seq"],                  # CPU-only scheduler
    ["kpz", "--scheduler", "bogus"],
    ["kpz", "--p", "1.5"],
    ["kmc", "--conc", "1.5"],
    ["kmc", "--eps", "-1"],
    ["kpz", "--mcs", "-3"],
    ["kpz", "--no-such-flag"],
    [],
])
def test_invalid_arguments_exit_2(argv, capsys):
    assert parse_and_run(argv) == 2
    err = capsys.readouterr().err
    assert "usage" in err.lower()


def test_csv_round_trip():
    cfg = ExperimentConfig("kmc", 64, 10, seed=3, realizations=2, conc=0.325, eps=1.5)
    rows = [Row(0, "open_bonds_per_particle", 8.123456789012345, 0, 0, 0.0, 0),
            Row(10, "open_bonds_per_particle", 6.5, 1310720, 12345, 12.5, 1)]
    buf = io.StringIO()
    write_csv(cfg, rows, buf)
    text = buf.getvalue()
    assert text.splitlines()[0].startswith("# ")
    meta, back = read_csv(text)
    assert back == rows
    assert meta["model"] == "kmc" and meta["size"] == "64" and meta["conc"] == "0.325"
    header = [ln for ln in text.splitlines() if not ln.startswith("#")][0]
    assert tuple(header.split(",")) == CSV_COLUMNS


def test_sample_schedule():
    cfg = ExperimentConfig("kpz", 64, 100)
    ts = cfg.sample_times()
    assert ts[0] == 0 and ts[-1] == 100 and ts == sorted(set(ts))
    assert ExperimentConfig("kpz", 64, 0).sample_times() == [0]
    assert ExperimentConfig("kpz", 64, 50, samples=[10, 20, 99]).sample_times() == [10, 20, 50]


@pytest.mark.gpu
def test_kpz_flat_single_row(tmp_path):
    """`kpz --size 64 --p 1 --q 0 --mcs 0` -> one sample, W^2 = 0.5."""
    out = tmp_path / "kpz.csv"
    assert parse_and_run(["kpz", "--size", "64", "--p", "1", "--q", "0", "--mcs", "0", "--out", str(out)]) == 0
    meta, rows = read_csv(out.read_text())
    w2 = [r for r in rows if r.observable_name == "W2"]
    assert len(w2) == 1 and w2[0].t == 0 and w2[0].value == 0.5
    h = [r for r in rows if r.observable_name == "mean_height"]
    assert h[0].value == -1.0


@pytest.mark.gpu
def test_kpz_series_accounting(tmp_path):
    """Accounting: the attempts column is the device count; with the
    default sub = 4 plan it is t * N on average (sd L per MCS, Poisson tile counts),
    with sub = 1 (the paper's scheme) exactly t * N -- see test_kpz_series_accounting_sub1."""
    out = tmp_path / "kpz.csv"
    assert parse_and_run(["kpz", "--size", "256", "--mcs", "30", "--realizations", "2", "--out", str(out)]) == 0
    _, rows = read_csv(out.read_text())
    assert {r.realization_id for r in rows} == {0, 1}
    for r in rows:
        assert abs(r.attempts - r.t * 256 * 256) < 6 * 256 * max(1, r.t) ** 0.5
    ts = [r.t for r in rows if r.realization_id == 0 and r.observable_name == "W2"]
    assert ts == sorted(set(ts)) and ts[-1] == 30


@pytest.mark.gpu
def test_kpz_series_accounting_sub1(tmp_path):
    """Accounting exactness with the paper's scheme (--sub 1): attempts = t * N."""
    out = tmp_path / "kpz1.csv"
    assert parse_and_run(["kpz", "--size", "256", "--mcs", "12", "--sub", "1", "--out", str(out)]) == 0
    _, rows = read_csv(out.read_text())
    assert rows and all(r.attempts == r.t * 256 * 256 for r in rows)


@pytest.mark.gpu
def test_kmc_quench_first_sample(tmp_path):
    """`kmc --size 64 --conc 0.325 --eps 1.5` -> first open-bonds sample 8.1 +- 0.1."""
    out = tmp_path / "kmc.csv"
    assert parse_and_run(["kmc", "--size", "64", "--conc", "0.325", "--eps", "1.5", "--mcs", "20",
                          "--scheduler", "doubletile", "--out", str(out)]) == 0
    _, rows = read_csv(out.read_text())
    assert rows[0].t == 0 and abs(rows[0].value - 8.1) < 0.1
    assert rows[-1].t == 20 and rows[-1].value < rows[0].value


@pytest.mark.gpu
@pytest.mark.parametrize("model", ["kpz", "kmc"])
def test_concurrent_realizations_equal_sequential(model):
    """Realizations in flight together on their own streams give the series of running
    them one after another (only wall_ms differs)."""
    from paper_1204_5072_b200.harness import run_experiment

    kw = dict(p=0.95, q=0.05) if model == "kpz" else dict(conc=0.5, eps=1.5, both_active=True)
    size = 128 if model == "kpz" else 32
    rows = {}
    for conc in (1, 3):
        cfg = ExperimentConfig(model, size, 12, seed=9, realizations=5, concurrency=conc, **kw)
        rows[conc] = [(r.t, r.observable_name, r.value, r.attempts, r.successes, r.realization_id)
                      for r in run_experiment(cfg)]
    assert rows[1] == rows[3]
    assert {x[-1] for x in rows[1]} == set(range(5))
