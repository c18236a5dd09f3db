"""Row f3 (output): the epivec-timeseries-v1 / summary CSV layouts against
the reference's own output (tests/golden/series.npz, made by
tests/golden/make_golden.py series), and the numpy oracle of `summarize`
against the reference's quartiles.  CPU only."""

from pathlib import Path

import numpy as np
import pytest

from oracle import series_np
from paper_2110_04421_b200.errors import ConfigError
from paper_2110_04421_b200.series import (CSV_COLUMNS, SUMMARY_METRICS, RunResult, load_results,
                                          summary_to_csv, summary_to_long_csv)

G = np.load(Path(__file__).parent / "golden" / "series.npz")


def _text(key):
    return bytes(G[key]).decode()


def test_run_result_csv_matches_reference():
    r = RunResult(replication=0, seed=int(G["run_seed"]), data=G["run_data"])
    assert r.to_csv() == _text("run_csv")
    back = RunResult.from_csv(_text("run_csv"))
    assert back.seed == r.seed and back.replication == 0
    assert np.array_equal(back.data, G["run_data"])
    assert np.array_equal(back.column("new_infections"), G["run_data"][:, CSV_COLUMNS.index("new_infections")])


def test_from_csv_errors_like_reference():
    with pytest.raises(ConfigError, match="not a epivec-timeseries-v1 file"):
        RunResult.from_csv("step\n")
    bad = _text("run_csv").replace("new_infections", "new_cases")
    with pytest.raises(ConfigError, match="column mismatch"):
        RunResult.from_csv(bad)


def test_load_results(tmp_path):
    with pytest.raises(ConfigError, match="no run_"):
        load_results(tmp_path)
    for i in range(3):
        RunResult(replication=i, seed=10 + i, data=G["runs_data"][i]).to_csv()
        (tmp_path / f"run_{i:03d}.csv").write_text(
            RunResult(replication=i, seed=10 + i, data=G["runs_data"][i]).to_csv())
    rs = load_results(tmp_path)
    assert [r.replication for r in rs] == [0, 1, 2]
    assert np.array_equal(rs[2].data, G["runs_data"][2])


def _summary(q):
    return {m: q[i] for i, m in enumerate(SUMMARY_METRICS)}


def test_oracle_summary_and_csv_layouts_match_reference():
    q = series_np.summarize_stacked(G["runs_data"])
    assert summary_to_csv(_summary(q)) == _text("sum_wide")
    assert summary_to_long_csv(_summary(q)) == _text("sum_long")


@pytest.mark.parametrize("key", [k for k in G.files if k.startswith("synth_")])
def test_oracle_quartiles_bitwise_reference(key):
    _, R, H, seed = key.split("_")
    data = np.random.default_rng(int(seed)).integers(0, 100_000, size=(int(R), int(H), 19), dtype=np.int64)
    assert np.array_equal(series_np.summarize_stacked(data), G[key])
