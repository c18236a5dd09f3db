"""Time-series output in the reference's schemas (SURVEY.md §8(f) row f3,
output part): `RunResult` with the `epivec-timeseries-v1` CSV
(`runner.py:31-74`), the replication summary (`runner.py:195-207`) and its
wide / long CSV layouts (`runner.py:210-238`), `load_results`
(`runner.py:241-246`).

The rows come from the device records (`ConfigSimulation.result()`: columns
0-18 of the `[horizon, 24]` record are the CSV columns in order), and
`summarize` computes the quartiles across replications on the device
(`epi_quartiles`, bitwise `np.percentile`), from host `RunResult`s or
straight from a stacked device record tensor (`summarize_device`).
Names, argument meaning and error messages follow the reference.
"""

from __future__ import annotations

import io
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native as N
from .errors import ConfigError
from .stages import Stage

SCHEMA = "epivec-timeseries-v1"
STAGE_COLUMNS = [f"n_{s.name.lower()}" for s in Stage]
CSV_COLUMNS = (["step"] + STAGE_COLUMNS
               + ["cumulative_infections", "cumulative_deaths", "in_hospital_or_icu",
                  "new_infections", "tests_administered", "doses_given",
                  "notifications_sent"])
SUMMARY_METRICS = [c for c in CSV_COLUMNS if c != "step"]
QUANTILES = ("q25", "q50", "q75")


@dataclass
class RunResult:
    """Per-step time series of one replication (runner.py:41-74)."""

    replication: int
    seed: int
    data: np.ndarray        # (horizon, len(CSV_COLUMNS)) int64
    n_edges_total: int = 0
    wall_seconds: float = 0.0

    def column(self, name: str) -> np.ndarray:
        return self.data[:, CSV_COLUMNS.index(name)]

    def to_csv(self) -> str:
        lines = [f"# schema={SCHEMA}", f"# replication={self.replication} seed={self.seed}",
                 ",".join(CSV_COLUMNS)]
        lines += [",".join(str(int(v)) for v in row) for row in self.data]
        return "\n".join(lines) + "\n"

    @classmethod
    def from_csv(cls, text: str) -> "RunResult":
        lines = text.splitlines()
        if not lines or lines[0] != f"# schema={SCHEMA}":
            raise ConfigError(f"not a {SCHEMA} file")
        meta = dict(part.split("=") for part in lines[1][2:].split(" "))
        if lines[2].split(",") != CSV_COLUMNS:
            raise ConfigError("time-series column mismatch with schema")
        rows = [[int(v) for v in line.split(",")] for line in lines[3:] if line]
        data = np.array(rows, dtype=np.int64).reshape(len(rows), len(CSV_COLUMNS))
        return cls(replication=int(meta["replication"]), seed=int(meta["seed"]), data=data)


def load_results(run_dir: str | Path) -> list[RunResult]:
    run_dir = Path(run_dir)
    paths = sorted(run_dir.glob("run_*.csv"))
    if not paths:
        raise ConfigError(f"no run_*.csv files under {run_dir}")
    return [RunResult.from_csv(p.read_text()) for p in paths]


def summarize_device(records, columns=None) -> dict[str, np.ndarray]:
    """Quartiles across replications of a stacked device record tensor
    `records` [R, horizon, C] int64 (C >= 19, CSV columns first): metric ->
    (horizon, 3) float64 [q25, q50, q75], computed by `epi_quartiles`."""
    import torch
    if records.device.type != "cuda":
        raise ConfigError("summarize_device needs device records (the quartile kernel runs on the GPU)")
    if records.dim() != 3 or records.dtype != torch.int64:
        raise ConfigError("records must be an int64 [replications, horizon, columns] tensor")
    names = SUMMARY_METRICS if columns is None else list(columns)
    idx = [CSV_COLUMNS.index(m) for m in names]
    rec = records.contiguous()
    R, H, C = rec.shape
    cols = torch.tensor(idx, dtype=torch.int32, device=rec.device)
    out = torch.empty((len(idx), H, 3), dtype=torch.float64, device=rec.device)
    N.check(N.lib().epi_quartiles(N.ptr(rec), int(R), int(H), int(C), N.ptr(cols), len(idx), N.ptr(out),
                                  N.stream_handle()))
    host = out.cpu().numpy()
    return {m: host[i] for i, m in enumerate(names)}


def summarize(results: list[RunResult]) -> dict[str, np.ndarray]:
    """Quartiles across replications: metric -> (horizon, 3) array [q25, q50, q75]
    (runner.py:195-207), on the device, for any number of replications
    (epi_quartiles: shared-memory sort up to 4096, bisection beyond).  Like
    every path of this package it needs the GPU: there is deliberately no
    host fallback (bitwise the reference's np.percentile either way)."""
    import torch
    if not results:
        raise ConfigError("summarize needs at least one replication")
    horizon = results[0].data.shape[0]
    for r in results:
        if r.data.shape[0] != horizon:
            raise ConfigError("replications disagree on horizon")
    stacked = np.stack([np.asarray(r.data, dtype=np.int64) for r in results])
    return summarize_device(torch.from_numpy(stacked).cuda())


def summary_to_csv(summary: dict[str, np.ndarray]) -> str:
    """Wide layout: one row per step, three columns per metric (runner.py:210-224)."""
    header = ["step"] + [f"{m}_{q}" for m in SUMMARY_METRICS for q in QUANTILES]
    lines = ["# schema=epivec-summary-v1", ",".join(header)]
    horizon = next(iter(summary.values())).shape[0]
    for step in range(horizon):
        lines.append(",".join([str(step)] + [repr(float(v)) for m in SUMMARY_METRICS for v in summary[m][step]]))
    return "\n".join(lines) + "\n"


def summary_to_long_csv(summary: dict[str, np.ndarray]) -> str:
    """Plot-ready long layout: step, metric, quantile, value (runner.py:227-238)."""
    lines = ["# schema=epivec-summary-long-v1", "step,metric,quantile,value"]
    horizon = next(iter(summary.values())).shape[0]
    for m in SUMMARY_METRICS:
        block = summary[m]
        for step in range(horizon):
            lines += [f"{step},{m},{q},{repr(float(v))}" for q, v in zip(QUANTILES, block[step])]
    return "\n".join(lines) + "\n"
