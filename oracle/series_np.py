"""Numpy restatement of the reference's replication summary — TEST
INFRASTRUCTURE (only tests/ may import it).

`summarize` (`pkg/src/epivec/runner.py:195-207`): per metric, the quartiles
[q25, q50, q75] across replications of every step, `np.percentile` with
numpy's default "linear" method.  The device kernel (`epi_quartiles`) is
checked against this and against the reference's own output
(tests/golden/series.npz).
"""

from __future__ import annotations

import numpy as np

METRICS = 18          # CSV columns 1..18 (every column but "step")


def summarize_stacked(data: np.ndarray) -> np.ndarray:
    """data int64 [R, horizon, >= 19] -> float64 [18, horizon, 3]."""
    out = np.empty((METRICS, data.shape[1], 3))
    for m in range(METRICS):
        stacked = data[:, :, 1 + m].T                      # (horizon, R), runner.py:204
        out[m] = np.percentile(stacked, [25, 50, 75], axis=1).T
    return out
