"""The persistent fused run (k_fused_run: all merged days of epi_sim_run in
one launch, a grid barrier per day) against the per-day merged kernels:
bitwise equal records, codes and state, including runs split at arbitrary
days, mixed with single steps, and replayed from a CUDA graph."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize
from paper_2110_04421_b200.defaults import default_disease, default_progression
from paper_2110_04421_b200.interventions import InterventionConfig
from paper_2110_04421_b200.sim import ConfigSimulation

pytestmark = pytest.mark.gpu

COLS = ("stage", "infected_at", "next_transition_at", "next_stage")


def _pair(cfg, n, seeds, seed, horizon):
    spec = ConfigNetworkSpec.config(cfg, n_agents=n, initial_infections=seeds)
    pop = synthesize(spec, 5)
    d, t, iv = default_disease(), default_progression(), InterventionConfig()
    mk = lambda p: ConfigSimulation(pop, d, t, iv, seed, mode="fused", horizon=horizon, persistent=p)
    return mk(True), mk(False)


def _same(a, b):
    assert np.array_equal(a.rec.cpu().numpy(), b.rec.cpu().numpy()), \
        np.argwhere(a.rec.cpu().numpy() != b.rec.cpu().numpy())[:5]
    assert torch.equal(a._codes_buf, b._codes_buf)
    ha, hb = a.host_columns(), b.host_columns()
    for c in COLS:
        assert np.array_equal(getattr(ha, c), getattr(hb, c)), c


@pytest.mark.parametrize("cfg,n,seeds", [(1, 100_000, 100), (0, 10_000, 10), (1, 6007, 300), (1, 129, 20)])
def test_persistent_run_equals_per_day(cfg, n, seeds):
    a, b = _pair(cfg, n, seeds, 21, 180)
    a.run()
    b.run()
    r = a.rec.cpu().numpy()
    assert r[:, 1].sum() > 0                      # infections happened
    _same(a, b)


def test_persistent_split_runs_and_steps():
    a, b = _pair(1, 20_011, 200, 5, 120)
    for chunk in (1, 37, 2, 0, 50):
        a.run(chunk)
        b.run(chunk)
    a.step(); b.step()
    a.step(); b.step()
    a.run(); b.run()
    _same(a, b)


def test_persistent_graph_replay_equals_run():
    a, b = _pair(1, 30_000, 60, 9, 90)
    a.capture()
    a.replay()
    a.replay()                                    # reset inside the graph: same result twice
    b.run()
    _same(a, b)
