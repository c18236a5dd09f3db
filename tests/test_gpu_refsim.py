"""The reference's own scenario on the device (refsim.py): population mirror
+ device seeding vs the reference's recorded initialize_run state, then the
device step loop (device realizer + GpuEngine) vs the oracle engine on the
restated realizer's graphs, bitwise."""

import dataclasses

import numpy as np
import pytest

from golden_io import Trajectory
from oracle import engine_np, refnet_np
from paper_2110_04421_b200.defaults import POPULATION
from paper_2110_04421_b200.graph import StepGraph
from paper_2110_04421_b200.state import COLUMN_SPECS

pytestmark = pytest.mark.gpu

MEANS = POPULATION["networks"]["occupation_mean_interactions"]
BETA = POPULATION["networks"]["rewire_beta"]


def _sim(tr):
    from paper_2110_04421_b200.refsim import ReferenceNativeSimulation
    z = tr.z
    infected = int(np.sum(z["init_infected_at"] == 0))
    return ReferenceNativeSimulation(len(z["init_age_band"]), seed=tr.seed, initial_infections=infected,
                                     horizon=int(z["horizon"]), disease=tr.disease, table=tr.table,
                                     interventions=tr.iv)


@pytest.mark.parametrize("name", ["noiv", "alliv", "nonster"])
def test_initial_state_equals_reference_initialize_run(name):
    tr = Trajectory(name)
    sim = _sim(tr)
    sim.engine.sync_to_host()
    for c, _, _ in COLUMN_SPECS:
        assert np.array_equal(getattr(sim.cols, c), tr.z[f"init_{c}"]), c


@pytest.mark.parametrize("name", ["noiv", "alliv"])
def test_device_loop_bitwise_vs_oracle(name):
    tr = Trajectory(name)
    sim = _sim(tr)
    sim.engine.vaccination_open = bool(tr.z["vaccination_open"])
    cols_o = tr.initial_cols()
    eo = engine_np.OracleEngine(cols_o, tr.disease, tr.table, tr.iv, tr.seed)
    eo.vaccination_open = bool(tr.z["vaccination_open"])
    hh, occ, deg = sim.cols.household_id, sim.cols.occupation, sim.cols.random_degree
    for t in range(25):
        s, d, k = refnet_np.realize(tr.seed, t, hh, occ, deg, MEANS, BETA, cols_o.stage == 10)
        ev_o = eo.step(StepGraph(t, s, d, k))
        ev_g = sim.step()
        assert dataclasses.astuple(ev_g) == dataclasses.astuple(ev_o), t
    sim.engine.sync_to_host()
    for c in ("stage", "infected_at", "next_stage", "next_transition_at", "quarantine_until",
              "vaccine_status", "immune"):
        assert np.array_equal(getattr(sim.cols, c), getattr(cols_o, c)), c
    assert sim.interactions > 0


def test_device_resident_run_equals_step_by_step():
    """run() (records on the device, one sync per step) == step() events."""
    import dataclasses as dc
    tr = Trajectory("noiv")
    a, b = _sim(tr), _sim(tr)
    ev_a = [a.step() for _ in range(20)]
    ev_b = b.run(20)
    assert [dc.astuple(x) for x in ev_a] == [dc.astuple(x) for x in ev_b]
    a.engine.sync_to_host()
    b.engine.sync_to_host()
    assert np.array_equal(a.cols.stage, b.cols.stage)
    assert a.interactions == b.interactions


def test_native_loop_in_chunks_equals_one_run():
    """epi_refnet_run over [0,7) + [7,20) + the rest == one call, bitwise
    (records, edge counts and final state)."""
    import dataclasses as dc
    tr = Trajectory("noiv")
    a, b = _sim(tr), _sim(tr)
    ev_a = a.run(7) + a.run(13) + a.run()
    ev_b = b.run()
    assert [dc.astuple(x) for x in ev_a] == [dc.astuple(x) for x in ev_b]
    a.engine.sync_to_host()
    b.engine.sync_to_host()
    for c in ("stage", "infected_at", "next_stage", "next_transition_at"):
        assert np.array_equal(getattr(a.cols, c), getattr(b.cols, c)), c


def test_native_loop_output_overflow_is_an_error():
    """A realizer output smaller than the step's graph: the native loop writes
    nothing out of bounds (the graph load only sees the edges written) and
    run() raises ConfigError at its end."""
    import torch
    from paper_2110_04421_b200.errors import ConfigError
    tr = Trajectory("noiv")
    sim = _sim(tr)
    small = 64
    r = sim.realizer
    r._src, r._dst, r._kind = r._src[:small].clone(), r._dst[:small].clone(), r._kind[:small].clone()
    with pytest.raises(ConfigError, match="capacity"):
        sim.run(3)
    torch.cuda.synchronize()


def test_native_loop_rejects_exposure_notification():
    """The contact log needs host-known edge counts: run() with DEN enabled is
    a ConfigError before any step; step() still works."""
    from paper_2110_04421_b200.errors import ConfigError
    tr = Trajectory("alliv")
    assert tr.iv.den_enabled
    sim = _sim(tr)
    with pytest.raises(ConfigError):
        sim.run(2)
    assert sim.clock == 0
    sim.step()
    assert sim.clock == 1
