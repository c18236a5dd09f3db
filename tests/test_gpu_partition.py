"""Agent-range partition emulated on one GPU: P ranks with their own contexts,
row ranges and code buffers, codes exchanged by device copies each day.  The
result must be bitwise identical to the unpartitioned run (each row is owned
and summed by exactly one rank in a fixed order)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize
from paper_2110_04421_b200.defaults import default_disease, default_progression
from paper_2110_04421_b200.interventions import InterventionConfig, TestKind
from paper_2110_04421_b200.partition import run_emulated
from paper_2110_04421_b200.sim import ConfigSimulation

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode,precision,world", [("fused", "f32", 2), ("csr", "f32", 3),
                                                  ("csr", "f64", 2), ("fused", "f32", 5)])
def test_partitioned_equals_single(mode, precision, world):
    spec = ConfigNetworkSpec.config(1, n_agents=6007, initial_infections=60)
    pop = synthesize(spec, 4)
    iv = InterventionConfig(quarantine_enabled=True, testing_enabled=True,
                            test_kind=TestKind("q", 0.5, 1, 2))
    d, t = default_disease(), default_progression()
    days = 45
    ref = ConfigSimulation(pop, d, t, iv, 99, mode=mode, precision=precision, horizon=days)
    ref.run()
    sims, rec = run_emulated(pop, d, t, iv, 99, world, days, mode=mode, precision=precision)
    assert np.array_equal(rec.cpu().numpy(), ref.rec.cpu().numpy())
    full = ref.host_columns()
    for s in sims:
        lo, hi = s.plan.rows(s.rank)
        mine = s.host_columns()
        for c in ("stage", "infected_at", "next_transition_at", "quarantine_until", "test_result_at"):
            assert np.array_equal(getattr(mine, c)[lo:hi], getattr(full, c)[lo:hi]), (s.rank, c)


@pytest.mark.parametrize("precision,world", [("f64", 2), ("f32", 3)])
def test_partitioned_den_and_vaccination_equal_single(precision, world):
    """Row f2: exposure notification and vaccination across agent ranges, the
    in-step exchanges emulated by host threads; bitwise equal to P = 1."""
    from paper_2110_04421_b200.interventions import DenConfig, VaccinePolicy
    from paper_2110_04421_b200.partition import run_threaded
    spec = ConfigNetworkSpec.config(1, n_agents=6007, initial_infections=60)
    pop = synthesize(spec, 8)
    iv = InterventionConfig(quarantine_enabled=True, testing_enabled=True,
                            test_kind=TestKind("cfg2", 0.3, 1, 2), den_enabled=True,
                            den=DenConfig(0.6), vaccination_enabled=True,
                            vaccine=VaccinePolicy(daily_rate=0.02, dose1_efficacy=0.5,
                                                  dose2_efficacy=0.9, dose_gap=7,
                                                  start_trigger=0.002))
    d, t = default_disease(), default_progression()
    days = 40
    ref = ConfigSimulation(pop, d, t, iv, 77, mode="csr", precision=precision, horizon=days)
    ref.run()
    r = ref.rec.cpu().numpy()
    assert r[:, 17].sum() > 0 and r[:, 18].sum() > 0          # doses given, notifications sent
    sims, rec = run_threaded(pop, d, t, iv, 77, world, days, mode="csr", precision=precision)
    assert np.array_equal(rec.cpu().numpy(), r), np.argwhere(rec.cpu().numpy() != r)[:5]
    full = ref.host_columns()
    for s in sims:
        lo, hi = s.plan.rows(s.rank)
        mine = s.host_columns()
        for c in ("stage", "infected_at", "next_transition_at", "quarantine_until", "vaccine_status",
                  "dose1_at", "immune", "den_test_due_at"):
            assert np.array_equal(getattr(mine, c)[lo:hi], getattr(full, c)[lo:hi]), (s.rank, c)


def _config1_pop(n=20_011, seeds=200):
    spec = ConfigNetworkSpec.config(1, n_agents=n, initial_infections=seeds)
    return synthesize(spec, 6)


def test_native_nccl_day_loop_world1_equals_single_and_replays_as_graph():
    """The native partitioned day loop over NCCL (epi_comm, one rank on this
    GPU): per-day in-place all-gather inside epi_sim_run, tomorrow's sigma
    tables on the side stream; bitwise equal to the plain run (push tables
    on, and off), and a CUDA-graph replay of the whole run equals eager."""
    from paper_2110_04421_b200.partition import NcclComm, PartitionedSimulation, PartitionPlan
    pop = _config1_pop()
    d, t, iv = default_disease(), default_progression(), InterventionConfig()
    days = 60
    ref = ConfigSimulation(pop, d, t, iv, 31, mode="fused", horizon=days)
    ref.run()
    nopush = ConfigSimulation(pop, d, t, iv, 31, mode="fused", horizon=days, push_max=0)
    nopush.run()
    assert np.array_equal(nopush.rec.cpu().numpy(), ref.rec.cpu().numpy())
    comm = NcclComm(1, 0, NcclComm.unique_id())
    plan = PartitionPlan(pop.n_agents, 1)
    ps = PartitionedSimulation(pop, d, t, iv, 31, plan, 0, comm=comm, mode="fused", horizon=days, push_max=0)
    ps.run()
    assert np.array_equal(ps.rec.cpu().numpy(), ref.rec.cpu().numpy())
    ps.capture()
    ps.replay()
    assert np.array_equal(ps.rec.cpu().numpy(), ref.rec.cpu().numpy())
    assert np.array_equal(ps.host_columns().stage, ref.host_columns().stage)


def test_sigma_ahead_on_and_off_bitwise():
    """Tomorrow's sigma tables built ahead on the side stream or in line:
    identical runs, including runs split at arbitrary days and reset."""
    pop = _config1_pop(9001, 90)
    d, t, iv = default_disease(), default_progression(), InterventionConfig()
    a = ConfigSimulation(pop, d, t, iv, 5, mode="fused", horizon=50, push_max=0)
    b = ConfigSimulation(pop, d, t, iv, 5, mode="fused", horizon=50, push_max=0)
    b._lib.epi_set_sigma_ahead(b._ctx, 0)
    for chunk in (7, 1, 13):
        a.run(chunk)
        b.run(chunk)
    a.step(); b.step()
    a.reset(); a.run(3)
    b.reset(); b.run(3)
    a.run(); b.run()
    assert np.array_equal(a.rec.cpu().numpy(), b.rec.cpu().numpy())
    assert torch.equal(a._codes_buf, b._codes_buf)


@pytest.mark.parametrize("world", [2, 3])
def test_threaded_ranks_native_day_loop_equal_single(world):
    """P emulated ranks (host threads, own streams) with the per-day code
    all-gather requested by the native loop (EPI_X_GATHER_U16 callback),
    fused mode, sigma tables ahead: bitwise equal to P = 1."""
    from paper_2110_04421_b200.partition import run_threaded
    pop = _config1_pop(12_007, 120)
    d, t, iv = default_disease(), default_progression(), InterventionConfig()
    days = 40
    ref = ConfigSimulation(pop, d, t, iv, 17, mode="fused", horizon=days)
    ref.run()
    sims, rec = run_threaded(pop, d, t, iv, 17, world, days, mode="fused")
    assert np.array_equal(rec.cpu().numpy(), ref.rec.cpu().numpy())
    full = ref.host_columns()
    for s in sims:
        lo, hi = s.plan.rows(s.rank)
        assert np.array_equal(s.host_columns().stage[lo:hi], full.stage[lo:hi])
