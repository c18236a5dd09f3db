"""Differential fuzzing: GPU engine / generator vs the golden-pinned oracle on
random parameters, intervention settings, graphs (empty, duplicate edges,
ragged sizes) and network specs.  Bar: bitwise."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import confignet_np, engine_np, rng_np
from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize
from paper_2110_04421_b200.defaults import PROGRESSION, default_progression
from paper_2110_04421_b200.disease import DiseaseParams
from paper_2110_04421_b200.engine import GpuEngine
from paper_2110_04421_b200.graph import StepGraph
from paper_2110_04421_b200.interventions import (TEST_KINDS, DenConfig, ImmunityMode,
                                                 InterventionConfig, Strategy, TestKind,
                                                 VaccinePolicy)
from paper_2110_04421_b200.progression import ProgressionTable
from paper_2110_04421_b200.sim import ConfigSimulation
from paper_2110_04421_b200.state import DYNAMIC_COLUMNS, AgentColumns

pytestmark = pytest.mark.gpu


def _constant_table(rng):
    d = {"edges": []}
    for e in PROGRESSION["edges"]:
        e = dict(e)
        if "duration" in e:
            e["duration"] = {"family": "constant", "days": float(rng.integers(1, 6))}
        d["edges"].append(e)
    return ProgressionTable.from_dict(d)


def _random_setup(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.choice([1, 2, 7, 64, 150, 333]))
    disease = DiseaseParams(float(rng.uniform(0.5, 12)), rng.uniform(0.2, 2.0, 9),
                            float(rng.uniform(0, 1)), rng.uniform(0.3, 3, 3),
                            float(rng.uniform(0.5, 12)), float(rng.uniform(3, 9)),
                            float(rng.uniform(1, 4)))
    table = default_progression() if rng.random() < 0.5 else _constant_table(rng)
    testing = bool(rng.random() < 0.7)
    iv = InterventionConfig(
        quarantine_enabled=bool(rng.random() < 0.7),
        quarantine_duration=int(rng.integers(1, 15)),
        quarantine_dropout=float(rng.choice([0.0, 0.3, 1.0])),
        testing_enabled=testing,
        test_kind=TEST_KINDS[str(rng.choice(list(TEST_KINDS)))] if rng.random() < 0.5
        else TestKind("fz", float(rng.uniform(0, 1)), 1, int(rng.integers(1, 4))),
        false_positive_prob=float(rng.choice([0.0, 0.1])),
        den_enabled=testing and bool(rng.random() < 0.6),
        den=DenConfig(float(rng.uniform(0, 1)), float(rng.uniform(0, 1)), int(rng.integers(1, 8))),
        vaccination_enabled=bool(rng.random() < 0.7),
        vaccine=VaccinePolicy(strategy=Strategy(int(rng.integers(0, 3))),
                              dose1_efficacy=float(rng.uniform(0, 1)),
                              dose2_efficacy=float(rng.uniform(0, 1)),
                              dose1_latency=int(rng.integers(0, 4)),
                              dose2_latency=int(rng.integers(0, 3)),
                              dose_gap=int(rng.integers(1, 5)),
                              daily_rate=float(rng.choice([0.0, 0.02, 0.1, 0.5])),
                              start_trigger=float(rng.choice([0.0, 0.01, 0.05])),
                              immunity_mode=ImmunityMode(int(rng.integers(0, 2))),
                              elderly_band=int(rng.integers(0, 9))))
    cols = AgentColumns.allocate(n)
    cols.age_band[:] = rng.integers(0, 9, n)
    eseed = int(rng.integers(0, 2**63))
    k = max(1, n // 10)
    ids = np.sort(rng.choice(n, size=k, replace=False))
    entry = engine_np.pick(table.rules[0], cols.age_band[ids], rng_np.uniforms(eseed, 0, 3, ids))
    cols.stage[ids] = entry
    cols.infected_at[ids] = 0
    nxt, d = engine_np.schedule(table, entry, cols.age_band[ids], rng_np.uniforms(eseed, 0, 4, ids),
                                rng_np.uniforms(eseed, 0, 5, ids))
    cols.next_stage[ids] = nxt
    cols.next_transition_at[ids] = d
    if iv.den_enabled:
        cols.has_den_app[:] = rng_np.uniforms(eseed, 0, 10, np.arange(n)) < iv.den.app_adoption
    return rng, n, disease, table, iv, cols, eseed


def _random_graph(rng, n, step):
    if n < 2 or rng.random() < 0.1:
        return StepGraph.empty(step)
    e = int(rng.integers(0, 6 * n))
    src = rng.integers(0, n, e).astype(np.int32)
    dst = rng.integers(0, n, e).astype(np.int32)
    keep = src != dst
    if rng.random() < 0.3:           # duplicated edges
        src, dst = np.concatenate([src, src]), np.concatenate([dst, dst])
        keep = np.concatenate([keep, keep])
    src, dst = src[keep], dst[keep]
    return StepGraph(step, src, dst, rng.integers(0, 3, len(src)).astype(np.int8))


@pytest.mark.parametrize("seed", range(24))
def test_engine_fuzz_bitwise(seed):
    rng, n, disease, table, iv, cols, eseed = _random_setup(seed)
    cols_o = cols.copy()
    eng = GpuEngine(cols, disease, table, iv, eseed)
    ora = engine_np.OracleEngine(cols_o, disease, table, iv, eseed)
    for step in range(20):
        g = _random_graph(rng, n, step)
        ev_g, ev_o = eng.step(g), ora.step(g)
        got = (ev_g.n_edges, ev_g.new_infections, ev_g.deaths, ev_g.hospitalizations,
               ev_g.tests_administered, ev_g.doses_given, ev_g.notifications_sent)
        want = (ev_o.n_edges, ev_o.new_infections, ev_o.deaths, ev_o.hospitalizations,
                ev_o.tests_administered, ev_o.doses_given, ev_o.notifications_sent)
        assert got == want, (seed, step, got, want)
        for c in DYNAMIC_COLUMNS:
            a, b = getattr(cols, c), getattr(cols_o, c)
            assert np.array_equal(a, b), (seed, step, c, np.flatnonzero(a != b)[:5])
        assert eng.vaccination_open == ora.vaccination_open


@pytest.mark.parametrize("seed", range(10))
def test_generator_fuzz_bitwise(seed):
    rng = np.random.default_rng(100 + seed)
    hh = tuple(sorted(set(int(x) for x in rng.integers(1, 33, 4))))
    probs = rng.dirichlet(np.ones(len(hh)))
    spec = ConfigNetworkSpec(
        n_agents=[2, 61, 1000, 4097, 5][seed % 5],
        household_sizes=hh, household_probs=tuple(float(p) for p in probs / probs.sum()),
        worker_bands=tuple(int(b) for b in rng.choice(9, int(rng.integers(0, 9)), replace=False)),
        wp_min=int(rng.integers(2, 20)), wp_max=int(rng.integers(20, 255)),
        colleague_draws=int(rng.choice([0, 1, 8, 9, 32])),
        random_mean=float(rng.uniform(0, 12)), random_slots=int(rng.choice([0, 1, 16, 17, 32])),
        initial_infections=0)
    pop = synthesize(spec, int(rng.integers(0, 2**62)))
    from paper_2110_04421_b200.defaults import default_disease
    sim = ConfigSimulation(pop, default_disease(), default_progression(), InterventionConfig(),
                           int(rng.integers(0, 2**63)), precision="f64")
    dead = np.zeros(spec.n_agents, bool)
    g = sim.realize_graph(0).sorted_canonical()
    src, dst, kind = confignet_np.realize(pop, sim.seed, 0, dead)
    assert np.array_equal(g.dst, dst) and np.array_equal(g.src, src) and np.array_equal(g.kind, kind)


@pytest.mark.parametrize("seed", range(8))
def test_message_pass_fuzz_within_1e5(seed):
    """North-star part (a) on random network specs (row layouts from empty to
    ~80 messages, ragged N, states reached by random numbers of fused days):
    the fp32 message pass vs the oracle hazard on the restated graph."""
    import torch
    from paper_2110_04421_b200 import roofline
    from paper_2110_04421_b200.graph import StepGraph
    rng = np.random.default_rng(500 + seed)
    hh = tuple(sorted(set(int(x) for x in rng.integers(1, 33, 3))))
    probs = rng.dirichlet(np.ones(len(hh)))
    spec = ConfigNetworkSpec(
        n_agents=int(rng.choice([33, 500, 3001, 7777])),
        household_sizes=hh, household_probs=tuple(float(p) for p in probs / probs.sum()),
        worker_bands=tuple(int(b) for b in rng.choice(9, int(rng.integers(0, 9)), replace=False)),
        wp_min=int(rng.integers(2, 20)), wp_max=int(rng.integers(20, 255)),
        colleague_draws=int(rng.choice([0, 1, 4, 8])),
        random_mean=float(rng.uniform(0, 12)), random_slots=int(rng.choice([0, 1, 8, 16])),
        initial_infections=int(rng.integers(1, 30)))
    sim = roofline.prepare(spec.n_agents, warm_days=int(rng.integers(1, 12)), spec=spec)
    t = sim.clock
    lam = torch.empty(spec.n_agents, dtype=torch.float32, device="cuda")
    rec = torch.zeros(24, dtype=torch.int64, device="cuda")
    roofline.gather(sim, lam, rec)
    cols = sim.host_columns()
    src, dst, kind = confignet_np.realize(sim.population, sim.seed, t, cols.stage == 10)
    ref = engine_np.hazard(cols, sim.disease, t, StepGraph(t, src, dst, kind), True)
    got = lam.cpu().numpy().astype(np.float64)
    nz = ref > 0
    assert np.all(np.abs(got[nz] - ref[nz]) <= 1e-5 * ref[nz])
    assert np.all(got[~nz] == 0)
    assert int(rec[19]) == len(src)


@pytest.mark.parametrize("seed", range(8))
def test_sparse_rows_fuzz_bitwise(seed):
    """Sparse in-rows (infectious sources only, in-edges counted from the
    out-edges) on random network specs and dispersed epidemics: 40 fused days
    bitwise equal -- records, codes, stages -- to the inverse bijections and
    to the full push tables (persistent run), whole population and 2
    emulated ranks."""
    from paper_2110_04421_b200.defaults import default_disease
    from paper_2110_04421_b200.partition import run_threaded
    rng = np.random.default_rng(900 + seed)
    hh = tuple(sorted(set(int(x) for x in rng.integers(1, 12, 3))))
    probs = rng.dirichlet(np.ones(len(hh)))
    spec = ConfigNetworkSpec(
        n_agents=int(rng.choice([64, 999, 4096, 20011])),
        household_sizes=hh, household_probs=tuple(float(p) for p in probs / probs.sum()),
        worker_bands=tuple(int(b) for b in rng.choice(9, int(rng.integers(0, 9)), replace=False)),
        wp_min=int(rng.integers(2, 20)), wp_max=int(rng.integers(20, 255)),
        colleague_draws=int(rng.choice([0, 1, 4, 8])),
        random_mean=float(rng.uniform(0, 12)), random_slots=16,
        initial_infections=int(rng.integers(1, 60)))
    pop = synthesize(spec, int(rng.integers(0, 2**62)))
    d, t, iv = default_disease(), default_progression(), InterventionConfig()
    seed_sim = int(rng.integers(0, 2**63))
    mk = lambda **kw: ConfigSimulation(pop, d, t, iv, seed_sim, mode="fused", horizon=40, **kw)
    full, inv, sp = mk(), mk(push_max=0, sparse_push=False), mk(push_max=0)
    for s in (full, inv, sp):
        s.run()
    for s in (full, inv):
        assert np.array_equal(sp.rec.cpu().numpy(), s.rec.cpu().numpy())
        assert torch.equal(sp._codes_buf, s._codes_buf)
    _, rec2 = run_threaded(pop, d, t, iv, seed_sim, 2, 40, mode="fused")
    assert np.array_equal(rec2.cpu().numpy(), sp.rec.cpu().numpy())
