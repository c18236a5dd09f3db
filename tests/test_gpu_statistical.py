"""North-star parity contract 3: daily infection / mortality curves from
independent seeds are statistically indistinguishable between the GPU fast
path (fused mode, fp32 hazard) and the reference algorithm (the golden-pinned
oracle, fp64, same network definition) — SURVEY.md §8(c).

R replicas per side, config 0 (10k agents), without interventions and with
every intervention (the GPU's DEN regenerates past contacts, the oracle keeps
a contact log); two-sample Kolmogorov-Smirnov on final attack rate, peak day
and final deaths, Welch t on cumulative infections at days 30/60/90/120 (and
on tests, doses and notifications with interventions); Bonferroni-corrected
alpha = 0.01."""

import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

torch = pytest.importorskip("torch")
scipy_stats = pytest.importorskip("scipy.stats")

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

R = 20
HORIZON = 150
CHECK_DAYS = (30, 60, 90, 120)


def _interventions(name):
    from paper_2110_04421_b200.interventions import (DenConfig, InterventionConfig, TestKind,
                                                     VaccinePolicy)
    if name == "none":
        return InterventionConfig()
    return InterventionConfig(quarantine_enabled=True, testing_enabled=True,
                              test_kind=TestKind("stat", 0.3, 1, 2), den_enabled=True,
                              den=DenConfig(0.5), vaccination_enabled=True,
                              vaccine=VaccinePolicy(daily_rate=0.01, dose1_efficacy=0.5,
                                                    dose2_efficacy=0.9, dose_gap=21,
                                                    start_trigger=0.005))


def _oracle_replica(args):
    seed, iv_name = args
    from oracle import confignet_np, engine_np, rng_np
    from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize
    from paper_2110_04421_b200.defaults import default_disease, default_progression
    from paper_2110_04421_b200.graph import StepGraph
    from paper_2110_04421_b200.sim import initial_columns
    pop = synthesize(ConfigNetworkSpec.config(0), 0)
    table = default_progression()
    cols = initial_columns(pop)
    ids = pop.seeds
    entry = engine_np.pick(table.rules[0], cols.age_band[ids], rng_np.uniforms(seed, 0, 3, ids))
    cols.stage[ids] = entry
    cols.infected_at[ids] = 0
    nxt, d = engine_np.schedule(table, entry, cols.age_band[ids], rng_np.uniforms(seed, 0, 4, ids),
                                rng_np.uniforms(seed, 0, 5, ids))
    cols.next_stage[ids] = nxt
    cols.next_transition_at[ids] = d
    iv = _interventions(iv_name)
    if iv.den_enabled:      # runner.py:86-89, as the device's epi_assign_app
        cols.has_den_app[:] = rng_np.uniforms(seed, 0, 10, np.arange(cols.n_agents)) < iv.den.app_adoption
    eng = engine_np.OracleEngine(cols, default_disease(), table, iv, seed)
    rows = []
    for t in range(HORIZON):
        s, dd, k = confignet_np.realize(pop, seed, t, cols.stage == 10, canonical=False)
        ev = eng.step(StepGraph(t, s, dd, k))
        rows.append(engine_np.series_row(cols, ev))
    return np.array(rows)


def _metrics(series):
    """series: [R, days, 19] -> dict of per-replica metrics."""
    cum_inf = series[:, :, 12]
    new_inf = series[:, :, 15]
    deaths = series[:, :, 13]
    n = series[0, 0, 1:12].sum()
    out = {"attack": cum_inf[:, -1] / n, "peak_day": new_inf.argmax(axis=1),
           "deaths": deaths[:, -1], **{f"cum{d}": cum_inf[:, d] for d in CHECK_DAYS}}
    for name, col in (("tests", 16), ("doses", 17), ("notified", 18)):
        if series[:, :, col].sum() > 0:
            out[name] = series[:, :, col].sum(axis=1)
    return out


@pytest.mark.parametrize("iv_name", ["none", "all"])
def test_curves_statistically_indistinguishable_from_reference_algorithm(iv_name):
    from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize
    from paper_2110_04421_b200.defaults import default_disease, default_progression
    from paper_2110_04421_b200.keyed import replication_seed
    from paper_2110_04421_b200.sim import ConfigSimulation
    pop = synthesize(ConfigNetworkSpec.config(0), 0)
    gpu = []
    for r in range(R):
        sim = ConfigSimulation(pop, default_disease(), default_progression(), _interventions(iv_name),
                               replication_seed(0, r), mode="fused", horizon=HORIZON)
        sim.run()
        gpu.append(sim.time_series())
    gpu = np.stack(gpu)
    with ProcessPoolExecutor(max_workers=min(R, os.cpu_count() or 1)) as pool:
        cpu = np.stack(list(pool.map(_oracle_replica, [(replication_seed(1, r), iv_name)
                                                        for r in range(R)])))
    mg, mc = _metrics(gpu), _metrics(cpu)
    welch = [f"cum{d}" for d in CHECK_DAYS] + [k for k in ("tests", "doses", "notified") if k in mg]
    if iv_name == "all":
        assert all(k in mg and k in mc for k in ("tests", "doses", "notified")), (mg.keys(), mc.keys())
    alpha = 0.01 / (3 + len(welch))
    report = {}
    for key in ("attack", "peak_day", "deaths"):
        report[key] = scipy_stats.ks_2samp(mg[key], mc[key]).pvalue
    for key in welch:
        report[key] = scipy_stats.ttest_ind(mg[key], mc[key], equal_var=False).pvalue
    print({k: round(float(v), 4) for k, v in report.items()},
          "attack gpu/cpu", mg["attack"].mean(), mc["attack"].mean())
    for k, p in report.items():
        assert p > alpha or np.isnan(p), (k, p, report)
