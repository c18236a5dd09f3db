"""The UNMODIFIED reference engine on the config networks -- TEST / BENCH
INFRASTRUCTURE (the reference arm of bench.py, the CPU side of the
statistical parity fixtures).  Never imported by the product package.

`epivec` (the reference, installed into baseline/_ref by
tools/install_reference.sh, or /root/reference/pkg/src in the build
container) provides the engine, the parameter objects, the keyed RNG and
the CSV row (`Engine`, engine.py:55-347; `_record_row`, runner.py:101-116).
The reference has no knob for the BASELINE.json networks, so
each day's StepGraph comes from the pinned CPU restatement of the config
generator (`oracle/confignet_np.py`), exactly as the reference's own loop
(runner.py:145-152) would take it from its GraphRealizer.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
REF_DIRS = (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src"))


def import_epivec():
    """The reference package: baseline/_ref first (travels to the GPU box)."""
    try:
        import epivec  # noqa: F401
    except ImportError:
        for d in REF_DIRS:
            if (d / "epivec").is_dir():
                sys.path.insert(0, str(d))
                break
        import epivec  # noqa: F401
    import epivec
    return epivec


def reference_interventions(enabled: bool, dose_gap: int = 21):
    """BASELINE.json configs[2] through the reference's own classes
    (SURVEY §8(d) mapping)."""
    import_epivec()
    from epivec.interventions import DenConfig, InterventionConfig, TestKind, VaccinePolicy
    if not enabled:
        return InterventionConfig()
    return InterventionConfig(quarantine_enabled=True, testing_enabled=True,
                              test_kind=TestKind("cfg2", 0.05, 2, 2), den_enabled=True,
                              den=DenConfig(0.5), vaccination_enabled=True,
                              vaccine=VaccinePolicy(daily_rate=0.01, dose1_efficacy=0.5,
                                                    dose2_efficacy=0.9, dose_gap=dose_gap))


class ReferenceReplica:
    """One replication of a config network driven by `epivec.engine.Engine`.

    Initial infections: the population's seed ids, entered with the
    reference's step-0 keyed draws exactly as `population.seed_infections`
    makes them (population.py:166-176); DEN apps as runner.py:86-89.
    """

    def __init__(self, spec, seed: int, interventions=None, pop=None, check_invariants=False):
        import_epivec()
        from epivec import rng as keyed
        from epivec.engine import Engine
        from epivec.rng import Purpose
        from epivec.scenario import default_scenario
        from epivec.state import AgentColumns

        from paper_2110_04421_b200.confignet import synthesize

        self.spec = spec
        self.pop = pop if pop is not None else synthesize(spec, 0)
        self.seed = int(seed)
        sc = default_scenario()
        disease, table = sc.disease, sc.progression
        iv = interventions if interventions is not None else reference_interventions(False)
        n = spec.n_agents
        cols = AgentColumns.allocate(n)
        cols.age_band[:] = self.pop.age_band
        cols.household_id[:] = self.pop.household_id
        cols.occupation[:] = (self.pop.wp_id >= 0).astype(np.int16)
        cols.random_degree[:] = spec.random_mean
        ids = np.sort(np.asarray(self.pop.seeds, dtype=np.int64))
        entry = table.entry_stages(cols.age_band[ids],
                                   keyed.uniforms(seed, 0, Purpose.ENTRY_STAGE, ids))
        cols.stage[ids] = entry
        cols.infected_at[ids] = 0
        nxt, delay = table.schedule_transitions(
            entry, cols.age_band[ids], keyed.uniforms(seed, 0, Purpose.PROGRESSION_BRANCH, ids),
            keyed.uniforms(seed, 0, Purpose.PROGRESSION_DELAY, ids))
        cols.next_stage[ids] = nxt
        cols.next_transition_at[ids] = delay
        if iv.den_enabled:
            u = keyed.uniforms(seed, 0, Purpose.DEN_APP, np.arange(n, dtype=np.int64))
            cols.has_den_app[:] = u < iv.den.app_adoption
        self.cols = cols
        self.engine = Engine(cols, disease, table, iv, seed, check_invariants=check_invariants)
        self.day = 0

    def step(self):
        """One day: realize (restated config generator) + Engine.step.
        Returns the reference's StepEvents."""
        from epivec.graphs import StepGraph

        from oracle import confignet_np
        t = self.day
        s, d, k = confignet_np.realize(self.pop, self.seed, t, self.cols.stage == 10, canonical=False)
        ev = self.engine.step(StepGraph(t, s, d, k))
        self.day += 1
        return ev

    def run(self, horizon: int) -> np.ndarray:
        """`horizon` days -> int64 [horizon, 19] rows (runner.py:101-116)."""
        from epivec.runner import CSV_COLUMNS, _record_row
        data = np.zeros((horizon, len(CSV_COLUMNS)), dtype=np.int64)
        for t in range(horizon):
            ev = self.step()
            _record_row(data, t, self.cols, ev)
        return data


class ReferenceNativeReplica:
    """The reference's own benchmark scenario (`epivec bench`, runner.py:268-289):
    default population, its GraphRealizer (households, per-occupation
    Watts-Strogatz, stub pairing) and its Engine -- all the reference's code,
    one replication (`initialize_run`, runner.py:81-98)."""

    def __init__(self, n_agents: int, base_seed: int, index: int = 0, initial_infections=None):
        import_epivec()
        from epivec.engine import Engine
        from epivec.runner import initialize_run, replication_seed
        from epivec.scenario import default_scenario
        kw = {} if initial_infections is None else {"initial_infections": initial_infections}
        cfg = default_scenario(n_agents=n_agents, horizon=180, replications=1, base_seed=base_seed, **kw)
        self.seed = replication_seed(cfg.base_seed, index)
        self.cols, self.realizer = initialize_run(cfg, self.seed)
        self.engine = Engine(self.cols, cfg.disease, cfg.progression, cfg.interventions, self.seed,
                             check_invariants=False)
        self.day = 0

    def step(self):
        g = self.realizer.realize(self.day, self.cols.stage == 10)
        ev = self.engine.step(g)
        self.day += 1
        return ev
