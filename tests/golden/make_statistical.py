"""Reference side of the statistical curve-parity test:
R = 32 replications per case of the UNMODIFIED reference engine
(`epivec.engine.Engine`, /root/reference/pkg/src) on the config networks,
180 days each, recorded with the reference's own `_record_row`
(runner.py:101-116) -> tests/golden/stat_<case>.npz, int32 [R, 180, 19].

The reference has no knob for the BASELINE.json networks, so
each day's StepGraph comes from the pinned CPU restatement of the config
generator (`oracle/confignet_np.py`), and the engine -- the thing whose
curves are compared -- is the reference's own, fed the reference's own
DiseaseParams / ProgressionTable / InterventionConfig objects.  Initial
infections: the population's seed ids, then the reference's step-0 keyed
draws exactly as `population.seed_infections` (population.py:166-176) makes
them; DEN apps as runner.py:86-89.  Replication r uses seed
replication_seed(1, r); the GPU side of the test uses replication_seed(0, r)
(independent seeds).

Run in the build container (needs /root/reference):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_statistical.py [case ...]
"""

from __future__ import annotations

import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

R = 32
HORIZON = 180
CASES = {
    # name: (config, interventions, dose gap)
    "config0": (0, False, 0),
    "config1": (1, False, 0),
    "config2_gap21": (1, True, 21),
    "config2_gap84": (1, True, 84),
}


def reference_interventions(enabled, gap):
    """BASELINE.json configs[2] through the reference's own classes
    (SURVEY §8(d) mapping)."""
    from epivec.interventions import DenConfig, InterventionConfig, TestKind, VaccinePolicy
    if not enabled:
        return InterventionConfig()
    return InterventionConfig(quarantine_enabled=True, testing_enabled=True,
                              test_kind=TestKind("cfg2", 0.05, 2, 2), den_enabled=True,
                              den=DenConfig(0.5), vaccination_enabled=True,
                              vaccine=VaccinePolicy(daily_rate=0.01, dose1_efficacy=0.5,
                                                    dose2_efficacy=0.9, dose_gap=gap))


def reference_defaults():
    from epivec.scenario import default_scenario
    sc = default_scenario()
    return sc.disease, sc.progression


def one_replica(args):
    case, r = args
    from epivec import rng as keyed
    from epivec.engine import Engine
    from epivec.graphs import StepGraph
    from epivec.rng import Purpose
    from epivec.runner import CSV_COLUMNS, _record_row, replication_seed
    from epivec.state import AgentColumns
    from oracle import confignet_np
    from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize

    cfg, iv_on, gap = CASES[case]
    spec = ConfigNetworkSpec.config(cfg)
    pop = synthesize(spec, 0)
    seed = replication_seed(1, r)
    disease, table = reference_defaults()
    iv = reference_interventions(iv_on, gap)
    n = spec.n_agents
    cols = AgentColumns.allocate(n)
    cols.age_band[:] = pop.age_band
    cols.household_id[:] = pop.household_id
    cols.occupation[:] = (pop.wp_id >= 0).astype(np.int16)
    cols.random_degree[:] = spec.random_mean
    ids = np.sort(pop.seeds.astype(np.int64))
    entry = table.entry_stages(cols.age_band[ids], keyed.uniforms(seed, 0, Purpose.ENTRY_STAGE, ids))
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
    eng = Engine(cols, disease, table, iv, seed, check_invariants=False)
    data = np.zeros((HORIZON, len(CSV_COLUMNS)), dtype=np.int64)
    for t in range(HORIZON):
        s, d, k = confignet_np.realize(pop, seed, t, cols.stage == 10, canonical=False)
        ev = eng.step(StepGraph(t, s, d, k))
        _record_row(data, t, cols, ev)
    return r, data.astype(np.int32)


def main(cases):
    for case in cases:
        t0 = time.time()
        with ProcessPoolExecutor(max_workers=os.cpu_count() or 1) as pool:
            out = dict(pool.map(one_replica, [(case, r) for r in range(R)]))
        series = np.stack([out[r] for r in range(R)])
        np.savez_compressed(HERE / f"stat_{case}.npz", series=series,
                            seeds_base=np.int64(1), horizon=np.int64(HORIZON))
        print(case, series.shape, f"{time.time() - t0:.0f}s", "attack",
              series[:, -1, 12].mean() / series[0, 0, 1:12].sum(), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
