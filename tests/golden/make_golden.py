"""Generate golden vectors by running the UNMODIFIED reference (epivec).

Run in the build container only (needs /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py independent   (row f4 fixtures)
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py series        (row f3 output fixtures)

Writes small .npz fixtures next to this script.  The GPU box never reads
/root/reference; tests load these fixtures instead.
"""

import json
import sys
from dataclasses import asdict
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from epivec import rng as R                                     # noqa: E402
from epivec.engine import Engine                                # noqa: E402
from epivec.interventions import priority_sort_key, Strategy    # noqa: E402
from epivec.runner import initialize_run, replication_seed      # noqa: E402
from epivec.scenario import (default_disease_dict, default_population_dict,  # noqa: E402
                             default_progression_dict, scenario_from_dict)
from epivec.state import DYNAMIC_COLUMNS                        # noqa: E402
from epivec.transmission import day_weight_table                # noqa: E402

OUT = Path(__file__).resolve().parent
ALL_COLS = ("age_band", "occupation", "household_id", "random_degree") + DYNAMIC_COLUMNS


def rng_fixture():
    keys = [(0, 0, 1, 0, 0), (0, 0, 1, 1, 0), (42, 7, 3, 12345, 0),
            (2 ** 64 - 1, 179, 11, 9999999, 2), (15266282343978493897, 5, 5, 77, 0)]
    scalar = np.array([R.uniform(*k) for k in keys])
    prefixes = np.array([R.key_prefix(s, t, p) for s, t, p, _, _ in keys], dtype=np.uint64)
    ids = np.arange(0, 50_000, 7, dtype=np.int64)
    vec = {f"vec_{s}_{t}_{p}_{k}": R.uniforms(s, t, p, ids, k)
           for s, t, p, k in [(0, 0, 1, 0), (123456789, 17, 5, 0), (2 ** 63 + 5, 3, 11, 2)]}
    seeds = np.array([R.derive_seed(0, 64, 0), R.derive_seed(42, 64, 3),
                      R.derive_seed(7, 67, 12, 5)], dtype=np.uint64)
    np.savez_compressed(OUT / "rng.npz", keys=np.array(keys, dtype=np.uint64),
                        scalar=scalar, prefixes=prefixes, ids=ids, derived=seeds, **vec)


def progression_fixture():
    from epivec.progression import ProgressionTable
    d = default_progression_dict()
    table = ProgressionTable.from_dict(d)
    n = 40_000
    ids = np.arange(n, dtype=np.int64)
    u_b = R.uniforms(99, 4, 4, ids)
    u_d = R.uniforms(99, 4, 5, ids)
    ages = (ids % 9).astype(np.int8)
    out = {}
    for s in range(1, 8):
        stages = np.full(n, s, dtype=np.int8)
        nxt, delay = table.schedule_transitions(stages, ages, u_b, u_d)
        out[f"next_{s}"], out[f"delay_{s}"] = nxt, delay
    out["entry"] = table.entry_stages(ages, R.uniforms(99, 4, 3, ids))
    # draws near the extremes of the unit interval
    edge_u = np.array([0.0, 2.0 ** -53, 1e-12, 0.5, 1 - 2.0 ** -53, 1 - 1e-12])
    for s in range(1, 8):
        st = np.full(len(edge_u), s, dtype=np.int8)
        a = np.zeros(len(edge_u), dtype=np.int8)
        out[f"edge_next_{s}"], out[f"edge_delay_{s}"] = table.schedule_transitions(st, a, edge_u, edge_u)
    np.savez_compressed(OUT / "progression.npz", ages=ages,
                        edge_u=edge_u, table_json=json.dumps(d), **out)
    weights = {f"w_{m}_{s}": day_weight_table(m, s)
               for m, s in [(5, 2), (7, 3), (3, 1), (10, 4.5), (6.5, 2.2)]}
    np.savez_compressed(OUT / "day_weights.npz", **weights)


def priority_fixture():
    rng = np.random.default_rng(5)
    n = 5000
    ages = rng.integers(0, 9, n).astype(np.int8)
    dose2 = rng.random(n) < 0.4
    ids = np.sort(rng.choice(10 * n, n, replace=False)).astype(np.int64)
    out = {f"order_{int(s)}": priority_sort_key(s, 6, ages, dose2, ids) for s in Strategy}
    np.savez_compressed(OUT / "priority.npz", ages=ages, dose2=dose2, ids=ids, **out)


def _iv_dict(iv):
    d = asdict(iv)
    d["test_kind"] = asdict(iv.test_kind)
    d["vaccine"]["strategy"] = int(iv.vaccine.strategy)
    d["vaccine"]["immunity_mode"] = int(iv.vaccine.immunity_mode)
    return d


def trajectory_fixture(name, n, horizon, seed, interventions, infections=8, record_gather=()):
    pop = default_population_dict()
    pop["n_agents"] = n
    cfg = scenario_from_dict({"population": pop, "horizon": horizon, "replications": 1,
                              "base_seed": seed, "initial_infections": infections,
                              "interventions": interventions}, name=name)
    rseed = replication_seed(cfg.base_seed, 0)
    cols, realizer = initialize_run(cfg, rseed)
    init = {f"init_{c}": getattr(cols, c).copy() for c in ALL_COLS}
    eng = Engine(cols, cfg.disease, cfg.progression, cfg.interventions, rseed)
    srcs, dsts, kinds, ev_rows, states, hz = [], [], [], [], {c: [] for c in DYNAMIC_COLUMNS}, {}
    for step in range(horizon):
        g = realizer.realize(step, cols.stage == 10)
        if step in record_gather:
            hz[f"hazard_{step}"] = eng.gather_exposure(g)
        ev = eng.step(g)
        srcs.append(g.src); dsts.append(g.dst); kinds.append(g.kind)
        ev_rows.append([ev.n_edges, ev.new_infections, ev.deaths, ev.hospitalizations,
                        ev.tests_administered, ev.doses_given, ev.notifications_sent])
        for c in DYNAMIC_COLUMNS:
            states[c].append(getattr(cols, c).copy())
    offs = np.concatenate(([0], np.cumsum([len(s) for s in srcs])))
    np.savez_compressed(
        OUT / f"traj_{name}.npz", seed=np.uint64(rseed), horizon=horizon,
        edge_offsets=offs, src=np.concatenate(srcs), dst=np.concatenate(dsts),
        kind=np.concatenate(kinds), events=np.array(ev_rows, dtype=np.int64),
        disease_json=json.dumps(default_disease_dict()),
        table_json=json.dumps(default_progression_dict()),
        iv_json=json.dumps(_iv_dict(cfg.interventions)),
        vaccination_open=eng.vaccination_open,
        **init, **{f"state_{c}": np.stack(v) for c, v in states.items()}, **hz)


def independent_fixture(name, n, horizon, seed, interventions, infections=8):
    """The reference's naive oracle in independent-edges mode (oracle.py:185-192:
    one Bernoulli per incident edge, keyed INFECTION_EDGE draws k = j over the
    sorted contributions), on its own reference-realizer graphs."""
    from epivec.oracle import OracleSim, agents_from_columns
    pop = default_population_dict()
    pop["n_agents"] = n
    cfg = scenario_from_dict({"population": pop, "horizon": horizon, "replications": 1,
                              "base_seed": seed, "initial_infections": infections,
                              "interventions": interventions}, name=name)
    rseed = replication_seed(cfg.base_seed, 0)
    cols, realizer = initialize_run(cfg, rseed)
    init = {f"init_{c}": getattr(cols, c).copy() for c in ALL_COLS}
    sim = OracleSim(agents_from_columns(cols), cfg.disease, cfg.progression, cfg.interventions,
                    rseed, mode=OracleSim.INDEPENDENT)
    srcs, dsts, kinds, states = [], [], [], {c: [] for c in DYNAMIC_COLUMNS}
    for step in range(horizon):
        g = realizer.realize(step, sim.column("stage") == 10)
        sim.step(g)
        srcs.append(g.src); dsts.append(g.dst); kinds.append(g.kind)
        for c in DYNAMIC_COLUMNS:
            states[c].append(sim.column(c).astype(getattr(cols, c).dtype))
    offs = np.concatenate(([0], np.cumsum([len(s) for s in srcs])))
    np.savez_compressed(
        OUT / f"traj_{name}.npz", seed=np.uint64(rseed), horizon=horizon,
        edge_offsets=offs, src=np.concatenate(srcs), dst=np.concatenate(dsts),
        kind=np.concatenate(kinds), events=np.zeros((horizon, 7), dtype=np.int64),
        disease_json=json.dumps(default_disease_dict()),
        table_json=json.dumps(default_progression_dict()),
        iv_json=json.dumps(_iv_dict(cfg.interventions)),
        vaccination_open=sim.vaccination_open,
        **init, **{f"state_{c}": np.stack(v) for c, v in states.items()})


ALL_IV = {
    "quarantine": {"enabled": True, "dropout_prob": 0.05},
    "testing": {"enabled": True, "kind": "rt-pcr"},
    "den": {"enabled": True, "app_adoption": 0.4, "compliance_prob": 0.8},
    "vaccination": {"enabled": True, "strategy": "delayed", "daily_rate": 0.01,
                    "start_trigger": 0.01, "immunity_mode": "sterilizing"},
}
NONSTER_IV = {
    "quarantine": {"enabled": True, "dropout_prob": 0.3},
    "testing": {"enabled": True, "kind": "rapid-poc", "false_positive_prob": 0.02},
    "den": {"enabled": True, "app_adoption": 0.7, "compliance_prob": 0.9, "lookback": 3},
    "vaccination": {"enabled": True, "strategy": "delayed-except-elderly",
                    "daily_rate": 0.05, "start_trigger": 0.0, "dose1_latency": 0,
                    "dose2_latency": 0, "dose_gap": 3, "dose1_efficacy": 0.6,
                    "dose2_efficacy": 0.9, "immunity_mode": "non-sterilizing"},
}
STD_IV = {
    "quarantine": {"enabled": True, "dropout_prob": 0.0, "duration": 5},
    "testing": {"enabled": True, "kind": "rapid-antigen"},
    "vaccination": {"enabled": True, "strategy": "standard", "daily_rate": 0.02,
                    "start_trigger": 0.02, "dose_gap": 4, "dose1_latency": 2},
}


def series_fixture():
    """Row f3 (output): the reference's RunResult CSV, summarize() quartiles
    and both summary CSV layouts, from real replications and from synthetic
    ensembles (regenerated in the test from the same numpy seed)."""
    from epivec.runner import (RunResult, run_replication, summarize, summary_to_csv,
                               summary_to_long_csv)
    cfg = scenario_from_dict({"population": dict(default_population_dict(), n_agents=300), "horizon": 15,
                              "base_seed": 2, "replications": 7, "initial_infections": 10})
    runs = [run_replication(cfg, i) for i in range(7)]
    summ = summarize(runs)
    out = {"run_data": runs[0].data, "run_seed": runs[0].seed, "run_csv": np.frombuffer(runs[0].to_csv().encode(), np.uint8),
           "runs_data": np.stack([r.data for r in runs]),
           "sum_wide": np.frombuffer(summary_to_csv(summ).encode(), np.uint8),
           "sum_long": np.frombuffer(summary_to_long_csv(summ).encode(), np.uint8)}
    for R, H, seed in ((1, 4, 10), (2, 4, 11), (5, 6, 12), (1000, 5, 13), (4096, 2, 14)):
        data = np.random.default_rng(seed).integers(0, 100_000, size=(R, H, 19), dtype=np.int64)
        s = summarize([RunResult(replication=i, seed=0, data=data[i]) for i in range(R)])
        out[f"synth_{R}_{H}_{seed}"] = np.stack([s[m] for m in s])
    np.savez_compressed(OUT / "series.npz", **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["series"]:
        series_fixture()
        sys.exit(0)
    if sys.argv[1:] == ["independent"]:
        independent_fixture("indep_noiv", 800, 45, 21, {}, infections=20)
        independent_fixture("indep_alliv", 300, 30, 4, ALL_IV, infections=8)
        sys.exit(0)
    rng_fixture()
    progression_fixture()
    priority_fixture()
    trajectory_fixture("noiv", 2000, 60, 3, {}, infections=20, record_gather=(10, 30, 45))
    trajectory_fixture("alliv", 300, 40, 1, ALL_IV, infections=8, record_gather=(20,))
    trajectory_fixture("nonster", 200, 30, 11, NONSTER_IV, infections=10)
    trajectory_fixture("stdvax", 250, 35, 5, STD_IV, infections=10)
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
