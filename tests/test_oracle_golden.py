"""Pin the CPU oracle (and host-side table builders) to vectors produced by
the unmodified reference (tests/golden/make_golden.py)."""

import json

import numpy as np
import pytest

from oracle import engine_np, rng_np
from paper_2110_04421_b200 import keyed
from paper_2110_04421_b200.disease import day_weight_table
from paper_2110_04421_b200.interventions import Strategy, priority_sort_key
from paper_2110_04421_b200.progression import ProgressionTable

from golden_io import Trajectory, compare_state, load


def test_rng_scalar_and_prefix_golden():
    z = load("rng.npz")
    for key, want, pre in zip(z["keys"].tolist(), z["scalar"], z["prefixes"].tolist()):
        s, t, p, a, k = key
        assert rng_np.uniform(s, t, p, a, k) == want
        assert keyed.uniform(s, t, p, a, k) == want
        assert rng_np.prefix(s, t, p) == pre == keyed.key_prefix(s, t, p)
    d = z["derived"].tolist()
    assert keyed.derive_seed(0, 64, 0) == d[0] == keyed.replication_seed(0, 0)
    assert keyed.derive_seed(42, 64, 3) == d[1]
    assert keyed.derive_seed(7, 67, 12, 5) == d[2]


def test_rng_vectors_golden():
    z = load("rng.npz")
    ids = z["ids"]
    for name in z.files:
        if name.startswith("vec_"):
            s, t, p, k = (int(x) for x in name[4:].split("_"))
            assert np.array_equal(rng_np.uniforms(s, t, p, ids, k), z[name])


def test_day_weights_golden():
    z = load("day_weights.npz")
    for name in z.files:
        m, s = (float(x) for x in name[2:].split("_"))
        assert np.array_equal(day_weight_table(m, s), z[name])


def _table():
    z = load("progression.npz")
    return z, ProgressionTable.from_dict(json.loads(str(z["table_json"])))


def test_oracle_schedule_golden():
    z, table = _table()
    ids = np.arange(len(z["ages"]), dtype=np.int64)
    u_b, u_d = rng_np.uniforms(99, 4, 4, ids), rng_np.uniforms(99, 4, 5, ids)
    for s in range(1, 8):
        nxt, delay = engine_np.schedule(table, np.full(len(ids), s, np.int8), z["ages"], u_b, u_d)
        assert np.array_equal(nxt, z[f"next_{s}"]) and np.array_equal(delay, z[f"delay_{s}"])
    entry = engine_np.pick(table.rules[0], z["ages"], rng_np.uniforms(99, 4, 3, ids))
    assert np.array_equal(entry, z["entry"])


def _device_delay(table, stage, age, u_b, u_d):
    """Host restatement of the device lookup (csrc/epi_common.cuh) for the CPU
    suite: branch by cumulative table, delay = 1 + #(tau <= u)."""
    dev = table.device_tables()
    nt = dev["n_targets"][stage]
    j = min(int((u_b >= dev["cum"][stage, age, :nt]).sum()), nt - 1)
    tau = dev["taus"][dev["spec_of"][stage, j]]
    return dev["targets"][stage, j], 1 + int(np.searchsorted(tau, u_d, side="right"))


def test_threshold_tables_reproduce_reference_delays():
    z, table = _table()
    dev = table.device_tables()
    ids = np.arange(len(z["ages"]), dtype=np.int64)
    u_b, u_d = rng_np.uniforms(99, 4, 4, ids), rng_np.uniforms(99, 4, 5, ids)
    for s in range(1, 8):
        nt = dev["n_targets"][s]
        cum = dev["cum"][s][z["ages"]][:, :nt]
        j = np.minimum((u_b[:, None] >= cum).sum(1), nt - 1)
        spec = dev["spec_of"][s][j]
        delay = np.empty(len(ids), np.int64)
        for sp in np.unique(spec):
            m = spec == sp
            delay[m] = 1 + np.searchsorted(dev["taus"][sp], u_d[m], side="right")
        assert np.array_equal(dev["targets"][s][j], z[f"next_{s}"])
        assert np.array_equal(delay, z[f"delay_{s}"])
        for i, u in enumerate(z["edge_u"]):
            nxt, d = _device_delay(table, s, 0, u, u)
            assert (nxt, d) == (z[f"edge_next_{s}"][i], z[f"edge_delay_{s}"][i])


@pytest.mark.parametrize("strategy", list(Strategy))
def test_priority_golden(strategy):
    z = load("priority.npz")
    want = z[f"order_{int(strategy)}"]
    assert np.array_equal(engine_np.priority_order(strategy, 6, z["ages"], z["dose2"], z["ids"]), want)
    assert np.array_equal(priority_sort_key(strategy, 6, z["ages"], z["dose2"], z["ids"]), want)


@pytest.mark.parametrize("name", ["noiv", "alliv", "nonster", "stdvax"])
def test_oracle_replays_reference_trajectory(name):
    tr = Trajectory(name)
    cols = tr.initial_cols()
    eng = engine_np.OracleEngine(cols, tr.disease, tr.table, tr.iv, tr.seed)
    for step in range(tr.horizon):
        g = tr.graph(step)
        want_h = tr.hazard(step)
        if want_h is not None:
            assert np.array_equal(eng.gather_exposure(g), want_h)
        ev = eng.step(g)
        got = [ev.n_edges, ev.new_infections, ev.deaths, ev.hospitalizations,
               ev.tests_administered, ev.doses_given, ev.notifications_sent]
        assert got == tr.events[step].tolist(), f"events differ at step {step}"
        compare_state(cols, tr, step)
    assert eng.vaccination_open == bool(tr.z["vaccination_open"])


@pytest.mark.parametrize("name", ["noiv", "alliv"])
def test_reference_realizer_restatement_reproduces_recorded_graphs(name):
    """oracle/graphs_np restates GraphRealizer draw for draw (graphs.py:176-240)."""
    from oracle.graphs_np import ReferenceRealizer
    from paper_2110_04421_b200.defaults import POPULATION
    tr = Trajectory(name)
    z = tr.z
    rr = ReferenceRealizer(tr.seed, z["init_household_id"], z["init_occupation"],
                           z["init_random_degree"], POPULATION["networks"]["occupation_mean_interactions"],
                           POPULATION["networks"]["rewire_beta"])
    for step in range(min(tr.horizon, 12)):
        dead = (z["init_stage"] if step == 0 else tr.state(step - 1, "stage")) == 10
        s, d, k = rr.realize(step, dead)
        g = tr.graph(step)
        assert np.array_equal(s, g.src) and np.array_equal(d, g.dst) and np.array_equal(k, g.kind)


@pytest.mark.parametrize("name", ["indep_noiv", "indep_alliv"])
def test_oracle_independent_edges_mode_replays_reference(name):
    """Row f4: the reference's naive oracle in independent-edges mode
    (oracle.py:185-192), recorded by make_golden.py, replayed bitwise."""
    tr = Trajectory(name)
    cols = tr.initial_cols()
    eng = engine_np.OracleEngine(cols, tr.disease, tr.table, tr.iv, tr.seed,
                                 infection_mode="independent")
    for step in range(tr.horizon):
        eng.step(tr.graph(step))
        compare_state(cols, tr, step)
    assert int(np.sum(cols.infected_at != -1)) > int(np.sum(tr.z["init_infected_at"] != -1))
