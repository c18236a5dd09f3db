"""GPU parity of the drop-in engine (graph-in mode) against the oracle and the
reference-generated trajectories.  Bar: bitwise for every state column and
event count; fp32 hazard within 1e-5 relative."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import engine_np, rng_np
from paper_2110_04421_b200 import _native as N
from paper_2110_04421_b200.engine import GpuEngine
from paper_2110_04421_b200.errors import InvariantViolation
from paper_2110_04421_b200.graph import StepGraph
from paper_2110_04421_b200.interventions import InterventionConfig
from paper_2110_04421_b200.stages import NetworkKind, Stage
from paper_2110_04421_b200.state import AgentColumns

from golden_io import Trajectory, compare_state, load

pytestmark = pytest.mark.gpu


def test_device_uniforms_match_reference_vectors():
    lib = N.lib()
    z = load("rng.npz")
    ids = torch.from_numpy(z["ids"]).cuda()
    for name in z.files:
        if not name.startswith("vec_"):
            continue
        s, t, p, k = (int(x) for x in name[4:].split("_"))
        out = torch.empty(ids.numel(), dtype=torch.float64, device="cuda")
        N.check(lib.epi_uniforms(s & (2**64 - 1), t, p, N.ptr(ids), ids.numel(), k, N.ptr(out),
                                 N.stream_handle()))
        assert np.array_equal(out.cpu().numpy(), z[name]), name
    out = torch.empty(5, dtype=torch.float64, device="cuda")
    for key, want in zip(z["keys"].tolist(), z["scalar"]):
        s, t, p, a, k = key
        one = torch.tensor([a], dtype=torch.int64, device="cuda")
        N.check(lib.epi_uniforms(s, t, p, N.ptr(one), 1, k, N.ptr(out), N.stream_handle()))
        assert out[0].item() == want


@pytest.mark.parametrize("name", ["noiv", "alliv", "nonster", "stdvax"])
def test_engine_replays_reference_trajectory_bitwise(name):
    tr = Trajectory(name)
    cols = tr.initial_cols()
    eng = GpuEngine(cols, tr.disease, tr.table, tr.iv, tr.seed)
    for step in range(tr.horizon):
        g = tr.graph(step)
        want_h = tr.hazard(step)
        if want_h is not None:
            got_h = eng.gather_exposure(g)
            assert np.array_equal(got_h, want_h), f"hazard differs at step {step}"
            h32 = eng.gather_exposure_f32(g).astype(np.float64)
            nz = want_h > 0
            assert np.all(np.abs(h32[nz] - want_h[nz]) <= 1e-5 * want_h[nz])
            assert np.all(h32[~nz] == 0)
        ev = eng.step(g)
        got = [ev.n_edges, ev.new_infections, ev.deaths, ev.hospitalizations,
               ev.tests_administered, ev.doses_given, ev.notifications_sent]
        assert got == tr.events[step].tolist(), f"events differ at step {step}: {got}"
        compare_state(cols, tr, step)
    assert eng.vaccination_open == bool(tr.z["vaccination_open"])


def test_engine_matches_oracle_on_random_graphs_with_injected_hazard():
    tr = Trajectory("alliv")
    rng = np.random.default_rng(3)
    cols_g, cols_o = tr.initial_cols(), tr.initial_cols()
    eng = GpuEngine(cols_g, tr.disease, tr.table, tr.iv, tr.seed)
    ora = engine_np.OracleEngine(cols_o, tr.disease, tr.table, tr.iv, tr.seed)
    for step in range(tr.horizon):
        g = tr.graph(step)
        perm = rng.permutation(g.n_edges)
        shuffled = StepGraph(step, g.src[perm], g.dst[perm], g.kind[perm])
        ev_g, ev_o = eng.step(shuffled), ora.step(g)
        assert ev_g.new_infections == ev_o.new_infections
        for c in ("stage", "infected_at", "next_stage", "next_transition_at",
                  "quarantine_until", "vaccine_status", "immune", "den_test_due_at"):
            assert np.array_equal(getattr(cols_g, c), getattr(cols_o, c)), (step, c)


def test_injected_uniforms_drive_stage_and_timer_bitwise():
    """Stage/timer update given the same injected uniforms and hazard."""
    tr = Trajectory("noiv")
    cols_g, cols_o = tr.initial_cols(), tr.initial_cols()
    n = tr.n
    eng = GpuEngine(cols_g, tr.disease, tr.table, tr.iv, seed=0)
    rng = np.random.default_rng(11)
    for step in range(20):
        hz = rng.exponential(0.3, n) * (rng.random(n) < 0.5)
        draws = {p: rng.integers(0, 2**53, n).astype(np.float64) * 2.0**-53 for p in (1, 3, 4, 5)}
        inj = {p: torch.from_numpy(v).cuda() for p, v in draws.items()}
        eng.step_with_hazard(hz, injected=inj)
        # oracle phases 1-2 with the same draws
        c = cols_o
        target = engine_np.target_mask(c, True)
        hit = np.flatnonzero(target & (draws[1] < 1.0 - np.exp(-np.where(target, hz, 0.0))))
        entry = engine_np.pick(tr.table.rules[0], c.age_band[hit], draws[3][hit])
        c.stage[hit] = entry
        c.infected_at[hit] = step
        nxt, d = engine_np.schedule(tr.table, entry, c.age_band[hit], draws[4][hit], draws[5][hit])
        c.next_stage[hit] = nxt
        c.next_transition_at[hit] = step + d
        due = np.flatnonzero(c.next_transition_at == step)
        dest = c.next_stage[due].copy()
        c.stage[due] = dest
        fin = (dest == 8) | (dest == 10)
        c.next_stage[due[fin]] = -1
        c.next_transition_at[due[fin]] = -1
        rest = due[~fin]
        nxt, d = engine_np.schedule(tr.table, c.stage[rest], c.age_band[rest], draws[4][rest], draws[5][rest])
        c.next_stage[rest] = nxt
        c.next_transition_at[rest] = step + d
        for col in ("stage", "infected_at", "next_stage", "next_transition_at"):
            assert np.array_equal(getattr(cols_g, col), getattr(cols_o, col)), (step, col)


def test_hard_errors():
    cols = AgentColumns.allocate(3)
    eng = GpuEngine(cols, Trajectory("noiv").disease, Trajectory("noiv").table, InterventionConfig(), 0)
    with pytest.raises(InvariantViolation, match="clock"):
        eng.step(StepGraph.empty(5))
    bad = StepGraph(0, np.array([0], np.int32), np.array([7], np.int32), np.zeros(1, np.int8))
    with pytest.raises(InvariantViolation, match="n_agents"):
        eng.step(bad)
    loop = StepGraph(0, np.array([1], np.int32), np.array([1], np.int32), np.zeros(1, np.int8))
    with pytest.raises(InvariantViolation, match="self-loop"):
        eng.step(loop)
    ev = eng.step(StepGraph.empty(0))
    assert ev.n_edges == 0 and ev.new_infections == 0 and eng.clock == 1


def test_rejected_graph_leaves_the_engine_intact():
    """Out-of-range indices (huge and negative dst) are rejected without
    touching memory outside the row tables: the next valid graph still gives
    the hazard of a fresh engine bitwise."""
    tr = Trajectory("noiv")
    g = tr.graph(0)
    a = GpuEngine(tr.initial_cols(), tr.disease, tr.table, InterventionConfig(), tr.seed)
    b = GpuEngine(tr.initial_cols(), tr.disease, tr.table, InterventionConfig(), tr.seed)
    n = tr.n
    for d in (n, n + 70_000, 2 ** 31 - 1, -5):
        bad = StepGraph(0, np.concatenate([g.src, [0]]).astype(np.int32),
                        np.concatenate([g.dst, [d]]).astype(np.int32),
                        np.concatenate([g.kind, [0]]).astype(np.int8))
        with pytest.raises(InvariantViolation, match="n_agents"):
            a.step(bad)
    assert a.clock == 0
    assert np.array_equal(a.gather_exposure(g), b.gather_exposure(g))
    assert np.array_equal(a.gather_exposure(g), tr.hazard(0)) if tr.hazard(0) is not None else True


def test_star_graph_gather_equals_formula():
    from paper_2110_04421_b200.disease import edge_hazard
    tr = Trajectory("noiv")
    n_leaves = 6
    cols = AgentColumns.allocate(n_leaves + 1)
    cols.stage[0] = int(Stage.MILD_SYMPTOMATIC)
    cols.infected_at[0] = 0
    cols.next_stage[0] = int(Stage.RECOVERED)
    cols.next_transition_at[0] = 10_000
    eng = GpuEngine(cols, tr.disease, tr.table, InterventionConfig(), 0)
    eng.clock = 4
    leaves = np.arange(1, n_leaves + 1, dtype=np.int32)
    hub = np.zeros(n_leaves, dtype=np.int32)
    g = StepGraph(4, np.concatenate([hub, leaves]), np.concatenate([leaves, hub]),
                  np.full(2 * n_leaves, int(NetworkKind.RANDOM), np.int8))
    h = eng.gather_exposure(g)
    assert np.all(h[1:] == edge_hazard(4, False, 0, 2, tr.disease))
    assert h[0] == 0.0


@pytest.mark.parametrize("name", ["indep_noiv", "indep_alliv"])
def test_engine_independent_edges_mode_replays_reference_oracle(name):
    """Row f4: GpuEngine in the reference oracle's independent-edges mode
    (oracle.py:185-192) replays the recorded reference trajectory bitwise."""
    from golden_io import compare_state
    from paper_2110_04421_b200.engine import GpuEngine
    tr = Trajectory(name)
    cols = tr.initial_cols()
    eng = GpuEngine(cols, tr.disease, tr.table, tr.iv, tr.seed, infection_mode="independent")
    for step in range(tr.horizon):
        eng.step(tr.graph(step))
        compare_state(cols, tr, step)


@pytest.mark.parametrize("seed", [0, 1])
def test_gather_canonical_order_on_skewed_rows(seed):
    """Graph load canonical order (k_rows_sort: register networks for rows of
    <= 8 / 16 / 32 entries, insertion beyond) on rows of 0..90 in-edges with
    duplicates and all kinds, shuffled: fp64 hazard bitwise vs the oracle."""
    tr = Trajectory("noiv")
    rng = np.random.default_rng(seed)
    n = 400
    cols = AgentColumns.allocate(n)
    inf = rng.random(n) < 0.5
    cols.stage[inf] = int(Stage.MILD_SYMPTOMATIC)
    cols.infected_at[inf] = rng.integers(0, 6, int(inf.sum()))
    cols.next_stage[inf] = int(Stage.RECOVERED)
    cols.next_transition_at[inf] = 10_000
    cols.age_band[:] = rng.integers(0, 9, n)
    lens = np.concatenate([np.arange(91), rng.integers(0, 40, n - 91)])
    dst = np.repeat(np.arange(n, dtype=np.int32), lens)
    src = rng.integers(0, n - 1, len(dst)).astype(np.int32)
    src[src >= dst] += 1                                  # no self loops
    kind = rng.integers(0, 3, len(dst)).astype(np.int8)
    assert np.unique(np.stack([src, dst, kind]), axis=1).shape[1] < len(dst)   # duplicate edges present
    p = rng.permutation(len(dst))
    g = StepGraph(6, src[p], dst[p], kind[p])
    eng = GpuEngine(cols.copy(), tr.disease, tr.table, InterventionConfig(), 0)
    eng.clock = 6
    want = engine_np.hazard(cols, tr.disease, 6, g, True)
    assert np.count_nonzero(want) > n // 4
    assert np.array_equal(eng.gather_exposure(g), want)


def test_gather_canonical_order_on_hub_rows():
    """Hubs: rows of 33 .. 100 000 in-edges go to the block sort
    (k_rows_sort_long: shared-memory bitonic tiles + merge-path passes); the
    fp64 hazard, summed in canonical (dst, src, kind) order, stays bitwise
    equal to the oracle's lexsort + bincount (engine.py:98-108)."""
    tr = Trajectory("noiv")
    rng = np.random.default_rng(5)
    n = 200_000
    cols = AgentColumns.allocate(n)
    long = [33, 64, 100, 1000, 8191, 8192, 8193, 20_000, 100_000]
    inf = rng.random(n) < 0.3
    inf[:len(long)] = False                               # the hubs are susceptible targets
    cols.stage[inf] = int(Stage.MILD_SYMPTOMATIC)
    cols.infected_at[inf] = rng.integers(0, 6, int(inf.sum()))
    cols.next_stage[inf] = int(Stage.RECOVERED)
    cols.next_transition_at[inf] = 10_000
    cols.age_band[:] = rng.integers(0, 9, n)
    lens = np.concatenate([long, rng.integers(0, 12, n - len(long))])
    dst = np.repeat(np.arange(n, dtype=np.int32), lens)
    src = rng.integers(0, n - 1, len(dst)).astype(np.int32)
    src[src >= dst] += 1
    kind = rng.integers(0, 3, len(dst)).astype(np.int8)
    p = rng.permutation(len(dst))
    g = StepGraph(6, src[p], dst[p], kind[p])
    eng = GpuEngine(cols.copy(), tr.disease, tr.table, InterventionConfig(), 0)
    eng.clock = 6
    want = engine_np.hazard(cols, tr.disease, 6, g, True)
    got = eng.gather_exposure(g)
    assert np.count_nonzero(want[:len(long)]) == len(long)
    assert np.array_equal(got, want), np.flatnonzero(got != want)[:10]
    # a second load on the same engine (long-row list reset between loads)
    g2 = StepGraph(6, src[::-1].copy(), dst[::-1].copy(), kind[::-1].copy())
    assert np.array_equal(eng.gather_exposure(g2), want)


@pytest.mark.parametrize("case", ["stage_range", "no_timestamp", "neg_hazard"])
def test_invariant_flags_raise(case):
    """state.py:90-102 through the device flags (rec_agent -> EPI_REC_FLAGS):
    a stage outside 0..10 and a non-susceptible, non-vaccinated agent without
    an infection timestamp raise InvariantViolation when checking (and pass
    silently when not, as the reference's check_invariants=False); a negative
    hazard (engine.py:157-158) raises in every mode."""
    tr = Trajectory("noiv")
    for check in (True, False):
        cols = AgentColumns.allocate(64)
        if case == "stage_range":
            cols.stage[5] = 11
        elif case == "no_timestamp":
            cols.stage[9] = int(Stage.RECOVERED)          # infected_at stays NEVER
        eng = GpuEngine(cols, tr.disease, tr.table, InterventionConfig(), 0, check_invariants=check)
        if case == "neg_hazard":
            hz = np.zeros(64)
            hz[3] = -1e-3
            with pytest.raises(InvariantViolation, match="negative hazard"):
                eng.step_with_hazard(hz)
            continue
        msg = "stage out of range" if case == "stage_range" else "without infection timestamp"
        if check:
            with pytest.raises(InvariantViolation, match=msg):
                eng.step(StepGraph.empty(0))
        else:
            eng.step(StepGraph.empty(0))
            assert eng.clock == 1


def test_engine_refuses_steps_after_invalidation():
    tr = Trajectory("noiv")
    eng = GpuEngine(AgentColumns.allocate(8), tr.disease, tr.table, InterventionConfig(), 0)
    eng.invalidate("realizer failed at step 0: edge output capacity exceeded")
    with pytest.raises(InvariantViolation, match="invalid"):
        eng.step(StepGraph.empty(0))


def test_recycled_context_buffers_replay_bitwise():
    """Contexts return their device buffers to a process-wide cache on
    destruction and the next context of the same sizes reuses them
    (epi_destroy): the reference trajectory with every intervention replays
    bitwise on engines built one after another, each on buffers the previous
    one left dirty, with engines of other sizes built in between."""
    import gc
    tr = Trajectory("alliv")
    for rep in range(4):
        cols = tr.initial_cols()
        eng = GpuEngine(cols, tr.disease, tr.table, tr.iv, tr.seed)
        for step in range(tr.horizon):
            ev = eng.step(tr.graph(step))
            got = [ev.n_edges, ev.new_infections, ev.deaths, ev.hospitalizations,
                   ev.tests_administered, ev.doses_given, ev.notifications_sent]
            assert got == tr.events[step].tolist(), f"rep {rep}: events differ at step {step}"
            compare_state(cols, tr, step)
        del eng
        gc.collect()
        # engines of other sizes in between, stepped once (their dirty
        # buffers join the cache too)
        rng = np.random.default_rng(rep)
        for n in (17, 300 + rep):
            other = AgentColumns.allocate(n)
            e2 = GpuEngine(other, tr.disease, tr.table, tr.iv, tr.seed)
            src = rng.integers(0, n, 4 * n).astype(np.int32)
            dst = (src + 1 + rng.integers(0, n - 1, 4 * n)) % n
            e2.step(StepGraph(0, src, dst.astype(np.int32), np.zeros(4 * n, np.int8)))
            del e2
        gc.collect()
