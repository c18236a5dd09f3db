"""The TIMED kernels against the oracle, on the values they consume.

The bench times the fp32 fused day kernels: `k_fused_step` (day 0 of a run,
and every day of the per-day path), `k_fused_run` (days 1.. of a persistent
run, config 1) and `k_iv_run` (days 1.. of a persistent intervention run,
config 2).  They build lambda from per-kind push-table sums, a different
factorisation from the csr/graph-in kernels, so they get their own checks:

1. lambda: the hazard each kernel feeds its Bernoulli (exported through
   `epi_set_lambda_probe`) is within 1e-5 relative of the oracle's
   `gather_exposure` (engine.py:77-117) on the restated generator's graph of
   the same day, evaluated on the device's own state of that day, for every
   agent of a 100k-agent config-1 population, on days from the first to the
   last, the epidemic peak included; exact zeros where the oracle is zero.
2. stage/timer (and, with interventions, every DYNAMIC_COLUMN): the oracle
   engine stepped from the device's state of day t with the device's lambda
   injected (the same keyed draws, engine.py:153-347) equals the device's
   state of day t + 1 bit for bit, and the day's events equal the record row.

The device state of day t comes from `reset(); run(t)`: the run is
deterministic (bitwise equal reruns, tests/test_gpu_persistent.py), and in
`run(t + 1)` day t is executed by the persistent kernel whenever t >= 1.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import confignet_np, engine_np
from paper_2110_04421_b200.confignet import ConfigNetworkSpec
from paper_2110_04421_b200.graph import StepGraph
from paper_2110_04421_b200.interventions import (DenConfig, InterventionConfig, TestKind,
                                                 VaccinePolicy)
from paper_2110_04421_b200.sim import ConfigSimulation
from paper_2110_04421_b200.state import DYNAMIC_COLUMNS

pytestmark = pytest.mark.gpu

REL = 1e-5          # north_star: per-agent lambda within 1e-5 relative (fp32)
DEAD = 10


def config2_interventions(dose_gap=21):
    """BASELINE.json configs[2] through the reference's knobs."""
    return InterventionConfig(quarantine_enabled=True, testing_enabled=True,
                              test_kind=TestKind("cfg2", 0.05, 2, 2), den_enabled=True,
                              den=DenConfig(0.5), vaccination_enabled=True,
                              vaccine=VaccinePolicy(daily_rate=0.01, dose1_efficacy=0.5,
                                                    dose2_efficacy=0.9, dose_gap=dose_gap))


def _state_at(sim, t):
    """Device state at the start of day t (and the vaccination latch)."""
    sim.reset()
    if t:
        sim.run(t)
    torch.cuda.synchronize()
    return sim.host_columns(), bool(int(sim.vax[0].item()))


def _lambda_of_day(sim, t):
    """The fp32 hazard of day t as the kernels consume it, plus the state and
    record of the following day; day t runs inside k_fused_run / k_iv_run
    when t >= 1 (persistent runs), inside k_fused_step otherwise."""
    buf = sim.lambda_probe(t, 1)
    sim.reset()
    sim.run(t + 1)
    torch.cuda.synchronize()
    lam = buf[0].cpu().numpy()
    sim.lambda_probe(0, 0)
    return lam, sim.host_columns(), sim.records()[t]


def check_lambda(got, ref):
    """|got - ref| <= 1e-5 * ref where the oracle is positive, exact zero
    elsewhere.  Returns the number of positive hazards compared."""
    assert not np.isnan(got).any(), "agents without an exported hazard"
    nz = ref > 0
    rel = np.abs(got[nz].astype(np.float64) - ref[nz]) / ref[nz]
    bad = np.flatnonzero(nz)[rel > REL]
    assert not len(bad), (f"{len(bad)} agents beyond 1e-5: agent {bad[0]} got {got[bad[0]]!r} "
                          f"want {ref[bad[0]]!r} (max rel {rel.max():.3g})")
    zbad = np.flatnonzero(~nz & (got != 0))
    assert not len(zbad), f"agent {zbad[0]}: got {got[zbad[0]]!r}, oracle 0"
    return int(nz.sum())


class _InjectedHazard(engine_np.OracleEngine):
    """The oracle engine with the device's hazard injected into phase 1."""

    def __init__(self, *a, lam, **kw):
        super().__init__(*a, **kw)
        self.lam = lam.astype(np.float64)

    def gather_exposure(self, graph):
        return self.lam


def _graph(sim, t, cols):
    s, d, k = confignet_np.realize(sim.population, sim.seed, t, cols.stage == DEAD)
    return StepGraph(t, s, d, k)


def _check_day(sim, t, iv):
    cols, vax_open = _state_at(sim, t)
    lam, nxt, rec = _lambda_of_day(sim, t)
    g = _graph(sim, t, cols)
    ref = engine_np.hazard(cols, sim.disease, t, g, int(iv.vaccine.immunity_mode) == 0)
    n_pos = check_lambda(lam, ref)
    # stage/timer bitwise with the device's lambda and the same keyed draws
    eng = _InjectedHazard(cols, sim.disease, sim.table, iv, sim.seed, lam=lam)
    eng.clock = t
    eng.vaccination_open = vax_open
    if eng.ring is not None:
        for s in range(max(0, t - iv.den.lookback), t):
            eng.ring.push(_graph(sim, s, _state_at(sim, s)[0]))
    ev = eng.step(g)
    for c in DYNAMIC_COLUMNS:
        a, b = getattr(cols, c), getattr(nxt, c)
        if not np.array_equal(a, b):
            i = int(np.flatnonzero(a != b)[0])
            raise AssertionError(f"day {t} column {c} agent {i}: device {b[i]!r} oracle {a[i]!r}")
    row = engine_np.series_row(cols, ev)
    assert np.array_equal(rec[:19], row), (t, rec[:19], row)
    assert int(rec[19]) == ev.n_edges, (t, int(rec[19]), ev.n_edges)
    return n_pos


@pytest.fixture(scope="module")
def sim1():
    spec = ConfigNetworkSpec.config(1)
    sim = ConfigSimulation.create(spec, seed=11, mode="fused", horizon=180)
    assert sim.uses_persistent_run()
    return sim


@pytest.fixture(scope="module")
def peak_day(sim1):
    sim1.reset()
    sim1.run()
    return int(np.argmax(sim1.records()[:, 15]))      # new infections per day


def test_config1_peak_is_inside_the_horizon(peak_day):
    assert 20 < peak_day < 170


@pytest.mark.parametrize("day", [0, 1, 15, "peak", 60, 120, 178])
def test_fused_run_lambda_and_update_vs_oracle_config1(sim1, peak_day, day):
    t = peak_day if day == "peak" else day
    n_pos = _check_day(sim1, t, sim1.iv)
    if 1 <= t <= peak_day:
        assert n_pos > 0


def test_fused_step_per_day_path_lambda_vs_oracle():
    """The per-day k_fused_step path (persistent off): used on day 0 of every
    run, for populations above the persistent kernel's cap, and partitioned."""
    spec = ConfigNetworkSpec.config(1, n_agents=30_011, initial_infections=300)
    sim = ConfigSimulation.create(spec, seed=3, mode="fused", horizon=60, persistent=False)
    assert not sim.uses_persistent_run()
    for t in (5, 40):
        assert _check_day(sim, t, sim.iv) > 0


@pytest.mark.parametrize("gap", [21, 84])
def test_iv_run_lambda_and_update_vs_oracle_config2(gap):
    iv = config2_interventions(gap)
    spec = ConfigNetworkSpec.config(1, n_agents=60_000, initial_infections=100)
    sim = ConfigSimulation.create(spec, seed=4, mode="fused", horizon=180, interventions=iv)
    sim.run()
    rec = sim.records()
    peak = int(np.argmax(rec[:, 15]))
    assert rec[:, 17].sum() > 0 and rec[:, 16].sum() > 0      # doses given, tests administered
    for t in (1, 25, peak, 150):
        _check_day(sim, t, iv)


def test_csr_f32_message_pass_update_lambda_vs_oracle():
    """csr mode's fused message pass + update (k_msg_pass<1>)."""
    spec = ConfigNetworkSpec.config(1, n_agents=20_000, initial_infections=200)
    sim = ConfigSimulation.create(spec, seed=8, mode="csr", precision="f32", horizon=60)
    for t in (0, 30):
        _check_day(sim, t, sim.iv)


def test_lambda_check_detects_a_wrong_factor_or_a_missing_edge(sim1, peak_day):
    """The 1e-5 bar has the power to see one wrong per-kind factor or one
    missing in-edge: the same comparison fails against a perturbed oracle."""
    t = peak_day
    cols, _ = _state_at(sim1, t)
    lam, _, _ = _lambda_of_day(sim1, t)
    g = _graph(sim1, t, cols)
    ster = True
    d = sim1.disease
    old = d.network_scale.copy()
    try:
        d.network_scale[1] = old[1] * (1 + 4e-5)          # occupation factor off by 4e-5
        with pytest.raises(AssertionError):
            check_lambda(lam, engine_np.hazard(cols, d, t, g, ster))
    finally:
        d.network_scale[:] = old
    # drop one valid in-edge of one target
    ref = engine_np.hazard(cols, d, t, g, ster)
    tt = t - cols.infected_at[g.src].astype(np.int64)
    ok = (engine_np.INFECTIOUS[cols.stage[g.src]] & (tt >= 1) & (tt <= d.t_max)
          & (ref[g.dst] > 0) & (cols.quarantine_until[g.src] <= t))
    e = int(np.flatnonzero(ok)[0])
    keep = np.ones(len(g.src), bool)
    keep[e] = False
    g2 = StepGraph(t, g.src[keep], g.dst[keep], g.kind[keep])
    with pytest.raises(AssertionError):
        check_lambda(lam, engine_np.hazard(cols, d, t, g2, ster))
