"""Row f3: config-population synthesis on the device, bitwise against the
host restatement (confignet.synthesize), and a device-built simulation equal
to a host-built one."""

import time

import numpy as np
import pytest

from paper_2110_04421_b200.confignet import ConfigNetworkSpec, DevicePopulation, synthesize

pytestmark = pytest.mark.gpu

SPECS = {
    "config0": dict(n_agents=10_000, worker_bands=(), initial_infections=10),
    "config1": dict(n_agents=100_000),
    "ragged": dict(n_agents=1_237, initial_infections=30),
    "one_agent": dict(n_agents=1, initial_infections=1),
    "big_households": dict(n_agents=20_011, household_sizes=(24, 32), household_probs=(0.5, 0.5)),
    "no_draws": dict(n_agents=5_000, colleague_draws=0),
    "narrow_workplaces": dict(n_agents=50_000, wp_min=2, wp_max=3, worker_bands=(0, 1, 2, 3, 4, 5, 6, 7, 8)),
    "wide_workplaces": dict(n_agents=50_000, wp_min=200, wp_max=255),
    "no_seeds": dict(n_agents=3_000, initial_infections=0),
}
FIELDS = ("age_band", "household_id", "hh_off", "hh_size", "wp_id", "wp_local", "wp_base", "wp_size",
          "wp_members", "seeds")


@pytest.mark.parametrize("name", sorted(SPECS))
@pytest.mark.parametrize("seed", [0, 12345])
def test_device_population_bitwise(name, seed):
    spec = ConfigNetworkSpec.config(1, **SPECS[name])
    want = synthesize(spec, seed)
    got = DevicePopulation(spec, seed).to_host()
    for f in FIELDS:
        a, b = getattr(got, f), getattr(want, f)
        assert a.shape == b.shape and np.array_equal(a.astype(np.int64), b.astype(np.int64)), f


def test_device_population_drives_the_same_simulation():
    from paper_2110_04421_b200.sim import ConfigSimulation
    spec = ConfigNetworkSpec.config(1, n_agents=20_000, initial_infections=40)
    a = ConfigSimulation.create(spec, seed=4, mode="fused", horizon=40)
    b = ConfigSimulation.create(spec, seed=4, mode="fused", horizon=40, on_device=True)
    a.run()
    b.run()
    assert np.array_equal(a.records(), b.records())


def test_ten_million_agents_in_milliseconds():
    import torch
    spec = ConfigNetworkSpec.config(3)
    DevicePopulation(ConfigNetworkSpec.config(1, n_agents=1000), 0)    # warm-up (module load)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pop = DevicePopulation(spec, 0)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    assert dt < 1.0, dt
    assert int(pop.seeds.numel()) == spec.initial_infections
    assert 18.5 < float(pop.wp_size.double().mean()) < 31.5
