"""Population mirror (population.py:43-177) vs the reference's recorded
initialize_run outputs (tests/golden/traj_*.npz, made by make_golden.py)."""

import numpy as np
import pytest

from golden_io import load as load_npz
from paper_2110_04421_b200.errors import ConfigError
from paper_2110_04421_b200.population import PopulationSpec, choose_seeds, synthesize
from paper_2110_04421_b200.state import AgentColumns

TRAJ = ["noiv", "alliv", "nonster", "stdvax"]


@pytest.mark.parametrize("name", TRAJ)
def test_synthesis_matches_reference(name):
    d = load_npz(f"traj_{name}.npz")
    n = len(d["init_age_band"])
    cols = synthesize(PopulationSpec.default(n), int(d["seed"]))
    for c in ("age_band", "occupation", "household_id", "random_degree"):
        assert np.array_equal(getattr(cols, c), d[f"init_{c}"]), c


@pytest.mark.parametrize("name", TRAJ)
def test_seed_choice_matches_reference(name):
    d = load_npz(f"traj_{name}.npz")
    n = len(d["init_age_band"])
    cols = synthesize(PopulationSpec.default(n), int(d["seed"]))
    infected = np.nonzero(d["init_infected_at"] == 0)[0]
    ids = choose_seeds(cols, len(infected), int(d["seed"]))
    assert np.array_equal(ids, infected)


def test_spec_validation():
    with pytest.raises(ConfigError):
        PopulationSpec.default(0)
    from paper_2110_04421_b200.defaults import POPULATION
    bad = dict(POPULATION, age_distribution=[0.5] * 9)
    with pytest.raises(ConfigError):
        PopulationSpec.from_dict(bad)
    cols = AgentColumns.allocate(3)
    with pytest.raises(ConfigError):
        choose_seeds(cols, 4, 0)
