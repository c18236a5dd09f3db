"""Packaged default parameter sets (placeholders, not clinically fitted).

Values restate the reference's shipped defaults
(`pkg/src/epivec/data/disease_params.json:3-9`,
`data/progression_table.json:4-67`, `data/population_spec.json:4-22`) as
Python literals so the GPU box needs no reference checkout.
"""

AGE_BANDS = 9

DISEASE = {
    "rate_scale": 3.3,
    "age_susceptibility": [0.40, 0.45, 0.70, 0.80, 0.90, 1.00, 1.10, 1.20, 1.30],
    "asymptomatic_factor": 0.55,
    "network_scale": {"household": 2.0, "occupation": 1.0, "random": 1.0},
    "mean_daily_interactions": 11.0,
    "infectiousness_mean_days": 7.0,
    "infectiousness_sd_days": 3.0,
}


def _edge(src, dst, probs, dur=None):
    e = {"from": src, "to": dst, "probability": list(probs)}
    if dur is not None:
        e["duration"] = dur
    return e


def _gamma(mean, sd):
    return {"family": "gamma", "mean": mean, "sd": sd}


_ONES = [1.0] * AGE_BANDS
_INCUBATION = {"family": "lognormal", "mu": 1.504, "sigma": 0.35}

PROGRESSION = {"edges": [
    _edge("susceptible", "asymptomatic",
          [0.50, 0.45, 0.42, 0.40, 0.38, 0.35, 0.32, 0.30, 0.30]),
    _edge("susceptible", "presymptomatic_mild",
          [0.49, 0.54, 0.56, 0.57, 0.57, 0.57, 0.55, 0.50, 0.42]),
    _edge("susceptible", "presymptomatic_severe",
          [0.01, 0.01, 0.02, 0.03, 0.05, 0.08, 0.13, 0.20, 0.28]),
    _edge("asymptomatic", "recovered", _ONES, _gamma(8.0, 3.0)),
    _edge("presymptomatic_mild", "mild_symptomatic", _ONES, _INCUBATION),
    _edge("presymptomatic_severe", "severe_symptomatic", _ONES, _INCUBATION),
    _edge("mild_symptomatic", "recovered", _ONES, _gamma(8.0, 3.0)),
    _edge("severe_symptomatic", "hospitalized",
          [0.30, 0.30, 0.35, 0.40, 0.45, 0.55, 0.65, 0.75, 0.85], _gamma(4.0, 1.5)),
    _edge("severe_symptomatic", "recovered",
          [0.70, 0.70, 0.65, 0.60, 0.55, 0.45, 0.35, 0.25, 0.15], _gamma(10.0, 3.0)),
    _edge("hospitalized", "critical_icu",
          [0.10, 0.10, 0.12, 0.15, 0.20, 0.25, 0.30, 0.35, 0.40], _gamma(3.0, 1.0)),
    _edge("hospitalized", "recovered",
          [0.90, 0.90, 0.88, 0.85, 0.80, 0.75, 0.70, 0.65, 0.60], _gamma(8.0, 2.5)),
    _edge("critical_icu", "dead",
          [0.25, 0.25, 0.28, 0.30, 0.35, 0.42, 0.50, 0.60, 0.70], _gamma(5.0, 2.0)),
    _edge("critical_icu", "recovered",
          [0.75, 0.75, 0.72, 0.70, 0.65, 0.58, 0.50, 0.40, 0.30], _gamma(7.0, 2.5)),
]}


def default_disease():
    from .disease import DiseaseParams
    return DiseaseParams.from_dict(DISEASE)


def default_progression():
    from .progression import ProgressionTable
    return ProgressionTable.from_dict(PROGRESSION)


# Synthetic population spec (data/population_spec.json:4-22), used by the
# reference-native scenarios (population.py:43-108).
POPULATION = {
    "n_agents": 10_000,
    "age_distribution": [0.12, 0.13, 0.14, 0.13, 0.13, 0.13, 0.10, 0.07, 0.05],
    "household_size_distribution": {"sizes": [1, 2, 3, 4, 5, 6],
                                    "probabilities": [0.28, 0.34, 0.15, 0.13, 0.07, 0.03]},
    "occupation_distribution": [0.09, 0.08, 0.07, 0.07, 0.06, 0.06, 0.05, 0.05, 0.05, 0.05,
                                0.04, 0.04, 0.04, 0.04, 0.04, 0.03, 0.03, 0.03, 0.02, 0.02,
                                0.02, 0.01, 0.01],
    "occupation_eligible_age_bands": [2, 3, 4, 5, 6],
    "random_degree_by_age": [2.0, 3.5, 4.5, 4.5, 4.5, 4.0, 3.5, 2.5, 2.0],
    "networks": {
        "occupation_mean_interactions": [10, 8, 12, 6, 8, 10, 8, 6, 14, 8, 6, 10, 4, 8, 12, 6, 8,
                                         10, 4, 6, 8, 12, 6],
        "rewire_beta": 0.1,
    },
}
