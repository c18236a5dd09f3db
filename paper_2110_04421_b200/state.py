"""Columnar agent state (host mirror of `pkg/src/epivec/state.py:21-112`).

The same 22 columns, dtypes and NEVER sentinels; the device copy
(`device.DeviceColumns`) holds one CUDA buffer per column with identical
dtype, so host<->device transfers are flat memcpys.
"""

from __future__ import annotations

from dataclasses import dataclass, fields

import numpy as np

from .errors import InvariantViolation
from .stages import N_STAGES, NEVER, Stage, VaccineStatus

# (name, dtype, fill) for every per-agent column, in device-struct order
COLUMN_SPECS = (
    ("age_band", np.int8, 0),
    ("occupation", np.int16, 0),
    ("household_id", np.int32, 0),
    ("random_degree", np.float64, 0.0),
    ("stage", np.int8, int(Stage.SUSCEPTIBLE)),
    ("infected_at", np.int32, NEVER),
    ("next_transition_at", np.int32, NEVER),
    ("next_stage", np.int8, NEVER),
    ("quarantine_until", np.int32, NEVER),
    ("quarantine_started_at", np.int32, NEVER),
    ("has_den_app", np.bool_, False),
    ("vaccine_status", np.int8, int(VaccineStatus.PRE_VACCINATION)),
    ("dose1_at", np.int32, NEVER),
    ("dose2_at", np.int32, NEVER),
    ("immune", np.bool_, False),
    ("immunity_check_at", np.int32, NEVER),
    ("immunity_check_prob", np.float64, 0.0),
    ("immunity_check_dose", np.int8, 0),
    ("test_sample_at", np.int32, NEVER),
    ("test_result_at", np.int32, NEVER),
    ("test_positive", np.bool_, False),
    ("den_test_due_at", np.int32, NEVER),
)

DYNAMIC_COLUMNS = (
    "stage", "infected_at", "next_transition_at", "next_stage",
    "quarantine_until", "quarantine_started_at", "has_den_app",
    "vaccine_status", "dose1_at", "dose2_at", "immune",
    "immunity_check_at", "immunity_check_prob", "immunity_check_dose",
    "test_sample_at", "test_result_at", "test_positive", "den_test_due_at",
)


@dataclass
class AgentColumns:
    n_agents: int
    age_band: np.ndarray
    occupation: np.ndarray
    household_id: np.ndarray
    random_degree: np.ndarray
    stage: np.ndarray
    infected_at: np.ndarray
    next_transition_at: np.ndarray
    next_stage: np.ndarray
    quarantine_until: np.ndarray
    quarantine_started_at: np.ndarray
    has_den_app: np.ndarray
    vaccine_status: np.ndarray
    dose1_at: np.ndarray
    dose2_at: np.ndarray
    immune: np.ndarray
    immunity_check_at: np.ndarray
    immunity_check_prob: np.ndarray
    immunity_check_dose: np.ndarray
    test_sample_at: np.ndarray
    test_result_at: np.ndarray
    test_positive: np.ndarray
    den_test_due_at: np.ndarray

    @classmethod
    def allocate(cls, n: int) -> "AgentColumns":
        return cls(n, **{name: np.full(n, fill, dtype=dt) for name, dt, fill in COLUMN_SPECS})

    def copy(self) -> "AgentColumns":
        return AgentColumns(self.n_agents, **{name: getattr(self, name).copy()
                                              for name, _, _ in COLUMN_SPECS})

    def stage_counts(self) -> np.ndarray:
        return np.bincount(self.stage, minlength=N_STAGES)

    def quarantined(self, step: int) -> np.ndarray:
        return self.quarantine_until > step

    def check_invariants(self, step: int) -> None:
        counts = self.stage_counts()
        if counts.sum() != self.n_agents:
            raise InvariantViolation(
                f"step {step}: stage counts sum to {counts.sum()} != {self.n_agents}")
        if (self.stage < 0).any() or (self.stage >= N_STAGES).any():
            raise InvariantViolation(f"step {step}: stage out of range")
        bad = ((self.stage != int(Stage.SUSCEPTIBLE)) & (self.stage != int(Stage.VACCINATED))
               & (self.infected_at == NEVER))
        if bad.any():
            raise InvariantViolation(
                f"step {step}: non-susceptible agent without infection timestamp")
