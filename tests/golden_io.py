"""Load the reference-generated fixtures into the mirror types."""

import json
from pathlib import Path

import numpy as np

from paper_2110_04421_b200.disease import DiseaseParams
from paper_2110_04421_b200.graph import StepGraph
from paper_2110_04421_b200.interventions import (DenConfig, ImmunityMode, InterventionConfig,
                                                 Strategy, TestKind, VaccinePolicy)
from paper_2110_04421_b200.progression import ProgressionTable
from paper_2110_04421_b200.state import COLUMN_SPECS, DYNAMIC_COLUMNS, AgentColumns

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name):
    return np.load(GOLDEN / name)


def interventions_from_json(s):
    d = json.loads(s)
    d["test_kind"] = TestKind(**d["test_kind"])
    d["den"] = DenConfig(**d["den"])
    v = d["vaccine"]
    v["strategy"] = Strategy(v["strategy"])
    v["immunity_mode"] = ImmunityMode(v["immunity_mode"])
    d["vaccine"] = VaccinePolicy(**v)
    return InterventionConfig(**d)


class Trajectory:
    def __init__(self, name):
        z = load(f"traj_{name}.npz")
        self.z = z
        self.seed = int(z["seed"])
        self.horizon = int(z["horizon"])
        self.disease = DiseaseParams.from_dict(json.loads(str(z["disease_json"])))
        self.table = ProgressionTable.from_dict(json.loads(str(z["table_json"])))
        self.iv = interventions_from_json(str(z["iv_json"]))
        self.offsets = z["edge_offsets"]
        self.events = z["events"]
        self.n = len(z["init_stage"])

    def initial_cols(self):
        cols = AgentColumns.allocate(self.n)
        for name, _, _ in COLUMN_SPECS:
            getattr(cols, name)[:] = self.z[f"init_{name}"]
        return cols

    def graph(self, step):
        a, b = self.offsets[step], self.offsets[step + 1]
        return StepGraph(step, self.z["src"][a:b], self.z["dst"][a:b], self.z["kind"][a:b])

    def state(self, step, col):
        return self.z[f"state_{col}"][step]

    def hazard(self, step):
        key = f"hazard_{step}"
        return self.z[key] if key in self.z.files else None


def compare_state(cols, traj, step):
    for c in DYNAMIC_COLUMNS:
        got, want = getattr(cols, c), traj.state(step, c)
        if not np.array_equal(got, want):
            bad = int(np.flatnonzero(got != want)[0])
            raise AssertionError(f"step {step} column {c} agent {bad}: "
                                 f"got {got[bad]!r} want {want[bad]!r}")
