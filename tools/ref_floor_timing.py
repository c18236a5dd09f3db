"""Where the wall time of the reference's throughput-floor test goes
(test_oracle.py TestThroughputFloor: runner.bench at 10k agents x 3 steps,
GpuEngine vs the reference oracle): python tools/ref_floor_timing.py"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT / "baseline" / "_ref"), str(ROOT)]

import numpy as np  # noqa: E402
import torch  # noqa: E402
from epivec import runner  # noqa: E402
from epivec.scenario import default_population_dict, scenario_from_dict  # noqa: E402
from epivec.stages import Stage  # noqa: E402

from paper_2110_04421_b200.engine import GpuEngine  # noqa: E402

pop = default_population_dict()
pop["n_agents"] = 10_000
config = scenario_from_dict({"population": pop, "horizon": 3, "replications": 1, "base_seed": 2,
                             "initial_infections": 8, "interventions": {}}, name="oracle-test")
torch.zeros(1, device="cuda")
for rep in range(4):
    seed = runner.replication_seed(config.base_seed, 0)
    cols, realizer = runner.initialize_run(config, seed)
    t = {}
    t0 = time.perf_counter()
    eng = GpuEngine(cols, config.disease, config.progression, config.interventions, seed, check_invariants=False)
    t["construct"] = time.perf_counter() - t0
    t["realize"] = t["step"] = 0.0
    for step in range(config.horizon):
        a = time.perf_counter()
        graph = realizer.realize(step, cols.stage == int(Stage.DEAD))
        b = time.perf_counter()
        eng.step(graph)
        c = time.perf_counter()
        t["realize"] += b - a
        t["step"] += c - b
    t["total"] = time.perf_counter() - t0
    oa = time.perf_counter()
    rep_o = runner.bench(config, use_oracle=True)
    t["oracle_total"] = time.perf_counter() - oa
    print({k: round(v * 1e3, 2) for k, v in t.items()}, "ms", flush=True)
