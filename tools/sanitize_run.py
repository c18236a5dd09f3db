"""Small runs of every native path for compute-sanitizer:

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_run.py

2k-agent config-1 population: the persistent fused run (k_fused_run, its
hand-rolled grid barrier), the persistent intervention run (k_iv_run), the
csr fp64 path, the non-push fused path with the side-stream sigma tables,
the graph-in engine (counting sort + long-row block sort + fp64 pass), and
the reference-native realizer (k_ref_* incl. the rewiring rounds)."""

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize  # noqa: E402
from paper_2110_04421_b200.defaults import default_disease, default_progression  # noqa: E402
from paper_2110_04421_b200.interventions import (DenConfig, InterventionConfig, TestKind,  # noqa: E402
                                                 VaccinePolicy)
from paper_2110_04421_b200.sim import ConfigSimulation  # noqa: E402


def main():
    spec = ConfigNetworkSpec.config(1, n_agents=2000, initial_infections=60)
    pop = synthesize(spec, 3)
    d, t = default_disease(), default_progression()
    iv_all = InterventionConfig(quarantine_enabled=True, testing_enabled=True,
                                test_kind=TestKind("cfg2", 0.3, 1, 2), den_enabled=True, den=DenConfig(0.5),
                                vaccination_enabled=True,
                                vaccine=VaccinePolicy(daily_rate=0.02, dose1_efficacy=0.5, dose2_efficacy=0.9,
                                                      dose_gap=7, start_trigger=0.002))
    out = {}
    runs = {
        "fused_persistent": dict(iv=InterventionConfig(), mode="fused"),
        "iv_persistent": dict(iv=iv_all, mode="fused"),
        "csr_f64": dict(iv=iv_all, mode="csr", precision="f64"),
        "fused_nopush_sigma_ahead": dict(iv=InterventionConfig(), mode="fused", push_max=0, persistent=False),
    }
    for name, kw in runs.items():
        iv = kw.pop("iv")
        sim = ConfigSimulation(pop, d, t, iv, 11, horizon=30, **kw)
        sim.run()
        torch.cuda.synchronize()
        out[name] = int(sim.records()[:, 15].sum())
    # graph-in engine on a hub graph (long-row sort) + the reference realizer
    from paper_2110_04421_b200.engine import GpuEngine
    from paper_2110_04421_b200.graph import StepGraph
    from paper_2110_04421_b200.refnet import GpuRealizer
    from paper_2110_04421_b200.state import AgentColumns
    rng = np.random.default_rng(0)
    n = 3000
    cols = AgentColumns.allocate(n)
    cols.stage[:300] = 4
    cols.infected_at[:300] = 0
    cols.next_stage[:300] = 8
    cols.next_transition_at[:300] = 1000
    lens = np.concatenate([[9000, 40], rng.integers(0, 6, n - 2)])
    dst = np.repeat(np.arange(n, dtype=np.int32), lens)
    src = rng.integers(0, n - 1, len(dst)).astype(np.int32)
    src[src >= dst] += 1
    kind = rng.integers(0, 3, len(dst)).astype(np.int8)
    eng = GpuEngine(cols, d, t, InterventionConfig(), 0)
    eng.clock = 3
    lam = eng.gather_exposure(StepGraph(3, src, dst, kind))
    out["hub_lambda_sum"] = float(lam.sum())
    hh = np.arange(n) // 3
    occ = np.where(rng.random(n) < 0.6, rng.integers(1, 5, n), 0).astype(np.int8)
    r = GpuRealizer(5, hh, occ, np.full(n, 4.0, np.float32), [6.0, 10.0, 4.0, 8.0], 1.0)
    out["refnet_edges"] = int(r.realize(0, np.zeros(n, bool)).n_edges)
    torch.cuda.synchronize()
    print("sanitize_run ok", out)


if __name__ == "__main__":
    main()
