"""Run `days` simulated days of a config network without CUDA graphs so ncu
can attribute every launch (`--mode csr|fused`, `--agents N`)."""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="fused")
    ap.add_argument("--agents", type=int, default=100_000)
    ap.add_argument("--days", type=int, default=60)
    ap.add_argument("--precision", default="f32")
    ap.add_argument("--iv", default="none", help="none | config2 (bench.workload_iv)")
    a = ap.parse_args()
    import torch
    from paper_2110_04421_b200.confignet import ConfigNetworkSpec
    from paper_2110_04421_b200.sim import ConfigSimulation
    spec = ConfigNetworkSpec.config(1, n_agents=a.agents,
                                    initial_infections=max(1, a.agents // 1000))
    from bench import workload_iv
    sim = ConfigSimulation.create(spec, seed=11, mode=a.mode, precision=a.precision, horizon=a.days,
                                  interventions=workload_iv(a.iv))
    sim.run()
    torch.cuda.synchronize()
    print("last day record:", sim.records()[-1].tolist())


if __name__ == "__main__":
    main()
