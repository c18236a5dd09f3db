"""Config 3 (10M agents, BASELINE.json configs[3]) on one GPU for `--days`
days without CUDA graphs, so ncu can attribute every launch:
ncu -k regex:k_fused_step --launch-skip 60 --launch-count 1 python tools/profile_c3.py --days 62"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--days", type=int, default=62)
    ap.add_argument("--no-sparse", action="store_true")
    a = ap.parse_args()
    import torch
    from bench import workload_spec
    from paper_2110_04421_b200.sim import ConfigSimulation
    sim = ConfigSimulation.create(workload_spec("config3"), seed=0, mode="fused", horizon=a.days,
                                  sparse_push=not a.no_sparse, on_device=True)
    sim.run()
    torch.cuda.synchronize()
    print("last day record:", sim.records()[-1].tolist())


if __name__ == "__main__":
    main()
