"""Small runs of every kernel family in one process (fused / csr / fp64
simulation, CUDA-graph replay, message pass, device population, partitioned
interventions on emulated ranks, the reference-native scenario):
python tools/all_paths_smoke.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2110_04421_b200 import roofline
    from paper_2110_04421_b200.confignet import ConfigNetworkSpec, DevicePopulation, synthesize
    from paper_2110_04421_b200.defaults import default_disease, default_progression
    from paper_2110_04421_b200.interventions import (DenConfig, InterventionConfig, TestKind,
                                                     VaccinePolicy)
    from paper_2110_04421_b200.partition import run_threaded
    from paper_2110_04421_b200.refsim import ReferenceNativeSimulation
    from paper_2110_04421_b200.sim import ConfigSimulation
    spec = ConfigNetworkSpec.config(1, n_agents=3001, initial_infections=40)
    for mode, prec in (("fused", "f32"), ("csr", "f32"), ("csr", "f64")):
        sim = ConfigSimulation.create(spec, seed=3, mode=mode, precision=prec, horizon=12)
        sim.run()
    sim = ConfigSimulation.create(spec, seed=3, mode="fused", horizon=12)
    sim.capture()
    sim.replay()
    lam = torch.empty(spec.n_agents, dtype=torch.float32, device="cuda")
    s2 = roofline.prepare(spec.n_agents, warm_days=5, spec=spec)
    roofline.gather(s2, lam)
    DevicePopulation(spec, 5)
    iv = InterventionConfig(quarantine_enabled=True, testing_enabled=True,
                            test_kind=TestKind("t", 0.3, 1, 2), den_enabled=True, den=DenConfig(0.6),
                            vaccination_enabled=True,
                            vaccine=VaccinePolicy(daily_rate=0.02, dose_gap=5, start_trigger=0.0))
    ConfigSimulation.create(spec, seed=4, mode="csr", precision="f64", interventions=iv, horizon=10).run()
    run_threaded(synthesize(spec, 4), default_disease(), default_progression(), iv, 4, 2, 8, mode="csr",
                 precision="f32")
    ReferenceNativeSimulation(2000, initial_infections=10, horizon=8).run()
    torch.cuda.synchronize()
    print("all paths ok")


if __name__ == "__main__":
    main()
