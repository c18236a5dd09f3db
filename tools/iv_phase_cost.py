"""k_iv_run cost by intervention subset (config 1 population, 180 days, CUDA
graph replays, L2 flushed in between): python tools/iv_phase_cost.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize  # noqa: E402
from paper_2110_04421_b200.defaults import default_disease, default_progression  # noqa: E402
from paper_2110_04421_b200.interventions import (DenConfig, InterventionConfig, TestKind,  # noqa: E402
                                                 VaccinePolicy)
from paper_2110_04421_b200.sim import ConfigSimulation  # noqa: E402

tk = TestKind("cfg2", 0.05, 2, 2)
vp = VaccinePolicy(daily_rate=0.01, dose1_efficacy=0.5, dose2_efficacy=0.9, dose_gap=21)
subsets = {
    "none (k_fused_run)": InterventionConfig(),
    "quarantine+testing": InterventionConfig(quarantine_enabled=True, testing_enabled=True, test_kind=tk),
    "quarantine+testing+DEN": InterventionConfig(quarantine_enabled=True, testing_enabled=True, test_kind=tk,
                                                 den_enabled=True, den=DenConfig(0.5)),
    "vaccination": InterventionConfig(vaccination_enabled=True, vaccine=vp),
    "all (config 2)": InterventionConfig(quarantine_enabled=True, testing_enabled=True, test_kind=tk,
                                         den_enabled=True, den=DenConfig(0.5), vaccination_enabled=True,
                                         vaccine=vp),
}
pop = synthesize(ConfigNetworkSpec.config(1), 0)
flush = torch.empty(384 * 1024 * 1024 // 4, device="cuda")
for name, iv in subsets.items():
    a = ConfigSimulation(pop, default_disease(), default_progression(), iv, 3, mode="fused", persistent=True)
    assert a.uses_persistent_run()
    a.capture()
    for _ in range(3):
        a.replay()
    torch.cuda.synchronize()
    ms = []
    for k in range(10):
        flush.fill_(float(k))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a.replay()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    rec = a.rec.cpu().numpy()
    print(f"{name:28s} {np.median(ms):.3f} ms/sim  tests {rec[:, 16].sum()} notified {rec[:, 18].sum()} "
          f"doses {rec[:, 17].sum()} cum_inf {rec[-1, 12]}", flush=True)
