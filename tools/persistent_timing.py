import sys, torch
sys.path.insert(0, '.')
from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize
from paper_2110_04421_b200.defaults import default_disease, default_progression
from paper_2110_04421_b200.interventions import InterventionConfig
from paper_2110_04421_b200.sim import ConfigSimulation
spec = ConfigNetworkSpec.config(1)
pop = synthesize(spec, 0)
for p in (False, True, False, True):
    s = ConfigSimulation(pop, default_disease(), default_progression(), InterventionConfig(), 3, mode="fused", persistent=p)
    s.capture()
    for _ in range(3): s.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): s.replay()
    e1.record(); torch.cuda.synchronize()
    print("persistent" if p else "per-day   ", round(e0.elapsed_time(e1) / 20, 3), "ms/sim", int(s.rec[:, 1].sum()))
