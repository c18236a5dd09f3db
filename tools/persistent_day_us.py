"""Mean device time per day of the persistent run (days 1..179 of config 1)."""
import sys, os, torch
sys.path.insert(0, '.')
from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize
from paper_2110_04421_b200.defaults import default_disease, default_progression
from paper_2110_04421_b200.interventions import InterventionConfig
from paper_2110_04421_b200.sim import ConfigSimulation
spec = ConfigNetworkSpec.config(1)
pop = synthesize(spec, 0)
s = ConfigSimulation(pop, default_disease(), default_progression(), InterventionConfig(), 3, mode="fused")
s.reset(); s.run(1); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(5):
    s.reset(); s.run(1); torch.cuda.synchronize()
    e0.record(); s.run(); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print("k_fused_run:", round(best * 1000 / 179, 2), "us per day (days 1-179 of config 1)")
