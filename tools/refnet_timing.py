"""Wall time of consecutive reference-native replications in one process
(the first ones pay lazy kernel loading and allocator growth)."""
import sys, time; sys.path.insert(0, ".")
import torch
from paper_2110_04421_b200.refsim import ReferenceNativeSimulation
for i in [1, 1, 2, 2, 3]:
    sim = ReferenceNativeSimulation(100_000, base_seed=i, initial_infections=10, horizon=180)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ev = sim.run(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(i, f"{(t1-t0)*1e3:.1f} ms", sim.interactions, sum(e.new_infections for e in ev), flush=True)
