"""One reference-native replication (for ncu captures of its kernels)."""
import sys; sys.path.insert(0, ".")
import torch
from paper_2110_04421_b200.refsim import ReferenceNativeSimulation
sim = ReferenceNativeSimulation(100_000, base_seed=5, initial_infections=10, horizon=180)
sim.run(); torch.cuda.synchronize()
print("interactions", sim.interactions)
