"""Kernel-time breakdown of one reference-native replication (refnet
workload) under torch.profiler (CUPTI): per-kernel device time, total busy
device time vs the wall time of the replication."""
import sys, time; sys.path.insert(0, ".")
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2110_04421_b200.refsim import ReferenceNativeSimulation

for i in (1, 2):
    sim = ReferenceNativeSimulation(100_000, base_seed=i, initial_infections=10, horizon=180)
    sim.run(); torch.cuda.synchronize()
sim = ReferenceNativeSimulation(100_000, base_seed=3, initial_infections=10, horizon=180)
torch.cuda.synchronize(); t0 = time.perf_counter()
sim.run(); torch.cuda.synchronize()
print(f"unprofiled wall {(time.perf_counter() - t0) * 1e3:.1f} ms")
sim = ReferenceNativeSimulation(100_000, base_seed=4, initial_infections=10, horizon=180)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    sim.run(); torch.cuda.synchronize()
    wall = time.perf_counter() - t0
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
busy = sum(e.device_time for e in ev) / 1e3
print(f"profiled wall {wall * 1e3:.1f} ms, device busy {busy:.1f} ms, {len(ev)} device ops")
print(prof.key_averages().table(sort_by="device_time_total", row_limit=30, max_name_column_width=60))
