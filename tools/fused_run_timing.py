"""Config-1 persistent fused run: ms per 180-day simulation (CUDA-graph
replays, L2 flushed in between) and bitwise agreement with the per-day
kernels.  python tools/fused_run_timing.py [replays] [--iv]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize  # noqa: E402
from paper_2110_04421_b200.defaults import default_disease, default_progression  # noqa: E402
from paper_2110_04421_b200.interventions import InterventionConfig  # noqa: E402
from paper_2110_04421_b200.sim import ConfigSimulation  # noqa: E402

iv = InterventionConfig()
if "--iv" in sys.argv:
    from bench import workload_iv
    iv = workload_iv("config2")
reps = int(next((a for a in sys.argv[1:] if a.isdigit()), "20"))
cfg = 0 if "--config0" in sys.argv else 1
spec = ConfigNetworkSpec.config(cfg)
pop = synthesize(spec, 0)
flush = torch.empty(384 * 1024 * 1024 // 4, device="cuda")
mk = lambda p: ConfigSimulation(pop, default_disease(), default_progression(), iv, 3, mode="fused", persistent=p)
a, b = mk(True), mk(False)
assert a.uses_persistent_run()
b.run()
for rnd in range(2):
    a.capture()
    for _ in range(3):
        a.replay()
    torch.cuda.synchronize()
    ms = []
    for k in range(reps):
        flush.fill_(float(k))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a.replay()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    same = np.array_equal(a.rec.cpu().numpy(), b.rec.cpu().numpy())
    print(f"{'k_iv_run' if iv.testing_enabled else 'k_fused_run'} run {rnd}: {np.median(ms):.3f} ms/sim "
          f"(min {min(ms):.3f}), bitwise equal to the per-day kernels: {same}", flush=True)
