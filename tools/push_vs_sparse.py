"""Full push tables vs sparse push rows vs inverse slot walks, per-day fused
path, by population size: python tools/push_vs_sparse.py [n ...]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2110_04421_b200.confignet import ConfigNetworkSpec, DevicePopulation  # noqa: E402
from paper_2110_04421_b200.defaults import default_disease, default_progression  # noqa: E402
from paper_2110_04421_b200.interventions import InterventionConfig  # noqa: E402
from paper_2110_04421_b200.sim import ConfigSimulation  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [200000, 500000, 1000000, 1300000, 2000000]
flush = torch.empty(384 * 1024 * 1024 // 4, device="cuda")
for n in sizes:
    pop = DevicePopulation(ConfigNetworkSpec.config(1, n_agents=n, initial_infections=max(1, n // 1000)), 0)
    out = []
    for name, kw in (("push", dict(push_max=1 << 30)), ("sparse", dict(push_max=0)),
                     ("inverse", dict(push_max=0, sparse_push=False))):
        s = ConfigSimulation(pop, default_disease(), default_progression(), InterventionConfig(), 3,
                             mode="fused", persistent=False, **kw)
        s.capture()
        s.replay()
        ms = []
        for k in range(3):
            flush.fill_(float(k))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s.replay()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        out.append(f"{name} {np.median(ms):8.3f}")
        del s
        torch.cuda.empty_cache()
    print(f"n {n:8d} ms/sim: " + "  ".join(out), flush=True)
