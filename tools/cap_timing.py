"""Per-day (k_fused_step) vs persistent (k_fused_run) fused path by population
size around the persistent residency cap (704 agents per SM):
python tools/cap_timing.py [n ...]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize  # noqa: E402
from paper_2110_04421_b200.defaults import default_disease, default_progression  # noqa: E402
from paper_2110_04421_b200.interventions import InterventionConfig  # noqa: E402
from paper_2110_04421_b200.sim import ConfigSimulation  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [100000, 104000, 150000, 200000, 300000]
flush = torch.empty(384 * 1024 * 1024 // 4, device="cuda")
for n in sizes:
    pop = synthesize(ConfigNetworkSpec.config(1, n_agents=n), 0)
    for persistent in (True, False):
        s = ConfigSimulation(pop, default_disease(), default_progression(), InterventionConfig(), 3,
                             mode="fused", persistent=persistent)
        s.capture()
        for _ in range(2):
            s.replay()
        ms = []
        for k in range(5):
            flush.fill_(float(k))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s.replay()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = np.median(ms)
        print(f"n {n:7d} persistent={persistent!s:5s} uses_run={s.uses_persistent_run()!s:5s} "
              f"{t:.3f} ms/sim  {t * 1e3 / 180 / n * 1e5:.2f} us per day per 100k agents", flush=True)
