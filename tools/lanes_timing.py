"""k_fused_run agents-per-warp sweep (epi_set_run_lanes): config 1, CUDA-graph
replays with an L2 flush between them, ms per 180-day simulation; the records
must be identical for every lane count."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize  # noqa: E402
from paper_2110_04421_b200.defaults import default_disease, default_progression  # noqa: E402
from paper_2110_04421_b200.interventions import InterventionConfig  # noqa: E402
from paper_2110_04421_b200.sim import ConfigSimulation  # noqa: E402

spec = ConfigNetworkSpec.config(1)
pop = synthesize(spec, 0)
flush = torch.empty(384 * 1024 * 1024 // 4, device="cuda")
ref = None
lanes_list = [int(x) for x in (sys.argv[1:] or ["32", "30", "29", "32"])]
for lanes in lanes_list:
    s = ConfigSimulation(pop, default_disease(), default_progression(), InterventionConfig(), 3, mode="fused")
    s._lib.epi_set_run_lanes(s._ctx, lanes)
    assert s.uses_persistent_run(), lanes
    s.capture()
    for _ in range(3):
        s.replay()
    torch.cuda.synchronize()
    ms = []
    for k in range(20):
        flush.fill_(float(k))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.replay()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    rec = s.rec.cpu().numpy()
    same = ref is None or np.array_equal(rec, ref)
    ref = rec if ref is None else ref
    print(f"lanes {lanes:2d}: {np.median(ms):.3f} ms/sim (min {min(ms):.3f})  identical={same}", flush=True)
