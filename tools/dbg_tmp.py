import os, sys, ctypes, numpy as np
os.environ["EPI_DBG"] = "1"
sys.path.insert(0, '.')
import torch
from bench import workload_iv
from paper_2110_04421_b200 import _native as N
from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize
from paper_2110_04421_b200.defaults import default_disease, default_progression
from paper_2110_04421_b200.sim import ConfigSimulation
spec = ConfigNetworkSpec.config(1)
pop = synthesize(spec, 0)
s = ConfigSimulation(pop, default_disease(), default_progression(), workload_iv("config2"), 3, mode="fused")
for _ in range(3):
    s.reset(); s.run(); torch.cuda.synchronize()
h = np.zeros(200 * 148 * 8, dtype=np.uint64)
assert N.lib().epi_dbg_copy(ctypes.c_void_p(h.ctypes.data), ctypes.c_size_t(h.nbytes)) == 0
d = h.reshape(200, 148, 8).astype(np.int64)[:178]
t0 = d[:, :, 0].min(axis=1)[:, None]
names = {0: "day start", 1: "A done", 5: "after bar1", 6: "B done", 2: "C start", 3: "C done/D start", 4: "D done"}
for k in (0, 1, 5, 6, 2, 3, 4):
    x = (d[:, :, k] - t0) / 1e3
    print(f"{names[k]:16s} mean {x.mean():6.2f}  max-per-day mean {x.max(axis=1).mean():6.2f}")
print("day length", np.diff(d[:, 0, 0]).mean() / 1e3)
