"""k_iv_run phase timeline (config 2, 180 days) from a -DEPI_IV_TRACE build:
EPI_B200_LIB=build/trace/libepib200.so python tools/iv_timeline.py
Per day and block, %globaltimer at: 0 day start, 1 end of phase A, 2 after
barrier 1, 3 after the DEN regeneration, 4 end of the end barrier's window,
5 after the end barrier.  Prints per-phase means over days (us)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import workload_iv  # noqa: E402
from paper_2110_04421_b200 import _native  # noqa: E402
from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize  # noqa: E402
from paper_2110_04421_b200.defaults import default_disease, default_progression  # noqa: E402
from paper_2110_04421_b200.sim import ConfigSimulation  # noqa: E402

D, B, K = 200, 160, 6
pop = synthesize(ConfigNetworkSpec.config(1), 0)
a = ConfigSimulation(pop, default_disease(), default_progression(), workload_iv("config2"), 3, mode="fused",
                     persistent=True)
for _ in range(3):
    a.run()
torch.cuda.synchronize()
buf = np.zeros(D * B * K, dtype=np.uint64)
lib = _native.load_library()
fn = lib.epi_debug_iv_trace
fn.restype, fn.argtypes = C.c_int, [C.c_void_p, C.c_longlong]
assert fn(buf.ctypes.data, buf.size) == 0
tr = buf.reshape(D, B, K).astype(np.float64)
nb = 148
days = [d for d in range(1, 179) if tr[d, 0, 0] > 0]
tr = tr[days, :nb] / 1e3          # us
t0 = tr[:, :, 0].min(axis=1, keepdims=True)
rel = tr - t0[:, :, None]
def st(x):
    return f"mean {x.mean():6.2f} max {x.max():6.2f}"
print(f"days {len(days)}")
print("phase A per block            ", st(rel[:, :, 1] - rel[:, :, 0]))
print("day start skew               ", st(rel[:, :, 0]))
print("end of A (latest block)      ", st(rel[:, :, 1].max(axis=1)))
print("after barrier 1 (per block)  ", st(rel[:, :, 2]))
print("DEN regen per block          ", st(rel[:, :, 3] - rel[:, :, 2]))
eb = np.all(tr[:, :, 4] > 0, axis=1) & np.all(tr[:, :, 5] > 0, axis=1)   # days with an end barrier
print(f"days with an end barrier {int(eb.sum())}")
print("end window per block         ", st(rel[eb][:, :, 4] - rel[eb][:, :, 3]))
print("end window end (latest)      ", st(rel[eb][:, :, 4].max(axis=1)))
print("after end barrier (first)    ", st(rel[eb][:, :, 5].min(axis=1)))
ne = ~eb & np.all(tr[:, :, 4] > 0, axis=1)                                 # days without one
print(f"days without an end barrier {int(ne.sum())}")
if ne.any():
    print("finish per block (no end bar)", st(rel[ne][:, :, 4] - rel[ne][:, :, 3]))
nxt = np.diff(tr[:, 0, 0])
print("day length (block 0 starts)  ", st(nxt[nxt < 1e3]))
ok = nxt < 1e3
print("  with an end barrier        ", st(nxt[ok & eb[:-1]]))
print("  without                    ", st(nxt[ok & ne[:-1]]))
for q in (10, 30, 60, 90, 120, 170):
    i = min(q, len(days) - 1)
    r = rel[i]
    print(f"day {days[i]:3d}: A max {r[:, 1].max():6.2f} mean {(r[:, 1] - r[:, 0]).mean():6.2f}  bar1 {r[:, 2].min():6.2f}"
          f"  regen max {(r[:, 3] - r[:, 2]).max():6.2f} end-win max {r[:, 4].max():6.2f}  end {r[:, 5].min():6.2f}")
