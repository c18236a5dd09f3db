"""Per-day device time vs population size (fused and csr modes).
PUSH_MAX=<agents> overrides the push-table cut-off (epi_set_push_max);
HOT_WINDOW=0 drops the L2-persisting window over the codes."""
import ctypes
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch
    from paper_2110_04421_b200 import _native as N
    from paper_2110_04421_b200.confignet import ConfigNetworkSpec
    from paper_2110_04421_b200.engine import _u64
    from paper_2110_04421_b200.sim import ConfigSimulation
    sizes = [int(x) for x in (sys.argv[1:] or ["100000", "300000", "1000000", "3000000"])]
    out = []
    for n in sizes:
        for mode in ("fused", "csr"):
            days = 40
            spec = ConfigNetworkSpec.config(1, n_agents=n, initial_infections=max(10, n // 100))
            pm = os.environ.get("PUSH_MAX")
            sim = ConfigSimulation.create(spec, seed=3, mode=mode, horizon=days,
                                          push_max=int(pm) if pm is not None else None)
            if os.environ.get("HOT_WINDOW") == "0":
                N.check(sim._lib.epi_set_hot_window(sim._ctx, None, 0))
            evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(days)]
            for d in evs:
                for e in d:
                    e.record()
            torch.cuda.synchronize()
            for t in range(days):
                h = (ctypes.c_void_p * 4)(*[e.cuda_event for e in evs[t]])
                st = sim.state.struct()
                N.check(sim._lib.epi_sim_step_timed(
                    sim._ctx, ctypes.byref(st), t, _u64(sim.seed), 0 if mode == "csr" else 1, N.F32,
                    N.ptr(sim.codes[t & 1]), N.ptr(sim.codes[(t + 1) & 1]), N.ptr(sim.rec[t]),
                    N.ptr(sim.vax), ctypes.addressof(h), N.stream_handle()))
            torch.cuda.synchronize()
            sim.clock = days
            gen = np.mean([evs[t][0].elapsed_time(evs[t][1]) for t in range(5, days)])
            pas = np.mean([evs[t][1].elapsed_time(evs[t][2]) for t in range(5, days)])
            E = float(sim.records()[5:, 19].mean())
            r = dict(n=n, mode=mode, push_max=pm, gen_us=1e3 * gen, main_us=1e3 * pas, edges=E,
                     edges_per_us=E / (1e3 * (gen + pas)))
            print(json.dumps(r), flush=True)
            out.append(r)
            del sim
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
