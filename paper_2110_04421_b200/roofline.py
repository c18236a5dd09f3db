"""Message-pass roofline probe (north-star part (a) on its own).

Builds a config population, advances it `warm_days` so the state is
mid-epidemic, generates day t's pre-joined message CSR (epi_net_generate),
then times the message pass alone (epi_net_gather, float hazard out) with
CUDA events.  Algorithmic bytes per launch:

    B_K1 = 2 E (one 16-bit message per directed edge)
         + 11 N (row length 4, stage 1, immune 1, age 1, hazard out 4).
"""

from __future__ import annotations

import ctypes

from . import _native as N
from .confignet import ConfigNetworkSpec, synthesize
from .defaults import default_disease, default_progression
from .engine import _u64
from .interventions import InterventionConfig
from .sim import ConfigSimulation


def prepare(n_agents: int, warm_days: int = 60, seed: int = 5, spec: ConfigNetworkSpec | None = None):
    if spec is None:
        spec = ConfigNetworkSpec.config(1, n_agents=n_agents,
                                        initial_infections=max(10, n_agents // 1000))
    sim = ConfigSimulation(synthesize(spec, 0), default_disease(), default_progression(),
                           InterventionConfig(), seed, mode="fused", horizon=warm_days + 1)
    sim.run(warm_days)
    t = sim.clock
    N.check(sim._lib.epi_net_generate(sim._ctx, t, _u64(sim.seed), N.ptr(sim.codes[t & 1]),
                                      N.stream_handle()))
    return sim


def gather(sim, lam, rec=None):
    t = sim.clock
    st = sim.state.struct()
    N.check(sim._lib.epi_net_gather(sim._ctx, ctypes.byref(st), t, N.ptr(sim.codes[t & 1]),
                                    N.ptr(lam), N.ptr(rec), N.stream_handle()))


def message_pass_roofline(n_agents: int = 10_000_000, warm_days: int = 60, reps: int = 20,
                          flush_l2: bool = True, peak_gbps: float | None = None) -> dict:
    import torch
    sim = prepare(n_agents, warm_days)
    lam = torch.empty(n_agents, dtype=torch.float32, device=sim.device)
    rec = torch.zeros(N.REC_LEN, dtype=torch.int64, device=sim.device)
    gather(sim, lam, rec)
    edges = int(rec[N.REC["edges"]].item())
    flush = torch.empty(384 * 1024 * 1024 // 4, dtype=torch.float32, device=sim.device) \
        if flush_l2 else None
    for _ in range(3):
        gather(sim, lam)
    torch.cuda.synchronize()
    pairs = []
    for i in range(reps):
        if flush is not None:
            flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        gather(sim, lam)
        b.record()
        pairs.append((a, b))
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in pairs)
    med = ms[len(ms) // 2]
    alg = 2 * edges + 11 * n_agents
    out = {"kernel": "k_msg_pass<0>: message pass alone (tile-packed 16-bit pre-joined "
                     "messages, rows padded to 4-message half-groups, 16-byte register-prefetched "
                     "loads, group-parallel fp32 half sums + per-row half-group sum)",
           "n_agents": n_agents, "day": sim.clock, "edges": edges, "ms_median": med,
           "ms_min": ms[0], "alg_bytes": alg, "achieved": alg / (med / 1e3) / 1e9,
           "unit": "GB/s", "l2_flushed_between_reps": bool(flush_l2)}
    if peak_gbps:
        out["peak"] = peak_gbps
        out["frac"] = out["achieved"] / peak_gbps
    return out


if __name__ == "__main__":
    import json
    import sys
    for n in [int(x) for x in (sys.argv[1:] or ["100000", "1000000", "10000000"])]:
        print(json.dumps(message_pass_roofline(n)), flush=True)
