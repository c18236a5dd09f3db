"""Timeline of partitioned days (torch.profiler / CUPTI: every kernel of the
process, every stream), for DESIGN.md §7:

  * 1 rank over native NCCL (epi_comm, world 1) and
  * 2 ranks emulated on one GPU (host threads, own streams; the code
    all-gather through the EPI_X_GATHER_U16 callback)

on a config-1-network population of --agents agents with push tables off
(the path of every partitioned rank).  Prints, per day, each kernel's start
and end (us, relative to the day's first kernel) and stream, so the side
stream's sigma tables for tomorrow can be seen overlapping today's
k_fused_step and the exchange.

    python tools/timeline_partition.py --agents 2000000 --days 6 > gpurun_out/timeline.txt
"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2110_04421_b200.confignet import DevicePopulation, ConfigNetworkSpec  # noqa: E402
from paper_2110_04421_b200.defaults import default_disease, default_progression  # noqa: E402
from paper_2110_04421_b200.interventions import InterventionConfig  # noqa: E402
from paper_2110_04421_b200.partition import NcclComm, PartitionedSimulation, PartitionPlan  # noqa: E402


def kernels(prof):
    out = []
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        out.append((e.time_range.start, e.time_range.end, e.name, getattr(e, "device_resource_id", None)))
    return sorted(out)


def show(title, ev, days_marker="k_fused_step"):
    print(f"== {title}")
    t0 = None
    day = -1
    for s, e, name, stream in ev:
        short = name.split("(")[0].replace("void ", "").replace("epi::", "")
        if days_marker in short:
            day += 1
        if t0 is None:
            t0 = s
        print(f"  day~{day:2d} stream {stream!s:>4} {short[:46]:46s} {s - t0:10.1f} .. {e - t0:10.1f} us "
              f"({e - s:7.1f})")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--agents", type=int, default=2_000_000)
    ap.add_argument("--days", type=int, default=6)
    a = ap.parse_args()
    spec = ConfigNetworkSpec.config(1, n_agents=a.agents, initial_infections=max(100, a.agents // 1000))
    pop = DevicePopulation(spec, 0)
    d, t, iv = default_disease(), default_progression(), InterventionConfig()
    # 1 rank, native NCCL
    comm = NcclComm(1, 0, NcclComm.unique_id())
    plan = PartitionPlan(spec.n_agents, 1)
    sim = PartitionedSimulation(pop, d, t, iv, 3, plan, 0, comm=comm, mode="fused", horizon=40, push_max=0)
    sim.run(20)                                  # into the epidemic
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        sim.run(a.days)
        torch.cuda.synchronize()
    show(f"1 rank, native NCCL, {a.agents} agents, days 20-{20 + a.days - 1}", kernels(prof))
    # 2 ranks emulated on one GPU: built first, then only their days profiled
    import threading
    from paper_2110_04421_b200.partition import ThreadExchange
    plan2 = PartitionPlan(spec.n_agents, 2)
    ex = ThreadExchange(plan2)
    streams = [torch.cuda.Stream() for _ in range(2)]
    sims = []
    for r in range(2):
        with torch.cuda.stream(streams[r]):
            sims.append(PartitionedSimulation(pop, d, t, iv, 3, plan2, r, ex.for_rank(r), mode="fused",
                                              horizon=40))
    torch.cuda.synchronize()

    def rank_main(r, days):
        with torch.cuda.stream(streams[r]):
            if days is None:
                sims[r].reset()
            else:
                sims[r].run(days)
            streams[r].synchronize()

    def both(days):
        th = [threading.Thread(target=rank_main, args=(r, days)) for r in range(2)]
        for x in th:
            x.start()
        for x in th:
            x.join()
    both(None)
    both(20)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof2:
        both(a.days)
        torch.cuda.synchronize()
    show(f"2 emulated ranks (host threads, own streams, code exchange by the EPI_X_GATHER_U16 callback: "
         f"device copies), {a.agents} agents, days 20-{20 + a.days - 1}", kernels(prof2))


if __name__ == "__main__":
    main()
