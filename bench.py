"""Benchmark: BASELINE.json metric on config 1 (100k agents, 180 days).

One bench "step" = one complete 180-day simulation of config 1 (households +
workplaces + Poisson(5) random contacts, 100 seeds, no interventions), i.e.
one pass of the hot path over every day: per-day edge generation, message
pass, fused infection/progression update and the per-day record.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--mode csr|fused] [--workload config1|config0]

`value` = agent-interactions/s (directed edges x days, the reference's own
definition, runner.py:269,287) over all ranks, device-timed with CUDA events
(max over ranks).  `e2e` = the same through the public API from pinned host
buffers: initial state H2D + 180 days + time-series D2H, every step.
`--impl reference` times the unmodified reference engine (epivec, installed
into baseline/_ref) on the same workload, all host cores, each process
walking through whole 180-day replications.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HORIZON = 180
DOSE_GAP = [21]      # config2 second-dose delay (set from --dose-gap)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", choices=["csr", "fused", "auto"], default="auto")
    ap.add_argument("--workload", choices=["config1", "config0", "config2", "config3", "config4",
                                           "refnet"],
                    default="config1")
    ap.add_argument("--dose-gap", type=int, default=21, help="config2: second-dose delay (21 or 84)")
    ap.add_argument("--replicas", type=int, default=128, help="config4: replicas per GPU")
    ap.add_argument("--streams", type=int, default=8, help="config4: concurrent streams")
    ap.add_argument("--replica-mode", default="persistent", choices=["concurrent", "persistent"],
                    help="config4: one persistent run per replica, one after another on one "
                         "stream (default), or per-day kernels of replicas on concurrent streams")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--precision", choices=["f32", "f64"], default="f32",
                    help="f64 = canonical-order fp64 message pass (csr mode only): bitwise the "
                         "reference engine's hazard")
    ap.add_argument("--no-partition", action="store_true",
                    help="skip the config-3 agent-range partition measured beside the headline")
    ap.add_argument("--no-message-pass", action="store_true",
                    help="skip the 10M-agent message-pass roofline probe")
    return ap.parse_args()


def workload_spec(name):
    from paper_2110_04421_b200.confignet import ConfigNetworkSpec
    return ConfigNetworkSpec.config({"config0": 0, "config1": 1, "config2": 2, "config3": 3,
                                     "config4": 4}[name])


def workload_iv(name, dose_gap=21):
    """BASELINE.json configs[2] (SURVEY §8(d) mapping): quarantine 14 days,
    testing of symptomatic agents (detection 5 %, 2-day result delay), DEN with
    app adoption 0.5, two-dose vaccination 1 %/day, efficacy 0.5 / 0.9, second
    dose after `dose_gap` days; no interventions for the other configs."""
    from paper_2110_04421_b200.interventions import (DenConfig, InterventionConfig, TestKind,
                                                     VaccinePolicy)
    if name != "config2":
        return InterventionConfig()
    return InterventionConfig(quarantine_enabled=True, testing_enabled=True,
                              test_kind=TestKind("cfg2", 0.05, 2, 2), den_enabled=True,
                              den=DenConfig(0.5), vaccination_enabled=True,
                              vaccine=VaccinePolicy(daily_rate=0.01, dose1_efficacy=0.5,
                                                    dose2_efficacy=0.9, dose_gap=dose_gap))


def workload_string(a):
    """config.workload -- identical in both arms (ours / --impl reference)."""
    if a.workload == "config2":
        return ("config2 (BASELINE.json configs[2]): config 1 + quarantine 14 d, testing "
                f"(5 %, 2-day delay), DEN (app 0.5), vaccination 1 %/day, efficacy 0.5/0.9, "
                f"dose gap {a.dose_gap} d")
    if a.workload == "config0":
        return ("config0 (BASELINE.json configs[0]): 10k agents, 180 days, households U{1..6} + "
                "Poisson(5) random contacts, 10 seeds, no interventions")
    return ("config1 (BASELINE.json configs[1]): 100k agents, 180 days, households U{1..6} + "
            "workplaces U{10..50} x 8 colleague draws + Poisson(5) random contacts, 100 seeds, "
            "no interventions")


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


# ---------------------------------------------------------------------------
# CPU reference arm: oracle port of Engine.step + the config-network
# restatement, one replica per process, bounded number of days.
def _cpu_worker(args):
    """cpu_baseline of our arm: the unmodified reference engine (baseline/_ref)
    on one core, one replica of the workload, days 0.. until `seconds`."""
    workload, seed, seconds = args
    sys.path.insert(0, str(ROOT))
    from oracle.epivec_driver import ReferenceNativeReplica, ReferenceReplica, reference_interventions
    if workload == "refnet":
        rep = ReferenceNativeReplica(REFNET_AGENTS, seed, 0, REFNET_SEEDS)
    else:
        rep = ReferenceReplica(workload_spec(workload), seed,
                               reference_interventions(workload == "config2", DOSE_GAP[0]))
    t0 = time.perf_counter()
    edges = days = 0
    while days < HORIZON and (time.perf_counter() - t0) < seconds:
        edges += rep.step().n_edges
        days += 1
    return edges, days, time.perf_counter() - t0


REFNET_AGENTS, REFNET_SEEDS = 100_000, 10   # epivec bench --agents 100000 (scenario.py:53)


def _ref_worker(conn, workload, dose_gap, base):
    """A host process driving the UNMODIFIED reference engine
    (`epivec.engine.Engine` from baseline/_ref) over whole 180-day
    replications of the workload, one after another.  Each command
    ("advance", seconds) simulates days until the budget is spent -- so over
    the run every worker walks through the whole horizon, more than once --
    and replies (directed edges, days, seconds)."""
    sys.path.insert(0, str(ROOT))
    from oracle.epivec_driver import ReferenceReplica, import_epivec, reference_interventions
    from paper_2110_04421_b200.confignet import synthesize
    import_epivec()
    from epivec.runner import replication_seed
    rep_i = 0
    if workload == "refnet":
        from oracle.epivec_driver import ReferenceNativeReplica

        def fresh():
            nonlocal rep_i
            rep_i += 1
            return ReferenceNativeReplica(REFNET_AGENTS, base, rep_i, REFNET_SEEDS)
    else:
        spec = workload_spec(workload)
        pop = synthesize(spec, 0)
        iv = reference_interventions(workload == "config2", dose_gap)

        def fresh():
            nonlocal rep_i
            rep_i += 1
            return ReferenceReplica(spec, replication_seed(base, rep_i), iv, pop=pop)
    rep = fresh()
    conn.send("ready")
    while True:
        cmd = conn.recv()
        if cmd is None:
            return
        t0 = time.perf_counter()
        edges = days = 0
        while time.perf_counter() - t0 < cmd:
            if rep.day >= HORIZON:
                rep = fresh()       # a new replication (building it is inside the timed budget)
            edges += rep.step().n_edges
            days += 1
        conn.send((edges, days, time.perf_counter() - t0))


def run_reference(a):
    """The reference arm: the unmodified reference engine on the host cores.
    One step = every host process advances its own chain of whole 180-day
    replications for a bounded slice of time (all processes in parallel);
    value = directed edges gathered / wall time of the steps."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    try:
        from oracle.epivec_driver import import_epivec
        import_epivec()
    except ImportError as e:
        print(json.dumps({"impl": "reference", "unavailable": f"the reference (epivec) is not installed in "
                          f"baseline/_ref (tools/install_reference.sh): {e}"}), flush=True)
        return
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    # the whole --steps K --warmup W run within a few minutes
    per_step = max(2.0, min(a.cpu_seconds / 2, 200.0 / max(1, a.steps + a.warmup)))
    ctx = mp.get_context("fork")
    pipes, procs = [], []
    for w in range(cores):
        here, there = ctx.Pipe()
        p = ctx.Process(target=_ref_worker, args=(there, a.workload, a.dose_gap, 7000 + w), daemon=True)
        p.start()
        pipes.append(here)
        procs.append(p)
    for c in pipes:
        assert c.recv() == "ready"
    steps = []
    days_done = 0
    for i in range(a.warmup + a.steps):
        t0 = time.perf_counter()
        for c in pipes:
            c.send(per_step)
        res = [c.recv() for c in pipes]
        wall = time.perf_counter() - t0
        if i >= a.warmup:
            steps.append((sum(r[0] for r in res), wall))
            days_done += sum(r[1] for r in res)
    for c in pipes:
        c.send(None)
    for p in procs:
        p.join(timeout=10)
    e = sum(s_[0] for s_ in steps)
    w = sum(s_[1] for s_ in steps)
    v = e / w
    graphs = ("the reference's own GraphRealizer, runner.initialize_run" if a.workload == "refnet" else
              "oracle/confignet_np restatement of the config generator")
    sample = (f"each step: {cores} processes x {per_step:.1f}s of the unmodified reference engine "
              f"(epivec.engine.Engine from baseline/_ref, fp64) stepping whole 180-day replications "
              f"in sequence (graphs: {graphs}); "
              f"{days_done} simulated days over the timed steps ({days_done / max(1, cores):.0f} "
              f"per process" + ("; every process covers the whole horizon" if days_done >= cores * HORIZON
                                else "; early days of the horizon only: a short run") + ")")
    line = {
        "impl": "reference", "metric": "agent-interactions/sec", "value": v,
        "unit": "agent-interactions/s", "n_gpus": a.gpus, "steps": len(steps), "warmup": a.warmup,
        "ms_per_step": 1000 * w / max(1, len(steps)), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": REFNET_DESC if a.workload == "refnet" else workload_string(a),
                   "parallelism": f"{cores} host processes"},
        "cpu_baseline": {"value": v, "unit": "agent-interactions/s", "cores": cores,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": "agent-interactions/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_single(workload, seconds):
    try:
        e, days, t = _cpu_worker((workload, 12345, seconds))
    except ImportError as err:
        return {"value": None, "unit": "agent-interactions/s", "cores": 1, "kind": "reference",
                "sample": f"unavailable: the reference (epivec) is not installed in baseline/_ref ({err})"}
    return {"value": e / t, "unit": "agent-interactions/s", "cores": 1, "kind": "reference",
            "sample": f"unmodified reference engine (epivec.engine.Engine, baseline/_ref) on the "
                      f"restated config generator, 1 replica, days 0-{days - 1} of 180 "
                      f"({e} directed edges in {t:.1f}s), single process"}


# ---------------------------------------------------------------------------
class ClockSampler:
    """NVML polling thread (2 ms period) over the timed region: SM clock and
    the throttle reasons nvidia-smi reports as clocks_event_reasons."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index):
        import threading
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception as e:  # noqa: BLE001
            self.nv, self.err = None, str(e)
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.002)

    def stop(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvml unavailable: {self.err}"]}
        self._stop.set()
        self.t.join(timeout=2)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def run_ours(a):
    import torch
    from paper_2110_04421_b200 import _native as N
    from paper_2110_04421_b200.confignet import synthesize
    from paper_2110_04421_b200.defaults import default_disease, default_progression
    from paper_2110_04421_b200.interventions import InterventionConfig
    from paper_2110_04421_b200.keyed import replication_seed
    from paper_2110_04421_b200.sim import ConfigSimulation

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    spec = workload_spec(a.workload)
    disease, table, iv = default_disease(), default_progression(), workload_iv(a.workload, a.dose_gap)
    pop = synthesize(spec, 0)
    n_sims = a.warmup + a.steps
    modes = ["csr", "fused"] if a.mode == "auto" else [a.mode]
    if a.precision == "f64":
        modes = ["csr"]                  # fused mode is fp32 only

    def make(mode, i):
        seed = replication_seed(0, rank * 100_000 + i)
        return ConfigSimulation(pop, disease, table, iv, seed, mode=mode, precision=a.precision,
                                horizon=HORIZON)

    # L2 flush buffer (> 126 MB L2), written between timed simulations
    flush = torch.empty(384 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def time_mode(mode):
        sims = [make(mode, i) for i in range(n_sims)]
        for s in sims:
            s.capture()
        torch.cuda.synchronize()
        for s in sims[:a.warmup]:
            s.replay()
        torch.cuda.synchronize()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        clk = ClockSampler(local_rank)
        t0 = time.perf_counter()
        for k, s in enumerate(sims[a.warmup:]):
            flush.fill_(float(k))
            starts[k].record()
            s.replay()
            ends[k].record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        if dist:
            dist.barrier()
        clocks = clk.stop()
        ms = [st.elapsed_time(en) for st, en in zip(starts, ends)]
        edges = sum(int(s.records()[:, N.REC["edges"]].sum()) for s in sims[a.warmup:])
        return dict(mode=mode, ms=ms, edges=edges, wall=wall, clocks=clocks, sims=sims)

    results = [time_mode(m) for m in modes]
    best = min(results, key=lambda r: sum(r["ms"]) / max(1, r["edges"]))
    ms_total = sum(best["ms"])
    if dist:
        t = torch.tensor([ms_total], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        e = torch.tensor([best["edges"]], device="cuda", dtype=torch.float64)
        dist.all_reduce(e)
        edges_all = float(e.item())
    else:
        edges_all = float(best["edges"])
    value = edges_all / (ms_total / 1000.0)

    # --- per-kernel device times (instrumented, same inputs) -> roofline
    profs = {r["mode"]: kernel_profile(r["sims"][a.warmup], r["mode"]) for r in results}
    prof = profs[best["mode"]]
    # --- end to end through the public API from pinned host buffers (every
    # rank; whole-job value = summed edges / max time over the ranks)
    e2e = end_to_end(make(best["mode"], 0), a, make(best["mode"], 0))
    serial = end_to_end(make(best["mode"], 0), a)      # copy in, run, copy out: nothing hidden
    if dist:
        t = torch.tensor([e2e["ms_per_step"], e2e["edges_per_step"]], device="cuda", dtype=torch.float64)
        dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:])
        e2e["ms_per_step"], e2e["edges_per_step"] = float(t[0]), float(t[1])
        e2e["value"] = e2e["edges_per_step"] / (e2e["ms_per_step"] / 1000.0)
        e2e["h2d_bytes_per_step"] *= world
        e2e["d2h_bytes_per_step"] *= world
    e2e.pop("edges_per_step")
    e2e["serial"] = {"value": serial["value"], "ms_per_step": serial["ms_per_step"], "copies": serial["copies"]}

    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    roof = prof["roofline"]
    roof["peak"] = peak
    roof["frac"] = roof["achieved"] / peak
    roof["peak_source"] = "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.65 TB/s"
    tfile = ROOT / "profiles" / "r02_traffic.json"
    if tfile.exists():
        tr = json.loads(tfile.read_text()).get(roof["kernel"])
        if tr:
            roof["traffic"] = tr["dram_bytes_read"] + tr["dram_bytes_write"]
            roof["traffic_source"] = tr["source"]
            # HBM is not what binds these kernels: their working set is
            # L2-resident; the ncu ceilings that do bind ride along
            if "ceilings" in tr:
                roof["binding_ceilings"] = tr["ceilings"]

    # north_star's multi-GPU path: config 3 partitioned over the same ranks
    # (strong scaling), measured beside the headline at every N
    part = None
    if not a.no_partition and a.workload == "config1":
        part = measure_partition(min(a.steps, 5), min(a.warmup, 2) or 1, rank, local_rank, world, dist)
    if rank != 0:
        return
    line = {
        "metric": "agent-interactions/sec", "value": value, "unit": "agent-interactions/s",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms_total / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": a.precision, "data": "synthetic",
        "config": {
            "workload": workload_string(a),
            "mode": best["mode"], "step": "one full 180-day simulation (CUDA graph replay)",
            "kernel_path": prof.get("path", "one kernel sequence per day"),
            "replicas": f"{a.steps} timed replications per GPU, distinct seeds",
            "l2": "flushed between timed simulations (384 MB write)",
            "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
        },
        "wall_s_per_sim": ms_total / a.steps / 1000.0,
        "undirected_contacts_per_s": value / 2,
        # end-to-end HBM GB/s = algorithmic bytes of all the
        # day kernels / device time per simulation
        "hbm_gbs_end_to_end": prof["alg_bytes_per_sim"] / (ms_total / a.steps / 1e3) / 1e9,
        "modes": {r["mode"]: {"ms_per_sim": sum(r["ms"]) / len(r["ms"]),
                              "interactions_per_s": r["edges"] / (sum(r["ms"]) / 1000)}
                  for r in results},
        "kernels": {m: p["kernels"] for m, p in profs.items()},
        "roofline": roof,
        "e2e": e2e,
        "gpu_launches": prof["launches_per_sim"] * a.steps,
        "clocks": best["clocks"],
    }
    if not a.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline_single(a.workload, a.cpu_seconds)
    if part is not None:
        line["partition_config3"] = {k: v for k, v in part.items() if v is not None or k != "e2e"}
    if not a.no_message_pass and world == 1:
        # north-star part (a) alone at BASELINE config-3 scale (10M agents):
        # the HBM-bound kernel of the decomposition, streamed 16-bit messages
        from paper_2110_04421_b200.roofline import message_pass_roofline
        mp = message_pass_roofline(10_000_000, peak_gbps=peak)
        tr = json.loads(tfile.read_text()).get("k_msg_pass<0> message pass (10M agents)") \
            if tfile.exists() else None
        mp["traffic"] = (tr["dram_bytes_read"] + tr["dram_bytes_write"]) if tr else None
        mp["bound"] = "hbm"
        line["roofline_message_pass_config3"] = mp
    print(json.dumps(line), flush=True)


def kernel_profile(sim, mode):
    """Per-kernel CUDA-event times over one full simulation (non-graph run with
    events between the launches of every day; a persistent run: events around
    day 0 and around the one k_fused_run launch of the other days)."""
    import ctypes
    import torch
    from paper_2110_04421_b200 import _native as N
    from paper_2110_04421_b200.engine import _u64
    if mode == "fused" and sim.uses_persistent_run():
        return persistent_profile(sim)
    sim.reset()
    torch.cuda.synchronize()
    lib = sim._lib
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(sim.horizon)]
    for day in evs:
        for e in day:
            e.record()           # materialise the cudaEvent_t
    torch.cuda.synchronize()
    for t in range(sim.horizon):
        handles = (ctypes.c_void_p * 4)(*[e.cuda_event for e in evs[t]])
        st = sim.state.struct()
        N.check(lib.epi_sim_step_timed(
            sim._ctx, ctypes.byref(st), t, _u64(sim.seed), 0 if mode == "csr" else 1,
            N.F64_CANONICAL if sim.precision == "f64" else N.F32,
            N.ptr(sim.codes[t & 1]), N.ptr(sim.codes[(t + 1) & 1]), N.ptr(sim.rec[t]),
            N.ptr(sim.vax), ctypes.addressof(handles), N.stream_handle()))
    torch.cuda.synchronize()
    sim.clock = sim.horizon
    gen = [evs[t][0].elapsed_time(evs[t][1]) for t in range(sim.horizon)]
    pas = [evs[t][1].elapsed_time(evs[t][2]) for t in range(sim.horizon)]
    ivt = [evs[t][2].elapsed_time(evs[t][3]) for t in range(sim.horizon)]
    rec = sim.records()
    E = rec[:, N.REC["edges"]].astype(np.float64)
    n = sim.n
    iv = sim.iv
    has_iv = iv.testing_enabled or iv.quarantine_enabled or iv.den_enabled or iv.vaccination_enabled
    total_ms = sum(gen) + sum(pas) + (sum(ivt) if has_iv else 0.0)
    kernels = {}
    if mode == "csr":
        # generator writes a 2 B pre-joined message per edge + 4 B row length
        # and reads 2 B code/agent; message pass + update streams the 2 B
        # messages: B_K1 = 2E + 10N (SURVEY §8(d) with 2-byte messages instead
        # of 4-byte src ids, no code gathers) + 16N state r/w
        b_gen = 2 * E + 6 * n
        b_pass = 2 * E + 10 * n + 16 * n
        kernels["k_day_tables+k_net_realize"] = {"ms_per_launch": sum(gen) / len(gen),
                                    "share": sum(gen) / total_ms,
                                    "alg_GBps": float(np.sum(b_gen) / (sum(gen) / 1e3) / 1e9)}
        kernels["k_pass_update"] = {"ms_per_launch": sum(pas) / len(pas),
                                    "share": sum(pas) / total_ms,
                                    "alg_GBps": float(np.sum(b_pass) / (sum(pas) / 1e3) / 1e9)}
        if has_iv:
            kernels["interventions (per-phase kernels)"] = {"ms_per_launch": sum(ivt) / len(ivt),
                                                            "share": sum(ivt) / total_ms}
        dom = "k_pass_update" if sum(pas) >= sum(gen) else "k_day_tables+k_net_realize"
        byt = b_pass if dom == "k_pass_update" else b_gen
        ms = pas if dom == "k_pass_update" else gen
        launches = 3
    else:
        # merged fused kernel: state r/w 16 N + own code 2 N + push rows
        # (rin 32 B + rout ids 64 B) + rin clear 32 B + next-day scatter ~16 B
        b = (16 + 2 + 32 + 64 + 32 + 16) * n
        kernels["day0_tables+keys"] = {"ms_per_launch": sum(gen) / len(gen), "share": sum(gen) / total_ms}
        kernels["k_fused_step"] = {"ms_per_launch": sum(pas) / len(pas), "share": sum(pas) / total_ms,
                                   "alg_GBps": float(b * len(pas) / (sum(pas) / 1e3) / 1e9)}
        dom, byt, ms, launches = "k_fused_step", b * np.ones_like(E), pas, 1
        extra = 2
        if has_iv:
            # fused intervention day: k_fused_step (+ testing), k_den_regen,
            # k_iv_post_chunks, k_finish_iv (+ doses, death days, tomorrow's
            # push tables); day 0 also k_day_keys + k_day_tables (+ k_died_update)
            den = iv.den_enabled and iv.testing_enabled
            post = iv.den_enabled or iv.quarantine_enabled or iv.vaccination_enabled
            kernels["interventions: k_den_regen + k_iv_post_chunks + k_finish_iv"] = {
                "ms_per_launch": sum(ivt) / len(ivt), "share": sum(ivt) / total_ms}
            launches = 2 + (1 if post else 0) + (1 if den else 0)
            extra = 1 + 2 + (1 if iv.den_enabled else 0) - (1 if den else 0)
    achieved = float(np.sum(byt) / (sum(ms) / 1e3) / 1e9)
    sim_bytes = float(np.sum(b_gen) + np.sum(b_pass)) if mode == "csr" else float(np.sum(b * np.ones_like(E)))
    return {"kernels": kernels,
            "launches_per_sim": launches * sim.horizon + (extra if mode != "csr" else 0),
            "alg_bytes_per_sim": sim_bytes,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "unit": "GB/s",
                         "traffic": None,
                         "bytes_model": "see DESIGN.md §4 (algorithmic bytes per launch)"}}


def persistent_profile(sim):
    """Day 0 (day tables + k_fused_step) and k_fused_run (days 1..179, one
    launch), CUDA events on the launching stream."""
    import torch
    from paper_2110_04421_b200 import _native as N
    sim.reset()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    sim.run(1)
    ev[1].record()
    sim.run()
    ev[2].record()
    torch.cuda.synchronize()
    day0, run = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    n, days = sim.n, sim.horizon - 1
    iv = sim.iv
    has_iv = iv.testing_enabled or iv.quarantine_enabled or iv.den_enabled or iv.vaccination_enabled
    # per agent-day, state in registers and the out-rows (rout) in shared
    # memory: own code write 2 + in-row read 32 + in-row clear 32 + next-day
    # scatter ~16 = 82 B; k_fused_run (up to 704 agents per SM) reads each
    # worker's 32-byte colleague row instead of gathering 16 codes: + 32 B
    # per worker.  On intervention days + the agent's state reloaded (16) and
    # the intervention columns read and written (testing, DEN, dropout,
    # doses, buckets: ~44) = 142 B
    workers = len(sim.population.wp_members) if sim.n <= 148 * 704 else 0
    b_day = 142 * n if has_iv else 82 * n + 32 * workers
    b_day0 = (16 + 2 + 32 + 64 + 32 + 16) * n + (32 + 10 + 1) * n      # + day-0 tables
    total = day0 + run
    name = "k_iv_run" if has_iv else "k_fused_run"
    d0name = "day0_tables+k_fused_step" + ("+intervention kernels" if has_iv else "")
    kernels = {d0name: {"ms_per_launch": day0, "share": day0 / total},
               name: {"ms_per_launch": run, "share": run / total, "days_per_launch": days,
                      "us_per_day": run * 1e3 / days, "alg_GBps": b_day * days / (run / 1e3) / 1e9}}
    achieved = b_day * days / (run / 1e3) / 1e9
    # ours per simulation: k_codes (reset), k_day_keys + k_day_tables + k_fused_step (day 0), the run;
    # intervention day 0 also k_died_update, k_iv_post_chunks, k_finish_iv
    launches = 5 + (3 if has_iv else 0)
    return {"kernels": kernels, "launches_per_sim": launches,
            "path": f"day 0: day tables + k_fused_step{' + intervention kernels' if has_iv else ''}; "
                    f"days 1-179: one persistent {name} launch",
            "alg_bytes_per_sim": float(b_day * days + b_day0),
            "roofline": {"bound": "hbm", "kernel": name, "achieved": achieved, "unit": "GB/s",
                         "traffic": None, "days_per_launch": days,
                         "bytes_model": f"{b_day / n:.1f} B per agent-day (DESIGN.md §4), x 179 days per launch"}}


def end_to_end(sim, a, sim2=None):
    """Public API from pinned host memory, every step: upload the initial
    state (all 22 columns, 7 MB), simulate 180 days, read the 19-column time
    series back.  With `sim2` the steps go through `sim.HostPipeline`: the
    copies of step k +- 1 run on a copy stream under the compute of step k."""
    import torch
    from paper_2110_04421_b200.sim import HostPipeline
    # the initial state in the device arena's layout, pinned: one copy in
    pinned = sim.initial.host_arena(sim.initial_host_columns())
    outs = [torch.empty((sim.horizon, 19), dtype=torch.int64).pin_memory() for _ in range(2)]
    h2d = int(pinned.numel())
    d2h = int(outs[0].numel() * outs[0].element_size())
    if sim2 is not None:
        pipe = HostPipeline([sim, sim2])
        k0 = 0
        for _ in range(a.warmup):
            pipe.submit(k0, pinned, outs[k0 & 1])
            k0 += 1
        pipe.drain()
        torch.cuda.synchronize()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for k in range(a.steps):
            pipe.submit(k0 + k, pinned, outs[(k0 + k) & 1])
        pipe.drain()
        en.record()
        torch.cuda.synchronize()
        mode = "pipelined: copies of the neighbouring steps under the compute (sim.HostPipeline)"
    else:
        sim.capture()

        def once():
            sim.initial.arena.copy_(pinned, non_blocking=True)
            sim.replay()
            outs[0].copy_(sim.rec[:, :19], non_blocking=True)
        for _ in range(a.warmup):
            once()
        torch.cuda.synchronize()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for _ in range(a.steps):
            once()
        en.record()
        torch.cuda.synchronize()
        mode = "serial: copy in, simulate, copy out"
    ms = st.elapsed_time(en) / a.steps
    edges = float(sim.records()[:, 19].sum())
    return {"value": edges / (ms / 1000.0), "unit": "agent-interactions/s",
            "ms_per_step": ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "edges_per_step": edges, "copies": mode}


def measure_partition(steps, warmup, rank, local_rank, world, dist, e2e_args=None):
    """Config 3 (10M agents, config-1 networks, 180 days): one simulation
    partitioned by agent range over the `world` ranks (strong scaling), the
    per-day code all-gather over native NCCL inside the native day loop, the
    whole run captured as one CUDA graph per rank; 1 rank = the whole
    population on one GPU.  Device time, max over the ranks."""
    import torch
    from paper_2110_04421_b200 import _native as N
    from paper_2110_04421_b200.confignet import DevicePopulation
    from paper_2110_04421_b200.defaults import default_disease, default_progression
    from paper_2110_04421_b200.interventions import InterventionConfig
    from paper_2110_04421_b200.keyed import replication_seed
    from paper_2110_04421_b200.partition import NcclComm, PartitionedSimulation, PartitionPlan
    from paper_2110_04421_b200.sim import ConfigSimulation
    spec = workload_spec("config3")
    pop = DevicePopulation(spec, 0)        # row f3: built on the device
    d, t, iv = default_disease(), default_progression(), InterventionConfig()
    seed = replication_seed(0, 0)
    if world > 1:
        plan = PartitionPlan(spec.n_agents, world)
        comm = NcclComm.from_process_group()
        sim = PartitionedSimulation(pop, d, t, iv, seed, plan, rank, comm=comm, mode="fused",
                                    horizon=HORIZON)
    else:
        sim = ConfigSimulation(pop, d, t, iv, seed, mode="fused", horizon=HORIZON)
    sim.capture()
    for _ in range(warmup):
        sim.replay()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = ClockSampler(local_rank)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(steps):
        sim.replay()
    en.record()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = st.elapsed_time(en)
    rec = sim.rec.clone()
    if dist:
        rec = reduce_partition_records(rec, world)
        tt = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    edges = float(rec[:, N.REC["edges"]].sum().item()) * steps
    e2e = None
    if e2e_args is not None and world == 1:
        # end to end through the public API: the 10M-agent initial state from
        # pinned host memory in, the time series out, every simulation
        e2e = end_to_end(sim, e2e_args)
        e2e.pop("edges_per_step", None)
    return {"e2e": e2e, "workload": "config3 (BASELINE.json configs[3]): 10M agents, config-1 networks, 180 days, "
                        "fused mode, no interventions",
            "value": edges / (ms / 1e3), "unit": "agent-interactions/s", "n_gpus": world,
            "steps": steps, "warmup": warmup, "ms_per_step": ms / steps, "scaling": "strong",
            "wall_s_per_sim": ms / steps / 1e3,
            "parallelism": (f"agent ranges x{world}: native NCCL all-gather of the 16-bit codes every "
                            "day inside the native day loop, tomorrow's sigma tables on a side stream, "
                            "one CUDA graph per rank" if world > 1 else "1 GPU"),
            "l2": "not flushed: every day touches the 10M-agent state (~160 MB hot, 700 MB total) and "
                  "tables, more than the 126 MB L2",
            "clocks": clocks}


def reduce_partition_records(rec, world):
    """Sum the ranks' partial day records (flags OR-ed, step kept)."""
    from paper_2110_04421_b200.partition import NcclCodeExchange, PartitionPlan
    plan = PartitionPlan(workload_spec("config3").n_agents, world)
    import torch.distributed as dist
    return NcclCodeExchange(plan, dist.get_rank()).reduce_records(rec)


def run_config3(a):
    """10M agents, agent-range partition over the ranks (strong scaling)."""
    import torch
    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    m = measure_partition(a.steps, a.warmup, rank, local_rank, world, dist, e2e_args=a)
    if rank == 0:
        clocks = m.pop("clocks")
        print(json.dumps({
            "metric": "agent-interactions/sec", "value": m["value"],
            "unit": "agent-interactions/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": m["ms_per_step"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": m["workload"], "parallelism": m["parallelism"], "l2": m["l2"]},
            "wall_s_per_sim": m["wall_s_per_sim"], "clocks": clocks, "e2e": m["e2e"]}), flush=True)


def run_config4(a):
    """Ensemble: R replicas per GPU of config 1, own seeds and rate scales,
    one CUDA graph per replica; no inter-GPU communication.  Default: each
    replica one persistent run (k_fused_run holds the whole GPU), replicas one
    after another on one stream; --replica-mode concurrent: per-day kernels on
    one block per SM, replicas on --streams concurrent streams."""
    import torch
    from paper_2110_04421_b200 import _native as N
    from paper_2110_04421_b200 import keyed
    from paper_2110_04421_b200.confignet import DevicePopulation
    from paper_2110_04421_b200.defaults import default_disease, default_progression
    from paper_2110_04421_b200.interventions import InterventionConfig
    from paper_2110_04421_b200.sim import ConfigSimulation
    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    spec = workload_spec("config4")
    pop = DevicePopulation(spec, 0)        # row f3: built on the device, shared by the replicas
    d0, t, iv = default_disease(), default_progression(), InterventionConfig()
    sims = []
    for i in range(a.replicas):
        r = rank * a.replicas + i
        u = keyed.uniform(0, 0, keyed.Purpose.REPLICATION, r, k=1)
        d = d0.with_rate(d0.rate_scale * (0.5 + u))
        # measured (replica-steps/s): persistent one after another 66.1 k;
        # concurrent on 8 streams with one block per SM 63.0 k (16 blocks
        # per SM: 59.4 k)
        sims.append(ConfigSimulation(pop, d, t, iv, keyed.replication_seed(0, r), mode="fused",
                                     horizon=HORIZON, persistent=a.replica_mode == "persistent",
                                     day_blocks_per_sm=1))
    n_streams = 1 if a.replica_mode == "persistent" else a.streams   # cooperative runs serialise anyway
    streams = [torch.cuda.Stream() for _ in range(n_streams)]
    for s in sims:
        s.capture()
    torch.cuda.synchronize()

    def sweep():
        for i, s in enumerate(sims):
            with torch.cuda.stream(streams[i % len(streams)]):
                s._graph.replay()
        for st_ in streams:
            torch.cuda.current_stream().wait_stream(st_)
    for _ in range(a.warmup):
        sweep()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = ClockSampler(local_rank)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(a.steps):
        sweep()
    en.record()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = st.elapsed_time(en)
    recs = torch.stack([s.rec for s in sims])                     # [R, days, 24]
    edges = float(recs[:, :, N.REC["edges"]].sum().item()) * a.steps
    new_inf = recs[:, :, N.REC["new_inf"]].double()
    if dist:
        tt = torch.tensor([ms, edges], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:])
        ms, edges = float(tt[0]), float(tt[1])
        allc = [torch.empty_like(new_inf) for _ in range(world)]
        dist.all_gather(allc, new_inf)
        new_inf = torch.cat(allc)
    # end to end through the public API: every replica's initial state from
    # pinned host memory in, its time series out, inside the timed region
    pinned = [s_.initial.host_arena(s_.initial_host_columns()) for s_ in sims]
    outs = [torch.empty((HORIZON, 19), dtype=torch.int64).pin_memory() for _ in sims]

    def sweep_e2e():
        for i, s_ in enumerate(sims):
            with torch.cuda.stream(streams[i % len(streams)]):
                s_.initial.arena.copy_(pinned[i], non_blocking=True)
                s_._graph.replay()
                outs[i].copy_(s_.rec[:, :19], non_blocking=True)
        for st_ in streams:
            torch.cuda.current_stream().wait_stream(st_)
    e_steps = max(1, min(a.steps, 3))
    sweep_e2e()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    st.record()
    for _ in range(e_steps):
        sweep_e2e()
    en.record()
    torch.cuda.synchronize()
    e_ms = st.elapsed_time(en)
    e_edges = float(torch.stack([s_.rec for s_ in sims])[:, :, N.REC["edges"]].sum().item()) * e_steps
    if dist:
        tt = torch.tensor([e_ms, e_edges], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:])
        e_ms, e_edges = float(tt[0]), float(tt[1])
    e2e = {"value": e_edges / (e_ms / 1e3), "unit": "agent-interactions/s", "ms_per_step": e_ms / e_steps,
           "steps": e_steps, "h2d_bytes_per_step": int(sum(int(x.numel()) for x in pinned)),
           "d2h_bytes_per_step": int(sum(o.numel() * o.element_size() for o in outs)),
           "copies": "serial per replica: its initial state in, its 180 days, its series out"}
    reps = a.replicas * world
    # replication quartiles of the daily infection curve on the device
    # (row f3 output: epi_quartiles, bitwise the reference's summarize)
    from paper_2110_04421_b200.series import summarize_device
    quart = summarize_device(recs, ["new_infections"])["new_infections"] if world == 1 else None
    if rank == 0:
        mean = new_inf.mean(0).cpu().numpy()
        std = new_inf.std(0).cpu().numpy()
        print(json.dumps({
            "metric": "agent-interactions/sec", "value": edges / (ms / 1e3),
            "unit": "agent-interactions/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"config4 (BASELINE.json configs[4]): {reps} replicas of config 1 "
                       "(shared static population, own seed, rate 3.3x[0.5,1.5]); one step = all "
                       "replicas x 180 days", "parallelism": f"{a.replicas} replicas/GPU ({a.replica_mode}) on "
                       f"{n_streams} stream(s) x {world} GPUs",
                       "l2": "not flushed: the replicas' states and push tables (~20 MB each) "
                       "exceed the 126 MB L2 many times over"},
            "replica_steps_per_s": reps * HORIZON * a.steps / (ms / 1e3),
            "daily_new_infections_mean": [round(float(x), 2) for x in mean],
            "daily_new_infections_std": [round(float(x), 2) for x in std],
            "daily_new_infections_quartiles": (None if quart is None else
                                               [[round(float(v), 2) for v in row] for row in quart]),
            "clocks": clocks, "e2e": e2e}), flush=True)


REFNET_DESC = ("refnet: the reference's own benchmark scenario (epivec bench --agents 100000 --steps "
               "180): default population_spec.json population (mirror of population.synthesize), "
               "households + per-occupation Watts-Strogatz (beta 0.1) + stub-pairing random network "
               "realized every step, 10 seeds, default disease/progression, fp64 canonical hazard")


def run_refnet(a):
    """The reference's own benchmark on the device: ReferenceNativeSimulation
    (population mirror, device realizer, GpuEngine resident).  One step = one
    180-step replication; interactions = directed edges gathered."""
    import torch
    from paper_2110_04421_b200.refsim import ReferenceNativeSimulation
    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")

    def make(i):
        return ReferenceNativeSimulation(REFNET_AGENTS, base_seed=1000 * rank + i,
                                         initial_infections=REFNET_SEEDS, horizon=HORIZON)
    # the first replications of a process pay one-time costs (lazy kernel
    # loading, allocator growth): at least two untimed ones
    for i in range(max(a.warmup, 2)):
        make(i).run()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = ClockSampler(local_rank)
    total_ms = 0.0
    edges = 0
    e2e_ms = 0.0
    h2d = 0
    for i in range(a.steps):
        # e2e: host population -> device (engine + realizer tables), seeding,
        # 180 steps (per-step events read back), final state -> host
        t0 = time.perf_counter()
        sim = make(a.warmup + i)
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        handle = sim.issue()       # the 180 steps (device work bracketed by the events)
        en.record()
        sim.finish(handle)         # flags, error bits, per-step events (host; inside e2e)
        sim.engine.sync_to_host()
        torch.cuda.synchronize()
        t_all = time.perf_counter() - t0
        total_ms += st.elapsed_time(en)
        edges += sim.interactions
        e2e_ms += 1e3 * (t_all - sim.host_setup_s)       # minus the host-only population draw
        h2d = sum(t.numel() * t.element_size() for t in sim.engine.dev.t.values())
    clocks = clk.stop()
    ms = total_ms
    if dist:
        tt = torch.tensor([ms, edges, e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:2])
        dist.all_reduce(tt[2:], op=dist.ReduceOp.MAX)
        ms, edges, e2e_ms = float(tt[0]), float(tt[1]), float(tt[2])
    if rank != 0:
        return
    line = {
        "metric": "agent-interactions/sec", "value": edges / (ms / 1e3),
        "unit": "agent-interactions/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": REFNET_DESC, "step": "one 180-step replication (GpuRealizer + "
                   "GpuEngine resident, records and edge counts on the device, no host sync "
                   "inside the 180 steps: the realizer's count feeds the graph load)",
                   "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
                   "l2": "not flushed; every step regenerates the graphs (> L2 traffic per step)"},
        "wall_s_per_sim": ms / a.steps / 1e3,
        "e2e": {"value": edges / (e2e_ms / 1e3), "unit": "agent-interactions/s",
                "ms_per_step": e2e_ms / a.steps, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": h2d + HORIZON * 8 * 24},
        "clocks": clocks,
    }
    if not a.no_cpu_baseline and world == 1:
        try:
            e, days, t = _cpu_worker(("refnet", 12345, a.cpu_seconds))
        except ImportError as err:
            e, days, t = 0, 0, float("nan")
            line["cpu_baseline_error"] = f"the reference (epivec) is not installed in baseline/_ref ({err})"
        line["cpu_baseline"] = {"value": e / t, "unit": "agent-interactions/s", "cores": 1,
                                "kind": "reference", "sample": f"the reference's own scenario "
                                f"(epivec initialize_run + GraphRealizer + Engine, baseline/_ref), "
                                f"1 replica, steps 0-{days - 1} of 180 ({e} directed edges in "
                                f"{t:.1f}s), single process"}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    DOSE_GAP[0] = a.dose_gap
    if a.impl == "reference":
        run_reference(a)
    elif a.workload == "config3":
        run_config3(a)
    elif a.workload == "config4":
        run_config4(a)
    elif a.workload == "refnet":
        run_refnet(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
