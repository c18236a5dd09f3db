"""Host-side cost of building one reference-native replication (the part of
the refnet e2e number that is not the 180 steps)."""
import sys, time; sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2110_04421_b200 import refsim
from paper_2110_04421_b200.defaults import default_disease, default_progression
from paper_2110_04421_b200.engine import GpuEngine
from paper_2110_04421_b200.interventions import InterventionConfig
from paper_2110_04421_b200.population import PopulationSpec, choose_seeds, synthesize
from paper_2110_04421_b200.refnet import GpuRealizer

spec = PopulationSpec.default(100_000)
for rep in range(4):
    T = {}
    t = time.perf_counter()
    cols = synthesize(spec, rep); T["synth"] = time.perf_counter() - t
    t = time.perf_counter()
    ids = choose_seeds(cols, 10, rep); T["seeds"] = time.perf_counter() - t
    t = time.perf_counter()
    eng = GpuEngine(cols, default_disease(), default_progression(), InterventionConfig(), rep,
                    check_invariants=False, resident=True); torch.cuda.synchronize()
    T["engine"] = time.perf_counter() - t
    t = time.perf_counter()
    eng.seed_infections(torch.from_numpy(ids).cuda()); torch.cuda.synchronize()
    T["seed_inf"] = time.perf_counter() - t
    t = time.perf_counter()
    r = GpuRealizer(rep, cols.household_id, cols.occupation, cols.random_degree,
                    spec.occupation_mean_interactions, spec.rewire_beta); torch.cuda.synchronize()
    T["realizer"] = time.perf_counter() - t
    t = time.perf_counter()
    sim = refsim.ReferenceNativeSimulation(100_000, base_seed=rep, initial_infections=10, horizon=180)
    torch.cuda.synchronize(); T["whole_ctor"] = time.perf_counter() - t - sim.host_setup_s
    t = time.perf_counter()
    sim.run(); torch.cuda.synchronize(); T["run"] = time.perf_counter() - t
    t = time.perf_counter()
    sim.engine.sync_to_host(); torch.cuda.synchronize(); T["to_host"] = time.perf_counter() - t
    t = time.perf_counter()
    del sim, eng, r; torch.cuda.synchronize(); T["del"] = time.perf_counter() - t
    print(" ".join(f"{k} {1e3 * v:.1f}" for k, v in T.items()), flush=True)
