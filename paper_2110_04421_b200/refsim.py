"""The reference's own scenario on the device: `epivec bench` / `run_replication`
with the reference-native networks (runner.py:81-98,
138-152, 268-289).

    population  : host mirror of population.synthesize + the seeding choice
                  (population.py), bitwise identical to the reference's;
    seeding     : entry stage + first transition scheduled on the device
                  (k_seed, the same keyed draws as population.py:168-177);
    per step    : GpuRealizer.realize(step, dead) -> device StepGraph
                  (households, per-occupation small world, stub pairing)
                  -> GpuEngine.step (graph-in: canonical CSR, fp64 message
                  pass bitwise equal to Engine.gather_exposure, phases).

The agent state stays on the device (`resident`); interactions are the
directed edges gathered, the reference's definition (runner.py:269, 287).
"""

from __future__ import annotations

import time

import numpy as np

from . import _native as N
from .defaults import default_disease, default_progression
from .engine import GpuEngine, StepEvents
from .errors import ConfigError
from .interventions import InterventionConfig
from .keyed import replication_seed
from .population import PopulationSpec, choose_seeds, synthesize
from .refnet import GpuRealizer


class ReferenceNativeSimulation:
    """One replication of the reference's default scenario (scenario.py
    defaults: disease, progression, population_spec.json) at `n_agents`."""

    def __init__(self, n_agents: int = 100_000, base_seed: int = 0, replication: int = 0,
                 initial_infections: int = 10, horizon: int = 180, disease=None, table=None,
                 interventions=None, spec: PopulationSpec | None = None, device=None,
                 seed: int | None = None):
        import torch
        self.spec = spec or PopulationSpec.default(n_agents)
        # the replication seed (runner.py:77-78), or an explicit one
        self.seed = replication_seed(base_seed, replication) if seed is None else int(seed)
        self.horizon = horizon
        self.iv = interventions or InterventionConfig()
        t0 = time.perf_counter()
        cols = synthesize(self.spec, self.seed)
        ids = choose_seeds(cols, initial_infections, self.seed)
        self.host_setup_s = time.perf_counter() - t0   # host-only population draw
        self.cols = cols
        self.engine = GpuEngine(cols, disease or default_disease(), table or default_progression(),
                                self.iv, self.seed, check_invariants=False, resident=True,
                                device=device)
        self.engine.seed_infections(torch.from_numpy(ids).to(self.engine.device))
        if self.iv.den_enabled:     # runner.py:86-89
            self.engine.assign_app(self.iv.den.app_adoption)
        self.realizer = GpuRealizer(self.seed, cols.household_id, cols.occupation, cols.random_degree,
                                    self.spec.occupation_mean_interactions, self.spec.rewire_beta,
                                    device=device)
        self.interactions = 0
        self.records = torch.zeros((horizon, N.REC_LEN), dtype=torch.int64, device=self.engine.device)

    @property
    def clock(self) -> int:
        return self.engine.clock

    def step(self):
        """One reference step: realize the day's networks for the alive agents,
        then Engine.step on them (runner.py:145-150)."""
        dead = self.engine.dev.t["stage"] == 10
        ev = self.engine.step(self.realizer.realize(self.engine.clock, dead))
        self.interactions += ev.n_edges
        return ev

    def run(self, steps: int | None = None):
        """The remaining steps with the state, the edge counts and the records
        on the device and no host synchronisation inside the loop (the
        realizer's edge count goes to the graph load on the device); graph
        flags and realizer errors checked once at the end.  Returns the
        StepEvents."""
        return self.finish(self.issue(steps))

    def issue(self, steps: int | None = None):
        """Issue the remaining steps (or `steps` of them) on the current
        stream and return a handle for finish(); nothing is synchronised."""
        import torch
        first = self.clock
        last = self.horizon if steps is None else min(self.horizon, first + steps)
        counts = torch.zeros((max(last - first, 1), 2), dtype=torch.int64, device=self.engine.device)
        if last > first:
            self.engine.advance_refnet(self.realizer, first, last, counts, self.records[first:last])
        return first, last, counts

    def finish(self, handle):
        """Wait for issued steps, check the graph flags and the realizer's
        error bits, and return their StepEvents."""
        first, last, counts = handle
        self.engine.check_graph_flags()
        errs = counts[:, 1].cpu().numpy() if last > first else np.zeros(0, np.int64)
        bad = np.flatnonzero(errs)
        if len(bad):
            # the reference raises at the step that fails; here the steps after
            # it already ran on a truncated graph: the state is unusable
            t = first + int(bad[0])
            err = int(errs[bad[0]])
            what = ("edge output capacity exceeded" if err & 1 else "dedupe hash table full" if err & 2
                    else "more than 2^31 random-network stubs" if err & 4
                    else "rewiring collision list overflow")
            self.engine.invalidate(f"realizer failed at step {t}: {what}")
            raise ConfigError(f"step {t}: {what} (state invalid; rebuild the simulation)")
        rec = self.records[first:last].cpu().numpy()
        neg = rec[:, N.REC["flags"]] & N.FLAG_NEG_HAZARD
        if neg.any():
            t = first + int(np.flatnonzero(neg)[0])
            self.engine.invalidate(f"negative hazard at step {t}")
            from .errors import InvariantViolation
            raise InvariantViolation(f"step {t}: negative hazard out of gather")
        events = [StepEvents.from_record(r) for r in rec]
        self.interactions += sum(ev.n_edges for ev in events)
        return events
