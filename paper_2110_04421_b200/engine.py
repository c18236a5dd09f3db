"""Drop-in replacement for the reference `Engine` (engine.py:55-347).

Same constructor, attributes (`cols`, `disease`, `table`, `iv`, `seed`,
`clock`, `vaccination_open`, `contact_log`, `check`) and methods
(`step(graph) -> StepEvents`, `gather_exposure(graph) -> float64[N]`); every
phase runs on the GPU through libepib200:

  step(graph):  graph -> device COO -> counting sort by destination + per-row
                   sorts (register networks, block sort for long rows) into
                   the canonical (dst, src, kind) CSR
                -> fp64 message pass in (dst, src, kind) order (bitwise equal
                   to the reference) fused with transmission + progression
                -> intervention phase kernels -> per-step record.

Compat mode (default) uploads the caller's `AgentColumns` before each call and
writes the new state back afterwards, because reference callers read and
even mutate `cols` between steps (runner.py:101-116, tests).  With
`resident=True` the state stays on the device and `sync_to_host()` /
`sync_to_device()` move it explicitly.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .device import DeviceColumns, pack_params
from .errors import InvariantViolation
from .state import DYNAMIC_COLUMNS


@dataclass
class StepEvents:
    """Per-step counts (engine.py:41-52)."""

    step: int
    n_edges: int = 0
    new_infections: int = 0
    deaths: int = 0
    hospitalizations: int = 0
    tests_administered: int = 0
    doses_given: int = 0
    notifications_sent: int = 0

    @classmethod
    def from_record(cls, rec) -> "StepEvents":
        r = N.REC
        return cls(int(rec[r["step"]]), int(rec[r["edges"]]), int(rec[r["new_inf"]]),
                   int(rec[r["deaths"]]), int(rec[r["hosp"]]), int(rec[r["tests"]]),
                   int(rec[r["doses"]]), int(rec[r["notify"]]))


class DeviceContactLog:
    """Stand-in for `ContactLog` (interventions.py:145-178): the edges live in
    a device ring inside the native context; this object reports its size."""

    def __init__(self, lookback: int):
        self.lookback = lookback
        self._n = 0

    def _pushed(self):
        self._n = min(self._n + 1, self.lookback)

    def __len__(self):
        return self._n


class GpuEngine:
    """Single-writer columnar engine for one replication, on one GPU."""

    def __init__(self, cols, disease, table, interventions, seed: int,
                 check_invariants: bool = True, resident: bool = False, device=None,
                 infection_mode: str = "aggregate"):
        import torch
        self._lib = N.lib()
        self.cols = cols
        self.disease = disease
        self.table = table
        self.iv = interventions
        self.seed = seed
        self.clock = 0
        self.check = check_invariants
        self.resident = resident
        self.contact_log = DeviceContactLog(interventions.den.lookback) \
            if interventions.den_enabled else None
        self._sterilizing = int(interventions.vaccine.immunity_mode) == 0
        self.n = cols.n_agents
        self.device = torch.device(device or "cuda")
        self._params = pack_params(disease, table, interventions, self.n)
        ctx = N._p()
        N.check(self._lib.epi_create(C_ref(self._params), self.n, C_ref(ctx)))
        self._ctx = ctx
        # "independent": the reference oracle's independent-edges mode
        # (oracle.py:185-192), validation only
        modes = {"aggregate": 0, "independent": 1}
        if infection_mode not in modes:
            from .errors import ConfigError
            raise ConfigError(f"unknown infection mode {infection_mode!r}")
        N.check(self._lib.epi_set_infection_mode(self._ctx, modes[infection_mode]))
        self.dev = DeviceColumns.from_host(cols, self.device)
        self._vax = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._rec = torch.zeros(N.REC_LEN, dtype=torch.int64, device=self.device)

    def invalidate(self, why: str) -> None:
        """Refuse every later step: a failure was detected after the state
        had already moved on (a device-side loop checked at its end)."""
        self._invalid = why

    def _usable(self):
        why = getattr(self, "_invalid", None)
        if why:
            raise InvariantViolation(f"engine state is invalid ({why}); rebuild it")

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx is not None and ctx.value:
            self._lib.epi_destroy(ctx)
            self._ctx = None

    # -- initial state on the device (population.py:168-177, runner.py:86-89)
    def seed_infections(self, ids) -> None:
        """Entry stage + first transition of the chosen agents (sorted ids,
        device int64 tensor), with the reference's keyed step-0 draws."""
        st = self.dev.struct()
        N.check(self._lib.epi_seed_infections(self._ctx, C_ref(st), _u64(self.seed), N.ptr(ids),
                                              int(ids.numel()), N.stream_handle()))
        if not self.resident:
            self.sync_to_host()

    def assign_app(self, adoption: float) -> None:
        """has_den_app = u(seed, 0, DEN_APP, id) < adoption."""
        st = self.dev.struct()
        N.check(self._lib.epi_assign_app(C_ref(st), _u64(self.seed), float(adoption),
                                         N.stream_handle()))
        if not self.resident:
            self.sync_to_host()

    # -- state movement ---------------------------------------------------
    def sync_to_device(self):
        self.dev.upload(self.cols)

    def sync_to_host(self):
        self.dev.download(self.cols, DYNAMIC_COLUMNS)

    @property
    def vaccination_open(self) -> bool:
        return bool(int(self._vax.item()))

    @vaccination_open.setter
    def vaccination_open(self, value: bool):
        self._vax.fill_(int(bool(value)))

    # -- graph upload + validation (engine.py:124-133) ----------------------
    def _load(self, graph, check: bool = True):
        import torch
        if _on_device(graph):
            src, dst, kind = graph.src, graph.dst, graph.kind
        else:
            src = torch.from_numpy(np.ascontiguousarray(graph.src, np.int32)).to(self.device)
            dst = torch.from_numpy(np.ascontiguousarray(graph.dst, np.int32)).to(self.device)
            kind = torch.from_numpy(np.ascontiguousarray(graph.kind, np.int8)).to(self.device)
        self._graph_tensors = (src, dst, kind)      # keep alive while the ctx refers to them
        s = N.stream_handle()
        N.check(self._lib.epi_graph_load(self._ctx, N.ptr(src), N.ptr(dst), N.ptr(kind),
                                         int(src.shape[0]), s))
        if check:
            self.check_graph_flags(graph)

    def check_graph_flags(self, graph=None):
        """Raise for the validation flags the graph loads set (engine.py:124-133);
        reads and clears the device flag word (a host sync)."""
        s = N.stream_handle()
        flags = N._i32()
        N.check(self._lib.epi_read_flags(self._ctx, C_ref(flags), s))
        f = flags.value
        if f & N.FLAG_INDEX:
            if graph is None:
                raise InvariantViolation(f"a graph references an agent >= n_agents {self.n}")
            src, dst = _host(graph.src), _host(graph.dst)
            top = max(int(np.max(src)), int(np.max(dst)))
            raise InvariantViolation(f"graph references agent {top} >= n_agents {self.n}")
        if f & N.FLAG_SELFLOOP:
            raise InvariantViolation("graph contains a self-loop")
        if f & N.FLAG_KIND:
            raise InvariantViolation("graph contains an unknown network kind")

    def gather_exposure(self, graph):
        """Summed hazard per agent, float64[N], bitwise equal to the reference."""
        import torch
        if not self.resident:
            self.sync_to_device()
        self._load(graph)
        out = torch.empty(self.n, dtype=torch.float64, device=self.device)
        st = self.dev.struct()
        N.check(self._lib.epi_gather(self._ctx, C_ref(st), int(self.clock), N.F64_CANONICAL,
                                     N.ptr(out), N.stream_handle()))
        return out.cpu().numpy()

    def gather_exposure_f32(self, graph):
        """fp32 fast-mode hazard (factored per-source message), float32[N]."""
        import torch
        if not self.resident:
            self.sync_to_device()
        self._load(graph)
        out = torch.empty(self.n, dtype=torch.float32, device=self.device)
        st = self.dev.struct()
        N.check(self._lib.epi_gather(self._ctx, C_ref(st), int(self.clock), N.F32,
                                     N.ptr(out), N.stream_handle()))
        return out.cpu().numpy()

    # -- the step (engine.py:121-151) -----------------------------------------
    def step(self, graph, injected=None) -> StepEvents:
        self._usable()
        if graph.step != self.clock:
            raise InvariantViolation(
                f"graph built for step {graph.step}, engine clock is {self.clock}")
        if not self.resident:
            self.sync_to_device()
        self._load(graph)
        st = self.dev.struct()
        inj = _injected_array(injected)
        N.check(self._lib.epi_step(self._ctx, C_ref(st), int(self.clock), _u64(self.seed),
                                   N.ptr(self._rec), N.ptr(self._vax), inj, int(self.check),
                                   N.stream_handle()))
        rec = self._rec.cpu().numpy()
        if not self.resident:
            self.sync_to_host()
        if self.contact_log is not None:
            self.contact_log._pushed()
        # a negative hazard is always an error (engine.py:157-158); the state
        # invariants (state.py:90-102) only when checking
        _raise_for_flags(int(rec[N.REC["flags"]]), self.clock, self.n, self.check)
        ev = StepEvents.from_record(rec)
        self.clock += 1
        return ev

    def advance(self, graph, record) -> None:
        """`step` for device-resident pipelines: no host synchronisation.  The
        day's record goes to the device int64[EPI_REC_LEN] tensor `record`
        (StepEvents.from_record reads it later); graph validation flags
        accumulate until `check_graph_flags()`."""
        self._usable()
        if graph.step != self.clock:
            raise InvariantViolation(
                f"graph built for step {graph.step}, engine clock is {self.clock}")
        if not self.resident:
            raise InvariantViolation("advance() needs resident=True")
        self._load(graph, check=False)
        st = self.dev.struct()
        N.check(self._lib.epi_step(self._ctx, C_ref(st), int(self.clock), _u64(self.seed),
                                   N.ptr(record), N.ptr(self._vax), None, 0, N.stream_handle()))
        if self.contact_log is not None:
            self.contact_log._pushed()
        self.clock += 1

    def advance_counted(self, step: int, src, dst, kind, count, record) -> None:
        """`advance` for a device-side edge producer: the first count[0]
        (device uint64) entries of the device arrays src/dst/kind are the
        step's edges — no host synchronisation at all (a realizer loop can be
        captured in a CUDA graph).  Graph flags accumulate as in advance()."""
        self._usable()
        if step != self.clock:
            raise InvariantViolation(f"graph built for step {step}, engine clock is {self.clock}")
        if not self.resident:
            raise InvariantViolation("advance_counted() needs resident=True")
        N.check(self._lib.epi_graph_load_counted(self._ctx, N.ptr(src), N.ptr(dst), N.ptr(kind), N.ptr(count),
                                                 int(src.shape[0]), N.stream_handle()))
        st = self.dev.struct()
        N.check(self._lib.epi_step(self._ctx, C_ref(st), int(self.clock), _u64(self.seed),
                                   N.ptr(record), N.ptr(self._vax), None, 0, N.stream_handle()))
        self.clock += 1

    def advance_refnet(self, realizer, first: int, last: int, counts, records) -> None:
        """Steps [first, last) of the reference's replication loop
        (runner.py:138-150) issued natively (`epi_refnet_run`): dead mask,
        realizer (dead agents read from the stage column), counted graph load
        and the step, per step, with no host
        synchronisation.  counts = device int64[last-first][2] (edges, realizer
        error bits), records = device int64[last-first][REC_LEN]."""
        import torch
        self._usable()
        if first != self.clock:
            raise InvariantViolation(f"graph built for step {first}, engine clock is {self.clock}")
        if not self.resident:
            raise InvariantViolation("advance_refnet() needs resident=True")
        if realizer.n_agents != self.cols.n_agents:
            raise InvariantViolation("realizer population size differs from the engine's")
        src, dst, kind = realizer.buffers()
        st = self.dev.struct()
        N.check(self._lib.epi_refnet_run(realizer._h, self._ctx, C_ref(st), _u64(realizer.seed), _u64(self.seed),
                                         int(first), int(last),
                                         N.ptr(src), N.ptr(dst), N.ptr(kind),
                                         int(src.shape[0]), N.ptr(counts), N.ptr(records), N.ptr(self._vax),
                                         N.stream_handle()))
        self.clock = last

    def step_with_hazard(self, hazard, injected=None) -> StepEvents:
        """Phases 1-6 with a caller-supplied float64 hazard (parity tests)."""
        self._usable()
        import torch
        if not self.resident:
            self.sync_to_device()
        h = torch.as_tensor(np.ascontiguousarray(hazard, np.float64)).to(self.device)
        st = self.dev.struct()
        N.check(self._lib.epi_step_with_hazard(self._ctx, C_ref(st), int(self.clock),
                                               _u64(self.seed), N.ptr(h), N.ptr(self._rec),
                                               N.ptr(self._vax), _injected_array(injected),
                                               N.stream_handle()))
        rec = self._rec.cpu().numpy()
        if not self.resident:
            self.sync_to_host()
        _raise_for_flags(int(rec[N.REC["flags"]]), self.clock, self.n, self.check)
        ev = StepEvents.from_record(rec)
        self.clock += 1
        return ev

    def last_record(self) -> np.ndarray:
        return self._rec.cpu().numpy()


def _on_device(graph) -> bool:
    """Any StepGraph-shaped object: the reference's (numpy arrays,
    graphs.py:30-51) or this package's (numpy or CUDA tensors)."""
    return not isinstance(graph.src, np.ndarray) and hasattr(graph.src, "data_ptr")


def _host(a) -> np.ndarray:
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


def _raise_for_flags(f: int, step: int, n: int, check: bool = True) -> None:
    if f & N.FLAG_NEG_HAZARD:
        raise InvariantViolation("negative hazard out of gather")
    if not check:
        return
    if f & N.FLAG_STAGE_RANGE:
        raise InvariantViolation(f"step {step}: stage out of range")
    if f & N.FLAG_NO_TIMESTAMP:
        raise InvariantViolation(f"step {step}: non-susceptible agent without infection timestamp")


def _u64(x: int) -> int:
    return int(x) & ((1 << 64) - 1)


def _injected_array(injected):
    """dict purpose -> device float64 tensor  ->  double*[12] (or None)."""
    if not injected:
        return None
    arr = (N._p * 12)()
    for k, t in injected.items():
        arr[int(k)] = N.ptr(t)
    _injected_array.keep = (arr, injected)
    import ctypes
    return ctypes.addressof(arr)


def C_ref(x):
    import ctypes
    return ctypes.byref(x)
