"""Device-resident simulation of the config networks (BASELINE.json 0-4).

One `ConfigSimulation` = one replication: static population layout on the
device, agent state in `DeviceColumns`, double-buffered 16-bit source codes,
and a [horizon, 24] int64 record buffer filled by the kernels (one row per
day, runner.py:101-116 columns plus edge/event counters).  `run()` issues
every day of the horizon with no host synchronisation; `capture()` records
the whole horizon into one CUDA graph and `replay()` relaunches it.

Modes:
  "csr"   — per day: generator kernel writes the padded dst-major CSR, then
            one fused message-pass + update kernel (north-star parts a-c);
  "fused" — per day: one kernel enumerates in-edges and consumes their
            source codes on the fly; no edge list ever reaches memory.
precision "f64" (csr only) = canonical-order fp64, bitwise equal to the
reference Engine driven by the same graphs; "f32" = fast mode.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .confignet import ConfigNetworkSpec, ConfigPopulation, DevicePopulation, synthesize
from .device import DeviceColumns, pack_params
from .engine import _u64
from .errors import ConfigError
from .graph import StepGraph
from .interventions import InterventionConfig
from .state import AgentColumns

SERIES_COLUMNS = slice(0, 19)


class DeviceNetwork:
    """Static config-network arrays on the device + the C `epi_net` view
    (from a host ConfigPopulation or a DevicePopulation)."""

    def __init__(self, pop: ConfigPopulation, device):
        import torch
        if not _TORCH_DT:
            _init_dtypes()

        def up(a, dt):
            if torch.is_tensor(a):      # DevicePopulation: already on the device
                return a.to(device=device, dtype=_TORCH_DT[np.dtype(dt)]).contiguous()
            return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(device)
        spec = pop.spec
        self.hh_off = up(pop.hh_off, np.uint8)
        self.hh_size = up(pop.hh_size, np.uint8)
        self.wp_id = up(pop.wp_id, np.int32)
        self.wp_local = up(pop.wp_local, np.uint8)
        self.wp_base = up(pop.wp_base if len(pop.wp_base) else np.zeros(1), np.int32)
        self.wp_size = up(pop.wp_size if len(pop.wp_size) else np.zeros(1), np.int32)
        self.wp_members = up(pop.wp_members if len(pop.wp_members) else np.zeros(1), np.int32)
        s = N.EpiNet()
        s.n_agents = spec.n_agents
        s.hh_off, s.hh_size = N.ptr(self.hh_off), N.ptr(self.hh_size)
        s.wp_id, s.wp_local = N.ptr(self.wp_id), N.ptr(self.wp_local)
        s.wp_base, s.wp_size = N.ptr(self.wp_base), N.ptr(self.wp_size)
        s.wp_members = N.ptr(self.wp_members)
        s.n_workplaces = pop.n_workplaces
        s.colleague_draws = spec.colleague_draws
        s.random_slots = spec.random_slots
        s.row_cap = spec.row_capacity
        s.n_member_slots = len(pop.wp_members)
        tab = pop.poisson_table()
        s.poisson_cdf[:len(tab)] = tab.tolist()
        self.struct = s
        self.row_cap = spec.row_capacity


_TORCH_DT = {}


def _init_dtypes():
    import torch
    _TORCH_DT.update({np.dtype(np.uint8): torch.uint8, np.dtype(np.int32): torch.int32,
                      np.dtype(np.int8): torch.int8, np.dtype(np.int64): torch.int64})


def initial_columns(pop: ConfigPopulation) -> AgentColumns:
    cols = AgentColumns.allocate(pop.n_agents)
    cols.age_band[:] = pop.age_band
    cols.household_id[:] = pop.household_id
    cols.occupation[:] = (pop.wp_id >= 0).astype(np.int16)
    cols.random_degree[:] = pop.spec.random_mean
    return cols


class ConfigSimulation:
    def __init__(self, pop: ConfigPopulation, disease, table, interventions, seed: int,
                 mode: str = "csr", precision: str = "f32", horizon: int = 180,
                 device=None, initial=None, push_max: int | None = None, persistent: bool = True,
                 iv_fusion: bool = True, day_blocks_per_sm: int = 0, sparse_push: bool = True):
        import torch
        if mode not in ("csr", "fused"):
            raise ConfigError(f"unknown mode {mode!r}")
        if precision not in ("f32", "f64"):
            raise ConfigError(f"unknown precision {precision!r}")
        if mode == "fused" and precision == "f64":
            raise ConfigError("fused mode is fp32-only")
        self._lib = N.lib()
        self.population = pop
        self.disease, self.table, self.iv = disease, table, interventions
        self.seed = int(seed)
        self.mode, self.precision = mode, precision
        self.horizon = horizon
        self.n = pop.n_agents
        self.device = torch.device(device or "cuda")
        self.net = DeviceNetwork(pop, self.device)
        self._params = pack_params(disease, table, interventions, self.n)
        ctx = N._p()
        N.check(self._lib.epi_create(ctypes.byref(self._params), self.n, ctypes.byref(ctx)))
        self._ctx = ctx
        N.check(self._lib.epi_net_attach(self._ctx, ctypes.byref(self.net.struct)))
        self._after_attach()
        if push_max is not None:
            N.check(self._lib.epi_set_push_max(self._ctx, int(push_max)))
        # beyond the push tables: sparse push rows (else 16 inverse slot walks per agent)
        N.check(self._lib.epi_set_sparse_push(self._ctx, int(bool(sparse_push))))
        # run(): merged fused days in one persistent launch (else one kernel per day)
        N.check(self._lib.epi_set_persistent(self._ctx, int(bool(persistent))))
        # fused-mode intervention days in 4 launches (else one kernel per phase)
        N.check(self._lib.epi_set_iv_fusion(self._ctx, int(bool(iv_fusion))))
        # per-day kernel grid cap (0 = default; 1 for replicas on concurrent streams)
        N.check(self._lib.epi_set_day_grid(self._ctx, int(day_blocks_per_sm)))
        self.state = DeviceColumns(self.n, self.device)
        self._codes_buf = self._alloc_codes()
        self.codes = [self._codes_buf[0], self._codes_buf[1]]
        # the random code gathers of every day stay L2-resident
        N.check(self._lib.epi_set_hot_window(self._ctx, N.ptr(self._codes_buf),
                                             self._codes_buf.numel() * 2))
        self.rec = torch.zeros((horizon, N.REC_LEN), dtype=torch.int64, device=self.device)
        self.vax = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.initial = initial if initial is not None else self._seeded_initial()
        self.reset()
        self._graph = None

    def _alloc_codes(self):
        """Both day parities in one buffer (one L2 window covers them)."""
        import torch
        return torch.zeros((2, self.n), dtype=torch.int16, device=self.device)

    def _after_attach(self):
        pass

    @classmethod
    def create(cls, spec: ConfigNetworkSpec, seed: int, disease=None, table=None,
               interventions=None, **kw) -> "ConfigSimulation":
        from .defaults import default_disease, default_progression
        pop = DevicePopulation(spec, seed) if kw.pop("on_device", False) else synthesize(spec, seed)
        return cls(pop, disease or default_disease(), table or default_progression(),
                   interventions or InterventionConfig(), seed, **kw)

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx is not None and ctx.value:
            self._lib.epi_destroy(ctx)
            self._ctx = None

    # -- initial state ------------------------------------------------------
    def _seeded_initial(self) -> DeviceColumns:
        import torch
        pop = self.population
        if isinstance(pop, DevicePopulation):
            # initial_columns on the device
            d = DeviceColumns(self.n, self.device)
            d.t["age_band"].copy_(pop.age_band[:self.n])
            d.t["household_id"].copy_(pop.household_id[:self.n])
            d.t["occupation"].copy_((pop.wp_id[:self.n] >= 0).to(torch.int16))
            d.t["random_degree"].fill_(pop.spec.random_mean)
            ids = pop.seeds.to(self.device)
        else:
            d = DeviceColumns.from_host(initial_columns(pop), self.device)
            ids = torch.from_numpy(pop.seeds.astype(np.int64)).to(self.device)
        st = d.struct()
        s = N.stream_handle()
        N.check(self._lib.epi_seed_infections(self._ctx, ctypes.byref(st), _u64(self.seed),
                                              N.ptr(ids), int(ids.numel()), s))
        if self.iv.den_enabled:
            N.check(self._lib.epi_assign_app(ctypes.byref(st), _u64(self.seed),
                                             float(self.iv.den.app_adoption), s))
        torch.cuda.current_stream().synchronize()
        return d

    def initial_host_columns(self) -> AgentColumns:
        return self.initial.to_host()

    def reset(self) -> None:
        """Back to day 0 (state copy + codes for step 0), all on the device."""
        self.state.copy_from(self.initial)
        self.vax.zero_()
        self.rec.zero_()
        st = self.state.struct()
        N.check(self._lib.epi_codes(self._ctx, ctypes.byref(st), ctypes.byref(self.net.struct),
                                    _u64(self.seed), 0, N.ptr(self.codes[0]), N.stream_handle()))
        self.clock = 0

    # -- stepping -------------------------------------------------------------
    def step(self) -> None:
        t = self.clock
        if t >= self.horizon:
            raise ConfigError(f"horizon {self.horizon} exhausted")
        st = self.state.struct()
        cur, nxt = self.codes[t & 1], self.codes[(t + 1) & 1]
        N.check(self._lib.epi_sim_step(
            self._ctx, ctypes.byref(st), t, _u64(self.seed), 0 if self.mode == "csr" else 1,
            N.F64_CANONICAL if self.precision == "f64" else N.F32, N.ptr(cur), N.ptr(nxt),
            N.ptr(self.rec[t]), N.ptr(self.vax), N.stream_handle()))
        self.clock = t + 1

    def run(self, days: int | None = None) -> None:
        """Advance `days` (default: to the horizon) in one native call."""
        d = self.horizon - self.clock if days is None else days
        if d <= 0:
            return
        if self.clock + d > self.horizon:
            raise ConfigError(f"horizon {self.horizon} exhausted")
        st = self.state.struct()
        t = self.clock
        N.check(self._lib.epi_sim_run(
            self._ctx, ctypes.byref(st), t, d, _u64(self.seed), 0 if self.mode == "csr" else 1,
            N.F64_CANONICAL if self.precision == "f64" else N.F32, N.ptr(self.codes[0]),
            N.ptr(self.codes[1]), N.ptr(self.rec[t]), N.ptr(self.vax), N.stream_handle()))
        self.clock = t + d

    def lambda_probe(self, first_step: int, n_days: int):
        """Export the fp32 hazard the step kernels consume on days
        [first_step, first_step + n_days) into a [n_days, n] device tensor
        (a test hook; n_days = 0 turns it off and returns None)."""
        import torch
        buf = None
        if n_days > 0:
            buf = torch.full((n_days, self.n), float("nan"), dtype=torch.float32, device=self.device)
        self._probe = buf
        N.check(self._lib.epi_set_lambda_probe(self._ctx, N.ptr(buf) if buf is not None else None,
                                               int(first_step), int(n_days)))
        return buf

    def uses_persistent_run(self) -> bool:
        """Whether run() sends its days after the first to k_fused_run."""
        r = self._lib.epi_run_persistent(self._ctx, 0 if self.mode == "csr" else 1,
                                         N.F64_CANONICAL if self.precision == "f64" else N.F32)
        N.check(min(r, 0))
        return r == 1

    def capture(self):
        """Record reset + the whole horizon as one CUDA graph."""
        import torch
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.reset()
            self.run()                      # warm-up outside capture
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            self.reset()
            self.run()
        self._graph = g
        return g

    def replay(self) -> None:
        if self._graph is None:
            self.capture()
        self._graph.replay()
        self.clock = self.horizon


    # -- outputs ----------------------------------------------------------------
    def records(self) -> np.ndarray:
        return self.rec[:self.clock].cpu().numpy()

    def time_series(self) -> np.ndarray:
        """[days, 19] rows in the reference CSV schema (runner.py:31-37)."""
        return self.records()[:, SERIES_COLUMNS]

    def result(self, replication: int = 0):
        """The run so far as the reference's `RunResult` (runner.py:41-74):
        the CSV columns of the device records, the directed edges gathered."""
        from .series import RunResult
        rec = self.records()
        return RunResult(replication=replication, seed=self.seed, data=rec[:, SERIES_COLUMNS].copy(),
                         n_edges_total=int(rec[:, N.REC["edges"]].sum()))

    def host_columns(self) -> AgentColumns:
        return self.state.to_host()

    def codes_for(self, step: int):
        return self.codes[step & 1]

    def realize_graph(self, step: int | None = None) -> StepGraph:
        """Edges of day `step` (default: the current day) as a device StepGraph,
        generated from the current codes (requires step == clock)."""
        import torch
        t = self.clock if step is None else step
        if t != self.clock:
            raise ConfigError("realize_graph only regenerates the current day")
        cap = self.net.row_cap
        entries = torch.empty(self.n * cap, dtype=torch.int32, device=self.device)
        row_len = torch.empty(self.n, dtype=torch.int32, device=self.device)
        N.check(self._lib.epi_net_realize(ctypes.byref(self.net.struct), _u64(self.seed), t,
                                          N.ptr(self.codes[t & 1]), N.ptr(entries),
                                          N.ptr(row_len), 1, N.stream_handle()))
        return csr_to_graph(t, entries, row_len, cap)


def csr_to_graph(step, entries, row_len, cap) -> StepGraph:
    import torch
    n = row_len.numel()
    lens = row_len.long()
    idx = torch.arange(cap, device=entries.device).unsqueeze(0) < lens.unsqueeze(1)
    e = entries.view(n, cap)[idx]
    dst = torch.arange(n, device=entries.device, dtype=torch.int32).unsqueeze(1).expand(n, cap)[idx]
    src = (e >> 2).to(torch.int32) & 0x3FFFFFFF
    kind = (e & 3).to(torch.int8)
    return StepGraph(step, src.contiguous(), dst.contiguous(), kind.contiguous())


def pinned_columns(cols: AgentColumns) -> dict:
    """The columns of a host `AgentColumns` as pinned tensors (the staging
    buffers of `run_from_host`)."""
    import torch
    from .state import COLUMN_SPECS
    out = {}
    for name, dt, _ in COLUMN_SPECS:
        arr = np.ascontiguousarray(getattr(cols, name), dtype=dt)
        out[name] = torch.from_numpy(arr.view(np.uint8) if arr.dtype == np.bool_ else arr).pin_memory()
    return out


class HostPipeline:
    """Whole simulations from host memory to host memory, pipelined: while
    one captured simulation runs on the compute stream, the next one's
    initial state is copied in (pinned host -> HBM, upload stream) and the
    previous one's time series copied out (HBM -> pinned host, download
    stream), so the copies hide under the compute.  Two simulations of the same population
    alternate (`sims`); step k runs sims[k % 2].

        pipe = HostPipeline([sim_a, sim_b])
        for k, cols in enumerate(batches):             # pinned_columns(...)
            pipe.submit(k, cols, out[k])               # out[k]: pinned int64 [horizon, 19]
        pipe.drain()
    """

    def __init__(self, sims):
        import torch
        if len(sims) != 2:
            raise ConfigError("HostPipeline alternates two simulations")
        self.sims = sims
        for s in sims:
            if s._graph is None:
                s.capture()
        self.up = torch.cuda.Stream()
        self.down = torch.cuda.Stream()
        self.main = torch.cuda.current_stream()
        self.done = [torch.cuda.Event(), torch.cuda.Event()]
        self.uploaded = [torch.cuda.Event(), torch.cuda.Event()]
        self.downloaded = [torch.cuda.Event(), torch.cuda.Event()]
        self._used = [False, False]

    def submit(self, k: int, host_cols, out) -> None:
        """host_cols: a pinned arena (`DeviceColumns.host_arena`, one copy)
        or a dict of pinned columns (`pinned_columns`)."""
        import torch
        i = k & 1
        s = self.sims[i]
        with torch.cuda.stream(self.up):
            if self._used[i]:
                self.up.wait_event(self.done[i])     # its previous run no longer reads `initial`
            if isinstance(host_cols, dict):
                for name, t in host_cols.items():
                    s.initial.t[name].copy_(t, non_blocking=True)
            else:
                s.initial.arena.copy_(host_cols, non_blocking=True)
            self.uploaded[i].record(self.up)
        self.main.wait_event(self.uploaded[i])
        if self._used[i]:
            self.main.wait_event(self.downloaded[i])   # its last records are out
        s.replay()
        self.done[i].record(self.main)
        self._used[i] = True
        with torch.cuda.stream(self.down):
            self.down.wait_event(self.done[i])
            out.copy_(s.rec[:, SERIES_COLUMNS], non_blocking=True)
            self.downloaded[i].record(self.down)

    def drain(self) -> None:
        """Make the compute stream wait for the last copies out."""
        self.main.wait_stream(self.down)
