"""Host -> device plumbing: parameter flattening and device-resident columns.

`pack_params` flattens DiseaseParams / ProgressionTable / InterventionConfig
(this package's or the reference's own classes: only attribute names are
used) into the POD `epi_params` of the C ABI.  `DeviceColumns` holds one CUDA
buffer per AgentColumns column with the same dtype (state.py:21-75), views
into one arena, so host <-> device transfers are flat copies and a whole
state copies in one.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .errors import ConfigError
from .progression import device_tables
from .state import COLUMN_SPECS, AgentColumns

_TORCH_DTYPES = None


def _torch_dtype(np_dtype):
    global _TORCH_DTYPES
    import torch
    if _TORCH_DTYPES is None:
        _TORCH_DTYPES = {np.dtype(np.int8): torch.int8, np.dtype(np.int16): torch.int16,
                         np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64,
                         np.dtype(np.float64): torch.float64, np.dtype(np.bool_): torch.uint8,
                         np.dtype(np.uint8): torch.uint8, np.dtype(np.uint16): torch.int16}
    return _TORCH_DTYPES[np.dtype(np_dtype)]


def pack_params(disease, table, interventions, n_agents: int) -> N.EpiParams:
    p = N.EpiParams()
    p.rate_scale = float(disease.rate_scale)
    p.asymptomatic_factor = float(disease.asymptomatic_factor)
    p.mean_daily_interactions = float(disease.mean_daily_interactions)
    p.age_susceptibility[:] = [float(x) for x in disease.age_susceptibility]
    p.network_scale[:] = [float(x) for x in disease.network_scale]
    w = np.asarray(disease.day_weights, dtype=np.float64)
    if len(w) - 1 > N.MAX_T:
        raise ConfigError(f"t_max={len(w) - 1} exceeds the device limit {N.MAX_T}")
    p.t_max = len(w) - 1
    p.day_weights[:len(w)] = w.tolist()
    iv = interventions
    p.sterilizing = int(int(iv.vaccine.immunity_mode) == 0)
    dev = table.device_tables() if hasattr(table, "device_tables") else device_tables(table)
    if len(dev["taus"]) > N.MAX_SPECS:
        raise ConfigError(f"progression table has {len(dev['taus'])} duration "
                          f"distributions; the device holds {N.MAX_SPECS}")
    for s in range(11):
        p.n_targets[s] = int(dev["n_targets"][s])
        for j in range(3):
            p.targets[s][j] = int(dev["targets"][s, j])
            p.spec_of[s][j] = int(dev["spec_of"][s, j])
            for a in range(9):
                p.cum[s][a][j] = float(dev["cum"][s, a, j])
    p.n_specs = len(dev["taus"])
    for i, tau in enumerate(dev["taus"]):
        p.tau_len[i] = len(tau)
        if len(tau):
            C.memmove(C.addressof(p.tau[i]), np.ascontiguousarray(tau, np.float64).ctypes.data,
                      8 * len(tau))
    p.quarantine_enabled = int(bool(iv.quarantine_enabled))
    p.quarantine_duration = int(iv.quarantine_duration)
    p.quarantine_dropout = float(iv.quarantine_dropout)
    p.testing_enabled = int(bool(iv.testing_enabled))
    p.turnaround_min = int(iv.test_kind.turnaround_min)
    p.turnaround_max = int(iv.test_kind.turnaround_max)
    p.detection_prob = float(iv.test_kind.detection_prob)
    p.false_positive_prob = float(iv.false_positive_prob)
    p.den_enabled = int(bool(iv.den_enabled))
    p.den_compliance = float(iv.den.compliance_prob)
    p.den_lookback = int(iv.den.lookback)
    v = iv.vaccine
    p.vaccination_enabled = int(bool(iv.vaccination_enabled))
    p.strategy = int(v.strategy)
    p.elderly_band = int(v.elderly_band)
    p.dose1_efficacy = float(v.dose1_efficacy)
    p.dose2_efficacy = float(v.dose2_efficacy)
    p.dose2_topup = float(v.dose2_topup_prob())
    p.dose1_latency = int(v.dose1_latency)
    p.dose2_latency = int(v.dose2_latency)
    p.dose_gap = int(v.dose_gap)
    p.dose_budget = int(np.rint(v.daily_rate * n_agents))            # interventions.py:107-108
    p.start_trigger_count = float(v.start_trigger) * n_agents         # engine.py:289
    return p


class DeviceColumns:
    """One CUDA tensor per AgentColumns column (identical dtypes), all views
    into one device arena (256-byte aligned columns), so copying a whole
    state -- reset() to the initial state, once per simulation and inside
    every captured run -- is one copy, not 22."""

    ALIGN = 256

    def __init__(self, n_agents: int, device=None):
        import torch
        self.n_agents = n_agents
        self.device = torch.device(device or "cuda")
        offs, at = [], 0
        for name, dt, _ in COLUMN_SPECS:
            offs.append(at)
            at += -(-(n_agents * np.dtype(dt).itemsize) // self.ALIGN) * self.ALIGN
        self.arena = torch.empty(max(at, self.ALIGN), dtype=torch.uint8, device=self.device)
        self.t = {}
        for (name, dt, fill), off in zip(COLUMN_SPECS, offs):
            nb = n_agents * np.dtype(dt).itemsize
            v = self.arena[off:off + nb].view(_torch_dtype(dt))
            v.fill_(fill)
            self.t[name] = v

    @classmethod
    def from_host(cls, cols, device=None) -> "DeviceColumns":
        d = cls(cols.n_agents, device)
        d.upload(cols)
        return d

    def upload(self, cols, names=None, non_blocking=False) -> None:
        import torch
        for name, dt, _ in COLUMN_SPECS:
            if names is not None and name not in names:
                continue
            host = np.ascontiguousarray(getattr(cols, name), dtype=dt)
            src = torch.from_numpy(host.view(np.uint8) if host.dtype == np.bool_ else host)
            self.t[name].copy_(src, non_blocking=non_blocking)

    def download(self, cols, names=None) -> None:
        for name, dt, _ in COLUMN_SPECS:
            if names is not None and name not in names:
                continue
            arr = self.t[name].cpu().numpy()
            getattr(cols, name)[:] = arr.view(np.bool_) if np.dtype(dt) == np.bool_ else arr

    def to_host(self) -> AgentColumns:
        cols = AgentColumns.allocate(self.n_agents)
        self.download(cols)
        return cols

    def host_arena(self, cols, pin: bool = True):
        """A host `AgentColumns` packed in this arena's layout (a pinned uint8
        tensor): uploading it is one copy (`arena.copy_(host, non_blocking)`)."""
        import torch
        buf = torch.zeros(self.arena.numel(), dtype=torch.uint8)
        base = self.arena.data_ptr()
        for name, dt, _ in COLUMN_SPECS:
            off = self.t[name].data_ptr() - base
            arr = np.ascontiguousarray(getattr(cols, name), dtype=dt)
            raw = arr.view(np.uint8).reshape(-1)
            buf[off:off + raw.size] = torch.from_numpy(raw.copy())
        return buf.pin_memory() if pin else buf

    def clone(self) -> "DeviceColumns":
        d = DeviceColumns(self.n_agents, self.device)
        d.arena.copy_(self.arena)
        return d

    def copy_from(self, other: "DeviceColumns") -> None:
        if other.n_agents != self.n_agents:
            raise ConfigError("state sizes differ")
        self.arena.copy_(other.arena)          # one copy for the 22 columns

    def struct(self) -> N.EpiState:
        s = N.EpiState()
        s.n_agents = self.n_agents
        for f in N.STATE_FIELDS:
            setattr(s, f, N.ptr(self.t[f]))
        return s

    def nbytes(self) -> int:
        return sum(int(v.numel() * v.element_size()) for v in self.t.values())
