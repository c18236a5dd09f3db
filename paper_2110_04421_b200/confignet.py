"""Synthetic populations and contact networks of BASELINE.json configs 0-4.

The reference has no knob for these networks (its random
network is stub pairing `graphs.py:138-168`, its occupations 23 Watts-Strogatz
graphs `graphs.py:86-129, 210-221`).  This module fixes a B200-first
definition whose in-edges can be enumerated *per destination* with no sort,
no atomics and no cross-GPU exchange, then feeds both the CUDA generator
(`csrc/epi_confignet.cuh`) and its CPU restatement (`oracle/confignet_np.py`).

Static layout (built once on the host, uploaded once):
  * agents are numbered so that every household is a contiguous id range;
    per agent `hh_off` (offset inside its household) and `hh_size` (u8);
  * workers (age bands 2..6, i.e. 20-69) are shuffled by a keyed hash and cut
    into workplaces of size U{wp_min..wp_max}; `wp_members` lists them
    workplace by workplace, per agent `wp_id` (-1 = none) and `wp_local`.

Per step t with graph seed g (the replication seed), dead agents excluded:
  household  : complete graph on the alive members;
  workplace  : sigma_{t,W} = keyed bijection of [0, m); shifts
               r_{t,W,j} in [1, m-1], j < colleague_draws; the worker at
               position p interacts with positions p + r_j and p - r_j (mod m);
  random     : for slot j < random_slots, pi_{t,j} = keyed bijection of
               [0, N); agent a with j < n_{t,a} (n ~ Poisson(random_mean)
               truncated at random_slots) interacts with pi_{t,j}(a) unless it
               is a itself.  The owner of b finds its in-partner via
               pi^{-1}(b) and checks n of that agent.
Every interaction is stored in both directions.

Keyed bijection of [0, n): 3-round Feistel network on the mixed-radix domain
[0, a*b), b = ceil(sqrt(n)), a = ceil(n/b), x = L*b + R,
    L <- (L + F(R, k0)) mod a;  R <- (R + F(L, k1)) mod b;  L <- (L + F(R, k2)) mod a
with F(v, k) = mulhi(g ^ (g >> 15), radix), g = (h ^ (h >> 16)) * 0x7FEB352D,
h = (v ^ k.x) * k.y (all mod 2^32),
cycle-walked back into
[0, n) (a*b - n < b, so a walk is needed with probability < 1/sqrt(n)).
Round keys: random slot j, round r: hash64(g, t, NET_RANDOM_PERM, j, r)
(low 32 bits = k.x, high 32 bits | 1 = k.y); workplace W: 16-bit fields of
hash64(g, t, NET_WORK_PERM, W, 0..1).  Shift r_j: 16-bit chunk (j & 3) of
hash64(g, t, NET_WORK_SHIFT, W, j >> 2), scaled as 1 + (v * (m-1)) >> 16.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import keyed
from .errors import ConfigError
from .keyed import Purpose
from .stages import N_AGE_BANDS

UNIFORM_AGES = tuple([1.0 / N_AGE_BANDS] * N_AGE_BANDS)
CONFIG_HOUSEHOLD_PROBS = (0.28, 0.35, 0.15, 0.13, 0.06, 0.03)


@dataclass(frozen=True)
class ConfigNetworkSpec:
    """Population + network knobs; defaults are BASELINE.json config 1."""

    n_agents: int = 100_000
    age_probs: tuple = UNIFORM_AGES
    household_sizes: tuple = (1, 2, 3, 4, 5, 6)
    household_probs: tuple = CONFIG_HOUSEHOLD_PROBS
    worker_bands: tuple = (2, 3, 4, 5, 6)
    wp_min: int = 10
    wp_max: int = 50
    colleague_draws: int = 8
    random_mean: float = 5.0
    random_slots: int = 16
    initial_infections: int = 100

    def __post_init__(self):
        if self.n_agents < 1 or self.n_agents >= (1 << 30):
            raise ConfigError("n_agents must be in [1, 2^30)")
        if abs(sum(self.age_probs) - 1.0) > 1e-9 or len(self.age_probs) != N_AGE_BANDS:
            raise ConfigError("age_probs must be 9 probabilities summing to 1")
        if abs(sum(self.household_probs) - 1.0) > 1e-9:
            raise ConfigError("household_probs must sum to 1")
        if min(self.household_sizes) < 1 or max(self.household_sizes) > 32:
            raise ConfigError("household sizes must be in [1, 32]")
        if not 2 <= self.wp_min <= self.wp_max <= 255:
            raise ConfigError("workplace sizes must satisfy 2 <= min <= max <= 255")
        if not 0 <= self.colleague_draws <= 32 or not 0 <= self.random_slots <= 32:
            raise ConfigError("colleague_draws / random_slots must be in [0, 32]")
        if self.random_mean < 0:
            raise ConfigError("random_mean must be >= 0")
        if not 0 <= self.initial_infections <= self.n_agents:
            raise ConfigError("initial_infections outside [0, n_agents]")

    @property
    def row_capacity(self) -> int:
        """Upper bound on in-edges of one agent (padded CSR row length)."""
        cap = (max(self.household_sizes) - 1) + 2 * self.colleague_draws \
            + 2 * self.random_slots
        return (cap + 7) // 8 * 8

    @classmethod
    def config(cls, index: int, **overrides) -> "ConfigNetworkSpec":
        """BASELINE.json configs: 0 (10k, no workplaces), 1/2 (100k), 3 (10M)."""
        base = {0: dict(n_agents=10_000, worker_bands=(), initial_infections=10),
                1: dict(n_agents=100_000), 2: dict(n_agents=100_000),
                3: dict(n_agents=10_000_000, initial_infections=1000),
                4: dict(n_agents=100_000)}[index]
        base.update(overrides)
        return cls(**base)


def poisson_cdf_table(mean: float, slots: int) -> np.ndarray:
    """F[k] = P(Poisson(mean) <= k), k < slots, summed in a fixed order so the
    device and the oracle compare draws against identical doubles."""
    out = np.zeros(max(slots, 1), dtype=np.float64)
    term = math.exp(-mean)
    acc = 0.0
    for k in range(slots):
        acc += term
        out[k] = acc
        term = term * mean / (k + 1)
    return out[:slots]


def _keyed_u(seed, purpose, idx, k=0):
    """Host-side keyed 64-bit hashes for one-time population setup (numpy)."""
    h0 = np.uint64(keyed.key_prefix(seed, 0, purpose))
    g = np.uint64(keyed.GOLDEN)
    c1, c2 = np.uint64(keyed.MIX1), np.uint64(keyed.MIX2)

    def mix(z):
        z = (z ^ (z >> np.uint64(30))) * c1
        z = (z ^ (z >> np.uint64(27))) * c2
        return z ^ (z >> np.uint64(31))
    with np.errstate(over="ignore"):
        a = np.asarray(idx, dtype=np.uint64)
        h = mix(h0 ^ (g * (a + np.uint64(1))))
        h = mix(h ^ (g * np.uint64(k + 1)))
    return h


@dataclass
class ConfigPopulation:
    spec: ConfigNetworkSpec
    seed: int
    age_band: np.ndarray      # int8[N]
    household_id: np.ndarray  # int32[N]
    hh_off: np.ndarray        # uint8[N]
    hh_size: np.ndarray       # uint8[N]
    wp_id: np.ndarray         # int32[N], -1 = not employed
    wp_local: np.ndarray      # uint8[N]
    wp_base: np.ndarray       # int32[W]
    wp_size: np.ndarray       # int32[W]
    wp_members: np.ndarray    # int32[sum wp_size]
    seeds: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))

    @property
    def n_agents(self) -> int:
        return self.spec.n_agents

    @property
    def n_workplaces(self) -> int:
        return len(self.wp_base)

    def poisson_table(self) -> np.ndarray:
        return poisson_cdf_table(self.spec.random_mean, self.spec.random_slots)


def synthesize(spec: ConfigNetworkSpec, seed: int) -> ConfigPopulation:
    """Static population for `seed` (host numpy; one-time setup, not per step)."""
    n = spec.n_agents
    ids = np.arange(n, dtype=np.int64)
    to_u = 1.0 / (1 << 53)
    # ages: inverse CDF of a keyed uniform
    u_age = (_keyed_u(seed, Purpose.POP_AGE, ids) >> np.uint64(11)).astype(np.float64) * to_u
    age = np.searchsorted(np.cumsum(spec.age_probs), u_age, side="right")
    age = np.minimum(age, N_AGE_BANDS - 1).astype(np.int8)
    # households: sequential size draws, contiguous id ranges, last one truncated
    sizes_all = np.asarray(spec.household_sizes, dtype=np.int64)
    cum_hh = np.cumsum(spec.household_probs)
    sizes = []
    covered = 0
    chunk = 0
    while covered < n:
        k = np.arange(chunk, chunk + max(1024, n // 2), dtype=np.int64)
        u = (_keyed_u(seed, Purpose.POP_HOUSEHOLD, k) >> np.uint64(11)).astype(np.float64) * to_u
        s = sizes_all[np.minimum(np.searchsorted(cum_hh, u, side="right"), len(sizes_all) - 1)]
        sizes.append(s)
        covered += int(s.sum())
        chunk += len(k)
    sizes = np.concatenate(sizes)
    ends = np.cumsum(sizes)
    n_hh = int(np.searchsorted(ends, n, side="left")) + 1
    sizes = sizes[:n_hh].copy()
    sizes[-1] -= int(ends[n_hh - 1]) - n
    starts = np.concatenate(([0], np.cumsum(sizes)[:-1]))
    household_id = np.repeat(np.arange(n_hh, dtype=np.int32), sizes)
    hh_off = (ids - starts[household_id]).astype(np.uint8)
    hh_size = sizes[household_id].astype(np.uint8)
    # workplaces: keyed shuffle of workers, cut into U{min..max} sized blocks
    workers = ids[np.isin(age, np.asarray(spec.worker_bands, dtype=np.int8))]
    wp_id = np.full(n, -1, dtype=np.int32)
    wp_local = np.zeros(n, dtype=np.uint8)
    if len(workers) and spec.colleague_draws > 0:
        keys = _keyed_u(seed, Purpose.POP_WORKPLACE, workers)
        members = workers[np.lexsort((workers, keys))].astype(np.int32)
        span = spec.wp_max - spec.wp_min + 1
        max_w = len(members) // spec.wp_min + 2
        uw = (_keyed_u(seed, Purpose.POP_WORKPLACE, np.arange(max_w), k=1)
              >> np.uint64(11)).astype(np.float64) * to_u
        wsz = spec.wp_min + (uw * span).astype(np.int64)
        wend = np.cumsum(wsz)
        n_w = int(np.searchsorted(wend, len(members), side="left")) + 1
        wsz = wsz[:n_w].copy()
        wsz[-1] -= int(wend[n_w - 1]) - len(members)
        wbase = np.concatenate(([0], np.cumsum(wsz)[:-1])).astype(np.int32)
        owner = np.repeat(np.arange(n_w, dtype=np.int32), wsz)
        wp_id[members] = owner
        wp_local[members] = (np.arange(len(members)) - wbase[owner]).astype(np.uint8)
        wp_size = wsz.astype(np.int32)
    else:
        members = np.empty(0, np.int32)
        wbase = np.empty(0, np.int32)
        wp_size = np.empty(0, np.int32)
    # initial infections: the `initial_infections` agents with the smallest keyed hash
    seeds = np.empty(0, np.int64)
    if spec.initial_infections:
        h = _keyed_u(seed, Purpose.POP_SEEDS, ids)
        seeds = np.sort(np.lexsort((ids, h))[:spec.initial_infections]).astype(np.int64)
    return ConfigPopulation(spec, seed, age, household_id, hh_off, hh_size, wp_id,
                            wp_local, wbase, wp_size, members, seeds)


class DevicePopulation:
    """The same population as `synthesize`, built on the device
    (csrc/epi_population.cuh, row f3): every array is a torch tensor with the
    ConfigPopulation name and dtype.  `to_host()` gives the ConfigPopulation."""

    def __init__(self, spec: ConfigNetworkSpec, seed: int, device=None):
        import ctypes

        import torch

        from . import _native as N
        self.spec, self.seed = spec, int(seed)
        dev = torch.device(device or "cuda")
        n = spec.n_agents
        workers = bool(spec.worker_bands) and spec.colleague_draws > 0
        max_w = n // spec.wp_min + 2

        def e(k, dt):
            return torch.empty(max(k, 1), dtype=dt, device=dev)
        self.age_band, self.household_id = e(n, torch.int8), e(n, torch.int32)
        self.hh_off, self.hh_size = e(n, torch.uint8), e(n, torch.uint8)
        self.wp_id, self.wp_local = e(n, torch.int32), e(n, torch.uint8)
        members, base, size = e(n, torch.int32), e(max_w, torch.int32), e(max_w, torch.int32)
        self.seeds = e(spec.initial_infections, torch.int64)
        counts = torch.zeros(2, dtype=torch.int64, device=dev)
        sp = N.EpiPopSpec()
        sp.n_agents = n
        sp.age_cum[:] = np.cumsum(spec.age_probs).tolist()
        sp.n_sizes = len(spec.household_sizes)
        sp.hh_sizes[:sp.n_sizes] = [int(x) for x in spec.household_sizes]
        sp.hh_cum[:sp.n_sizes] = np.cumsum(spec.household_probs).tolist()
        sp.worker_mask = sum(1 << int(b) for b in spec.worker_bands) if workers else 0
        sp.wp_min, sp.wp_max = spec.wp_min, spec.wp_max
        sp.n_seeds = spec.initial_infections
        out = N.EpiPopOut()
        for f, t in (("age_band", self.age_band), ("household_id", self.household_id),
                     ("hh_off", self.hh_off), ("hh_size", self.hh_size), ("wp_id", self.wp_id),
                     ("wp_local", self.wp_local), ("wp_members", members), ("wp_base", base),
                     ("wp_size", size), ("seeds", self.seeds), ("counts", counts)):
            setattr(out, f, N.ptr(t))
        N.check(N.lib().epi_pop_synthesize(ctypes.byref(sp), self.seed & ((1 << 64) - 1),
                                           ctypes.byref(out), N.stream_handle()))
        n_w, n_m = (int(x) for x in counts.cpu())
        self.wp_members, self.wp_base, self.wp_size = members[:n_m], base[:n_w], size[:n_w]
        self.seeds = self.seeds[:spec.initial_infections]

    @property
    def n_agents(self) -> int:
        return self.spec.n_agents

    @property
    def n_workplaces(self) -> int:
        return int(self.wp_base.numel())

    def poisson_table(self) -> np.ndarray:
        return poisson_cdf_table(self.spec.random_mean, self.spec.random_slots)

    def to_host(self) -> ConfigPopulation:
        def h(t):
            return t.cpu().numpy()
        return ConfigPopulation(self.spec, self.seed, h(self.age_band), h(self.household_id),
                                h(self.hh_off), h(self.hh_size), h(self.wp_id), h(self.wp_local),
                                h(self.wp_base), h(self.wp_size), h(self.wp_members), h(self.seeds))
