"""Agent-range partitioning of a config simulation across GPUs (§8(e)).

Rank r owns the contiguous agent rows [r*chunk, min(N, (r+1)*chunk)).  Every
in-edge of an owned destination is enumerable from the global 16-bit code
vector alone (confignet.py: keyed bijections, no cross-rank edge exchange), so
the only per-day exchange is one all-gather of the codes each rank just wrote
for its rows (2 bytes/agent, N*2/P bytes sent per rank).  Day records are
partial sums per rank, reduced once at the end.

The exchange is pluggable:
  NcclCodeExchange   torch.distributed all_gather_into_tensor (NCCL over
                     NVLink/NVSwitch on one 8xB200 node; gloo on CPU tests);
  LocalCodeExchange  P emulated ranks in one process on one GPU (device
                     copies), used to prove partition invariance bitwise.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _native as N
from .errors import ConfigError
from .sim import ConfigSimulation


@dataclass(frozen=True)
class PartitionPlan:
    n_agents: int
    world: int

    def __post_init__(self):
        if self.world < 1 or self.n_agents < self.world:
            raise ConfigError(f"cannot split {self.n_agents} agents over {self.world} ranks")
        if (self.world - 1) * self.chunk >= self.n_agents:
            raise ConfigError(f"{self.n_agents} agents are too few for {self.world} ranks "
                              "of 32-row tiles")

    @property
    def chunk(self) -> int:
        # multiple of 32 rows: warp tiles line up with the unpartitioned run,
        # so tile-local summation orders (and fp32 results) are identical
        return -(-self.n_agents // (32 * self.world)) * 32

    @property
    def padded(self) -> int:
        return self.chunk * self.world

    def rows(self, rank: int) -> tuple[int, int]:
        lo = rank * self.chunk
        return lo, min(self.n_agents, lo + self.chunk)


class NcclCodeExchange:
    """All-gather of each rank's code chunk through a torch.distributed group."""

    def __init__(self, plan: PartitionPlan, rank: int, group=None):
        self.plan, self.rank, self.group = plan, rank, group

    def exchange(self, codes):
        import torch
        import torch.distributed as dist
        c = self.plan.chunk
        mine = codes[self.rank * c:(self.rank + 1) * c]
        if hasattr(dist, "all_gather_into_tensor") and codes.is_cuda:
            dist.all_gather_into_tensor(codes, mine.clone(), group=self.group)
        else:   # gloo (CPU tests): no int16 support, widen to int32
            parts = [torch.empty(c, dtype=torch.int32) for _ in range(self.plan.world)]
            dist.all_gather(parts, mine.to(torch.int32), group=self.group)
            for r, p in enumerate(parts):
                codes[r * c:(r + 1) * c].copy_(p.to(codes.dtype))

    def reduce_records(self, rec):
        """Sum the per-rank partial day records (step column kept)."""
        import torch.distributed as dist
        step = rec[:, N.REC["step"]].clone()
        flags = rec[:, N.REC["flags"]].clone()
        dist.all_reduce(rec, group=self.group)
        rec[:, N.REC["step"]] = step
        dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=self.group)
        rec[:, N.REC["flags"]] = flags
        return rec


class LocalCodeExchange:
    """P emulated ranks in one process: chunks are copied device to device."""

    def __init__(self, plan: PartitionPlan):
        self.plan = plan
        self.buffers = {}

    def register(self, rank, sims):
        self.sims = sims

    def exchange_all(self, day_parity: int):
        c = self.plan.chunk
        bufs = [s.codes[day_parity] for s in self.sims]
        for r, src in enumerate(bufs):
            piece = src[r * c:(r + 1) * c]
            for q, dst in enumerate(bufs):
                if q != r:
                    dst[r * c:(r + 1) * c].copy_(piece)

    @staticmethod
    def reduce_records(sims):
        out = sims[0].rec.clone()
        for s in sims[1:]:
            out += s.rec
        out[:, N.REC["step"]] = sims[0].rec[:, N.REC["step"]]
        return out


class PartitionedSimulation(ConfigSimulation):
    """One rank of an agent-range partitioned config simulation."""

    def __init__(self, pop, disease, table, interventions, seed, plan: PartitionPlan, rank: int,
                 exchange=None, **kw):
        if interventions.den_enabled or interventions.vaccination_enabled:
            raise ConfigError("partitioned runs support quarantine/testing only "
                              "(DEN and vaccination need global state; SURVEY §8(f) f2)")
        self.plan, self.rank, self.exchange = plan, rank, exchange
        self._code_len = plan.padded
        super().__init__(pop, disease, table, interventions, seed, **kw)

    def _alloc_codes(self):
        import torch
        return torch.zeros((2, self._code_len), dtype=torch.int16, device=self.device)

    def _after_attach(self):
        lo, hi = self.plan.rows(self.rank)
        N.check(self._lib.epi_set_rows(self._ctx, lo, hi))

    def reset(self) -> None:
        super().reset()
        if isinstance(self.exchange, NcclCodeExchange):
            self.exchange.exchange(self.codes[0])

    def step(self) -> None:
        t = self.clock
        super().step()
        if isinstance(self.exchange, NcclCodeExchange):
            self.exchange.exchange(self.codes[(t + 1) & 1])

    def run(self, days: int | None = None) -> None:
        # one day at a time: the code exchange sits between days
        for _ in range(self.horizon - self.clock if days is None else days):
            self.step()


def run_emulated(pop, disease, table, interventions, seed, world: int, days: int, **kw):
    """P ranks on one GPU, days in lockstep; returns (sims, summed records)."""
    plan = PartitionPlan(pop.n_agents, world)
    ex = LocalCodeExchange(plan)
    sims = [PartitionedSimulation(pop, disease, table, interventions, seed, plan, r, ex,
                                  horizon=days, **kw) for r in range(world)]
    ex.register(None, sims)
    ex.exchange_all(0)
    for t in range(days):
        for s in sims:
            s.step()
        ex.exchange_all((t + 1) & 1)
    return sims, LocalCodeExchange.reduce_records(sims)
