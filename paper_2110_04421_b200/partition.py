"""Agent-range partitioning of a config simulation across GPUs (§8(e)).

Rank r owns the contiguous agent rows [r*chunk, min(N, (r+1)*chunk)).  Every
in-edge of an owned destination is enumerable from the global 16-bit code
vector alone (confignet.py: keyed bijections, no cross-rank edge exchange), so
the only per-day exchange is one all-gather of the codes each rank just wrote
for its rows (2 bytes/agent, N*2/P bytes sent per rank).  Day records are
partial sums per rank, reduced once at the end.

With exposure notification or vaccination a day
also needs three in-step exchanges, which the native step requests through
a callback (epi_set_exchange):
  * the DEN notifications: each rank regenerates the contacts of its own
    notifiers over the lookback days and marks them, whoever owns them; the
    marks are OR-reduced over the ranks (one byte per agent);
  * the vaccination eligibility histogram and active count (all-reduce of
    55 integers), so every rank computes the same cut bucket and budget;
  * the cut-bucket count of the lower-ranked (lower-id) ranges (exclusive
    scan of one integer), so the cut bucket is served in global id order.

The exchange is pluggable:
  NcclCodeExchange   torch.distributed (NCCL over NVLink/NVSwitch on one
                     8xB200 node; gloo on CPU tests);
  LocalCodeExchange  P emulated ranks in one process on one GPU (device
                     copies, days in lockstep), to prove partition invariance;
  ThreadExchange     P emulated ranks in P host threads on one GPU (streams
                     of their own, host barriers between the phases; no
                     kernel ever waits on another rank's kernel), for the
                     in-step exchanges of DEN and vaccination.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _native as N
from .errors import ConfigError
from .sim import ConfigSimulation

_X_GATHER_U8, _X_SUM_U64, _X_EXSCAN_I64, _X_OR_U8 = 1, 2, 3, 4


class _DevArray:
    """Zero-copy view of a raw device pointer (__cuda_array_interface__)."""

    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


def _view(ptr, count, typestr):
    import torch
    return torch.as_tensor(_DevArray(ptr, count, typestr), device="cuda")


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


def _or_fold(parts):
    """Bitwise OR of equally shaped integer tensors (the EPI_REC_FLAGS bits)."""
    import torch
    out = parts[0].clone()
    for p in parts[1:]:
        out = torch.bitwise_or(out, p)
    return out


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

    # -- in-step exchanges (DEN, vaccination) --------------------------------
    def gather_rows(self, t):
        """Every rank's owned rows of the global-indexed tensor `t`, everywhere."""
        import torch
        import torch.distributed as dist
        c = self.plan.chunk
        lo, hi = self.plan.rows(self.rank)
        mine = torch.zeros(c, dtype=t.dtype, device=t.device)
        mine[:hi - lo] = t[lo:hi]
        if t.is_cuda:
            full = torch.empty(self.plan.padded, dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(full, mine, group=self.group)
        else:   # gloo: widen
            parts = [torch.empty(c, dtype=torch.int32) for _ in range(self.plan.world)]
            dist.all_gather(parts, mine.to(torch.int32), group=self.group)
            full = torch.cat(parts).to(t.dtype)
        n = self.plan.n_agents
        t[:n].copy_(full[:n])

    def sum_(self, t):
        import torch.distributed as dist
        dist.all_reduce(t, group=self.group)

    def or_(self, t):
        """OR over the ranks of a byte array whose bytes are 0 or one common
        flag bit (the DEN marks): equal to the MAX, in place."""
        import torch
        import torch.distributed as dist
        if t.is_cuda:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        else:   # gloo: widen
            w = t.to(torch.int32)
            dist.all_reduce(w, op=dist.ReduceOp.MAX, group=self.group)
            t.copy_(w.to(t.dtype))

    def exscan_(self, t):
        """Exclusive prefix sum over the ranks (rank order), in place."""
        import torch
        import torch.distributed as dist
        parts = [torch.empty_like(t) for _ in range(self.plan.world)]
        dist.all_gather(parts, t.clone(), group=self.group)
        acc = torch.zeros_like(t)
        for r in range(self.rank):
            acc += parts[r]
        t.copy_(acc)

    def reduce_records(self, rec):
        """Sum the per-rank partial day records (step column kept; the flag
        column is a bitmask, OR-ed: NCCL has no bitwise-or reduction, so the
        flags are all-gathered and folded)."""
        import torch
        import torch.distributed as dist
        step = rec[:, N.REC["step"]].clone()
        flags = rec[:, N.REC["flags"]].clone()
        dist.all_reduce(rec, group=self.group)
        rec[:, N.REC["step"]] = step
        parts = [torch.empty_like(flags) for _ in range(self.plan.world)]
        dist.all_gather(parts, flags, group=self.group)
        rec[:, N.REC["flags"]] = _or_fold(parts)
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
        out[:, N.REC["flags"]] = _or_fold([s.rec[:, N.REC["flags"]] for s in sims])
        return out


class ThreadExchange:
    """P emulated ranks, one host thread and CUDA stream each, on one GPU.

    Every exchange: the rank synchronises its stream, publishes its buffer,
    waits at a host barrier, combines the published buffers into its own
    (device copies on its stream), synchronises again and waits at a second
    barrier, so no rank overwrites a buffer another rank is still reading."""

    def __init__(self, plan: PartitionPlan):
        import threading
        self.plan = plan
        self.barrier = threading.Barrier(plan.world)
        self.posted = [None] * plan.world

    def _post(self, rank, t):
        import torch
        torch.cuda.current_stream().synchronize()
        self.posted[rank] = t
        self.barrier.wait()

    def _done(self):
        import torch
        torch.cuda.current_stream().synchronize()
        self.barrier.wait()

    def for_rank(self, rank):
        ex = self

        class _Rank:
            def gather_rows(self, t):
                ex._post(rank, t)
                for q, other in enumerate(ex.posted):
                    if q != rank:
                        lo, hi = ex.plan.rows(q)
                        t[lo:hi].copy_(other[lo:hi])
                ex._done()

            def sum_(self, t):
                ex._post(rank, t.clone())
                acc = ex.posted[0].clone()
                for other in ex.posted[1:]:
                    acc += other
                t.copy_(acc)
                ex._done()

            def or_(self, t):
                ex._post(rank, t.clone())
                acc = ex.posted[0].clone()
                for other in ex.posted[1:]:
                    acc |= other
                t.copy_(acc)
                ex._done()

            def exscan_(self, t):
                ex._post(rank, t.clone())
                acc = torch_zeros_like(t)
                for q in range(rank):
                    acc += ex.posted[q]
                t.copy_(acc)
                ex._done()

            def exchange(self, codes):
                self.gather_rows(codes)
        return _Rank()


def torch_zeros_like(t):
    import torch
    return torch.zeros_like(t)


class PartitionedSimulation(ConfigSimulation):
    """One rank of an agent-range partitioned config simulation."""

    def __init__(self, pop, disease, table, interventions, seed, plan: PartitionPlan, rank: int,
                 exchange=None, **kw):
        needs_x = interventions.den_enabled or interventions.vaccination_enabled
        if needs_x and not hasattr(exchange, "sum_"):
            raise ConfigError("exposure notification and vaccination in a partitioned run need "
                              "an in-step exchange (NcclCodeExchange or ThreadExchange)")
        self.plan, self.rank, self.exchange = plan, rank, exchange
        self._code_len = plan.padded
        self._ready = False          # no exchange from inside the constructor's reset()
        super().__init__(pop, disease, table, interventions, seed, **kw)
        self._ready = True
        if needs_x:
            self._hook = N.XFN(self._on_exchange)      # kept alive with the simulation
            N.check(self._lib.epi_set_exchange(self._ctx, self._hook, None))

    def _on_exchange(self, _user, kind, buf, count, _stream):
        """Called by the native step (same thread, current stream)."""
        try:
            if kind == _X_GATHER_U8:
                self.exchange.gather_rows(_view(buf, count, "|u1"))
            elif kind == _X_SUM_U64:
                self.exchange.sum_(_view(buf, count, "<i8"))    # non-negative counts
            elif kind == _X_EXSCAN_I64:
                self.exchange.exscan_(_view(buf, count, "<i8"))
            elif kind == _X_OR_U8:
                self.exchange.or_(_view(buf, count, "|u1"))
            else:
                return 1
            return 0
        except Exception:  # noqa: BLE001 - reported through the C return code
            import traceback
            traceback.print_exc()
            return 1

    def _alloc_codes(self):
        import torch
        return torch.zeros((2, self._code_len), dtype=torch.int16, device=self.device)

    def _after_attach(self):
        lo, hi = self.plan.rows(self.rank)
        N.check(self._lib.epi_set_rows(self._ctx, lo, hi))

    def reset(self) -> None:
        super().reset()
        if self._ready and self.exchange is not None and not isinstance(self.exchange, LocalCodeExchange):
            self.exchange.exchange(self.codes[0])

    def step(self) -> None:
        t = self.clock
        super().step()
        if self.exchange is not None and not isinstance(self.exchange, LocalCodeExchange):
            self.exchange.exchange(self.codes[(t + 1) & 1])

    def capture(self):
        raise ConfigError("a partitioned simulation exchanges with its peers between and "
                          "inside days; run it day by day (run()) instead of as a CUDA graph")

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


def run_threaded(pop, disease, table, interventions, seed, world: int, days: int, **kw):
    """P ranks on one GPU in P host threads (own streams), with the in-step
    exchanges of DEN and vaccination; returns (sims, summed records)."""
    import threading

    import torch
    plan = PartitionPlan(pop.n_agents, world)
    ex = ThreadExchange(plan)
    sims = [None] * world
    errors = []
    build = threading.Lock()

    def rank_main(r):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                with build:          # contexts and tables are built one at a time
                    sims[r] = PartitionedSimulation(pop, disease, table, interventions, seed, plan, r,
                                                    ex.for_rank(r), horizon=days, **kw)
                ex.barrier.wait()
                sims[r].reset()      # exchanges the day-0 codes
                for _ in range(days):
                    sims[r].step()
                stream.synchronize()
        except BaseException as e:  # noqa: BLE001
            errors.append(e)
            ex.barrier.abort()
    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return sims, LocalCodeExchange.reduce_records(sims)
