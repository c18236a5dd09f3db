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

_X_GATHER_U8, _X_SUM_U64, _X_EXSCAN_I64, _X_OR_U8, _X_GATHER_U16 = 1, 2, 3, 4, 5


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


class NcclComm:
    """A native NCCL communicator (libepib200 `epi_comm`): the per-day code
    all-gather runs inside the native day loop (epi_set_code_exchange mode
    2), in place, on the simulation's stream -- no Python per day, no copy
    of the send chunk, and the partitioned run can be captured in a CUDA
    graph.  Rank 0 draws the NCCL unique id; `from_process_group` ships it
    over torch.distributed."""

    def __init__(self, world: int, rank: int, unique_id: bytes):
        import ctypes
        self._lib = N.lib()
        self.world, self.rank = world, rank
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(unique_id)
        h = N._p()
        N.check(self._lib.epi_comm_create(buf, world, rank, ctypes.byref(h)))
        self._h = h

    @staticmethod
    def unique_id() -> bytes:
        import ctypes
        buf = (ctypes.c_uint8 * 128)()
        N.check(N.lib().epi_comm_unique_id(buf))
        return bytes(buf)

    @classmethod
    def from_process_group(cls, group=None) -> "NcclComm":
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        box = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        return cls(world, rank, box[0])

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.epi_comm_destroy(h)
            self._h = None


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
                 exchange=None, comm: NcclComm | None = None, **kw):
        """`comm`: the per-day code all-gather over native NCCL (inside the
        day loop, capturable); otherwise `exchange` provides it (Python
        callback from the native loop: NcclCodeExchange over
        torch.distributed, ThreadExchange), or -- LocalCodeExchange -- the
        caller exchanges between lockstep days.  `exchange` also provides
        the in-step exchanges of DEN and vaccination."""
        needs_x = interventions.den_enabled or interventions.vaccination_enabled
        if needs_x and not hasattr(exchange, "sum_"):
            raise ConfigError("exposure notification and vaccination in a partitioned run need "
                              "an in-step exchange (NcclCodeExchange or ThreadExchange)")
        if comm is not None and (comm.world != plan.world or comm.rank != rank):
            raise ConfigError("the communicator's world/rank differ from the partition plan's")
        self.plan, self.rank, self.exchange, self.comm = plan, rank, exchange, comm
        self._code_len = plan.padded
        self._ready = False          # no exchange from inside the constructor's reset()
        super().__init__(pop, disease, table, interventions, seed, **kw)
        self._ready = True
        callback = exchange is not None and not isinstance(exchange, LocalCodeExchange)
        if needs_x or (callback and comm is None):
            self._hook = N.XFN(self._on_exchange)      # kept alive with the simulation
            N.check(self._lib.epi_set_exchange(self._ctx, self._hook, None))
        if comm is not None:
            N.check(self._lib.epi_set_code_exchange(self._ctx, comm._h, 2, plan.chunk))
        elif callback:
            N.check(self._lib.epi_set_code_exchange(self._ctx, None, 1, plan.chunk))
        self._native_gather = comm is not None or callback

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
            elif kind == _X_GATHER_U16:
                self.exchange.exchange(_view(buf, self.plan.padded, "<i2"))
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
        if self._ready and self._native_gather:
            # the day-0 codes of every rank (the native exchange, in place)
            N.check(self._lib.epi_allgather_codes(self._ctx, N.ptr(self.codes[0]), N.stream_handle()))

    # step() / run(): the native day loop ends every day with the code
    # exchange (epi_set_code_exchange), tomorrow's sigma tables built on a
    # side stream meanwhile

    def capture(self):
        if self.comm is None or self.iv.den_enabled or self.iv.vaccination_enabled:
            raise ConfigError("only a partitioned run over native NCCL without in-step exchanges "
                              "(DEN, vaccination) can be captured as a CUDA graph")
        return super().capture()


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
                sims[r].run()        # the native day loop; the code exchange ends every day
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
