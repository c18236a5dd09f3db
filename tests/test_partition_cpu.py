"""Host-side logic of the agent-range partition, multi-process on CPU (gloo)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_04421_b200 import _native as N
from paper_2110_04421_b200.errors import ConfigError
from paper_2110_04421_b200.partition import NcclCodeExchange, PartitionPlan


def test_plan_rows_cover_population_once():
    for n, w in [(10, 1), (200, 3), (100_000, 8), (6007, 5), (10_000_000, 8)]:
        plan = PartitionPlan(n, w)
        rows = [plan.rows(r) for r in range(w)]
        assert rows[0][0] == 0 and rows[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
        assert plan.padded >= n and plan.padded % w == 0 and plan.chunk % 32 == 0
    for n, w in [(3, 4), (7, 7), (32, 2)]:
        with pytest.raises(ConfigError):
            PartitionPlan(n, w)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = PartitionPlan(n, world)
    ex = NcclCodeExchange(plan, rank)
    codes = torch.zeros(plan.padded, dtype=torch.int16)
    lo, hi = plan.rows(rank)
    codes[lo:hi] = torch.arange(lo, hi, dtype=torch.int16) * 3 + 1   # this rank's rows
    ex.exchange(codes)
    rec = torch.zeros((4, N.REC_LEN), dtype=torch.int64)
    rec[:, N.REC["step"]] = torch.arange(4)
    rec[:, N.REC["edges"]] = 10 * (rank + 1)
    rec[:, N.REC["flags"]] = 8 << rank              # distinct flag bits per rank (a bitmask column)
    rec[0, N.REC["flags"]] = 8                      # the same bit on both ranks on day 0
    ex.reduce_records(rec)
    # in-step exchanges of DEN / vaccination (row f2)
    flags = torch.zeros(n, dtype=torch.uint8)
    flags[lo:hi] = (torch.arange(lo, hi) % 7 == 0).to(torch.uint8) * (2 + rank)
    ex.gather_rows(flags)
    hist = torch.arange(55, dtype=torch.int64) * (rank + 1)
    ex.sum_(hist)
    cut = torch.tensor([5 + 10 * rank], dtype=torch.int64)
    ex.exscan_(cut)
    marks = torch.zeros(n, dtype=torch.uint8)
    marks[rank::3] = 4                              # each rank notifies every third agent from its offset
    ex.or_(marks)
    q.put((rank, codes.numpy().copy(), rec.numpy().copy(), flags.numpy().copy(), hist.numpy().copy(),
           int(cut[0]), marks.numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [100, 1001])
def test_code_exchange_and_record_reduction_gloo_world2(n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=60) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = (np.arange(n, dtype=np.int16) * 3 + 1)
    plan = PartitionPlan(n, world)
    want_flags = np.zeros(n, np.uint8)
    for r in range(world):
        lo, hi = plan.rows(r)
        ids = np.arange(lo, hi)
        want_flags[lo:hi] = (ids % 7 == 0) * (2 + r)
    want_marks = np.zeros(n, np.uint8)
    for r in range(world):
        want_marks[r::3] = 4
    for rank, codes, rec, flags, hist, cut, marks in out:
        assert np.array_equal(marks, want_marks)
        assert np.array_equal(flags, want_flags)
        assert np.array_equal(hist, np.arange(55) * 3)
        assert cut == (0 if rank == 0 else 5)
        assert np.array_equal(codes[:n], want)
        assert np.array_equal(rec[:, N.REC["step"]], np.arange(4))
        assert np.all(rec[:, N.REC["edges"]] == 30)
        assert np.array_equal(rec[:, N.REC["flags"]], [8, 24, 24, 24])   # OR, not MAX / sum


def test_local_exchange_ors_the_flag_column():
    """the emulated ranks' record reduction ORs EPI_REC_FLAGS
    (8 + 8 must stay 8, not become 16 = another flag)."""
    from types import SimpleNamespace
    from paper_2110_04421_b200.partition import LocalCodeExchange
    recs = []
    for r, fl in enumerate((8, 8 | 32)):
        rec = torch.zeros((3, N.REC_LEN), dtype=torch.int64)
        rec[:, N.REC["step"]] = torch.arange(3)
        rec[:, N.REC["edges"]] = 5
        rec[:, N.REC["flags"]] = fl
        recs.append(SimpleNamespace(rec=rec))
    out = LocalCodeExchange.reduce_records(recs)
    assert torch.all(out[:, N.REC["flags"]] == 40)
    assert torch.all(out[:, N.REC["edges"]] == 10)
    assert torch.equal(out[:, N.REC["step"]], torch.arange(3))
