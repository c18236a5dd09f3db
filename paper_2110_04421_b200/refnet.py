"""Reference-native contact networks on the GPU.

`GpuRealizer` has the constructor and `realize(step, dead)` of the
reference's `GraphRealizer` (graphs.py:176-240) and returns a device-resident
`StepGraph`.  The three families are keyed parallel algorithms
(csrc/epi_refnet.cuh):
  * households — exact cliques over alive members (graphs.py:54-75);
  * occupations — ring lattice over each occupation's alive members with
    k = min(round_to_even(mean), 2*floor((m-1)/2)) (graphs.py:210-221), each
    lattice edge rewired with probability beta to a uniform non-neighbour;
  * random — stub pairing with floor(d) + Bernoulli(frac d) stubs and a keyed
    permutation of the stubs (graphs.py:138-168).
Duplicates resolve to the lowest edge / pair index, self pairs are dropped,
dead agents appear in no network.  The reference's PCG64 streams cannot be
reproduced in parallel, so parity with the reference generator is
statistical; parity with the CPU restatement of *this* algorithm
(oracle/refnet_np.py) is bitwise.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .engine import _u64
from .graph import StepGraph


def round_to_even(x: float) -> int:
    """graphs.py:171-173 (Python's half-to-even round)."""
    return int(2 * round(x / 2.0))


class GpuRealizer:
    def __init__(self, seed: int, household_id, occupation, random_degree,
                 occupation_mean_interactions, rewire_beta: float = 0.1, device=None):
        import torch
        self._lib = N.lib()
        self.seed = int(seed)
        hh = np.asarray(household_id, dtype=np.int64)
        occ = np.asarray(occupation, dtype=np.int64)
        deg = np.asarray(random_degree, dtype=np.float64)
        means = np.asarray(occupation_mean_interactions, dtype=np.float64)
        self.n_agents = n = len(hh)
        self.device = torch.device(device or "cuda")
        ids = np.arange(n, dtype=np.int64)
        # households: members grouped by id, per-agent start / size
        if n and np.all(hh[1:] >= hh[:-1]):
            order = ids                         # population.synthesize numbers households in order
        else:
            order = np.argsort(hh, kind="stable")
        sorted_hh = hh[order]
        # group boundaries in the sorted ids: start slot and size of each group
        starts = np.flatnonzero(np.concatenate(([True], sorted_hh[1:] != sorted_hh[:-1]))) if n else ids
        sizes = np.diff(np.append(starts, n))
        hh_start = np.empty(n, np.int32)
        hh_size = np.empty(n, np.int32)
        hh_start[order] = np.repeat(starts, sizes)
        hh_size[order] = np.repeat(sizes, sizes)
        # occupations 1..n_occ: members in ascending id order
        n_occ = len(means)
        emp = occ > 0
        occ_order = np.argsort(occ[emp], kind="stable")    # by occupation, ids ascending
        occ_members = ids[emp][occ_order]
        counts = np.bincount(occ[emp], minlength=n_occ + 1)[1:n_occ + 1]
        occ_start = np.concatenate(([0], np.cumsum(counts))).astype(np.int32)
        occ_k = np.array([round_to_even(float(x)) for x in means], dtype=np.int32)
        ks = np.minimum(occ_k, np.maximum(counts - 1, 0))
        ws_edges = int(np.sum(counts * np.maximum(ks, 0) // 2))
        max_stubs = int(np.sum(np.ceil(deg)))
        hh_edges = int(np.sum(hh_size.astype(np.int64) - 1))
        self.capacity = hh_edges + 2 * ws_edges + 2 * (max_stubs // 2) + 64
        slots = 1
        while slots < 2 * (ws_edges + max_stubs // 2) + 1024:
            slots <<= 1

        def up(a, dt):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(self.device)
        self._keep = dict(hh_members=up(order, np.int32), hh_start=up(hh_start, np.int32),
                          hh_size=up(hh_size, np.int32),
                          occ_members=up(occ_members if len(occ_members) else np.zeros(1), np.int32),
                          occ_start=up(occ_start, np.int32), occ_k=up(occ_k, np.int32),
                          random_degree=up(deg, np.float64))
        d = N.EpiRefnetDesc()
        d.n_agents = n
        d.hh_members = N.ptr(self._keep["hh_members"])
        d.hh_start = N.ptr(self._keep["hh_start"])
        d.hh_size = N.ptr(self._keep["hh_size"])
        d.n_occ = n_occ
        d.occ_members = N.ptr(self._keep["occ_members"])
        d.occ_start = N.ptr(self._keep["occ_start"])
        d.occ_k = N.ptr(self._keep["occ_k"])
        d.n_member_slots = len(occ_members)
        d.rewire_beta = float(rewire_beta)
        d.random_degree = N.ptr(self._keep["random_degree"])
        d.table_slots = slots
        self._desc = d
        h = N._p()
        N.check(self._lib.epi_refnet_create(ctypes.byref(d), ctypes.byref(h)))
        self._h = h
        self._src = torch.empty(self.capacity, dtype=torch.int32, device=self.device)
        self._dst = torch.empty(self.capacity, dtype=torch.int32, device=self.device)
        self._kind = torch.empty(self.capacity, dtype=torch.int8, device=self.device)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.epi_refnet_destroy(h)
            self._h = None

    def realize_counted(self, step: int, dead, count) -> None:
        """Edges of `step` into the realizer's buffers (src/dst/kind views:
        `buffers()`) without synchronising: count = device uint64[2] (edges,
        error bits 1 capacity / 2 dedupe table / 4 stub overflow)."""
        import torch
        if dead.dtype == torch.bool and dead.device == self.device and dead.is_contiguous():
            dead_t = dead.view(torch.uint8)          # same bytes (0/1), no conversion launch
        else:
            dead_t = dead.to(device=self.device, dtype=torch.uint8).contiguous()
        self._dead_keep = dead_t
        N.check(self._lib.epi_refnet_realize_counted(self._h, _u64(self.seed), int(step), N.ptr(dead_t),
                                                     N.ptr(self._src), N.ptr(self._dst), N.ptr(self._kind),
                                                     self.capacity, N.ptr(count), N.stream_handle()))

    def buffers(self):
        return self._src, self._dst, self._kind

    def realize(self, step: int, dead, copy: bool = True) -> StepGraph:
        """Edges of `step` for the given dead mask (bool[N], numpy or torch).
        copy=False returns views of the realizer's buffers, valid until the
        next call (a consumer that loads the graph at once)."""
        import torch
        if isinstance(dead, np.ndarray):
            dead_t = torch.from_numpy(np.ascontiguousarray(dead, dtype=np.uint8)).to(self.device)
        else:
            dead_t = dead.to(device=self.device, dtype=torch.uint8).contiguous()
        e = N._i64()
        N.check(self._lib.epi_refnet_realize(self._h, _u64(self.seed), int(step), N.ptr(dead_t),
                                             N.ptr(self._src), N.ptr(self._dst), N.ptr(self._kind),
                                             self.capacity, ctypes.byref(e), N.stream_handle()))
        m = int(e.value)
        if not copy:
            return StepGraph(step, self._src[:m], self._dst[:m], self._kind[:m])
        return StepGraph(step, self._src[:m].clone(), self._dst[:m].clone(), self._kind[:m].clone())
