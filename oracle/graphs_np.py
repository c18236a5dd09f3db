"""Restatement of the reference's per-step realizer — TEST INFRASTRUCTURE.

Follows pkg/src/epivec/graphs.py:54-240 draw for draw (numpy PCG64
substreams keyed by rng.py:103-113), so on the same numpy version its output
equals the reference's edge lists element for element; pinned against the
graphs recorded in tests/golden/traj_*.npz.  Used as the statistical
reference for the GPU reference-native generator (row f1).
"""

from __future__ import annotations

import numpy as np

from . import rng_np


def _substream(seed, purpose, *idx):
    """rng.py:103-113: PCG64 seeded with derive_seed(seed, purpose, *idx)."""
    h = rng_np.prefix(seed, 0, purpose)
    for i in idx:
        h = rng_np._fold_py(h, int(i))
    return np.random.Generator(np.random.PCG64(h))


def household_edges(household_id):
    """graphs.py:54-83: per household of m >= 2, every ordered member pair."""
    order = np.argsort(household_id, kind="stable")
    ids = household_id[order]
    cuts = np.flatnonzero(np.diff(ids)) + 1
    src, dst = [], []
    for group in np.split(order, cuts):
        m = len(group)
        if m < 2:
            continue
        src.append(np.repeat(group, m - 1))
        dst.append(np.broadcast_to(group, (m, m))[~np.eye(m, dtype=bool)])
    if not src:
        return np.empty(0, np.int32), np.empty(0, np.int32)
    return np.concatenate(src).astype(np.int32), np.concatenate(dst).astype(np.int32)


def small_world(n, k, beta, gen):
    """graphs.py:86-129: ring lattice + sequential rewiring at the source end."""
    half = k // 2
    base = np.arange(n, dtype=np.int64)
    us = np.tile(base, half)
    vs = np.concatenate([(base + j) % n for j in range(1, half + 1)])
    if beta > 0.0:
        chosen = np.flatnonzero(gen.random(len(us)) < beta)
        if len(chosen):
            taken = set((np.minimum(us, vs) * n + np.maximum(us, vs)).tolist())
            for i in chosen.tolist():
                u, v = int(us[i]), int(vs[i])
                taken.discard(min(u, v) * n + max(u, v))
                target = v
                for _ in range(8 * n):
                    w = int(gen.integers(0, n))
                    if w != u and (min(u, w) * n + max(u, w)) not in taken:
                        target = w
                        break
                vs[i] = target
                taken.add(min(u, target) * n + max(u, target))
    return us, vs


def stub_pairs(agents, degrees, gen):
    """graphs.py:138-168: floor + Bernoulli stubs, shuffle, pair, drop self /
    duplicate pairs (first occurrence kept)."""
    whole = np.floor(degrees).astype(np.int64)
    counts = whole + (gen.random(len(agents)) < degrees - whole)
    stubs = np.repeat(agents, counts)
    if len(stubs) < 2:
        return np.empty(0, np.int32), np.empty(0, np.int32)
    stubs = gen.permutation(stubs)
    if len(stubs) % 2:
        stubs = stubs[:-1]
    a, b = stubs[0::2].astype(np.int64), stubs[1::2].astype(np.int64)
    ok = a != b
    a, b = a[ok], b[ok]
    if len(a):
        span = int(max(a.max(), b.max())) + 1
        _, first = np.unique(np.minimum(a, b) * span + np.maximum(a, b), return_index=True)
        keep = np.sort(first)
        a, b = a[keep], b[keep]
    return a.astype(np.int32), b.astype(np.int32)


class ReferenceRealizer:
    """graphs.py:176-240."""

    def __init__(self, seed, household_id, occupation, random_degree, means, beta=0.1):
        self.seed = seed
        self.hh_src, self.hh_dst = household_edges(np.asarray(household_id))
        occupation = np.asarray(occupation)
        self.random_degree = np.asarray(random_degree, dtype=np.float64)
        self.groups = {int(j): np.flatnonzero(occupation == j).astype(np.int32)
                       for j in np.unique(occupation) if j > 0}
        self.means = {j: float(means[j - 1]) for j in self.groups}
        self.beta = float(beta)

    def realize(self, step, dead):
        S, D, K = [], [], []
        if len(self.hh_src):
            keep = ~(dead[self.hh_src] | dead[self.hh_dst])
            S.append(self.hh_src[keep]); D.append(self.hh_dst[keep])
            K.append(np.zeros(int(keep.sum()), np.int8))
        for j, members in self.groups.items():
            live = members[~dead[members]]
            m = len(live)
            k = min(int(2 * round(self.means[j] / 2.0)), 2 * ((m - 1) // 2))
            if m < 3 or k < 2:
                continue
            us, vs = small_world(m, k, self.beta, _substream(self.seed, 67, step, j))
            a, b = live[us], live[vs]
            S.append(np.concatenate([a, b]).astype(np.int32))
            D.append(np.concatenate([b, a]).astype(np.int32))
            K.append(np.ones(2 * len(a), np.int8))
        alive = np.flatnonzero(~dead).astype(np.int32)
        if len(alive) >= 2:
            a, b = stub_pairs(alive, self.random_degree[alive], _substream(self.seed, 68, step))
            S.append(np.concatenate([a, b]).astype(np.int32))
            D.append(np.concatenate([b, a]).astype(np.int32))
            K.append(np.full(2 * len(a), 2, np.int8))
        if not S:
            return np.empty(0, np.int32), np.empty(0, np.int32), np.empty(0, np.int8)
        return np.concatenate(S), np.concatenate(D), np.concatenate(K)
