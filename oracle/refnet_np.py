"""CPU restatement of the GPU reference-native generator — TEST INFRASTRUCTURE.

Specification: paper_2110_04421_b200/csrc/epi_refnet.cuh (header comment);
independent vectorised numpy implementation used as the bitwise checker of
the CUDA kernels (row f1).  Output: canonical (dst, src, kind) order.
"""

from __future__ import annotations

import numpy as np

from . import confignet_np, rng_np

P_WS, P_STUB, P_PERM = 81, 82, 83


def _dedupe_min(u, v, idx):
    """Keep, per undirected pair, only the entry with the smallest index."""
    if not len(u):
        return u, v
    key = np.minimum(u, v).astype(np.int64) << 31 | np.maximum(u, v).astype(np.int64)
    order = np.lexsort((idx, key))
    first = np.ones(len(order), bool)
    first[1:] = key[order][1:] != key[order][:-1]
    keep = order[first]
    return u[keep], v[keep]


def realize(seed, step, household_id, occupation, random_degree, means, beta, dead):
    dead = np.asarray(dead, dtype=bool)
    n = len(dead)
    hh = np.asarray(household_id, dtype=np.int64)
    occ = np.asarray(occupation, dtype=np.int64)
    deg = np.asarray(random_degree, dtype=np.float64)
    S, D, K = [], [], []
    # households: every ordered pair of alive co-members
    order = np.argsort(hh, kind="stable")
    cuts = np.flatnonzero(np.diff(hh[order])) + 1
    for g in np.split(order, cuts):
        g = g[~dead[g]]
        if len(g) >= 2:
            a = np.repeat(g, len(g))
            b = np.tile(g, len(g))
            ok = a != b
            S.append(a[ok]); D.append(b[ok]); K.append(np.zeros(int(ok.sum()), np.int8))
    # occupations
    for j in range(1, len(means) + 1):
        live = np.flatnonzero((occ == j) & ~dead)
        m = len(live)
        k = min(int(2 * round(float(means[j - 1]) / 2.0)), 2 * ((m - 1) // 2))
        if m < 3 or k < 2:
            continue
        half, span = k // 2, m - k - 1
        e = np.arange(half * m, dtype=np.int64)
        i, p = e // m + 1, e % m
        idx = (np.int64(j) << 40) | e
        rew = np.zeros(len(e), bool)
        if span > 0:
            rew = rng_np.uniforms(seed, step, P_WS, idx, 0) < beta
        q = (p + i) % m
        if rew.any():
            u1 = rng_np.uniforms(seed, step, P_WS, idx[rew], 1)
            q[rew] = (p[rew] + half + 1 + (u1 * span).astype(np.int64)) % m
        u, v = live[p], live[q]
        keep_u, keep_v = u[~rew], v[~rew]
        ru, rv = _dedupe_min(u[rew], v[rew], idx[rew])
        for a, b in ((keep_u, keep_v), (ru, rv)):
            S.append(np.concatenate([a, b])); D.append(np.concatenate([b, a]))
            K.append(np.ones(2 * len(a), np.int8))
    # stub pairing
    ids = np.arange(n, dtype=np.int64)
    whole = np.floor(deg)
    counts = (whole + (rng_np.uniforms(seed, step, P_STUB, ids) < deg - whole)).astype(np.int64)
    counts[dead] = 0
    off = np.concatenate(([0], np.cumsum(counts)))
    total = int(off[-1])
    if total >= 2:
        hs = [int(rng_np.hashes(seed, step, P_PERM, [0], r)[0]) for r in range(3)]
        k1 = [np.uint64(h & 0xFFFFFFFF) for h in hs]
        k2 = [np.uint64((h >> 32) | 1) for h in hs]
        a_, b_ = confignet_np.radix(total)
        pos = np.arange(2 * (total // 2), dtype=np.uint64)
        stub = confignet_np.walk(pos, total, k1, k2, np.uint64(a_), np.uint64(b_))
        owner = np.searchsorted(off, stub, side="right") - 1
        u, v = owner[0::2], owner[1::2]
        pair = np.arange(len(u), dtype=np.int64)
        ok = u != v
        ru, rv = _dedupe_min(u[ok], v[ok], pair[ok])
        S.append(np.concatenate([ru, rv])); D.append(np.concatenate([rv, ru]))
        K.append(np.full(2 * len(ru), 2, np.int8))
    if not S:
        return np.empty(0, np.int32), np.empty(0, np.int32), np.empty(0, np.int8)
    src = np.concatenate(S).astype(np.int32)
    dst = np.concatenate(D).astype(np.int32)
    kind = np.concatenate(K).astype(np.int8)
    o = np.lexsort((kind, src, dst))
    return src[o], dst[o], kind[o]
