"""CPU restatement of the GPU reference-native generator — TEST INFRASTRUCTURE.

Specification: paper_2110_04421_b200/csrc/epi_refnet.cuh (header comment);
rewired occupation edges are re-drawn on collision, never dropped, as the
reference's sequential rejection keeps n*k/2 edges (graphs.py:86-129);
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


WS_ROUNDS = 64


def _rewire_rounds(seed, step, live, idx, p, i, m, half, span):
    """Rewired lattice edges placed one-for-one (graphs.py:116-128 keeps the
    undirected edge count at n*k/2): round 0 proposes u_1, the lowest edge
    index keeps a contested pair; in round r >= 1 every unplaced edge
    proposes u_{1+r}, pairs placed earlier are taken, the lowest index wins
    among the round's new pairs; after WS_ROUNDS rounds an edge keeps its
    lattice pair (p, p + i)."""
    order = np.argsort(idx, kind="stable")
    idx, p, i = idx[order], p[order], i[order]
    taken = set()
    out_u = np.empty(len(idx), np.int64)
    out_v = np.empty(len(idx), np.int64)
    pending = np.arange(len(idx))
    for r in range(WS_ROUNDS + 1):
        if not len(pending):
            break
        ids = idx[pending]
        u1 = rng_np.uniforms(seed, step, P_WS, ids, 1 + r)
        q = (p[pending] + half + 1 + (u1 * span).astype(np.int64)) % m
        u, v = live[p[pending]], live[q]
        keys = (np.minimum(u, v).astype(np.int64) << 31) | np.maximum(u, v).astype(np.int64)
        won = np.zeros(len(pending), bool)
        seen = set()
        for t in range(len(pending)):            # ascending edge index
            k = int(keys[t])
            if k not in taken and k not in seen:
                won[t] = True
            seen.add(k)
        taken.update(int(k) for k in keys[won])
        out_u[pending[won]], out_v[pending[won]] = u[won], v[won]
        pending = pending[~won]
    if len(pending):                             # no free pair: the lattice pair
        out_u[pending] = live[p[pending]]
        out_v[pending] = live[(p[pending] + i[pending]) % m]
    return out_u, out_v


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
        ru, rv = _rewire_rounds(seed, step, live, idx[rew], p[rew], i[rew], m, half, span)
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
