"""CPU restatement of the config-network generator — TEST INFRASTRUCTURE.

Specification: `paper_2110_04421_b200/confignet.py` module docstring.  This
is an independent vectorised numpy implementation of the same definition
(the CUDA one is `paper_2110_04421_b200/csrc/epi_confignet.cuh`):
  * bijections are evaluated forward over the whole domain and inverted by
    scatter (the device evaluates the inverse rounds directly), so the two
    implementations cross-check each other's inverse;
  * keyed hashes come from `oracle.rng_np` (reference rng.py:60-100 chain).
Output: a StepGraph-like triple in canonical (dst, src, kind) order.
"""

from __future__ import annotations

import numpy as np

from . import rng_np

P_RCOUNT, P_RPERM, P_WPERM, P_WSHIFT = 72, 73, 74, 75
M32 = np.uint64(0xFFFFFFFF)


def _bits(n):
    """Domain bits k with 2^k >= n (k >= 1)."""
    return max(1, int(n - 1).bit_length())


def _round_fwd(x, mult, key, mask, s):
    x = (((x ^ key) * mult) & M32) & mask
    return x ^ (x >> s)


def walk_forward(n, mults, keys):
    """Cycle-walked keyed bijection of [0, n), evaluated for every x."""
    k = _bits(n)
    mask, s = np.uint64((1 << k) - 1), np.uint64((k + 1) >> 1)
    x = np.arange(n, dtype=np.uint64)
    out = x.copy()
    todo = np.arange(n)
    cur = x
    while len(todo):
        for m, kk in zip(mults, keys):
            cur = _round_fwd(cur, np.uint64(m), np.uint64(kk) & mask, mask, s)
        done = cur < np.uint64(n)
        out[todo[done]] = cur[done]
        todo, cur = todo[~done], cur[~done]
    return out.astype(np.int64)


def random_perm_keys(seed, step, slot):
    hs = [int(rng_np.hashes(seed, step, P_RPERM, [slot], r)[0]) for r in range(3)]
    return [(h & 0xFFFFFFFF) | 1 for h in hs], [h >> 32 for h in hs]


def work_perm_keys(seed, step, w):
    h = int(rng_np.hashes(seed, step, P_WPERM, [w], 0)[0])
    return ([((h >> (16 * r)) & 0xFF) | 1 for r in range(3)],
            [(h >> (16 * r + 8)) & 0xFF for r in range(3)])


def work_shifts(seed, step, w, m, draws):
    out = []
    for j in range(draws):
        h = int(rng_np.hashes(seed, step, P_WSHIFT, [w], j >> 2)[0])
        v = (h >> (16 * (j & 3))) & 0xFFFF
        out.append(1 + ((v * (m - 1)) >> 16))
    return out


def random_counts(seed, step, n, table, dead):
    u = rng_np.uniforms(seed, step, P_RCOUNT, np.arange(n))
    cnt = (u[:, None] >= table[None, :]).sum(axis=1) if len(table) else np.zeros(n, np.int64)
    cnt[dead] = 0
    return cnt


def realize(pop, seed, step, dead):
    """All directed edges of step `step` as (src, dst, kind), canonical order."""
    spec = pop.spec
    n = spec.n_agents
    dead = np.asarray(dead, dtype=bool)
    alive = ~dead
    S, D, K = [], [], []
    # households: complete graph on alive members (contiguous id ranges)
    ids = np.arange(n, dtype=np.int64)
    start = ids - pop.hh_off.astype(np.int64)
    for off in range(int(pop.hh_size.max()) if n else 0):
        c = start + off
        ok = (off < pop.hh_size) & (c != ids) & alive
        c_ok = np.where(ok, c, 0)
        ok &= alive[c_ok]
        S.append(c[ok]); D.append(ids[ok]); K.append(np.zeros(int(ok.sum()), np.int8))
    # workplaces
    for w in range(pop.n_workplaces):
        m = int(pop.wp_size[w])
        if m < 2:
            continue
        mem = pop.wp_members[pop.wp_base[w]:pop.wp_base[w] + m].astype(np.int64)
        mults, keys = work_perm_keys(seed, step, w)
        sigma = walk_forward(m, mults, keys)            # position -> local index
        pos = np.empty(m, dtype=np.int64)
        pos[sigma] = np.arange(m)                       # local index -> position
        for r in work_shifts(seed, step, w, m, spec.colleague_draws):
            for partner_pos in ((pos + r) % m, (pos - r) % m):
                src = mem[sigma[partner_pos]]
                ok = alive[mem] & alive[src]
                S.append(src[ok]); D.append(mem[ok]); K.append(np.ones(int(ok.sum()), np.int8))
    # random slots
    if n >= 2:
        cnt = random_counts(seed, step, n, pop.poisson_table(), dead)
        for j in range(spec.random_slots):
            mults, keys = random_perm_keys(seed, step, j)
            pi = walk_forward(n, mults, keys)
            inv = np.empty(n, dtype=np.int64)
            inv[pi] = ids
            ok = (j < cnt) & (pi != ids) & alive & alive[pi]
            S.append(pi[ok]); D.append(ids[ok]); K.append(np.full(int(ok.sum()), 2, np.int8))
            ok = (inv != ids) & (j < cnt[inv]) & alive
            S.append(inv[ok]); D.append(ids[ok]); K.append(np.full(int(ok.sum()), 2, np.int8))
    src = np.concatenate(S).astype(np.int32) if S else np.empty(0, np.int32)
    dst = np.concatenate(D).astype(np.int32) if D else np.empty(0, np.int32)
    kind = np.concatenate(K).astype(np.int8) if K else np.empty(0, np.int8)
    o = np.lexsort((kind, src, dst))
    return src[o], dst[o], kind[o]
