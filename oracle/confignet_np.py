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
    out = np.arange(n, dtype=np.uint64)
    todo = np.arange(n)
    cur = out.copy()
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


_BITLEN = np.array([max(1, int(x).bit_length()) for x in range(256)], dtype=np.uint64)


def workplace_sigma(pop, seed, step):
    """For every member slot (base_w + position): the local index sigma_w(position).
    Vectorised over all workplaces; per-element domain bits, masks and keys."""
    m_w = pop.wp_size.astype(np.int64)
    W = len(m_w)
    h = rng_np.hashes(seed, step, P_WPERM, np.arange(W), 0)
    owner = np.repeat(np.arange(W), m_w)
    pos = (np.arange(len(owner)) - pop.wp_base[owner]).astype(np.uint64)
    m_i = m_w[owner].astype(np.uint64)
    k_i = _BITLEN[np.maximum(m_w[owner] - 1, 0)]
    mask = (np.uint64(1) << k_i) - np.uint64(1)
    sh = (k_i + np.uint64(1)) >> np.uint64(1)
    mult = [((h[owner] >> np.uint64(16 * r)) & np.uint64(0xFF)) | np.uint64(1) for r in range(3)]
    key = [((h[owner] >> np.uint64(16 * r + 8)) & np.uint64(0xFF)) & mask for r in range(3)]
    out = pos.copy()
    todo = np.arange(len(pos))
    cur = pos.copy()
    while len(todo):
        for r in range(3):
            cur = (((cur ^ key[r][todo]) * mult[r][todo]) & M32) & mask[todo]
            cur = cur ^ (cur >> sh[todo])
        done = cur < m_i[todo]
        out[todo[done]] = cur[done]
        todo, cur = todo[~done], cur[~done]
    return out.astype(np.int64)


def work_shifts_all(pop, seed, step, draws):
    """r[w, j] = 1 + ((v * (m - 1)) >> 16), v = 16-bit chunk j&3 of hash (w, j>>2)."""
    W = pop.n_workplaces
    m = pop.wp_size.astype(np.uint64)
    out = np.zeros((W, draws), dtype=np.int64)
    for j in range(draws):
        h = rng_np.hashes(seed, step, P_WSHIFT, np.arange(W), j >> 2)
        v = (h >> np.uint64(16 * (j & 3))) & np.uint64(0xFFFF)
        out[:, j] = (np.uint64(1) + ((v * np.maximum(m, np.uint64(1)) - v) >> np.uint64(16))).astype(np.int64)
    return out


def random_counts(seed, step, n, table, dead):
    u = rng_np.uniforms(seed, step, P_RCOUNT, np.arange(n))
    cnt = (u[:, None] >= table[None, :]).sum(axis=1) if len(table) else np.zeros(n, np.int64)
    cnt[dead] = 0
    return cnt


def realize(pop, seed, step, dead, canonical=True):
    """All directed edges of step `step` as (src, dst, kind); canonical
    (dst, src, kind) order unless `canonical=False` (the timed CPU arm: the
    reference engine sorts the valid edges itself, engine.py:98)."""
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
    # workplaces (vectorised over all members)
    if pop.n_workplaces and spec.colleague_draws:
        base = pop.wp_base.astype(np.int64)
        m_w = pop.wp_size.astype(np.int64)
        owner = np.repeat(np.arange(pop.n_workplaces), m_w)
        sigma = workplace_sigma(pop, seed, step)            # slot base+p -> local index
        posof = np.empty(len(sigma), dtype=np.int64)
        posof[base[owner] + sigma] = np.arange(len(sigma)) - base[owner]
        shifts = work_shifts_all(pop, seed, step, spec.colleague_draws)
        mem = pop.wp_members.astype(np.int64)
        m_i = m_w[owner]
        ok_w = (m_i >= 2) & alive[mem]
        for j in range(spec.colleague_draws):
            r = shifts[owner, j]
            for sign in (1, -1):
                q = np.mod(posof + sign * r, np.maximum(m_i, 1))
                src = mem[base[owner] + sigma[base[owner] + q]]
                ok = ok_w & alive[src]
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
    if not canonical:
        return src, dst, kind
    o = np.lexsort((kind, src, dst))
    return src[o], dst[o], kind[o]
